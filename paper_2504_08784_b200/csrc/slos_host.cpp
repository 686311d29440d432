// C-ABI implementation (include/slos_planner.h) of the product planner.
//
// Host side = the work the reference does before/around its DP that is host-
// trivial or string-typed (SURVEY.md §7 hard part 6): validation
// (dp_scheduler.cpp:367-392), the chain std::stable_sort with its eps/forced/id
// comparator (:393-397, run here with libstdc++ so eps-tie behaviour is identical),
// floor_at / suffix_prefill (:399-408), edf_fallback's prefill order (:121-124),
// packing instances into SoA blobs, one H2D copy, the kernel pipeline
// (dp_kernel -> build_kernel -> compact_kernel), one D2H copy of the packed
// results, and capacity regrowth for the rare instance whose scratch estimate
// was too small. There is no CPU fallback: without an sm_100 device every entry
// point returns SLOS_ERR_NO_DEVICE.
#include <algorithm>
#include <array>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <numeric>
#include <set>
#include <chrono>
#include <condition_variable>
#include <functional>
#include <thread>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "slos_dev.h"
#include "slos_launch.h"
#include "../../include/slos_planner.h"
#include "../../include/slos_fit.h"

namespace slos {
struct GapBatchOut {
  double start_s, end_s;
  int64_t capacity, spec_step, decode_tokens, prefill_budget;
  int64_t per_tier[kMaxTiers];
  int32_t first_owner, n_owner;
};
struct GapParams {
  const PlannerDev* planner;
  const GapQueryDev* q;
  const double* ph;
  const int64_t* bl;
  const int64_t* rm;
  const int32_t* tr;
  const int32_t* ow;
  GapBatchOut* ob;
  int64_t* oo;
  unsigned char* work;
  GapOutDev* out;
};
struct SpecSolH {
  bool ok;
  int lengths[kMaxTiers];
  double bt;
  int64_t cap;
  int64_t decode;
  double tpt;
};
}  // namespace slos

using namespace slos;

// ------------------------------------------------------------------ state ---

struct slos_planner {
  PlannerDev dev;
  std::vector<slos_perf_term> terms;
  std::vector<double> tpot, slow;
  int L = 0;
  int tpot_window = 10;
  slos_planner_config cfg{};
  bool device_ok = true;  // representable on device (terms, tiers, spec length)
};

namespace {

thread_local std::string g_err;

int set_err(int code, const std::string& msg) {
  g_err = std::string(slos_status_slug(code)) + ": " + msg;
  return code;
}

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    size_t want = std::max(bytes, (size_t)1 << 20);
    want = want + want / 4;
    cudaError_t e = cudaMalloc(&p, want);
    if (e == cudaSuccess) cap = want;
    return e;
  }
};

struct PinBuf {
  void* p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap) return cudaSuccess;
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
    size_t want = std::max(bytes, (size_t)1 << 20);
    want = want + want / 4;
    cudaError_t e = cudaHostAlloc(&p, want, cudaHostAllocDefault);
    if (e == cudaSuccess) cap = want;
    return e;
  }
};

// Pinned result arenas, reference counted by the slos_result objects that point
// into them; recycled through a small pool.
struct ResultArena {
  std::atomic<int> refs{0};
  void* p = nullptr;
  size_t cap = 0;
  bool pinned = true;
};

struct Ctx {
  std::mutex mu;
  bool init = false;
  int status = SLOS_OK;
  std::string why;
  cudaStream_t stream = nullptr;
  size_t smem_optin = 0;  // opt-in dynamic shared memory per CTA (227 KB on B200)
  DevBuf d_in, d_scr, d_out, d_pack, d_wscr, d_small, d_fit;
  PinBuf h_in, h_small, h_fit;
  std::mutex pool_mu;
  std::vector<ResultArena*> pool;
};

Ctx& ctx() {
  static Ctx* c = new Ctx();  // never destroyed: results may outlive static teardown
  return *c;
}

// Host worker pool for the per-instance preparation (chain sort, capacity
// estimates, pair keys, SoA fill): instances are independent, so a batch's host
// work splits across cores like the kernels split across SMs.
class HostPool {
 public:
  static HostPool& get() {
    static HostPool* p = new HostPool();
    return *p;
  }
  // fn(lo, hi) over contiguous ranges of [0, n); runs inline for small n. Workers
  // spin for a short while after each job before sleeping, so the back-to-back
  // jobs of one upload do not pay a thread wake-up each.
  // time spent in run() and the number of runs (SLOS_HOST_TIMING breakdowns)
  double run_ms = 0.0;
  int runs = 0;
  // min_grain: fewest items per piece (16 for cheap items; 1 for items heavy enough
  // that even a few of them are worth every core, e.g. 2,000-decoder instances)
  void run(int n, const std::function<void(int, int)>& fn, int min_grain = 16) {
    const int T = (int)workers_.size() + 1;
    if (n < (min_grain < 16 ? 2 : 64) || T == 1) { fn(0, n); return; }
    struct Tm {
      HostPool* h;
      std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
      ~Tm() {
        h->run_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        ++h->runs;
      }
    } tm_{this};
    fn_ = &fn;
    n_ = n;
    next_.store(0, std::memory_order_relaxed);
    // chunks: ~8 per thread, at least 16 items (one shared counter: small chunks of
    // cheap items would serialise on it)
    grain_ = std::max(std::max(1, min_grain), n / (8 * T));
    busy_.store((int)workers_.size(), std::memory_order_relaxed);
    {
      std::lock_guard<std::mutex> l(mu_);
      gen_.fetch_add(1, std::memory_order_release);
    }
    cv_.notify_all();
    work();
    // wait for the workers (spinning: they are normally already awake)
    const auto t0 = std::chrono::steady_clock::now();
    while (busy_.load(std::memory_order_acquire) != 0) {
      if (std::chrono::steady_clock::now() - t0 > std::chrono::microseconds(200)) {
        std::unique_lock<std::mutex> l(mu_);
        done_.wait(l, [&] { return busy_.load(std::memory_order_acquire) == 0; });
        break;
      }
    }
    fn_ = nullptr;
  }

 private:
  HostPool() {
    const char* e = std::getenv("SLOS_HOST_THREADS");
    int t = e ? std::atoi(e) : (int)std::min(16u, std::max(1u, std::thread::hardware_concurrency()));
    for (int k = 1; k < t; ++k) workers_.emplace_back([this] { loop(); });
    for (auto& w : workers_) w.detach();
  }
  void work() {
    const int grain = grain_;
    for (;;) {
      const int lo = next_.fetch_add(grain);
      if (lo >= n_) break;
      (*fn_)(lo, std::min(n_, lo + grain));
    }
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      // a new job: spin ~0.5 ms first, then sleep on the condition variable
      const auto t0 = std::chrono::steady_clock::now();
      uint64_t g = gen_.load(std::memory_order_acquire);
      while (g == seen && std::chrono::steady_clock::now() - t0 < std::chrono::microseconds(500))
        g = gen_.load(std::memory_order_acquire);
      if (g == seen) {
        std::unique_lock<std::mutex> l(mu_);
        cv_.wait(l, [&] { return gen_.load(std::memory_order_acquire) != seen; });
        g = gen_.load(std::memory_order_acquire);
      }
      seen = g;
      work();
      if (busy_.fetch_sub(1, std::memory_order_acq_rel) == 1) {
        std::lock_guard<std::mutex> l(mu_);
        done_.notify_all();
      }
    }
  }
  std::vector<std::thread> workers_;
  int grain_ = 16;
  std::mutex mu_;
  std::condition_variable cv_, done_;
  const std::function<void(int, int)>* fn_ = nullptr;
  std::atomic<int> next_{0};
  int n_ = 0;
  std::atomic<int> busy_{0};
  std::atomic<uint64_t> gen_{0};
};

int ensure_device(Ctx& c) {
  if (c.init) return c.status;
  c.init = true;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    c.status = SLOS_ERR_NO_DEVICE;
    c.why = "no CUDA device (the product has no CPU fallback)";
    return c.status;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, dev);
  if (prop.major != 10) {
    c.status = SLOS_ERR_NO_DEVICE;
    c.why = std::string("device ") + prop.name + " is not sm_100 (B200)";
    return c.status;
  }
  int optin = 0;
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  c.smem_optin = (size_t)optin;
  e = cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    c.status = SLOS_ERR_CUDA;
    c.why = cudaGetErrorString(e);
    return c.status;
  }
  c.status = SLOS_OK;
  return SLOS_OK;
}

ResultArena* arena_get(Ctx& c, size_t bytes) {
  {
    // best fit among the pooled pinned arenas
    std::lock_guard<std::mutex> g(c.pool_mu);
    long best = -1;
    for (size_t i = 0; i < c.pool.size(); ++i)
      if (c.pool[i]->cap >= bytes && (best < 0 || c.pool[i]->cap < c.pool[(size_t)best]->cap)) best = (long)i;
    if (best >= 0) {
      ResultArena* a = c.pool[(size_t)best];
      c.pool.erase(c.pool.begin() + best);
      return a;
    }
  }
  ResultArena* a = new ResultArena();
  // power-of-two sizes so arenas of similar batches are reused (pinned
  // allocation costs milliseconds)
  size_t want = (size_t)1 << 16;
  while (want < bytes) want <<= 1;
  if (cudaHostAlloc(&a->p, want, cudaHostAllocDefault) != cudaSuccess) {
    a->p = std::malloc(want);  // pageable is still correct, only slower to fill
    if (!a->p) { delete a; return nullptr; }
    a->cap = want;
    a->pinned = false;
    return a;
  }
  a->cap = want;
  return a;
}

void arena_release(ResultArena* a) {
  Ctx& c = ctx();
  if (--a->refs != 0) return;
  if (!a->pinned) {
    std::free(a->p);
    delete a;
    return;
  }
  {
    // keep up to 16 pinned arenas / 8 GiB for reuse: pinned allocation and release
    // cost milliseconds and a pipelined batch holds one arena per chunk
    std::lock_guard<std::mutex> g(c.pool_mu);
    size_t held = 0;
    for (const ResultArena* x : c.pool) held += x->cap;
    if (c.pool.size() < 16 && held + a->cap <= ((size_t)8 << 30)) {
      c.pool.push_back(a);
    } else {
      cudaFreeHost(a->p);
      delete a;
    }
  }
}


// ------------------------------------------------------------ blob layout ---

struct Blob {
  size_t bytes = 0;
  template <typename T>
  size_t add(size_t count) {
    bytes = (bytes + 255) & ~(size_t)255;
    const size_t o = bytes;
    bytes += sizeof(T) * std::max<size_t>(count, 1);
    return o;
  }
};

// BatchPlanner::quantize_gap (batch_planner.cpp:136-139), host copy for the pair keys.
double host_quantize_gap(double g) {
  if (g <= 0) return 0.0;
  return std::floor(g * 1000.0 + 1e-6) / 1000.0;
}

// Instances with at most this many running decoders are reconstructed by one warp
// (measured crossover: warp-built C1 (48 decoders) and the C5 corpus are faster,
// block-built C2 (240 decoders) is faster). SLOS_BUILD_WARP_MAX_DEC overrides.
int build_warp_max_dec() {
  static const int v = [] {
    const char* e = std::getenv("SLOS_BUILD_WARP_MAX_DEC");
    return e ? std::atoi(e) : 96;
  }();
  return v;
}

// Parts of one solve whose DP / reconstruction are pipelined across streams
// (SLOS_SOLVE_PARTS overrides; 1 disables).
int solve_parts(int nv) {
  static const int env = [] {
    const char* e = std::getenv("SLOS_SOLVE_PARTS");
    return e ? std::atoi(e) : 2;
  }();
  static const int per = [] {  // fewest instances per part (SLOS_PART_MIN)
    const char* e = std::getenv("SLOS_PART_MIN");
    return e ? std::max(1, std::atoi(e)) : 128;
  }();
  int P = std::max(1, std::min(env, kMaxParts));
  if (nv < per * P) P = std::max(1, nv / per);
  return std::max(1, P);
}

// Direct bucket-table entries per DP CTA (shared memory); instances whose count
// space prod_l (items of tier l + 1) exceeds it hash instead.
constexpr int kDirectMax = 1024;
// Instances with (n_dec + 8) * (N + 1)^2 < kSmallCost (chain <= 14 items, a few
// dozen decoders: the C5 sweep family) run their admission DP in dp_kernel_small,
// 64-thread CTAs at 16 per SM; their direct bucket table holds kDirectSmall entries.
constexpr double kSmallCost = 2048.0;
// Instances with cost >= kBigCost (thousands of running decoders: the C4 family) run
// their admission DP in dp_kernel_big (512 threads, one CTA per SM); SLOS_DP_BIG_COST
// overrides (0 disables). A power of two, so the big instances are a prefix of the
// log2-bucketed cost-descending launch order.
// Batches of at most this many instances are latency bound (fewer instances than
// SMs): every instance gets the widest kernels (SLOS_LATENCY_BATCH overrides, 0 off).
bool latency_batch(int nv) {
  const char* e = std::getenv("SLOS_LATENCY_BATCH");  // read per upload: tests toggle it
  return nv <= (e ? std::atoi(e) : 148);
}

double dp_big_cost() {
  static const double v = [] {
    const char* e = std::getenv("SLOS_DP_BIG_COST");
    return e ? std::atof(e) : 262144.0;
  }();
  return v;
}
constexpr int kDirectSmall = 256;
bool dp_small_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("SLOS_DP_SMALL");
    return e ? std::atoi(e) != 0 : true;
  }();
  return on;
}

// Instances with at least this many running decoders are reconstructed by a
// 256-thread CTA (SLOS_BUILD_BIG_MIN_DEC overrides).
int build_big_min_dec() {
  static const int v = [] {
    const char* e = std::getenv("SLOS_BUILD_BIG_MIN_DEC");
    return e ? std::atoi(e) : 1024;
  }();
  return v;
}

bool integral(double v) { return std::isfinite(v) && v == std::floor(v) && std::fabs(v) < 4.0e15; }

struct Prep {  // host-side per-instance preparation
  int status = SLOS_OK;
  std::string why;
  int planner = 0;
  int N = 0, n_dec = 0, n_pre = 0;
  int last_forced = -1;
  bool have_rd = false;
  bool values_integral = true;
  std::vector<int> chain;  // encoded: >=0 running idx (forced), <0 -(pending+1)
  std::vector<int> pre;    // running indices, EDF order
  double span = 0.0;       // max gap bound for slot capacity
  double tail_bound = 0.0;
  int64_t max_rem = 0;
};

struct ChainKey {
  bool forced;
  const char* id;
  double deadline;
  int enc;
};

// prep_instance runs on HostPool workers: its message goes into the Prep and the
// calling thread reports it (g_err is thread-local)
int prep_err(Prep& pr, int code, const char* msg) {
  pr.why = std::string(slos_status_slug(code)) + ": " + msg;
  return code;
}

int prep_instance(const slos_planner* P, const slos_input* in, int unit_value, Prep& pr) {
  // Prep objects are reused across calls (their vectors keep their capacity)
  pr.planner = 0;
  pr.N = pr.n_dec = pr.n_pre = 0;
  pr.last_forced = -1;
  pr.have_rd = false;
  pr.values_integral = true;
  pr.span = pr.tail_bound = 0.0;
  pr.max_rem = 0;
  const int L = P->L;
  if (L > 8) return prep_err(pr, SLOS_ERR_INVALID_PARAMETERS, "at most 8 SLO tiers supported");
  if (in->n_running >= SLOS_ENTRY_MAX_REQS || in->n_pending >= SLOS_ENTRY_MAX_REQS)  // 24-bit entry refs
    return prep_err(pr, SLOS_ERR_INVALID_PARAMETERS, "too many requests for the plan entry format");
  if (!P->device_ok) return prep_err(pr, SLOS_ERR_RANGE, "planner not representable on device");
  thread_local std::vector<ChainKey> ch;  // capacity kept across calls
  ch.clear();
  ch.reserve((size_t)in->n_running + (size_t)in->n_pending);
  for (int i = 0; i < in->n_running; ++i) {
    const slos_running& r = in->running[i];
    if (r.prefill_remaining <= 0) continue;
    ch.push_back({true, r.id ? r.id : "", r.prefill_deadline, i});
  }
  for (int i = 0; i < in->n_pending; ++i) {
    const slos_pending& p = in->pending[i];
    ch.push_back({false, p.id ? p.id : "", p.prefill_deadline, -(i + 1)});
  }
  if (ch.size() > 250) return prep_err(pr, SLOS_ERR_INVALID_PARAMETERS, "admission chain too large");
  for (const ChainKey& k : ch) {
    const int tier = k.enc >= 0 ? in->running[k.enc].decode_tier : in->pending[-k.enc - 1].decode_tier;
    if (tier < 0 || tier >= L) return prep_err(pr, SLOS_ERR_INVALID_PARAMETERS, "bad SLO tier");
  }
  for (int i = 0; i < in->n_running; ++i) {
    const slos_running& r = in->running[i];
    if (r.prefill_remaining <= 0 && r.decode_remaining > 0 && (r.decode_tier < 0 || r.decode_tier >= L))
      return prep_err(pr, SLOS_ERR_INVALID_PARAMETERS, "vector::_M_range_check: running decode tier");
  }
  std::stable_sort(ch.begin(), ch.end(), [](const ChainKey& a, const ChainKey& b) {
    if (std::abs(a.deadline - b.deadline) > kTimeEps) return a.deadline < b.deadline;
    if (a.forced != b.forced) return a.forced;
    return std::strcmp(a.id, b.id) < 0;
  });
  pr.N = (int)ch.size();
  pr.chain.resize(ch.size());
  double maxdl = in->now, mindl = in->now;
  for (size_t k = 0; k < ch.size(); ++k) {
    pr.chain[k] = ch[k].enc;
    if (ch[k].forced) pr.last_forced = (int)k;
    maxdl = std::max(maxdl, ch[k].deadline);
    mindl = std::min(mindl, ch[k].deadline);
    const double v = ch[k].forced ? 0.0 : (unit_value ? 1.0 : in->pending[-ch[k].enc - 1].value);
    if (!integral(v)) pr.values_integral = false;
  }
  pr.span = std::max(0.0, maxdl - mindl);
  struct PreKey { int idx; double ddl; const char* id; };
  thread_local std::vector<PreKey> pre;  // capacity kept across calls
  pre.clear();
  double tb = 0.0;
  for (int i = 0; i < in->n_running; ++i) {
    const slos_running& r = in->running[i];
    if (r.prefill_remaining > 0) {
      pre.push_back({i, r.prefill_deadline, r.id ? r.id : ""});
    } else if (r.decode_remaining > 0) {
      pr.n_dec++;
      pr.have_rd = true;
      const double tp = P->tpot[r.decode_tier];
      tb = std::max(tb, (r.next_due_s - in->now) + tp);
      pr.max_rem = std::max(pr.max_rem, r.decode_remaining + std::max<int64_t>(0, r.backlog));
    }
  }
  std::stable_sort(pre.begin(), pre.end(), [](const PreKey& a, const PreKey& b) {
    if (std::abs(a.ddl - b.ddl) > kTimeEps) return a.ddl < b.ddl;
    return std::strcmp(a.id, b.id) < 0;
  });
  pr.n_pre = (int)pre.size();
  pr.pre.resize(pre.size());
  for (size_t k = 0; k < pre.size(); ++k) pr.pre[k] = pre[k].idx;
  double max_tpot = 0.0;
  for (int l = 0; l < L; ++l) max_tpot = std::max(max_tpot, P->tpot[l]);
  pr.tail_bound = std::max({2.0 * max_tpot, in->tail_horizon_s, tb, 0.0});
  if (pr.N == 0 && !(in->tail_horizon_s > kTimeEps)) {
    // untrimmed decode tail (dp_scheduler.cpp:311-315): every line to completion
    double full = 0.0;
    for (int i = 0; i < in->n_running; ++i) {
      const slos_running& r = in->running[i];
      if (r.prefill_remaining > 0 || r.decode_remaining <= 0) continue;
      const double tp = P->tpot[r.decode_tier];
      full = std::max(full, std::max(0.0, r.next_due_s - in->now) + (double)r.decode_remaining * tp);
    }
    pr.tail_bound = std::max(pr.tail_bound, full + max_tpot);
  }
  return SLOS_OK;
}

// capacities (scratch) per instance; `grow` multiplies them after an overflow
struct Caps {
  int64_t surv, cand, memo, batch, entry, work, gb, go;
};

int64_t pow2_at_least(int64_t x) {
  int64_t p = 1;
  while (p < x) p <<= 1;
  return p;
}

Caps estimate_caps(const slos_planner* P, const slos_input* in, const Prep& pr, int grow) {
  Caps c;
  const double t0 = P->tpot[0];
  const int64_t S_gap = (int64_t)std::ceil(pr.span / t0) + 6;
  const int64_t S_tail = (int64_t)std::ceil(pr.tail_bound / t0) + 6;
  const int64_t S = std::max<int64_t>({S_gap, S_tail, 16});
  const int64_t M = pr.n_dec + pr.N + 1;
  const int64_t g = (int64_t)1 << (2 * grow);
  const int64_t N1 = pr.N + 1;
  // small chains get small arenas (the DP clears its memo and bucket-hash slices
  // itself, so their size is write traffic per solve); overflow regrows (grow)
  c.surv = std::max<int64_t>(256, 16 * N1 * N1) * g;
  c.cand = pow2_at_least(std::max<int64_t>(64, 4 * N1 * N1) * g);
  c.memo = pow2_at_least(std::max<int64_t>(64, 8 * N1 * N1) * g);
  c.gb = (S + 8) << (2 * grow);
  c.go = M * c.gb;
  // plan output: gaps + tail, or the fallback (until every line completes)
  double max_tpot = 0.0;
  for (int l = 0; l < P->L; ++l) max_tpot = std::max(max_tpot, P->tpot[l]);
  int64_t pre_tokens = 0;
  for (int i = 0; i < in->n_running; ++i)
    if (in->running[i].prefill_remaining > 0) pre_tokens += in->running[i].prefill_remaining;
  const int64_t fb_batches = pr.max_rem * ((int64_t)std::ceil(max_tpot / t0) + 1) +
                             pre_tokens / std::max<int64_t>(1, P->cfg.max_chunk_tokens) + pr.n_pre + 16;
  c.batch = std::max<int64_t>((pr.N + 2) * (S + 4), std::min<int64_t>(fb_batches, 100000)) * (grow + 1) + 64;
  c.entry = std::max<int64_t>(c.batch * (pr.n_dec + pr.N + 1) / 2, 1024) * (grow + 1);
  const int64_t engine = S * (M + 1) * 4 + S * (64 + 8 * P->L) + M * 48 + 64 * M + (1 << 16);
  c.work = (M * 32 + (pr.N + 2) * 32 + 2 * c.gb * (int64_t)sizeof(GapBatchOut) + 16 * c.go + engine) * (grow + 1);
  return c;
}

void fill_planner_dev(slos_planner* p) {
  PlannerDev& d = p->dev;
  std::memset(&d, 0, sizeof d);
  p->device_ok = p->terms.size() <= (size_t)kMaxTerms && p->L <= kMaxTiers &&
                 (!p->cfg.speculative || p->cfg.spec_max_len <= kMaxSpecLen);
  d.n_terms = (int32_t)std::min<size_t>(p->terms.size(), kMaxTerms);
  for (int t = 0; t < d.n_terms; ++t) {
    d.k1[t] = p->terms[t].k1;
    d.k2[t] = p->terms[t].k2;
    d.b[t] = p->terms[t].b;
  }
  d.L = std::min(p->L, kMaxTiers);
  for (int l = 0; l < d.L; ++l) d.tpot[l] = p->tpot[l];
  d.margin1 = 1.0 + p->cfg.plan_margin;
  d.spec_alpha = p->cfg.spec_alpha;
  d.max_chunk = p->cfg.max_chunk_tokens;
  d.max_batch = p->cfg.max_batch_tokens;
  d.speculative = p->cfg.speculative ? 1 : 0;
  d.spec_max_len = std::min(p->cfg.spec_max_len, kMaxSpecLen);
  for (int sl = 1; sl <= d.spec_max_len; ++sl) d.acc[sl] = slos_expected_accepted(p->cfg.spec_alpha, sl);
}

// ---------------------------------------------------------- batch runner ---

struct Job {
  int k;      // index into the caller's arrays
  int grow;   // capacity growth step
};

struct Layout {
  size_t planners, inst, order, dec_idx, dec_tier, dec_bytier, dec_next, dec_backlog, dec_rem;
  size_t ch_deadline, ch_prefill, ch_tier, ch_memory, ch_value, ch_forced, ch_ref, ch_floor, ch_suffix;
  size_t pre_idx, pre_left, run_tier, recdef, recmap;
  size_t in_bytes;
  size_t s_counts, s_mem, s_pb, s_value, s_nadm, s_parent, s_arena, s_level;
  size_t c_src, c_j, c_memo, c_flag, c_bucket, c_pos, c_aux, c_counts, c_mem, c_pb, c_value, c_nadm;
  size_t c_bkey, c_bval, memo, bq, work, anchors, scr_bytes, atask, pair, groups, s_sb, s_bcnt, k_val, ctime, ccnt;
  int64_t n_atask;
  size_t memo_bytes, bkey_bytes, bval_bytes;
  size_t out, sel, ids, batches, entries, out_bytes;
};

struct Workspace {
  DevBuf d_in, d_scr, d_out, d_pack, d_wscr;
  PinBuf h_in, h_small;
  slos_planner* const* planners = nullptr;
  const slos_input* inputs = nullptr;
  int unit_value = 0;
  std::vector<Job> jobs;
  std::vector<int> valid;
  int nv = 0;
  Layout Ly;
  BatchArgs A;
  DpParams dp;
  size_t smem = 0;
  DpParams dp_small;              // dp_kernel_small (instances of cost < kSmallCost)
  size_t smem_small = 0;
  int small_lo[kMaxParts] = {0};  // first order position of each part that is small
  int big_hi[kMaxParts] = {0};    // end of each part's big prefix (dp_kernel_big)
  DpParams dp_big;                // dp_kernel_big
  size_t smem_big = 0;
  bool any_big = false;
  size_t anchor_smem = 0;
  int maxN = 0;
  cudaStream_t stream = nullptr;
  bool uploaded = false;
  bool solved = false;  // ev[2] marks the end of a solve
  int64_t launches = 0;  // kernels launched by the last solve
  int n_total = 0;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  cudaStream_t own_stream = nullptr;  // pipeline workspaces only
  int n_parts = 1;
  int part_lo[kMaxParts + 1] = {0};
  int atask_lo[kMaxParts + 1] = {0};  // anchor-task range of each part
  int atask_big[kMaxParts] = {0};     // end of each part's big-instance anchor tasks
  cudaEvent_t ev_anc[kMaxParts] = {nullptr};
  int qbase[kQueues] = {0};
  int qn[kQueues] = {0};
  cudaStream_t pstream[kMaxParts] = {nullptr};  // per-part streams, earlier parts higher priority
  cudaStream_t astream = nullptr;                // anchor / group kernels of every part
  cudaEvent_t ev_fork = nullptr, ev_dp[kMaxParts] = {nullptr}, ev_join[kMaxParts] = {nullptr};
  cudaEvent_t ev_bend[kMaxParts] = {nullptr};  // end of a part's reconstruction (SLOS_HOST_TIMING)
  // per-part collection (plan_all): each part's headers are copied on its stream
  // right after its reconstruction, so its compaction and D2H overlap later parts
  bool part_collect = false;
  // default records of every input (slos_workspace_records): uploaded only for the
  // workspace API; slos_plan_batch's pipeline and regrowth rounds do not read them
  bool records = true;
  int prio_shift = 0;  // pipeline workspaces after the first: streams this much lower
  std::vector<int32_t> ord;  // instance order: part p = ord[part_lo[p] .. part_lo[p+1])
  PinBuf h_hdr[kMaxParts], h_offs[kMaxParts];
  DevBuf d_packp[kMaxParts];
  cudaEvent_t ev_hdr[kMaxParts] = {nullptr}, ev_d2h[kMaxParts] = {nullptr};
  std::vector<Prep> prep;  // host preparation, reused across uploads
};

thread_local int64_t g_h2d = 0, g_d2h = 0;

bool host_timing() {
  static const bool on = std::getenv("SLOS_HOST_TIMING") != nullptr;
  return on;
}


// Host preparation + one H2D copy; the instances become device-resident.
int ws_upload(Ctx& c, Workspace& ws, slos_planner* const* planners, const slos_input* inputs,
              int unit_value, const std::vector<Job>& jobs, slos_result* outs, cudaStream_t stream) {
  ws.planners = planners;
  ws.inputs = inputs;
  ws.unit_value = unit_value;
  ws.jobs = jobs;
  ws.stream = stream ? stream : c.stream;
  ws.uploaded = false;
  ws.nv = 0;
  ws.valid.clear();
  const int n = (int)jobs.size();
  if (n == 0) return SLOS_OK;
  // ---- host preparation ----
  std::vector<Prep>& prep = ws.prep;  // reused: no per-instance heap traffic per call
  if (prep.size() < (size_t)n) prep.resize((size_t)n);
  std::vector<const slos_planner*> plist;
  std::vector<int> valid;
  int64_t TD = 0, TC = 0, TP = 0, TR = 0, TS = 0, TCd = 0, TM = 0, TW = 0, TSel = 0, TIds = 0, TB = 0, TE = 0;
  thread_local std::vector<Caps> caps_tl;  // lambdas below see it through the reference
  std::vector<Caps>& caps = caps_tl;  // per-call scratch kept across calls: large fresh
  caps.resize((size_t)n);                // vectors would page-fault on every call
  int maxN = 0, maxDec = 0, Lmax = 1;
  double S_need = 16;
  const auto t_a = std::chrono::steady_clock::now();
  if (host_timing()) { HostPool::get().runs = 0; HostPool::get().run_ms = 0.0; }
  // instances with hundreds of requests each: per-instance pieces, so a batch of a few
  // dozen (C4: 64 x 2,048 requests) still spreads over every core
  int grain = 16;
  if (n < 256) {  // (larger batches already make >= 16 pieces of 16)
    int64_t reqs = 0;
    for (int q = 0; q < n; ++q) reqs += (int64_t)inputs[jobs[q].k].n_running + inputs[jobs[q].k].n_pending;
    if (reqs >= 256 * (int64_t)n) grain = 1;
  }
  HostPool::get().run(n, [&](int lo, int hi) {
    for (int q = lo; q < hi; ++q) {
      const int k = jobs[q].k;
      Prep& pr = prep[q];
      pr.status = prep_instance(planners[k], &inputs[k], unit_value, pr);
      if (pr.status == SLOS_OK) caps[q] = estimate_caps(planners[k], &inputs[k], pr, jobs[q].grow);
    }
  }, grain);
  const auto t_a1 = std::chrono::steady_clock::now();
  // Totals over the valid instances: fixed chunks reduced in parallel and folded in
  // chunk order, so the valid list, the planner order (first appearance) and the
  // reported error (the last failing instance) are those of one serial pass.
  {
    struct Red {
      int64_t TD, TC, TP, TR, TS, TCd, TM, TW, TSel, TIds, TB, TE;
      int maxN, maxDec, Lmax, nvalid, last_bad, off;
      double S_need;
      std::vector<const slos_planner*> pl;  // distinct planners, first appearance
    };
    const int chunks = n < 4096 ? 1 : 256;
    thread_local std::vector<Red> red_tl;  // lambdas below see it through the reference
    std::vector<Red>& red = red_tl;
    red.resize((size_t)chunks);
    auto lo_of = [&](int ch) { return (int)((int64_t)ch * n / chunks); };
    auto reduce = [&](int ch) {
      Red& r = red[ch];
      r.TD = r.TC = r.TP = r.TR = r.TS = r.TCd = r.TM = r.TW = r.TSel = r.TIds = r.TB = r.TE = 0;
      r.maxN = 0; r.maxDec = 0; r.Lmax = 1; r.nvalid = 0; r.last_bad = -1; r.S_need = 16;
      r.pl.clear();
      for (int q = lo_of(ch); q < lo_of(ch + 1); ++q) {
        const int k = jobs[q].k;
        const slos_planner* P = planners[k];
        const Prep& pr = prep[q];
        if (pr.status != SLOS_OK) {
          std::memset(&outs[k], 0, sizeof(outs[k]));
          outs[k].status = pr.status;
          r.last_bad = q;
          continue;
        }
        if (r.pl.empty() || r.pl.back() != P) {
          bool seen = false;
          for (const slos_planner* x : r.pl) if (x == P) { seen = true; break; }
          if (!seen) r.pl.push_back(P);
        }
        ++r.nvalid;
        r.TD += pr.n_dec;
        r.TC += (pr.N + 1 + 3) & ~3;  // 16-byte aligned chain slices (the DP stages them by TMA)
        r.TP += pr.n_pre;
        r.TR += inputs[k].n_running;
        r.TS += caps[q].surv;
        r.TCd += caps[q].cand;
        r.TM += caps[q].memo;
        r.TW += (caps[q].work + 255) & ~(int64_t)255;
        r.TSel += pr.N + 1;
        r.TIds += 2 * (int64_t)inputs[k].n_pending + 1;
        r.TB += caps[q].batch;
        r.TE += caps[q].entry;
        r.maxN = std::max(r.maxN, pr.N);
        r.maxDec = std::max(r.maxDec, pr.n_dec);
        r.Lmax = std::max(r.Lmax, P->L);
        r.S_need = std::max(r.S_need, std::ceil(pr.span / P->tpot[0]) + 8);
      }
    };
    if (chunks == 1) reduce(0);
    else HostPool::get().run(chunks, [&](int c0, int c1) { for (int ch = c0; ch < c1; ++ch) reduce(ch); });
    int last_bad = -1, nvalid = 0;
    for (int ch = 0; ch < chunks; ++ch) {
      Red& r = red[ch];
      r.off = nvalid;
      nvalid += r.nvalid;
      if (r.last_bad >= 0) last_bad = r.last_bad;
      for (const slos_planner* P : r.pl) {
        bool seen = false;
        for (const slos_planner* x : plist) if (x == P) { seen = true; break; }
        if (!seen) plist.push_back(P);
      }
      TD += r.TD; TC += r.TC; TP += r.TP; TR += r.TR; TS += r.TS; TCd += r.TCd; TM += r.TM; TW += r.TW;
      TSel += r.TSel; TIds += r.TIds; TB += r.TB; TE += r.TE;
      maxN = std::max(maxN, r.maxN);
      maxDec = std::max(maxDec, r.maxDec);
      Lmax = std::max(Lmax, r.Lmax);
      S_need = std::max(S_need, r.S_need);
    }
    if (last_bad >= 0) g_err = prep[last_bad].why;  // on the calling thread
    valid.resize((size_t)nvalid);
    auto place = [&](int ch) {
      int x = red[ch].off;
      const slos_planner* lastP = nullptr;
      int lastpi = -1;
      for (int q = lo_of(ch); q < lo_of(ch + 1); ++q) {
        Prep& pr = prep[q];
        if (pr.status != SLOS_OK) continue;
        const slos_planner* P = planners[jobs[q].k];
        if (P != lastP) {
          lastP = P;
          for (size_t y = 0; y < plist.size(); ++y) if (plist[y] == P) { lastpi = (int)y; break; }
        }
        pr.planner = lastpi;
        valid[x++] = q;
      }
    };
    if (chunks == 1) place(0);
    else HostPool::get().run(chunks, [&](int c0, int c1) { for (int ch = c0; ch < c1; ++ch) place(ch); });
  }
  const auto t_b = std::chrono::steady_clock::now();
  const int nv = (int)valid.size();
  if (nv == 0) return SLOS_OK;
  const int Sc = (int)std::min<double>(S_need, 1 << 20);
  int64_t TA = 0, TT = 0, TPair = 0;  // anchor cache bytes, anchor tasks, pair records
  thread_local std::vector<int64_t> astride_tl;  // lambdas below see it through the reference
  std::vector<int64_t>& astride = astride_tl;
  astride.resize((size_t)n);
  {
    const int chunks = nv < 4096 ? 1 : 256;
    thread_local std::vector<std::array<int64_t, 3>> sums_tl;  // lambdas below see it through the reference
    std::vector<std::array<int64_t, 3>>& sums = sums_tl;
    sums.resize((size_t)chunks);
    auto body = [&](int ch) {
      int64_t a = 0, t = 0, pp = 0;
      for (int x = (int)((int64_t)ch * nv / chunks); x < (int)((int64_t)(ch + 1) * nv / chunks); ++x) {
        const int q = valid[x];
        const int N = prep[q].N;
        astride[q] = (int64_t)dp_anchor_stride(prep[q].n_dec, Sc, Lmax, N);
        a += astride[q] * (N + 1);
        t += N;
        pp += (int64_t)N * (N + 1) / 2;
      }
      sums[ch] = {a, t, pp};
    };
    if (chunks == 1) body(0);
    else HostPool::get().run(chunks, [&](int c0, int c1) { for (int ch = c0; ch < c1; ++ch) body(ch); });
    for (int ch = 0; ch < chunks; ++ch) { TA += sums[ch][0]; TT += sums[ch][1]; TPair += sums[ch][2]; }
  }
  const auto t_b1 = std::chrono::steady_clock::now();
  Layout& Ly = ws.Ly;
  Blob bi;
  Ly.planners = bi.add<PlannerDev>(plist.size());
  Ly.inst = bi.add<InstDev>(nv);
  Ly.order = bi.add<int32_t>(nv);
  Ly.atask = bi.add<int32_t>(2 * TT);
  Ly.pair = bi.add<uint8_t>(TPair);
  const size_t grec_hdr = dp_group_hdr_bytes();
  const size_t grec_stride = (grec_hdr + dp_group_stride(Sc, Lmax) + 127) & ~(size_t)127;
  Ly.dec_idx = bi.add<int32_t>(TD);
  Ly.dec_tier = bi.add<int32_t>(TD);
  Ly.dec_bytier = bi.add<int32_t>(TD);
  Ly.dec_next = bi.add<double>(TD);
  Ly.dec_backlog = bi.add<int64_t>(TD);
  Ly.dec_rem = bi.add<int64_t>(TD);
  Ly.ch_deadline = bi.add<double>(TC);
  Ly.ch_prefill = bi.add<int64_t>(TC);
  Ly.ch_tier = bi.add<int32_t>(TC);
  Ly.ch_memory = bi.add<int64_t>(TC);
  Ly.ch_value = bi.add<double>(TC);
  Ly.ch_forced = bi.add<int32_t>(TC);
  Ly.ch_ref = bi.add<int32_t>(TC);
  Ly.ch_floor = bi.add<int32_t>(TC);
  Ly.ch_suffix = bi.add<int64_t>(TC);
  Ly.pre_idx = bi.add<int32_t>(TP);
  Ly.pre_left = bi.add<int64_t>(TP);
  Ly.run_tier = bi.add<int32_t>(TR);
  Ly.recdef = ws.records ? bi.add<slos_record>(n) : 0;
  Ly.recmap = ws.records ? bi.add<int32_t>(nv) : 0;
  Ly.in_bytes = bi.bytes;
  Blob bs;
  Ly.s_counts = bs.add<uint64_t>(TS);
  Ly.s_mem = bs.add<int64_t>(TS);
  Ly.s_pb = bs.add<int64_t>(TS);
  Ly.s_value = bs.add<double>(TS);
  Ly.s_nadm = bs.add<int32_t>(TS);
  Ly.s_parent = bs.add<int32_t>(TS);
  Ly.s_arena = bs.add<int32_t>(TS);
  Ly.s_level = bs.add<int32_t>(TS);
  Ly.c_src = bs.add<int32_t>(TCd);
  Ly.c_j = bs.add<int32_t>(TCd);
  Ly.c_memo = bs.add<int32_t>(TCd);
  Ly.c_flag = bs.add<int32_t>(TCd);
  Ly.c_bucket = bs.add<int32_t>(TCd);
  Ly.c_pos = bs.add<int32_t>(TCd);
  Ly.c_aux = bs.add<int32_t>(TCd);
  Ly.c_counts = bs.add<uint64_t>(TCd);
  Ly.c_mem = bs.add<int64_t>(TCd);
  Ly.c_pb = bs.add<int64_t>(TCd);
  Ly.c_value = bs.add<double>(TCd);
  Ly.c_nadm = bs.add<int32_t>(TCd);
  Ly.c_bkey = bs.add<uint64_t>(2 * TCd);
  Ly.c_bval = bs.add<int32_t>(2 * TCd);
  Ly.memo = bs.add<MemoEnt>(TM);
  Ly.bq = bs.add<int32_t>(nv + 2 * kQueues);
  Ly.work = bs.add<unsigned char>(TW);
  Ly.anchors = bs.add<unsigned char>(TA);
  Ly.groups = bs.add<unsigned char>((size_t)TPair * grec_stride);
  Ly.s_sb = bs.add<int32_t>(TS);
  Ly.s_bcnt = bs.add<uint64_t>(TS);
  Ly.k_val = bs.add<int64_t>(TCd);
  Ly.ctime = bs.add<double>((size_t)nv * Lmax * Sc);
  Ly.ccnt = bs.add<int32_t>((size_t)nv * kMaxTiers);
  Ly.scr_bytes = bs.bytes;
  Blob bo;
  Ly.out = bo.add<OutHdr>(nv);
  Ly.sel = bo.add<int32_t>(TSel);
  Ly.ids = bo.add<int32_t>(TIds);
  Ly.batches = bo.add<slos_batch>(TB);
  Ly.entries = bo.add<slos_entry>(TE);
  Ly.out_bytes = bo.bytes;

  const auto t_b2 = std::chrono::steady_clock::now();
  cudaError_t e;
  if ((e = ws.h_in.ensure(Ly.in_bytes)) != cudaSuccess) return set_err(SLOS_ERR_CUDA, cudaGetErrorString(e));
  if ((e = ws.d_in.ensure(Ly.in_bytes)) != cudaSuccess) return set_err(SLOS_ERR_CUDA, cudaGetErrorString(e));
  if ((e = ws.d_scr.ensure(Ly.scr_bytes)) != cudaSuccess) return set_err(SLOS_ERR_CUDA, cudaGetErrorString(e));
  if ((e = ws.d_out.ensure(Ly.out_bytes)) != cudaSuccess) return set_err(SLOS_ERR_CUDA, cudaGetErrorString(e));
  const auto t_b3 = std::chrono::steady_clock::now();
  unsigned char* H = (unsigned char*)ws.h_in.p;
  auto hp = [&](size_t off) { return H + off; };
  PlannerDev* hP = (PlannerDev*)hp(Ly.planners);
  for (size_t x = 0; x < plist.size(); ++x) hP[x] = plist[x]->dev;
  InstDev* hI = (InstDev*)hp(Ly.inst);
  int32_t* h_dec_idx = (int32_t*)hp(Ly.dec_idx);
  int32_t* h_dec_tier = (int32_t*)hp(Ly.dec_tier);
  int32_t* h_dec_bytier = (int32_t*)hp(Ly.dec_bytier);
  double* h_dec_next = (double*)hp(Ly.dec_next);
  int64_t* h_dec_bl = (int64_t*)hp(Ly.dec_backlog);
  int64_t* h_dec_rem = (int64_t*)hp(Ly.dec_rem);
  double* h_dl = (double*)hp(Ly.ch_deadline);
  int64_t* h_pf = (int64_t*)hp(Ly.ch_prefill);
  int32_t* h_tr = (int32_t*)hp(Ly.ch_tier);
  int64_t* h_mm = (int64_t*)hp(Ly.ch_memory);
  double* h_vl = (double*)hp(Ly.ch_value);
  int32_t* h_fc = (int32_t*)hp(Ly.ch_forced);
  int32_t* h_rf = (int32_t*)hp(Ly.ch_ref);
  int32_t* h_fl = (int32_t*)hp(Ly.ch_floor);
  int64_t* h_sf = (int64_t*)hp(Ly.ch_suffix);
  int32_t* h_pre_idx = (int32_t*)hp(Ly.pre_idx);
  int64_t* h_pre_left = (int64_t*)hp(Ly.pre_left);
  int32_t* h_run_tier = (int32_t*)hp(Ly.run_tier);
  int n_small = 0;
  uint8_t* h_pair = (uint8_t*)hp(Ly.pair);
  thread_local std::vector<double> cost_tl;  // lambdas below see it through the reference
  std::vector<double>& cost = cost_tl;
  thread_local std::vector<uint8_t> kind_v_tl;  // lambdas below see it through the reference
  std::vector<uint8_t>& kind_v = kind_v_tl;  // compact copies for the serial ordering passes
  thread_local std::vector<int32_t> N_v_tl;  // lambdas below see it through the reference
  std::vector<int32_t>& N_v = N_v_tl;
  cost.resize((size_t)nv);
  kind_v.resize((size_t)nv);
  N_v.resize((size_t)nv);
  struct Off { int64_t D, C, P, R, S, Cd, M, W, Sel, Ids, B, E, A, Pair; };
  thread_local std::vector<Off> offs_tl;  // lambdas below see it through the reference
  std::vector<Off>& offs = offs_tl;
  offs.resize((size_t)nv);
  {
    // per-instance sizes and a chunk-local exclusive scan in parallel (the inputs are
    // scattered), the chunk bases folded in order, then the bases added in parallel
    auto add = [](Off& a, const Off& x) {
      a.D += x.D; a.C += x.C; a.P += x.P; a.R += x.R; a.S += x.S; a.Cd += x.Cd; a.M += x.M;
      a.W += x.W; a.Sel += x.Sel; a.Ids += x.Ids; a.B += x.B; a.E += x.E; a.A += x.A; a.Pair += x.Pair;
    };
    const int chunks = nv < 4096 ? 1 : 256;
    thread_local std::vector<Off> cbase_tl;  // lambdas below see it through the reference
    std::vector<Off>& cbase = cbase_tl;
    cbase.resize((size_t)chunks);
    auto lo_of = [&](int ch) { return (int)((int64_t)ch * nv / chunks); };
    auto sizes = [&](int ch) {
      Off acc{0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
      for (int v = lo_of(ch); v < lo_of(ch + 1); ++v) {
        const int q = valid[v];
        const Prep& pr = prep[q];
        const Caps& cp = caps[q];
        const slos_input* in = &inputs[jobs[q].k];
        Off x;
        x.D = pr.n_dec;
        x.C = (pr.N + 1 + 3) & ~3;
        x.P = pr.n_pre;
        x.R = in->n_running;
        x.S = cp.surv;
        x.Cd = cp.cand;
        x.M = cp.memo;
        x.W = (cp.work + 255) & ~(int64_t)255;
        x.Sel = pr.N + 1;
        x.Ids = 2 * (int64_t)in->n_pending + 1;
        x.B = cp.batch;
        x.E = cp.entry;
        x.A = astride[q] * (pr.N + 1);
        x.Pair = (int64_t)pr.N * (pr.N + 1) / 2;
        offs[v] = acc;
        add(acc, x);
      }
      cbase[ch] = acc;
    };
    if (chunks == 1) sizes(0);
    else HostPool::get().run(chunks, [&](int c0, int c1) { for (int ch = c0; ch < c1; ++ch) sizes(ch); });
    Off o{0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (int ch = 0; ch < chunks; ++ch) {
      const Off t = cbase[ch];
      cbase[ch] = o;
      add(o, t);
    }
    if (chunks > 1)
      HostPool::get().run(chunks, [&](int c0, int c1) {
        for (int ch = c0; ch < c1; ++ch)
          for (int v = lo_of(ch); v < lo_of(ch + 1); ++v) add(offs[v], cbase[ch]);
      });
  }
  const auto t_c = std::chrono::steady_clock::now();
  HostPool::get().run(nv, [&](int v_lo, int v_hi) {
  for (int v = v_lo; v < v_hi; ++v) {
    int64_t oD = offs[v].D, oC = offs[v].C, oP = offs[v].P, oR = offs[v].R, oS = offs[v].S, oCd = offs[v].Cd,
            oM = offs[v].M, oW = offs[v].W, oSel = offs[v].Sel, oIds = offs[v].Ids, oB = offs[v].B,
            oE = offs[v].E, oA = offs[v].A, oPair = offs[v].Pair;
    const int q = valid[v];
    const int k = jobs[q].k;
    const slos_input* in = &inputs[k];
    const Prep& pr = prep[q];
    const Caps& cp = caps[q];
    InstDev& I = hI[v];
    std::memset(&I, 0, sizeof I);
    I.now = in->now;
    I.tail_horizon = in->tail_horizon_s;
    I.mem_budget = in->memory_total - in->memory_standard_resident;
    I.planner = pr.planner;
    I.unit_value = unit_value;
    I.R_total = in->n_running;
    I.n_dec = pr.n_dec;
    I.N = pr.N;
    I.n_pre = pr.n_pre;
    I.n_pending = in->n_pending;
    I.last_forced = pr.last_forced;
    I.have_running_decode = pr.have_rd ? 1 : 0;
    I.values_integral = pr.values_integral ? 1 : 0;
    // A batch smaller than the SM count cannot fill the GPU: every instance gets the
    // widest reconstruction (256 threads) and admission DP (512 threads) for latency
    // (one C1 plan end to end 0.72 -> ~0.5 ms); larger batches pick by throughput.
    I.build_kind = pr.n_dec >= build_big_min_dec() ? 3
                   : latency_batch(nv)              ? 2
                   : (pr.n_dec <= build_warp_max_dec() ? 0 : 1);
    kind_v[v] = (uint8_t)I.build_kind;
    N_v[v] = pr.N;
    {  // direct bucket table when the count-vector space is small
      int64_t maxc[kMaxTiers] = {0};
      for (int x = 0; x < pr.N; ++x) {
        const int enc = pr.chain[x];
        const int t = enc >= 0 ? in->running[enc].decode_tier : in->pending[-enc - 1].decode_tier;
        if (t >= 0 && t < kMaxTiers) ++maxc[t];
      }
      const bool small = dp_small_enabled() &&
                         (double)(pr.n_dec + 8) * (double)(pr.N + 1) * (double)(pr.N + 1) < kSmallCost;
      const int dmax = small ? kDirectSmall : kDirectMax;
      int64_t D = 1;
      for (int l = 0; l < planners[k]->L && D <= dmax; ++l) {
        I.dstride[l] = (int32_t)D;
        D *= std::min<int64_t>(maxc[l], 250) + 1;
      }
      I.direct = D <= dmax ? 1 : 0;
    }
    I.off_dec = oD;
    I.off_chain = oC;
    I.off_pre = oP;
    I.off_run = oR;
    I.off_surv = oS; I.cap_surv = cp.surv;
    I.off_cand = oCd; I.cap_cand = cp.cand;
    I.off_memo = oM; I.cap_memo = cp.memo;
    I.off_sel = oSel;
    I.off_ids = oIds;
    I.off_batch = oB; I.cap_batch = cp.batch;
    I.off_entry = oE; I.cap_entry = cp.entry;
    I.off_work = oW; I.cap_work = cp.work;
    I.cap_gb = cp.gb;
    I.cap_go = cp.go;
    I.off_anchor = oA;
    I.anchor_stride = astride[q];
    I.off_pair = oPair;
    I.off_group = oPair * (int64_t)grec_stride;
    const int64_t oD0 = oD;
    for (int i = 0; i < in->n_running; ++i) {
      const slos_running& r = in->running[i];
      h_run_tier[oR + i] = r.decode_tier;
      if (r.prefill_remaining <= 0 && r.decode_remaining > 0) {
        h_dec_idx[oD] = i;
        h_dec_tier[oD] = r.decode_tier;
        h_dec_next[oD] = r.next_due_s;
        h_dec_bl[oD] = r.backlog;
        h_dec_rem[oD] = r.decode_remaining;
        ++oD;
      }
    }
    {  // decoders grouped by tier: a warp of the anchor due walk then walks lines of
       // one cadence (equal due counts) instead of the longest of mixed ones
      int32_t* bt = h_dec_bytier + oD0;
      int x = 0;
      const int nd = (int)(oD - oD0);
      for (int l = 0; l < kMaxTiers && x < nd; ++l)
        for (int k = 0; k < nd; ++k)
          if (h_dec_tier[oD0 + k] == l) bt[x++] = k;
      for (int k = 0; k < nd && x < nd; ++k)  // tiers outside [0, kMaxTiers) (rejected upstream)
        if (h_dec_tier[oD0 + k] < 0 || h_dec_tier[oD0 + k] >= kMaxTiers) bt[x++] = k;
    }
    for (int x = 0; x < pr.n_pre; ++x) {
      h_pre_idx[oP + x] = pr.pre[x];
      h_pre_left[oP + x] = in->running[pr.pre[x]].prefill_remaining;
    }
    int lf = -1;
    for (int x = 0; x < pr.N; ++x) {
      const int enc = pr.chain[x];
      const int64_t o = oC + x;
      h_fl[o] = lf;
      if (enc >= 0) {
        const slos_running& r = in->running[enc];
        h_dl[o] = r.prefill_deadline;
        h_pf[o] = r.prefill_remaining;
        h_tr[o] = r.decode_tier;
        h_mm[o] = 0;
        h_vl[o] = 0.0;
        h_fc[o] = 1;
        h_rf[o] = enc;
        lf = x;
      } else {
        const slos_pending& p = in->pending[-enc - 1];
        h_dl[o] = p.prefill_deadline;
        h_pf[o] = p.prefill_tokens;
        h_tr[o] = p.decode_tier;
        h_mm[o] = p.memory_units;
        h_vl[o] = unit_value ? 1.0 : p.value;
        h_fc[o] = 0;
        h_rf[o] = enc;
      }
    }
    {  // memo-key sharing per DP pair (j, i): the kernel's key (a_us, raw_us), or the
       // ms-quantised gap without running decoders (dp_scheduler.cpp:423-424,
       // batch_planner.cpp:411); a pair whose key no other pair has gets its own keys
      struct PK { uint64_t k0, k1; int64_t idx; };
      std::vector<PK> keys;
      uint8_t* hpair = h_pair + oPair;
      std::memset(hpair, 0, (size_t)pr.N * (pr.N + 1) / 2);
      for (int i = 0; i < pr.N; ++i) {
        for (int j = h_fl[oC + i]; j < i; ++j) {
          const double a = j < 0 ? in->now : h_dl[oC + j];
          const double d = h_dl[oC + i] - a;
          const double raw = (0.0 < d) ? d : 0.0;
          PK k;
          if (pr.have_rd) {
            k.k0 = (uint64_t)std::llround(a * 1e6);
            k.k1 = (uint64_t)std::llround(raw * 1e6);
          } else {
            const double gap = host_quantize_gap(host_quantize_gap(raw));
            k.k0 = 0xFFFFFFFFFFFFFFFFULL;
            k.k1 = (uint64_t)std::llround(gap * 1000.0);
          }
          k.idx = pair_index(pr.N, j + 1, i);
          keys.push_back(k);
        }
      }
      std::sort(keys.begin(), keys.end(), [](const PK& x, const PK& y) {
        return x.k0 != y.k0 ? x.k0 < y.k0 : x.k1 < y.k1;
      });
      for (size_t x = 0; x < keys.size();) {
        size_t y = x + 1;
        while (y < keys.size() && keys[y].k0 == keys[x].k0 && keys[y].k1 == keys[x].k1) ++y;
        if (y - x > 1) {
          for (size_t z = x; z < y; ++z) hpair[keys[z].idx] = 1;
          I.has_shared = 1;
        }
        x = y;
      }
    }
    h_sf[oC + pr.N] = 0;
    for (int x = pr.N - 1; x >= 0; --x) h_sf[oC + x] = h_sf[oC + x + 1] + h_pf[oC + x];
    cost[v] = (double)(pr.n_dec + 8) * (double)(pr.N + 1) * (double)(pr.N + 1);
  }
  }, grain);
  const auto t_d = std::chrono::steady_clock::now();
  auto t_d1 = t_d, t_d2 = t_d;
  int32_t* h_order = (int32_t*)hp(Ly.order);
  {
    // launch order, heaviest first (load balance only: results do not depend on it).
    // Large batches bucket by log2(cost) instead of sorting (O(n), stable).
    thread_local std::vector<int32_t> ord_tl;  // lambdas below see it through the reference
    std::vector<int32_t>& ord = ord_tl;
    ord.resize((size_t)nv);
    if (nv <= 4096) {
      for (int v = 0; v < nv; ++v) ord[v] = v;
      std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return cost[a] > cost[b]; });
    } else {
      constexpr int kB = 64;
      thread_local std::vector<uint8_t> key_tl;
      std::vector<uint8_t>& key = key_tl;
      key.resize((size_t)nv);
      // stable counting sort over fixed chunks: per-chunk histograms in parallel,
      // positions by (bucket, chunk), scatter in parallel (each chunk in order)
      constexpr int kCh = 128;
      thread_local std::vector<std::array<int, kB>> hist_tl;  // lambdas below see it through the reference
      std::vector<std::array<int, kB>>& hist = hist_tl;
      hist.resize(kCh);
      auto clo = [&](int ch) { return (int)((int64_t)ch * nv / kCh); };
      HostPool::get().run(kCh, [&](int c0, int c1) {
        for (int ch = c0; ch < c1; ++ch) {
          std::array<int, kB>& h = hist[ch];
          h.fill(0);
          for (int v = clo(ch); v < clo(ch + 1); ++v) {
            const int e = std::min(kB - 1, std::max(0, std::ilogb(std::max(1.0, cost[v]))));
            key[v] = (uint8_t)(kB - 1 - e);
            ++h[key[v]];
          }
        }
      });
      int run = 0;
      for (int b = 0; b < kB; ++b)
        for (int ch = 0; ch < kCh; ++ch) {
          const int x = hist[ch][b];
          hist[ch][b] = run;
          run += x;
        }
      HostPool::get().run(kCh, [&](int c0, int c1) {
        for (int ch = c0; ch < c1; ++ch) {
          std::array<int, kB>& h = hist[ch];
          for (int v = clo(ch); v < clo(ch + 1); ++v) ord[h[key[v]]++] = v;
        }
      });
    }
    std::memcpy(h_order, ord.data(), sizeof(int32_t) * (size_t)nv);
    ws.ord.assign(ord.begin(), ord.end());
    t_d1 = std::chrono::steady_clock::now();
    // solve parts: contiguous ranges of the cost-descending order (every part gets
    // a share of the heavy instances); each part's DP and reconstruction are
    // launched on their own stream so one part's reconstruction overlaps the next
    // part's DP (ws_solve)
    const int P = solve_parts(nv);
    ws.n_parts = P;
    int qcount[kQueues] = {0};
    for (int p = 0; p <= P; ++p) ws.part_lo[p] = (int)((int64_t)p * nv / P);
    // the small instances are a suffix of each part (cost-descending order; the
    // bucketed order keys on ilogb(cost) and kSmallCost is a power of two)
    // (cost is non-increasing along the order at power-of-two thresholds, so both
    // boundaries are partition points: binary searches instead of scans of the part)
    auto first_where = [&](int lo, int hi, auto pred) {  // first x in [lo, hi) with pred(x), else hi
      while (lo < hi) {
        const int mid = lo + (hi - lo) / 2;
        if (pred(mid)) hi = mid; else lo = mid + 1;
      }
      return lo;
    };
    for (int p = 0; p < P; ++p) {
      int x = ws.part_lo[p + 1];
      if (dp_small_enabled())
        x = first_where(ws.part_lo[p], x, [&](int z) { return cost[ord[z]] < kSmallCost; });
      ws.small_lo[p] = x;
      int y = ws.part_lo[p];
      const double big_thr = latency_batch(nv) ? 0.0 : dp_big_cost();
      if (big_thr > 0 || latency_batch(nv))
        y = first_where(y, x, [&](int z) { return !(cost[ord[z]] >= big_thr); });
      ws.big_hi[p] = y;
    }
    // chain lengths per chunk of the order (the anchor-task scan below), summed in the
    // same pass as the queue sizes
    constexpr int kOrdCh = 128;
    thread_local std::vector<int64_t> cs_tl;  // lambdas below see it through the reference
    std::vector<int64_t>& cs = cs_tl;
    cs.resize(kOrdCh + 1);
    {  // queue sizes (per part and reconstruction kind) and each instance's part, over
       // fixed chunks of the order in parallel
      constexpr int kCh = kOrdCh;
      thread_local std::vector<std::array<int, kQueues>> qc_tl;  // lambdas below see it through the reference
      std::vector<std::array<int, kQueues>>& qc = qc_tl;
      qc.resize(kCh);
      auto clo = [&](int ch) { return (int)((int64_t)ch * nv / kCh); };
      auto body = [&](int ch) {
        std::array<int, kQueues>& c = qc[ch];
        c.fill(0);
        int p = 0;
        int64_t a = 0;
        for (int x = clo(ch); x < clo(ch + 1); ++x) {
          while (x >= ws.part_lo[p + 1]) ++p;
          const int v = ord[x];
          hI[v].part = p;
          ++c[kBuildKinds * p + kind_v[v]];
          a += N_v[v];
        }
        cs[ch + 1] = a;
      };
      if (nv < 4096) { for (int ch = 0; ch < kCh; ++ch) body(ch); }
      else HostPool::get().run(kCh, [&](int c0, int c1) { for (int ch = c0; ch < c1; ++ch) body(ch); });
      for (int ch = 0; ch < kCh; ++ch)
        for (int q = 0; q < kQueues; ++q) qcount[q] += qc[ch][q];
    }
    int qb = 2 * kQueues;  // the counters come first
    for (int q = 0; q < kQueues; ++q) {
      ws.qbase[q] = qb;
      ws.qn[q] = qcount[q];
      qb += qcount[q];
    }
    // anchor tasks (instance, anchor j), j = -1 .. N-2, grouped by solve part so each
    // part's anchor/group kernels run on its own stream ahead of its DP
    t_d2 = std::chrono::steady_clock::now();
    int32_t* t = (int32_t*)hp(Ly.atask);
    thread_local std::vector<int64_t> aoff_tl;  // lambdas below see it through the reference
    std::vector<int64_t>& aoff = aoff_tl;  // first task of the instance at order position y
    aoff.resize((size_t)nv + 1);
    {  // exclusive scan of the chain lengths in launch order (chunk sums from the pass
       // above), each chunk then writing its offsets and its anchor tasks
      constexpr int kCh = kOrdCh;
      auto clo = [&](int ch) { return (int)((int64_t)ch * nv / kCh); };
      auto fill = [&](int ch) {
        int64_t a = cs[ch];
        for (int y = clo(ch); y < clo(ch + 1); ++y) {
          const int v = ord[y];
          aoff[y] = a;
          for (int j = -1; j < N_v[v] - 1; ++j, ++a) { t[2 * a] = v; t[2 * a + 1] = j; }
        }
      };
      cs[0] = 0;
      for (int ch = 0; ch < kCh; ++ch) cs[ch + 1] += cs[ch];
      if (nv >= 4096) HostPool::get().run(kCh, [&](int c0, int c1) { for (int ch = c0; ch < c1; ++ch) fill(ch); });
      else for (int ch = 0; ch < kCh; ++ch) fill(ch);
      aoff[nv] = cs[kCh];
    }
    for (int p = 0; p <= P; ++p) ws.atask_lo[p] = (int)aoff[ws.part_lo[p]];
    for (int p = 0; p < P; ++p) ws.atask_big[p] = (int)aoff[ws.big_hi[p]];
    Ly.n_atask = aoff[nv];
  }
  if (ws.records) {
    slos_record* rd = (slos_record*)hp(Ly.recdef);
    HostPool::get().run(n, [&](int lo, int hi) {
      std::memset(rd + lo, 0, sizeof(slos_record) * (size_t)(hi - lo));
      for (int q = lo; q < hi; ++q) rd[q].status = prep[q].status;
    });
    int32_t* rm = (int32_t*)hp(Ly.recmap);
    std::memcpy(rm, valid.data(), sizeof(int32_t) * (size_t)nv);
  }
  const auto t_e = std::chrono::steady_clock::now();
  ws.n_total = n;
  g_h2d += (int64_t)Ly.in_bytes;
  // ---- device pipeline ----
  unsigned char* DI = (unsigned char*)ws.d_in.p;
  unsigned char* DS = (unsigned char*)ws.d_scr.p;
  unsigned char* DO = (unsigned char*)ws.d_out.p;
  cudaStream_t s = ws.stream;
  cudaMemcpyAsync(DI, H, Ly.in_bytes, cudaMemcpyHostToDevice, s);
  if (std::getenv("SLOS_HOST_TIMING")) {
    const auto t_f = std::chrono::steady_clock::now();
    auto ms = [](std::chrono::steady_clock::time_point x, std::chrono::steady_clock::time_point y) {
      return std::chrono::duration<double, std::milli>(y - x).count();
    };
    std::fprintf(stderr, "[slos upload] n %d: prep run %.3f totals loop %.3f | order sort %.3f parts %.3f tasks+rec %.3f\n", n,
                 ms(t_a, t_a1), ms(t_a1, t_b), ms(t_d, t_d1), ms(t_d1, t_d2), ms(t_d2, t_e));
    std::fprintf(stderr, "[slos upload] n %d: prep %.3f, totals %.3f, layout %.3f (strides %.3f blobs %.3f ensure %.3f), fill %.3f, order/parts %.3f, h2d %.3f ms; host pool %d runs %.3f ms\n",
                 n, ms(t_a, t_b), 0.0, ms(t_b, t_c), ms(t_b, t_b1), ms(t_b1, t_b2), ms(t_b2, t_b3), ms(t_c, t_d),
                 ms(t_d, t_e), ms(t_e, t_f), HostPool::get().runs, HostPool::get().run_ms);
    HostPool::get().runs = 0;
    HostPool::get().run_ms = 0.0;
  }
  Ly.memo_bytes = sizeof(MemoEnt) * (size_t)TM;
  Ly.bkey_bytes = sizeof(uint64_t) * 2 * (size_t)TCd;
  Ly.bval_bytes = sizeof(int32_t) * 2 * (size_t)TCd;
  BatchArgs& A = ws.A;
  std::memset(&A, 0, sizeof A);
  A.planners = (const PlannerDev*)(DI + Ly.planners);
  A.inst = (const InstDev*)(DI + Ly.inst);
  A.order = (const int32_t*)(DI + Ly.order);
  A.atask = (const int32_t*)(DI + Ly.atask);
  A.n_atask = (int32_t)Ly.n_atask;
  A.n_inst = nv;
  {  // reconstruction queues split by planner kind when both are present (below)
    bool any_spec = false, any_ar = false;
    for (const slos_planner* pl : plist) (pl->dev.speculative ? any_spec : any_ar) = true;
    A.mixed_spec = any_spec && any_ar ? 1 : 0;
  }
  A.dec_idx = (const int32_t*)(DI + Ly.dec_idx);
  A.dec_tier = (const int32_t*)(DI + Ly.dec_tier);
  A.dec_bytier = (const int32_t*)(DI + Ly.dec_bytier);
  A.dec_next = (const double*)(DI + Ly.dec_next);
  A.dec_backlog = (const int64_t*)(DI + Ly.dec_backlog);
  A.dec_rem = (const int64_t*)(DI + Ly.dec_rem);
  A.ch_deadline = (const double*)(DI + Ly.ch_deadline);
  A.ch_prefill = (const int64_t*)(DI + Ly.ch_prefill);
  A.ch_tier = (const int32_t*)(DI + Ly.ch_tier);
  A.ch_memory = (const int64_t*)(DI + Ly.ch_memory);
  A.ch_value = (const double*)(DI + Ly.ch_value);
  A.ch_forced = (const int32_t*)(DI + Ly.ch_forced);
  A.ch_ref = (const int32_t*)(DI + Ly.ch_ref);
  A.ch_floor = (const int32_t*)(DI + Ly.ch_floor);
  A.ch_suffix = (const int64_t*)(DI + Ly.ch_suffix);
  A.pre_idx = (const int32_t*)(DI + Ly.pre_idx);
  A.pre_left = (const int64_t*)(DI + Ly.pre_left);
  A.run_tier = (const int32_t*)(DI + Ly.run_tier);
  A.s_counts = (uint64_t*)(DS + Ly.s_counts);
  A.s_mem = (int64_t*)(DS + Ly.s_mem);
  A.s_pb = (int64_t*)(DS + Ly.s_pb);
  A.s_value = (double*)(DS + Ly.s_value);
  A.s_nadm = (int32_t*)(DS + Ly.s_nadm);
  A.s_parent = (int32_t*)(DS + Ly.s_parent);
  A.s_arena = (int32_t*)(DS + Ly.s_arena);
  A.s_level = (int32_t*)(DS + Ly.s_level);
  A.c_src = (int32_t*)(DS + Ly.c_src);
  A.c_j = (int32_t*)(DS + Ly.c_j);
  A.c_memo = (int32_t*)(DS + Ly.c_memo);
  A.c_flag = (int32_t*)(DS + Ly.c_flag);
  A.c_bucket = (int32_t*)(DS + Ly.c_bucket);
  A.c_pos = (int32_t*)(DS + Ly.c_pos);
  A.c_aux = (int32_t*)(DS + Ly.c_aux);
  A.c_counts = (uint64_t*)(DS + Ly.c_counts);
  A.c_mem = (int64_t*)(DS + Ly.c_mem);
  A.c_pb = (int64_t*)(DS + Ly.c_pb);
  A.c_value = (double*)(DS + Ly.c_value);
  A.c_nadm = (int32_t*)(DS + Ly.c_nadm);
  A.c_bkey = (uint64_t*)(DS + Ly.c_bkey);
  A.c_bval = (int32_t*)(DS + Ly.c_bval);
  A.memo = (MemoEnt*)(DS + Ly.memo);
  A.work = DS + Ly.work;
  A.anchors = DS + Ly.anchors;
  A.pair_shared = (const uint8_t*)(DI + Ly.pair);
  A.groups = DS + Ly.groups;
  A.s_sb = (int32_t*)(DS + Ly.s_sb);
  A.s_bcnt = (uint64_t*)(DS + Ly.s_bcnt);
  A.k_val = (int64_t*)(DS + Ly.k_val);
  A.ctime = (double*)(DS + Ly.ctime);
  A.ccnt = (int32_t*)(DS + Ly.ccnt);
  A.bq = (int32_t*)(DS + Ly.bq);
  for (int q = 0; q < kQueues; ++q) { A.qbase[q] = ws.qbase[q]; A.qn[q] = ws.qn[q]; }
  (void)n_small;
  A.out = (OutHdr*)(DO + Ly.out);
  A.sel = (int32_t*)(DO + Ly.sel);
  A.ids = (int32_t*)(DO + Ly.ids);
  A.batches = (slos_batch*)(DO + Ly.batches);
  A.entries = (slos_entry*)(DO + Ly.entries);

  DpParams& dp = ws.dp;
  dp.a = A;
  dp.Lmax = Lmax;
  dp.Sc = Sc;
  const size_t stride = dp_warp_scr_stride(dp.Sc, Lmax);
  dp.wscr_stride = stride;
  // 4 CTAs of 256 threads per SM (64 registers/thread, SLOS_DP_MIN_BLOCKS)
  // dynamic shared memory cap per CTA (SLOS_DP_SMEM_KB overrides). Staging the
  // decoders (read only by the rare warp fallback) costs a CTA per SM at C2 sizes,
  // so it is off unless SLOS_DP_STAGE_DEC=1.
  static const size_t kSmemBudget = [] {
    const char* e = std::getenv("SLOS_DP_SMEM_KB");
    return (size_t)(e ? std::atoi(e) : 74) * 1024;
  }();
  static const bool kStageDec = [] {
    const char* e = std::getenv("SLOS_DP_STAGE_DEC");
    return e ? std::atoi(e) != 0 : false;
  }();
  dp.grec_hdr = grec_hdr;
  dp.grec_stride = grec_stride;
  dp.grec_stage = (grec_hdr + dp_group_eval_bytes(Sc, Lmax) + 15) & ~(size_t)15;
  ws.any_big = false;
  for (int p = 0; p < ws.n_parts; ++p) ws.any_big = ws.any_big || ws.big_hi[p] > ws.part_lo[p];
  dp.wscr_warps = ws.any_big ? kDpMaxWarpsHost : 8;
  if ((e = ws.d_wscr.ensure(stride * (size_t)dp.wscr_warps * (size_t)nv)) != cudaSuccess)
    return set_err(SLOS_ERR_CUDA, cudaGetErrorString(e));
  dp.wscr_global = (unsigned char*)ws.d_wscr.p;
  size_t& smem = ws.smem;
  // candidates per level kept in shared memory (SLOS_DP_TSM overrides). Bigger is
  // not better: what the 4 resident CTAs leave of the SM's 228 KB stays L1 for the
  // HBM scratch (survivors, group records, larger levels). Measured on C2 x 1024:
  // dp_kernel 1.81 ms at 192, 1.87 at 256, 2.07 at 512 (3 CTAs), 2.39 at 640.
  static const int kTsm = [] {
    const char* e = std::getenv("SLOS_DP_TSM");
    return e ? std::atoi(e) : 192;
  }();
  dp.Tsm = kTsm;
  dp.dtab = kDirectMax;
  auto fit = [&](int dec) { return dp_smem_bytes(maxN, dec, dp.Sc, Lmax, dp.Tsm, &dp.overlay_bytes, dp.dtab); };
  while (fit(0) > kSmemBudget && dp.Tsm > 64) {
    if (dp.Tsm > 256) dp.Tsm -= 32;
    else dp.Tsm /= 2;
  }
  smem = fit(0);
  dp.phase_cycles = nullptr;
  if (std::getenv("SLOS_PHASE_TIMING")) {
    static unsigned long long* dev_pc = nullptr;
    if (!dev_pc) {
      cudaMalloc(&dev_pc, 32 * sizeof(unsigned long long));
      cudaMemset(dev_pc, 0, 32 * sizeof(unsigned long long));
    }
    dp.phase_cycles = dev_pc;
  }
  dp.dec_smem_max = 0;
  if (kStageDec && fit(maxDec) <= kSmemBudget) dp.dec_smem_max = maxDec;
  smem = fit(dp.dec_smem_max);
  {  // dp_kernel_small: 64 threads, 16 CTAs per SM -> ~13 KB of shared memory each
    DpParams& ds = ws.dp_small;
    ds = dp;
    ds.dec_smem_max = 0;
    ds.dtab = kDirectSmall;
    static const int kTsmSmall = [] {
      const char* e = std::getenv("SLOS_DP_SMALL_TSM");
      return e ? std::atoi(e) : 48;
    }();
    ds.Tsm = kTsmSmall;
    ws.smem_small = dp_smem_bytes(std::min(maxN, kDpSmallMaxChainHost), 0, ds.Sc, Lmax, ds.Tsm, &ds.overlay_bytes,
                                  ds.dtab, true);
  }
  {  // dp_kernel_big: one 512-thread CTA per SM, so a large level stays on chip
    DpParams& db = ws.dp_big;
    db = dp;
    db.dec_smem_max = 0;
    static const int kTsmBig = [] {
      const char* e = std::getenv("SLOS_DP_BIG_TSM");
      return e ? std::atoi(e) : 1024;
    }();
    static const size_t kSmemBig = [] {
      const char* e = std::getenv("SLOS_DP_BIG_SMEM_KB");
      return (size_t)(e ? std::atoi(e) : 200) * 1024;
    }();
    db.Tsm = kTsmBig;
    auto fitb = [&] { return dp_smem_bytes(maxN, 0, db.Sc, Lmax, db.Tsm, &db.overlay_bytes, db.dtab, 2); };
    while (fitb() > std::min(kSmemBig, (size_t)c.smem_optin) && db.Tsm > 64) db.Tsm -= 64;
    ws.smem_big = fitb();
  }
  ws.anchor_smem = anchor_smem_bytes(maxN, dp.Sc, Lmax, &dp.anchor_scr_bytes);
  if (S_need > (double)(1 << 20) || smem > c.smem_optin || ws.anchor_smem > c.smem_optin ||
      (ws.any_big && ws.smem_big > c.smem_optin)) {
    // the slot grid of the widest deadline span does not fit a CTA's shared memory;
    // plan_all solves wide instances in their own slot classes, so only an instance
    // that alone exceeds it lands here (per-instance SLOS_ERR_RANGE, never a launch failure)
    ws.uploaded = false;
    ws.nv = 0;
    return set_err(SLOS_ERR_RANGE, "deadline span needs a slot grid of " + std::to_string((int64_t)S_need) +
                                       " slots, more than a CTA's shared memory holds");
  }
  ws.maxN = maxN;
  ws.valid = valid;
  ws.nv = nv;
  ws.uploaded = true;
  return SLOS_OK;
}

// Enqueue the kernel pipeline on the device-resident batch (no host sync).
int ws_solve(Workspace& ws, cudaStream_t stream) {
  if (!ws.uploaded || ws.nv == 0) return SLOS_OK;
  const cudaStream_t s = stream ? stream : ws.stream;
  const int nv = ws.nv;
  DpParams& dp = ws.dp;
  const size_t smem = ws.smem;
  unsigned char* DS = (unsigned char*)ws.d_scr.p;
  unsigned char* DO = (unsigned char*)ws.d_out.p;
  const Layout& Ly = ws.Ly;
  // scratch init is part of every solve (memo tables, bucket hashes, headers)
  for (int k = 0; k < 4; ++k)
    if (!ws.ev[k]) cudaEventCreate(&ws.ev[k]);
  cudaEventRecord(ws.ev[1], s);  // start of the solve (scratch init), stage_ms[3]
  if (host_timing())
    std::fprintf(stderr, "[slos solve] nv %d: memset memo %.1f MB, bkey %.1f MB, bval %.1f MB, hdr %.1f MB\n", nv,
                 Ly.memo_bytes / 1e6, Ly.bkey_bytes / 1e6, Ly.bval_bytes / 1e6, sizeof(OutHdr) * (double)nv / 1e6);
  // (the memo tables and HBM bucket hashes are cleared by dp_kernel, per instance
  // and only when used: a batch-wide memset wrote GBs for small instances)
  cudaMemsetAsync(DO + Ly.out, 0, sizeof(OutHdr) * nv, s);
  cudaMemsetAsync(DS + Ly.bq, 0, 2 * kQueues * sizeof(int32_t), s);
  cudaError_t e;
  if (!ws.ev_fork) {
    cudaEventCreateWithFlags(&ws.ev_fork, cudaEventDisableTiming);
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    // (SLOS_ANCHOR_PRIO_LOW: anchor/group kernels below the parts' DP and reconstruction)
    cudaStreamCreateWithPriority(&ws.astream, cudaStreamNonBlocking,
                                 std::getenv("SLOS_ANCHOR_PRIO_LOW") ? lo : std::min(lo, hi + ws.prio_shift));
    static const bool rev = std::getenv("SLOS_PART_PRIO_REV") != nullptr;
    for (int p = 0; p < kMaxParts; ++p) {
      cudaStreamCreateWithPriority(&ws.pstream[p], cudaStreamNonBlocking,
                                   rev ? std::max(hi + 1, lo - p) : std::min(lo, hi + 1 + p + ws.prio_shift));
      cudaEventCreate(&ws.ev_bend[p]);
      cudaEventCreate(&ws.ev_dp[p]);
      cudaEventCreate(&ws.ev_anc[p]);
      cudaEventCreateWithFlags(&ws.ev_join[p], cudaEventDisableTiming);
    }
  }
  cudaEventRecord(ws.ev[0], s);
  cudaEventRecord(ws.ev_fork, s);
  ws.launches = 0;  // kernels this solve launches (slos_workspace_launches)
  for (int p = 0; p < ws.n_parts; ++p) {
    const int nt = ws.atask_lo[p + 1] - ws.atask_lo[p];
    ws.launches += (ws.atask_big[p] > ws.atask_lo[p]) + (ws.atask_lo[p + 1] > ws.atask_big[p]) +
                   (nt > 0 && ws.maxN > 0) + (ws.big_hi[p] > ws.part_lo[p]) + (ws.small_lo[p] > ws.big_hi[p]) +
                   (ws.part_lo[p + 1] > ws.small_lo[p]);
    for (int kd = 0; kd < kBuildKinds; ++kd) ws.launches += ws.qn[kBuildKinds * p + kd] > 0;
  }
  BuildParams bp;
  bp.a = ws.A;
  // per-gap working set per CTA (SLOS_BUILD_SMEM_KB). Measured C2 x 1024 with 4
  // CTAs per SM (128 registers): build stage 0.69 ms at 44 KB, 0.61 at 32, 0.57 at
  // 24, 1.03 at 16 (gaps spill to HBM); at 3 CTAs per SM (168 registers) 0.81-0.83.
  static const size_t kBuildSmem = [] {
    const char* e = std::getenv("SLOS_BUILD_SMEM_KB");
    return (size_t)(e ? std::atoi(e) : 24) * 1024;
  }();
  bp.smem_bytes = kBuildSmem;
  static const size_t kBuildSmemBig = [] {  // build_kernel_big (SLOS_BUILD_BIG_SMEM_KB)
    const char* e = std::getenv("SLOS_BUILD_BIG_SMEM_KB");
    return (size_t)(e ? std::atoi(e) : 44) * 1024;
  }();
  bp.smem_big = kBuildSmemBig;
  static const size_t kBuildSmemWarp = [] {  // per CTA of 4 warp-built instances (SLOS_BUILD_WARP_SMEM_KB)
    const char* e = std::getenv("SLOS_BUILD_WARP_SMEM_KB");
    return (size_t)(e ? std::atoi(e) : 16) * 1024;
  }();
  bp.smem_warp = kBuildSmemWarp;
  bp.phase_cycles = dp.phase_cycles ? dp.phase_cycles + 16 : nullptr;
  // per part: admission DP, then its plan reconstruction, on the part's stream;
  // part p's reconstruction runs while part p+1's DP still occupies SMs
  // anchor caches and pair groups of every part, in part order, on the highest-
  // priority stream (throughput kernels: they fill the SMs the latency-bound DP
  // leaves idle and put each part's DP on its critical path as early as possible)
  cudaStreamWaitEvent(ws.astream, ws.ev_fork, 0);
  for (int p = 0; p < ws.n_parts; ++p) {
    DpParams dpa = dp;
    const int nt = ws.atask_lo[p + 1] - ws.atask_lo[p];
    // anchors of the big-instance prefix on 512-thread CTAs, the rest on 128
    dpa.task0 = ws.atask_lo[p];
    if ((e = launch_anchor(dpa, ws.atask_big[p] - ws.atask_lo[p], ws.anchor_smem, ws.astream, true)) != cudaSuccess)
      return set_err(SLOS_ERR_CUDA, cudaGetErrorString(e));
    dpa.task0 = ws.atask_big[p];
    if ((e = launch_anchor(dpa, ws.atask_lo[p + 1] - ws.atask_big[p], ws.anchor_smem, ws.astream)) != cudaSuccess)
      return set_err(SLOS_ERR_CUDA, cudaGetErrorString(e));
    dpa.task0 = ws.atask_lo[p];
    if ((e = launch_group(dpa, nt, ws.maxN, ws.astream)) != cudaSuccess)
      return set_err(SLOS_ERR_CUDA, cudaGetErrorString(e));
    cudaEventRecord(ws.ev_anc[p], ws.astream);
  }
  for (int p = 0; p < ws.n_parts; ++p) {
    const cudaStream_t sp = ws.pstream[p];
    cudaStreamWaitEvent(sp, ws.ev_anc[p], 0);
    DpParams dpb = ws.dp_big;
    dpb.blk0 = ws.part_lo[p];
    if ((e = launch_dp(dpb, ws.big_hi[p] - ws.part_lo[p], ws.smem_big, sp, 2)) != cudaSuccess)
      return set_err(SLOS_ERR_CUDA, cudaGetErrorString(e));
    DpParams dpp = dp;
    dpp.blk0 = ws.big_hi[p];
    if ((e = launch_dp(dpp, ws.small_lo[p] - ws.big_hi[p], smem, sp)) != cudaSuccess)
      return set_err(SLOS_ERR_CUDA, cudaGetErrorString(e));
    DpParams dps = ws.dp_small;
    dps.blk0 = ws.small_lo[p];
    dps.task0 = dpp.task0;
    if ((e = launch_dp(dps, ws.part_lo[p + 1] - ws.small_lo[p], ws.smem_small, sp, 1)) != cudaSuccess)
      return set_err(SLOS_ERR_CUDA, cudaGetErrorString(e));
    cudaEventRecord(ws.ev_dp[p], sp);
    bp.part = p;
    static const bool build_after_next = std::getenv("SLOS_BUILD_AFTER_NEXT_ANC") != nullptr;
    if (build_after_next && p + 1 < ws.n_parts) cudaStreamWaitEvent(sp, ws.ev_anc[p + 1], 0);
    const int q0 = kBuildKinds * p;
    if ((e = launch_build(bp, ws.qn[q0], ws.qn[q0 + 1], ws.qn[q0 + 2], ws.qn[q0 + 3], sp)) != cudaSuccess)
      return set_err(SLOS_ERR_CUDA, cudaGetErrorString(e));
    if (ws.part_collect) {  // this part's headers, as soon as its reconstruction ends
      if ((e = ws.h_hdr[p].ensure(sizeof(OutHdr) * nv)) != cudaSuccess) return set_err(SLOS_ERR_CUDA, cudaGetErrorString(e));
      if (!ws.ev_hdr[p]) cudaEventCreateWithFlags(&ws.ev_hdr[p], cudaEventDisableTiming);
      cudaMemcpyAsync(ws.h_hdr[p].p, DO + Ly.out, sizeof(OutHdr) * nv, cudaMemcpyDeviceToHost, sp);
      cudaEventRecord(ws.ev_hdr[p], sp);
    }
    if (host_timing()) cudaEventRecord(ws.ev_bend[p], sp);
    cudaEventRecord(ws.ev_join[p], sp);
    cudaStreamWaitEvent(s, ws.ev_join[p], 0);
  }
  cudaEventRecord(ws.ev[2], s);
  ws.solved = true;
  return SLOS_OK;
}

// end of the admission DP over all parts (ms after ev[0])
float dp_end_ms(Workspace& ws) {
  float t = 0.0f;
  for (int p = 0; p < ws.n_parts; ++p) {
    float x = 0.0f;
    cudaEventElapsedTime(&x, ws.ev[0], ws.ev_dp[p]);
    t = std::max(t, x);
  }
  return t;
}

void print_phase_debug(Workspace& ws, const std::vector<OutHdr>& hdr) {
  const int nv = ws.nv;
  const std::vector<int>& valid = ws.valid;
  const std::vector<Job>& jobs = ws.jobs;
  {
    unsigned long long pc[32];
    cudaMemcpy(pc, ws.dp.phase_cycles, sizeof pc, cudaMemcpyDeviceToHost);
    unsigned long long tot = 0;
    for (int k = 0; k < 14; ++k) tot += pc[k];
    static const char* names[12] = {"setup", "anchor", "anchor_dues", "memo", "group", "E1", "E2", "E3",
                                    "states", "buckets", "survivors", "terminal"};
    std::fprintf(stderr, "[slos phases] total %.3e cycles:", (double)tot);
    for (int k = 0; k < 12; ++k) std::fprintf(stderr, " %s %.1f%%", names[k], 100.0 * (double)pc[k] / (double)(tot ? tot : 1));
    std::fprintf(stderr, " | buckets sub: hash %.1f%% fast %.1f%% \n", 100.0 * (double)pc[12] / (double)(tot ? tot : 1),
                 100.0 * (double)pc[13] / (double)(tot ? tot : 1));
    unsigned long long bt = 0;
    for (int k = 16; k < 22; ++k) bt += pc[k];
    static const char* bn[6] = {"setup", "census", "tile_gap", "emit", "tail", "fallback"};
    std::fprintf(stderr, "[slos build phases] total %.3e cycles:", (double)bt);
    for (int k = 0; k < 6; ++k) std::fprintf(stderr, " %s %.1f%%", bn[k], 100.0 * (double)pc[16 + k] / (double)(bt ? bt : 1));
    std::fprintf(stderr, " | max instance %.3e cycles over %llu instances\n", (double)pc[22], pc[23]);
    std::fprintf(stderr, "[slos fallback] %.3e cycles over %llu batches\n", (double)pc[30], pc[31]);
    std::fprintf(stderr, "[slos E3a] keys %llu, eval mean %.0f max %llu cycles, key_of mean %.0f; dues==0 %llu, Lx>0 %llu\n",
                 pc[25], (double)pc[24] / (double)(pc[25] ? pc[25] : 1), pc[26],
                 (double)pc[27] / (double)(pc[25] ? pc[25] : 1), pc[28], pc[29]);
    std::vector<int> idx(nv);
    for (int v = 0; v < nv; ++v) idx[v] = v;
    std::sort(idx.begin(), idx.end(), [&](int x, int y) { return hdr[x].dbg_cycles > hdr[y].dbg_cycles; });
    {
      double bsum = 0.0, esum = 0.0, nbs = 0.0;
      for (int v = 0; v < nv; ++v) {
        bsum += (double)hdr[v].dbg_cycles;
        esum += (double)hdr[v].n_entries;
        nbs += (double)hdr[v].n_batches;
      }
      auto bq = [&](double f) { return (double)hdr[idx[std::min(nv - 1, (int)(f * nv))]].dbg_cycles; };
      std::fprintf(stderr, "[slos build instances] mean %.3e p50 %.3e p90 %.3e max %.3e cycles; mean batches %.1f entries %.1f\n",
                   bsum / nv, bq(0.5), bq(0.1), bq(0.0), nbs / nv, esum / nv);
    }
    for (int r = 0; r < std::min(nv, 6); ++r) {
      const OutHdr& h = hdr[idx[r]];
      std::fprintf(stderr, "  slow build #%d: job %d cycles %.3e batches %lld entries %lld infeasible %d admitted %d T %lld\n", r,
                   jobs[valid[idx[r]]].k, (double)h.dbg_cycles, (long long)h.n_batches, (long long)h.n_entries,
                   h.infeasible, h.n_admitted, (long long)h.ctr[0]);
    }
    std::sort(idx.begin(), idx.end(), [&](int x, int y) { return hdr[x].dbg_dp_cycles > hdr[y].dbg_dp_cycles; });
    double dsum = 0.0;
    for (int v = 0; v < nv; ++v) dsum += (double)hdr[v].dbg_dp_cycles;
    auto q = [&](double f) { return (double)hdr[idx[std::min(nv - 1, (int)(f * nv))]].dbg_dp_cycles; };
    std::fprintf(stderr, "[slos dp instances] mean %.3e p10 %.3e p50 %.3e p90 %.3e max %.3e cycles\n", dsum / nv, q(0.9),
                 q(0.5), q(0.1), q(0.0));
    for (int r = 0; r < std::min(nv, 6); ++r) {
      const OutHdr& h = hdr[idx[r]];
      std::fprintf(stderr, "  slow dp #%d: job %d cycles %.3e T %lld gap_evals %lld dues %lld states %lld admitted %d\n", r,
                   jobs[valid[idx[r]]].k, (double)h.dbg_dp_cycles, (long long)h.ctr[0], (long long)h.ctr[1],
                   (long long)h.ctr[2], (long long)h.ctr[4], h.n_admitted);
    }
  }
}

// One set of instances (positions x -> instance v = vlist[x]): capacity regrowth
// list, packed offsets, compaction on `s` and one async D2H into a result arena;
// fills the slos_result of each instance (the caller synchronises `s`).
int collect_set(Ctx& c, Workspace& ws, const OutHdr* hdr, const int32_t* vlist_h, const int32_t* vlist_d, int n,
                PinBuf& h_offs, DevBuf& d_pack, cudaStream_t s, slos_result* outs, std::vector<Job>& retry) {
  const auto tcs = std::chrono::steady_clock::now();
  const std::vector<int>& valid = ws.valid;
  const std::vector<Job>& jobs = ws.jobs;
  const BatchArgs& A = ws.A;
  cudaError_t e;
  auto vof = [&](int x) { return vlist_h ? vlist_h[x] : x; };
  thread_local std::vector<int64_t> boff_tl, eoff_tl, ioff_tl;  // kept across calls (no page faults)
  std::vector<int64_t>& boff = boff_tl;  // the pool's lambdas see them through these references
  std::vector<int64_t>& eoff = eoff_tl;
  std::vector<int64_t>& ioff = ioff_tl;
  boff.resize((size_t)n);  // every entry is written below (0 for unplanned instances)
  eoff.resize((size_t)n);
  ioff.resize((size_t)n);
  // packed layout per planned instance, from a 16-byte aligned start: batches,
  // entries, ids, each 16-byte aligned; the next instance starts at the next 16-byte
  // boundary. Chunk-local offsets in parallel, chunk bases folded in order.
  const int chunks = n < 4096 ? 1 : 128;
  struct CRed { size_t bytes; int good; size_t last_end; std::vector<Job> retry; };
  thread_local std::vector<CRed> cred_tl;  // lambdas below see it through the reference
  std::vector<CRed>& cred = cred_tl;
  cred.resize((size_t)chunks);
  auto lo_of = [&](int ch) { return (int)((int64_t)ch * n / chunks); };
  auto a16 = [](size_t x) { return (x + 15) & ~(size_t)15; };
  auto local = [&](int ch) {
    CRed& r = cred[ch];
    r.bytes = 0; r.good = 0; r.last_end = 0;
    r.retry.clear();
    size_t at = 0;  // aligned start of the next instance, relative to the chunk
    for (int x = lo_of(ch); x < lo_of(ch + 1); ++x) {
      const int v = vof(x);
      const int q = valid[v];
      const OutHdr& h = hdr[v];
      boff[x] = eoff[x] = ioff[x] = 0;
      if (h.status == SLOS_ERR_CAPACITY && jobs[q].grow < 6) {
        r.retry.push_back({jobs[q].k, jobs[q].grow + 1});
        continue;
      }
      if (h.status != SLOS_OK) continue;
      ++r.good;
      boff[x] = (int64_t)at;
      size_t e = a16(at + sizeof(slos_batch) * (size_t)h.n_batches);
      eoff[x] = (int64_t)e;
      e = a16(e + sizeof(slos_entry) * (size_t)h.n_entries);
      ioff[x] = (int64_t)e;
      r.last_end = e + sizeof(int32_t) * (size_t)(h.n_admitted + h.n_declined);
      at = a16(r.last_end);
    }
    r.bytes = at;
  };
  if (chunks == 1) local(0);
  else HostPool::get().run(chunks, [&](int c0, int c1) { for (int ch = c0; ch < c1; ++ch) local(ch); });
  size_t packed = 0, base = 0;
  int good = 0;
  thread_local std::vector<size_t> cbase_tl;
  std::vector<size_t>& cbase = cbase_tl;
  cbase.resize((size_t)chunks);
  for (int ch = 0; ch < chunks; ++ch) {
    CRed& r = cred[ch];
    cbase[ch] = base;
    if (r.good) packed = base + r.last_end;  // the end of the last planned instance
    base += r.bytes;
    good += r.good;
    retry.insert(retry.end(), r.retry.begin(), r.retry.end());
  }
  if (chunks > 1)
    HostPool::get().run(chunks, [&](int c0, int c1) {
      for (int ch = c0; ch < c1; ++ch) {
        const int64_t b = (int64_t)cbase[ch];
        if (b == 0) continue;
        for (int x = lo_of(ch); x < lo_of(ch + 1); ++x) {
          boff[x] += b;
          eoff[x] += b;
          ioff[x] += b;
        }
      }
    });
  const auto tc0 = std::chrono::steady_clock::now();
  ResultArena* ra = nullptr;
  if (good) {
    const size_t offs_bytes = sizeof(int64_t) * 3 * (size_t)n;
    if ((e = d_pack.ensure(packed + offs_bytes + 256)) != cudaSuccess) return set_err(SLOS_ERR_CUDA, cudaGetErrorString(e));
    if ((e = h_offs.ensure(offs_bytes)) != cudaSuccess) return set_err(SLOS_ERR_CUDA, cudaGetErrorString(e));
    int64_t* ho = (int64_t*)h_offs.p;
    std::memcpy(ho, boff.data(), sizeof(int64_t) * n);
    std::memcpy(ho + n, eoff.data(), sizeof(int64_t) * n);
    std::memcpy(ho + 2 * n, ioff.data(), sizeof(int64_t) * n);
    unsigned char* DP_ = (unsigned char*)d_pack.p;
    const size_t offs_at = (packed + 255) & ~(size_t)255;
    cudaMemcpyAsync(DP_ + offs_at, ho, offs_bytes, cudaMemcpyHostToDevice, s);
    CompactParams cpp;
    cpp.inst = A.inst;
    cpp.out = A.out;
    cpp.batches = A.batches;
    cpp.entries = A.entries;
    cpp.ids = A.ids;
    cpp.vlist = vlist_d;
    cpp.boff = (const int64_t*)(DP_ + offs_at);
    cpp.eoff = cpp.boff + n;
    cpp.ioff = cpp.boff + 2 * n;
    cpp.dst = DP_;
    if ((e = launch_compact(cpp, n, s)) != cudaSuccess) return set_err(SLOS_ERR_CUDA, cudaGetErrorString(e));
    ra = arena_get(c, packed + 64);
    if (!ra) return set_err(SLOS_ERR_ALLOC, "result arena");
    if ((e = cudaMemcpyAsync(ra->p, DP_, packed, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
      return set_err(SLOS_ERR_CUDA, cudaGetErrorString(e));
    g_d2h += (int64_t)packed;
    g_h2d += (int64_t)offs_bytes;
  }
  const auto tc1 = std::chrono::steady_clock::now();
  if (ra) ra->refs += good;  // one reference per result that points into the arena
  HostPool::get().run(n, [&](int lo, int hi) {
  for (int x = lo; x < hi; ++x) {
    const int v = vof(x);
    const int q = valid[v];
    const int k = jobs[q].k;
    const OutHdr& h = hdr[v];
    slos_result& r = outs[k];
    if (h.status == SLOS_ERR_CAPACITY && jobs[q].grow < 6) continue;  // retried
    std::memset(&r, 0, sizeof r);
    r.status = h.status;
    if (h.status != SLOS_OK) continue;
    unsigned char* base = (unsigned char*)ra->p;
    r.running_set_infeasible = h.infeasible;
    r.admitted_value = h.value;
    r.n_admitted = h.n_admitted;
    r.n_declined = h.n_declined;
    r.n_deferred = 0;
    r.admitted = (const int32_t*)(base + ioff[x]);
    r.declined = r.admitted + h.n_admitted;
    r.deferred = r.declined + h.n_declined;
    r.n_batches = h.n_batches;
    r.batches = (const slos_batch*)(base + boff[x]);
    r.n_entries = h.n_entries;
    r.entries = (const slos_entry*)(base + eoff[x]);
    r.exact_until_s = h.exact_until;
    r.counters.transitions = h.ctr[0];
    r.counters.gap_evals = h.ctr[1];
    r.counters.dues = h.ctr[2];
    r.counters.slots = h.ctr[3];
    r.counters.states = h.ctr[4];
    r.owner_ = ra;
  }
  });
  if (host_timing()) {
    auto ms = [](std::chrono::steady_clock::time_point x, std::chrono::steady_clock::time_point y) {
      return std::chrono::duration<double, std::milli>(y - x).count();
    };
    std::fprintf(stderr, "[slos collect_set] n %d: offsets %.3f, copies+compaction %.3f, results %.3f ms\n", n,
                 ms(tcs, tc0), ms(tc0, tc1), ms(tc1, std::chrono::steady_clock::now()));
  }
  return SLOS_OK;
}

// Headers back, capacity regrowth list, compaction and the D2H of the results.
// With per-part headers (ws.part_collect, copied by ws_solve on each part's
// stream) a part's compaction and D2H start as soon as ITS reconstruction ends,
// under the later parts' kernels; otherwise one set over the whole workspace.
int ws_collect_finish(Workspace& ws);

// The first half of a collection: headers, regrowth list, compaction and the async
// D2H into the result arena, the result pointers. With per-part headers the D2H is
// still in flight on return (ws_collect_finish waits for it), so the chunk pipeline
// prepares the next chunk on the host meanwhile.
int ws_collect_start(Ctx& c, Workspace& ws, slos_result* outs, std::vector<Job>& retry) {
  if (!ws.uploaded || ws.nv == 0) return SLOS_OK;
  const int nv = ws.nv;
  cudaError_t e;
  if (ws.part_collect) {
    for (int p = 0; p < ws.n_parts; ++p) {
      const auto t0 = std::chrono::steady_clock::now();
      if ((e = cudaEventSynchronize(ws.ev_hdr[p])) != cudaSuccess) return set_err(SLOS_ERR_CUDA, cudaGetErrorString(e));
      if (host_timing())
        std::fprintf(stderr, "[slos collect] part %d: header wait %.3f ms\n", p,
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
      g_d2h += (int64_t)(sizeof(OutHdr) * (size_t)nv);
      const int lo = ws.part_lo[p], n = ws.part_lo[p + 1] - lo;
      const auto t1 = std::chrono::steady_clock::now();
      const int r = collect_set(c, ws, (const OutHdr*)ws.h_hdr[p].p, ws.ord.data() + lo, ws.A.order + lo, n,
                                ws.h_offs[p], ws.d_packp[p], ws.pstream[p], outs, retry);
      if (r != SLOS_OK) return r;
      if (host_timing())
        std::fprintf(stderr, "[slos collect] part %d: collect_set %.3f ms (%d instances)\n", p,
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t1).count(), n);
      if (host_timing()) {
        if (!ws.ev_d2h[p]) cudaEventCreate(&ws.ev_d2h[p]);
        cudaEventRecord(ws.ev_d2h[p], ws.pstream[p]);
      }
    }
    return SLOS_OK;
  }
  const Layout& Ly = ws.Ly;
  const cudaStream_t s = ws.stream;
  unsigned char* DO = (unsigned char*)ws.d_out.p;
  if ((e = ws.h_small.ensure(sizeof(OutHdr) * nv)) != cudaSuccess) return set_err(SLOS_ERR_CUDA, cudaGetErrorString(e));
  OutHdr* hO = (OutHdr*)ws.h_small.p;
  // the headers are final only after the last solve's kernels, which may have run on
  // another stream than the upload's (slos_workspace_solve takes its own stream)
  if (ws.solved) cudaStreamWaitEvent(s, ws.ev[2], 0);
  cudaMemcpyAsync(hO, DO + Ly.out, sizeof(OutHdr) * nv, cudaMemcpyDeviceToHost, s);
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return set_err(SLOS_ERR_CUDA, cudaGetErrorString(e));
  std::vector<OutHdr> hdr(hO, hO + nv);
  g_d2h += (int64_t)(sizeof(OutHdr) * (size_t)nv);
  if (ws.dp.phase_cycles) print_phase_debug(ws, hdr);
  const int r = collect_set(c, ws, hdr.data(), nullptr, nullptr, nv, ws.h_offs[0], ws.d_pack, s, outs, retry);
  if (r != SLOS_OK) return r;
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return set_err(SLOS_ERR_CUDA, cudaGetErrorString(e));
  return SLOS_OK;
}

// The second half: wait for the result D2H of every part (per-part collection).
int ws_collect_finish(Workspace& ws) {
  if (!ws.uploaded || ws.nv == 0 || !ws.part_collect) return SLOS_OK;
  cudaError_t e;
  {
    const auto t0 = std::chrono::steady_clock::now();
    for (int p = 0; p < ws.n_parts; ++p)
      if ((e = cudaStreamSynchronize(ws.pstream[p])) != cudaSuccess) return set_err(SLOS_ERR_CUDA, cudaGetErrorString(e));
    if (host_timing())
      std::fprintf(stderr, "[slos collect] d2h wait %.3f ms\n",
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    if (host_timing()) {
      for (int p = 0; p < ws.n_parts; ++p) {
        float a = 0.0f, b = 0.0f, d = 0.0f;
        cudaEventElapsedTime(&a, ws.ev[0], ws.ev_dp[p]);
        cudaEventElapsedTime(&b, ws.ev[0], ws.ev_d2h[p]);
        cudaEventElapsedTime(&d, ws.ev[0], ws.ev[2]);
        std::fprintf(stderr, "[slos collect] part %d: dp end %.3f ms, d2h end %.3f ms (solve end %.3f ms)\n", p, a, b, d);
      }
    }
  }
  return SLOS_OK;
}

int ws_collect(Ctx& c, Workspace& ws, slos_result* outs, std::vector<Job>& retry) {
  const int r = ws_collect_start(c, ws, outs, retry);
  if (r != SLOS_OK) {
    cudaDeviceSynchronize();  // no D2H may outlive a failed collection
    return r;
  }
  return ws_collect_finish(ws);
}

}  // namespace

// ------------------------------------------------------------------ C-ABI ---

extern "C" {

const char* slos_status_slug(int s) {
  switch (s) {
    case SLOS_OK: return "ok";
    case SLOS_ERR_INVALID_PARAMETERS: return "invalid-parameters";
    case SLOS_ERR_INTERNAL_INCONSISTENCY: return "internal-inconsistency";
    case SLOS_ERR_INFEASIBLE_BUDGET: return "infeasible-budget";
    case SLOS_ERR_CUDA: return "cuda-error";
    case SLOS_ERR_CAPACITY: return "capacity";
    case SLOS_ERR_NO_DEVICE: return "no-device";
    case SLOS_ERR_ALLOC: return "alloc";
    case SLOS_ERR_RANGE: return "range";
    case 20: return "invalid-distribution-parameters";  // slos_trace.h
    case 21: return "invariant-violation";
    case 22: return "insufficient-samples";             // slos_fit.h
    case 23: return "degenerate-samples";
    default: return "error";
  }
}

const char* slos_last_error(void) { return g_err.c_str(); }
const char* slos_backend(void) { return "b200-cuda"; }

double slos_expected_accepted(double alpha, int32_t sl) {  // batch_planner.cpp:32-37
  if (sl < 1) return NAN;
  if (alpha >= 1.0) return (double)sl;
  if (alpha <= 0.0) return 1.0;
  return (1.0 - std::pow(alpha, sl)) / (1.0 - alpha);
}

void slos_planner_config_default(slos_planner_config* c) {
  c->max_chunk_tokens = 2048;
  c->max_batch_tokens = 16384;
  c->speculative = 0;
  c->spec_max_len = 8;
  c->spec_alpha = 0.8;
  c->plan_margin = 0.0;
}

int slos_planner_create(const slos_perf_term* terms, int32_t n_terms, const double* tpot,
                        const double* slow, int32_t n_tiers, int32_t tpot_window,
                        const slos_planner_config* cfg, slos_planner** out) {
  *out = nullptr;
  if (n_terms < 1) return set_err(SLOS_ERR_INVALID_PARAMETERS, "perf model needs at least one term");
  for (int i = 0; i < n_terms; ++i)
    if (terms[i].k1 < 0 || terms[i].k2 < 0 || terms[i].b < 0)
      return set_err(SLOS_ERR_INVALID_PARAMETERS, "perf model coefficients must be nonnegative");
  if (n_tiers < 1) return set_err(SLOS_ERR_INVALID_PARAMETERS, "slo config needs at least one tier");
  for (int i = 0; i < n_tiers; ++i) {
    if (tpot[i] <= 0) return set_err(SLOS_ERR_INVALID_PARAMETERS, "tpot tiers must be positive");
    if (i > 0 && tpot[i] < tpot[i - 1])
      return set_err(SLOS_ERR_INVALID_PARAMETERS, "tpot tiers must ascend from tightest to loosest");
    if (slow[i] < 1.0) return set_err(SLOS_ERR_INVALID_PARAMETERS, "ttft slowdown multipliers must be >= 1");
  }
  if (tpot_window < 1) return set_err(SLOS_ERR_INVALID_PARAMETERS, "tpot window must be >= 1");
  slos_planner_config c;
  if (cfg) c = *cfg; else slos_planner_config_default(&c);
  if (c.max_chunk_tokens < 1 || c.max_batch_tokens < 1)
    return set_err(SLOS_ERR_INVALID_PARAMETERS, "batch and chunk caps must be positive");
  if (c.max_chunk_tokens > INT32_MAX || c.max_batch_tokens > INT32_MAX)  // slos_entry is 32-bit
    return set_err(SLOS_ERR_INVALID_PARAMETERS, "batch and chunk caps must fit the 32-bit plan entries");
  if (c.speculative && c.spec_max_len > SLOS_ENTRY_MAX_SPEC)  // 7-bit entry spec_len
    return set_err(SLOS_ERR_INVALID_PARAMETERS, "spec_max_len must fit the plan entry format");
  if (c.plan_margin < 0) return set_err(SLOS_ERR_INVALID_PARAMETERS, "plan margin must be >= 0");
  slos_planner* p = new slos_planner();
  p->terms.assign(terms, terms + n_terms);
  p->tpot.assign(tpot, tpot + n_tiers);
  p->slow.assign(slow, slow + n_tiers);
  p->L = n_tiers;
  p->tpot_window = tpot_window;
  p->cfg = c;
  fill_planner_dev(p);
  *out = p;
  return SLOS_OK;
}

void slos_planner_destroy(slos_planner* p) { delete p; }

}  // extern "C"

struct slos_workspace {
  Workspace ws;
  std::vector<int> grow;  // per instance: capacity growth that made it fit
  bool has_inputs = false;
  int n = 0;
};

namespace {
Workspace& default_ws() {
  static Workspace* w = new Workspace();
  return *w;
}

// Three pipeline workspaces with their own streams (chunk i uses i % 3): chunk i+1's
// host preparation and H2D overlap chunk i's kernels, and chunk i's compaction + D2H
// overlap chunk i+1's kernels (copy engines vs SMs) and chunk i+2's host preparation.
constexpr int kPipeWs = 3;
Workspace& pipe_ws(int k) {
  static Workspace* w[kPipeWs] = {nullptr, nullptr, nullptr};
  if (!w[k]) {
    w[k] = new Workspace();
    {  // SLOS_CHUNK_PRIO=n: later chunks' kernel streams n priority levels lower
      const char* e = std::getenv("SLOS_CHUNK_PRIO");
      w[k]->prio_shift = (e && k > 0) ? std::atoi(e) : 0;
    }
    // the earlier chunk runs at higher priority so its D2H starts while the next
    // chunk's kernels still run
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    cudaStreamCreateWithPriority(&w[k]->own_stream, cudaStreamNonBlocking, k == 0 ? hi : lo);
  }
  return *w[k];
}

int pipeline_chunks(int n, double reqs_per_instance) {
  static const int env = [] {
    const char* e = std::getenv("SLOS_PIPELINE_CHUNKS");
    return e ? std::atoi(e) : 0;
  }();
  if (env > 0) return std::min(env, std::max(1, n));
  // measured: C2 x 1024 (heavy instances, GPU-bound): 2 chunks best; C5 x 65,536 (tiny
  // instances, host-preparation-bound; collection split around the next chunk's
  // preparation): 3 chunks 7.05-7.18 ms, 4: 7.25-7.33, 5: 7.4-7.5, 6: 7.7, 8: 8.3-8.6
  if (n < 512) return 1;
  if (n < 40000) return 2;
  // Three workspaces are live at once: chunks of instances with many requests (device
  // scratch grows with them: ~2 MB per C2 instance) stay at <= 10,923 instances so
  // the pipeline's footprint is no larger than two 16k-instance workspaces were.
  if (reqs_per_instance >= 64.0) return std::min(16, (n + 10922) / 10923);
  return std::min(8, n / 20000);
}

bool part_collect_enabled() {  // SLOS_PART_COLLECT=0: one collection per workspace
  static const bool on = [] {
    const char* e = std::getenv("SLOS_PART_COLLECT");
    return !(e && std::atoi(e) == 0);
  }();
  return on;
}

// Slot-grid need of one instance: ws_upload sizes every kernel's shared-memory slot
// grid (Sc) by the widest deadline span of its batch (prep_instance's span), so a
// single outlier -- a far-future pending deadline, a late forced prefill -- must not
// size everybody's grid. Same span as prep_instance (chain deadlines and now).
double slot_need(const slos_planner* P, const slos_input* in) {
  double maxdl = in->now, mindl = in->now;
  for (int i = 0; i < in->n_running; ++i)
    if (in->running[i].prefill_remaining > 0) {
      maxdl = std::max(maxdl, in->running[i].prefill_deadline);
      mindl = std::min(mindl, in->running[i].prefill_deadline);
    }
  for (int i = 0; i < in->n_pending; ++i) {
    maxdl = std::max(maxdl, in->pending[i].prefill_deadline);
    mindl = std::min(mindl, in->pending[i].prefill_deadline);
  }
  const double t0 = P->L > 0 ? P->tpot[0] : 1.0;
  const double s = std::ceil(std::max(0.0, maxdl - mindl) / t0) + 8;
  return std::isfinite(s) ? s : 1e18;
}

// Instances whose grid needs more slots than this are solved apart, in classes of
// similar width (SLOS_NARROW_SLOTS overrides).
double narrow_slots() {
  static const double v = [] {
    const char* e = std::getenv("SLOS_NARROW_SLOTS");
    return e ? std::atof(e) : 512.0;
  }();
  return v;
}

// Solve `jobs` with capacity regrowth (up to 8 rounds) in one workspace.
int solve_rounds(Ctx& c, Workspace& ws, slos_planner* const* planners, const slos_input* inputs,
                 int32_t unit_value, slos_result* outs, cudaStream_t stream, std::vector<Job> jobs) {
  std::vector<Job> retry;
  ws.part_collect = part_collect_enabled();
  ws.records = false;
  for (int round = 0; round < 8 && !jobs.empty(); ++round) {
    retry.clear();
    int r = ws_upload(c, ws, planners, inputs, unit_value, jobs, outs, stream);
    if (r == SLOS_OK) r = ws_solve(ws, stream);
    if (r == SLOS_OK) r = ws_collect(c, ws, outs, retry);
    if (r != SLOS_OK) {
      for (const Job& j : jobs) outs[j.k].status = r;
      return r;
    }
    jobs.swap(retry);
  }
  for (const Job& j : jobs) {
    std::memset(&outs[j.k], 0, sizeof(outs[j.k]));
    outs[j.k].status = SLOS_ERR_CAPACITY;
  }
  return SLOS_OK;
}

// Wide instances (slot_need > narrow_slots()), sorted by need, in classes whose widest
// member needs at most twice the narrowest; a class the shared memory cannot hold is
// retried one instance at a time so only the instances that alone exceed it fail.
int solve_wide(Ctx& c, Workspace& ws, slos_planner* const* planners, const slos_input* inputs,
               int32_t unit_value, slos_result* outs, cudaStream_t stream,
               std::vector<std::pair<double, int>>& wide) {
  std::sort(wide.begin(), wide.end());
  size_t a = 0;
  while (a < wide.size()) {
    size_t b = a + 1;
    while (b < wide.size() && wide[b].first <= 2.0 * wide[a].first) ++b;
    std::vector<Job> cls;
    for (size_t x = a; x < b; ++x) cls.push_back({wide[x].second, 0});
    int r = solve_rounds(c, ws, planners, inputs, unit_value, outs, stream, cls);
    if (r == SLOS_ERR_RANGE && cls.size() > 1) {
      for (const Job& j : cls) {
        r = solve_rounds(c, ws, planners, inputs, unit_value, outs, stream, {j});
        if (r != SLOS_OK && r != SLOS_ERR_RANGE) return r;
      }
    } else if (r != SLOS_OK && r != SLOS_ERR_RANGE) {
      return r;
    }
    a = b;
  }
  return SLOS_OK;
}

// full pipeline with capacity regrowth; caller holds ctx().mu
int plan_all(Ctx& c, Workspace& ws, slos_planner* const* planners, int32_t n, const slos_input* inputs,
             int32_t unit_value, slos_result* outs, cudaStream_t stream) {
  g_h2d = 0;
  g_d2h = 0;
  const auto t_p0 = std::chrono::steady_clock::now();
  // per-call job lists kept across calls (fresh 0.5 MB vectors page-fault on every
  // C5-size call)
  thread_local std::vector<Job> jobs_tl;
  std::vector<Job>& jobs = jobs_tl;
  jobs.clear();
  std::vector<Job> retry;
  std::vector<std::pair<double, int>> wide;
  {
    thread_local std::vector<double> need_tl;  // the workers see it through the reference
    std::vector<double>& need = need_tl;
    need.resize((size_t)n);
    HostPool::get().run(n, [&](int lo, int hi) {
      for (int k = lo; k < hi; ++k) need[k] = slot_need(planners[k], &inputs[k]);
    });
    if (host_timing())
      std::fprintf(stderr, "[slos pipeline] slot needs: %.3f ms\n",
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_p0).count());
    const double lim = narrow_slots();
    bool any_wide = false;
    for (int k = 0; k < n; ++k) any_wide |= need[k] > lim;
    if (!any_wide) {  // (the common case: the job list is the identity, filled in parallel)
      jobs.resize((size_t)n);
      HostPool::get().run(n, [&](int lo, int hi) { for (int k = lo; k < hi; ++k) jobs[k] = {k, 0}; });
    } else {
      jobs.reserve((size_t)n);
      for (int k = 0; k < n; ++k) {
        if (need[k] > lim) wide.push_back({need[k], k});
        else jobs.push_back({k, 0});
      }
    }
  }
  if (host_timing())
    std::fprintf(stderr, "[slos pipeline] %zu wide instances (job list at %.3f ms)\n", wide.size(),
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_p0).count());
  if (!wide.empty()) {
    const int r = solve_wide(c, ws, planners, inputs, unit_value, outs, stream, wide);
    if (r != SLOS_OK) {
      for (int k = 0; k < n; ++k) outs[k].status = r;
      return r;
    }
  }
  n = (int32_t)jobs.size();
  double reqs = 0.0;  // mean requests per instance (chunk sizing)
  if (n >= 40000) {
    for (int k = 0; k < n; ++k) reqs += (double)inputs[jobs[k].k].n_running + inputs[jobs[k].k].n_pending;
    reqs /= n;
  }
  const int K = pipeline_chunks(n, reqs);
  if (K > 1) {
    // order after the caller's prior work on `stream`
    static cudaEvent_t ev0 = nullptr;
    if (!ev0) cudaEventCreateWithFlags(&ev0, cudaEventDisableTiming);
    cudaEventRecord(ev0, stream ? stream : c.stream);
    if (host_timing())
      std::fprintf(stderr, "[slos pipeline] ev0 at %.3f ms\n",
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_p0).count());
    // chunk boundaries: with 2 chunks the first is the smaller (SLOS_PIPELINE_SPLIT):
    // the GPU starts after a short host preparation, the second chunk's preparation
    // overlaps the first's kernels, and both chunks' kernels then share the SMs
    static const double split = [] {
      const char* e = std::getenv("SLOS_PIPELINE_SPLIT");
      return e ? std::atof(e) : 0.3;  // measured C2 x 1024: 0.3 -> 4.5 ms, 0.5 -> 4.9 ms, 0.7 -> 5.2 ms
    }();
    thread_local std::vector<std::vector<Job>> chunk_tl;
    std::vector<std::vector<Job>>& chunk = chunk_tl;
    if ((int)chunk.size() < K) chunk.resize((size_t)K);
    // chunk i = jobs[ceil(i n / K), ceil((i+1) n / K)) (contiguous; jobs[k].k is the
    // caller's instance index)
    // With 3+ chunks the last one takes `tail` of an equal share (SLOS_PIPELINE_TAIL):
    // its kernels, D2H and collection are the part of the call nothing overlaps.
    static const double tail = [] {
      const char* e = std::getenv("SLOS_PIPELINE_TAIL");
      return e ? std::atof(e) : 1.0;
    }();
    for (int i = 0; i < K; ++i) {
      auto lo = [&](int x) {
        if (x == 0) return 0;
        if (x == K) return n;
        if (K == 2) return (int)(split * n);
        return (int)((double)n * x / (K - 1 + tail));
      };
      chunk[i].assign(jobs.begin() + lo(i), jobs.begin() + lo(i + 1));
    }
    if (host_timing())
      std::fprintf(stderr, "[slos pipeline] before the chunks: %.3f ms\n",
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_p0).count());
    // step i: upload + solve chunk i, start chunk i-1's collection (headers, compaction,
    // D2H enqueued), finish chunk i-2's (its D2H ran under chunk i's host preparation)
    auto fail = [&](int r) {
      cudaDeviceSynchronize();  // no D2H may outlive a failed call
      for (const Job& j : jobs) outs[j.k].status = r;
      return r;
    };
    for (int i = 0; i <= K + 1; ++i) {
      const auto t_a = std::chrono::steady_clock::now();
      if (i < K) {
        Workspace& w = pipe_ws(i % kPipeWs);
        cudaStreamWaitEvent(w.own_stream, ev0, 0);
        w.part_collect = part_collect_enabled();
        w.records = false;
        int r = ws_upload(c, w, planners, inputs, unit_value, chunk[i], outs, w.own_stream);
        if (r == SLOS_OK) r = ws_solve(w, w.own_stream);
        if (r != SLOS_OK) return fail(r);
      }
      const auto t_b = std::chrono::steady_clock::now();
      if (i >= 1 && i - 1 < K) {
        const int r = ws_collect_start(c, pipe_ws((i - 1) % kPipeWs), outs, retry);
        if (r != SLOS_OK) return fail(r);
      }
      if (i >= 2) {
        const int r = ws_collect_finish(pipe_ws((i - 2) % kPipeWs));
        if (r != SLOS_OK) return fail(r);
      }
      if (std::getenv("SLOS_HOST_TIMING")) {
        const auto t_c = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[slos pipeline] step %d: upload+enqueue %.3f ms, collect %.3f ms\n", i,
                     std::chrono::duration<double, std::milli>(t_b - t_a).count(),
                     std::chrono::duration<double, std::milli>(t_c - t_b).count());
      }
    }
    jobs.assign(retry.begin(), retry.end());  // (keeps the reused buffer)
    retry.clear();
    if (std::getenv("SLOS_HOST_TIMING")) std::fprintf(stderr, "[slos pipeline] %d chunks, %zu retried\n", K, jobs.size());
  }
  const int r = solve_rounds(c, ws, planners, inputs, unit_value, outs, stream, std::vector<Job>(jobs));
  if (r == SLOS_ERR_RANGE) return SLOS_OK;  // per-instance statuses already set
  return r;
}
}  // namespace

extern "C" {

int slos_plan_batch(slos_planner* const* planners, int32_t n, const slos_input* inputs,
                    int32_t unit_value, slos_result* outs, void* stream) {
  g_err.clear();  // a message always belongs to this call
  Ctx& c = ctx();
  std::lock_guard<std::mutex> g(c.mu);  // (the host pool serves one call at a time)
  const auto t0 = std::chrono::steady_clock::now();
  if (n > 0)
    HostPool::get().run(n, [&](int lo, int hi) { std::memset(outs + lo, 0, sizeof(*outs) * (size_t)(hi - lo)); });
  if (host_timing())
    std::fprintf(stderr, "[slos plan_batch] clear %d results: %.3f ms\n", n,
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  const int st = ensure_device(c);
  if (st != SLOS_OK) {
    set_err(st, c.why);
    for (int k = 0; k < n; ++k) outs[k].status = st;
    return st;
  }
  return plan_all(c, default_ws(), planners, n, inputs, unit_value, outs, (cudaStream_t)stream);
}

int slos_workspace_create(slos_workspace** out) {
  *out = nullptr;
  Ctx& c = ctx();
  std::lock_guard<std::mutex> g(c.mu);
  const int st = ensure_device(c);
  if (st != SLOS_OK) return set_err(st, c.why);
  *out = new slos_workspace();
  return SLOS_OK;
}

void slos_workspace_destroy(slos_workspace* b) {
  if (!b) return;
  Ctx& c = ctx();
  std::lock_guard<std::mutex> g(c.mu);
  cudaDeviceSynchronize();
  for (DevBuf* d : {&b->ws.d_in, &b->ws.d_scr, &b->ws.d_out, &b->ws.d_pack, &b->ws.d_wscr})
    if (d->p) cudaFree(d->p);
  for (PinBuf* h : {&b->ws.h_in, &b->ws.h_small})
    if (h->p) cudaFreeHost(h->p);
  delete b;
}

int slos_workspace_upload(slos_workspace* b, slos_planner* const* planners, int32_t n, const slos_input* inputs,
                      int32_t unit_value, slos_result* outs, void* stream) {
  g_err.clear();  // a message always belongs to this call
  for (int k = 0; k < n; ++k) std::memset(&outs[k], 0, sizeof(outs[k]));
  Ctx& c = ctx();
  std::lock_guard<std::mutex> g(c.mu);
  if ((int)b->grow.size() != n || b->ws.inputs != inputs) b->grow.assign(n, 0);
  std::vector<Job> jobs(n);
  for (int k = 0; k < n; ++k) jobs[k] = {k, b->grow[k]};
  b->n = n;
  b->has_inputs = true;
  g_h2d = 0;
  g_d2h = 0;
  return ws_upload(c, b->ws, planners, inputs, unit_value, jobs, outs, (cudaStream_t)stream);
}

int slos_workspace_solve(slos_workspace* b, void* stream) {
  g_err.clear();  // a message always belongs to this call
  Ctx& c = ctx();
  std::lock_guard<std::mutex> g(c.mu);
  return ws_solve(b->ws, (cudaStream_t)stream);
}

int slos_workspace_download(slos_workspace* b, slos_result* outs, void* stream) {
  g_err.clear();  // a message always belongs to this call
  Ctx& c = ctx();
  std::lock_guard<std::mutex> g(c.mu);
  std::vector<Job> retry;
  int r = ws_collect(c, b->ws, outs, retry);
  if (r != SLOS_OK || retry.empty()) return r;
  // Regrow the overflowed instances (rare), remember their capacities, then
  // re-upload the whole batch so the resident workspace fits from now on.
  std::vector<Job> jobs = retry;
  for (int round = 0; round < 8 && !jobs.empty(); ++round) {
    for (const Job& j : jobs) b->grow[j.k] = j.grow;
    std::vector<Job> again;
    r = ws_upload(c, b->ws, b->ws.planners, b->ws.inputs, b->ws.unit_value, jobs, outs, (cudaStream_t)stream);
    if (r == SLOS_OK) r = ws_solve(b->ws, (cudaStream_t)stream);
    if (r == SLOS_OK) r = ws_collect(c, b->ws, outs, again);
    if (r != SLOS_OK) return r;
    jobs.swap(again);
  }
  for (const Job& j : jobs) outs[j.k].status = SLOS_ERR_CAPACITY;
  std::vector<Job> all(b->n);
  for (int k = 0; k < b->n; ++k) all[k] = {k, b->grow[k]};
  std::vector<slos_result> scratch(b->n);
  return ws_upload(c, b->ws, b->ws.planners, b->ws.inputs, b->ws.unit_value, all, scratch.data(),
                   (cudaStream_t)stream);
}

int slos_workspace_records(slos_workspace* b, slos_record* out, void* stream) {
  g_err.clear();  // a message always belongs to this call
  Ctx& c = ctx();
  std::lock_guard<std::mutex> g(c.mu);
  Workspace& ws = b->ws;
  if (!ws.uploaded || !ws.records) return set_err(SLOS_ERR_INVALID_PARAMETERS, "nothing uploaded");
  const cudaStream_t s = stream ? (cudaStream_t)stream : ws.stream;
  unsigned char* DI = (unsigned char*)ws.d_in.p;
  cudaError_t e = cudaMemcpyAsync(out, DI + ws.Ly.recdef, sizeof(slos_record) * (size_t)ws.n_total,
                                  cudaMemcpyDeviceToDevice, s);
  if (e == cudaSuccess)
    e = launch_records(ws.A.out, (const int32_t*)(DI + ws.Ly.recmap), ws.nv, out, s);
  return e == cudaSuccess ? SLOS_OK : set_err(SLOS_ERR_CUDA, cudaGetErrorString(e));
}

int slos_workspace_kernel_ms(slos_workspace* b, float* ms2) {
  Workspace& ws = b->ws;
  ms2[0] = ms2[1] = 0.0f;
  if (!ws.ev[2]) return SLOS_OK;
  cudaEventSynchronize(ws.ev[2]);
  float all = 0.0f;
  cudaEventElapsedTime(&all, ws.ev[0], ws.ev[2]);
  ms2[0] = dp_end_ms(ws);
  ms2[1] = all - ms2[0];
  return SLOS_OK;
}

int slos_workspace_launches(slos_workspace* b, int64_t* n) {
  Ctx& c = ctx();
  std::lock_guard<std::mutex> g(c.mu);
  *n = b->ws.launches;
  return SLOS_OK;
}

int slos_workspace_stage_ms(slos_workspace* b, float* ms, int32_t n) {
  Workspace& ws = b->ws;
  float t[3] = {0.0f, 0.0f, 0.0f};
  if (ws.ev[2]) {
    cudaEventSynchronize(ws.ev[2]);
    float all = 0.0f;
    cudaEventElapsedTime(&all, ws.ev[0], ws.ev[2]);
    for (int p = 0; p < ws.n_parts; ++p) {  // anchor stage: until the last part's groups
      float x = 0.0f;
      cudaEventElapsedTime(&x, ws.ev[0], ws.ev_anc[p]);
      t[0] = std::max(t[0], x);
    }
    if (host_timing())
      for (int p = 0; p < ws.n_parts; ++p) {
        float a = 0.0f, d = 0.0f, b = 0.0f;
        cudaEventElapsedTime(&a, ws.ev[0], ws.ev_anc[p]);
        cudaEventElapsedTime(&d, ws.ev[0], ws.ev_dp[p]);
        cudaEventElapsedTime(&b, ws.ev[0], ws.ev_bend[p]);
        std::fprintf(stderr, "[slos stages] part %d: groups end %.3f, dp end %.3f, build end %.3f ms\n", p, a, d, b);
      }
    const float dp_end = dp_end_ms(ws);  // last part's DP (parts overlap: stages are
    t[1] = dp_end - t[0];                // timed to their last part's end)
    t[2] = all - dp_end;
  }
  float t3 = 0.0f;  // scratch init (memsets) before the kernels
  if (ws.ev[2]) cudaEventElapsedTime(&t3, ws.ev[1], ws.ev[0]);
  for (int k = 0; k < n && k < 3; ++k) ms[k] = t[k];
  if (n > 3) ms[3] = t3;
  return SLOS_OK;
}

// ---- the plan broker (include/slos_planner.h) --------------------------------
}  // extern "C"

struct slos_broker {
  struct Req {
    slos_planner* p;
    slos_input in;
    slos_result* out;
    bool done;
  };
  std::mutex mu;
  std::condition_variable cv;
  int32_t unit_value = 0;
  int active = 0;
  bool flushing = false;
  std::vector<Req*> queue;
  int64_t flushes = 0, plans = 0;
};

namespace {
// Called with the lock held by the thread that made `active` reach zero: run every
// queued plan as one slos_plan_batch (outside the lock, so clients may keep queueing
// for the next batch), then wake the callers, which are active again.
void broker_flush(slos_broker* b, std::unique_lock<std::mutex>& lk) {
  while (b->active == 0 && !b->flushing && !b->queue.empty()) {
    b->flushing = true;
    std::vector<slos_broker::Req*> batch;
    batch.swap(b->queue);
    lk.unlock();
    const int n = (int)batch.size();
    std::vector<slos_planner*> ps((size_t)n);
    std::vector<slos_input> ins((size_t)n);
    std::vector<slos_result> outs((size_t)n);
    for (int k = 0; k < n; ++k) {
      ps[k] = batch[k]->p;
      ins[k] = batch[k]->in;
    }
    const int st = slos_plan_batch(ps.data(), n, ins.data(), b->unit_value, outs.data(), nullptr);
    lk.lock();
    for (int k = 0; k < n; ++k) {
      *batch[k]->out = outs[k];
      if (st != SLOS_OK && outs[k].status == SLOS_OK) batch[k]->out->status = st;
      batch[k]->done = true;
    }
    b->active += n;
    b->flushing = false;
    b->flushes += 1;
    b->plans += n;
    b->cv.notify_all();
  }
}
}  // namespace

extern "C" {

int slos_broker_create(int32_t unit_value, slos_broker** out) {
  *out = new slos_broker();
  (*out)->unit_value = unit_value;
  return SLOS_OK;
}

void slos_broker_destroy(slos_broker* b) { delete b; }

void slos_broker_join(slos_broker* b) {
  std::lock_guard<std::mutex> g(b->mu);
  b->active += 1;
}

void slos_broker_leave(slos_broker* b) {
  std::unique_lock<std::mutex> lk(b->mu);
  b->active -= 1;
  broker_flush(b, lk);
}

int slos_broker_plan(slos_broker* b, slos_planner* p, const slos_input* in, slos_result* out) {
  g_err.clear();  // a message always belongs to this call (the batch may run on another thread)
  std::unique_lock<std::mutex> lk(b->mu);
  slos_broker::Req r{p, *in, out, false};
  b->queue.push_back(&r);
  b->active -= 1;
  broker_flush(b, lk);
  b->cv.wait(lk, [&] { return r.done; });
  if (out->status != SLOS_OK && g_err.empty()) set_err(out->status, "plan failed");
  return out->status;
}

void slos_broker_stats(slos_broker* b, int64_t* flushes, int64_t* plans) {
  std::lock_guard<std::mutex> g(b->mu);
  *flushes = b->flushes;
  *plans = b->plans;
}

void slos_last_transfer_bytes(int64_t* h2d, int64_t* d2h) {
  *h2d = g_h2d;
  *d2h = g_d2h;
}

int slos_plan(slos_planner* p, const slos_input* in, int32_t unit_value, slos_result* out) {
  slos_planner* const hs[1] = {p};
  const int st = slos_plan_batch(hs, 1, in, unit_value, out, nullptr);
  if (st != SLOS_OK) return st;
  if (out->status != SLOS_OK) {
    if (g_err.empty() || out->status == SLOS_ERR_CAPACITY) set_err(out->status, "plan failed");
    return out->status;
  }
  return SLOS_OK;
}

void slos_result_free(slos_result* r) {
  if (!r) return;
  if (r->owner_) arena_release((ResultArena*)r->owner_);
  std::memset(r, 0, sizeof *r);
}

// ---- tile_gap primitives (K1) ----------------------------------------------

int slos_tile_gap_batch(slos_planner* p, int32_t n, const slos_gap_query* qs, slos_gap_result* outs) {
  g_err.clear();  // a message always belongs to this call
  for (int k = 0; k < n; ++k) std::memset(&outs[k], 0, sizeof(outs[k]));
  if (n <= 0) return SLOS_OK;
  Ctx& c = ctx();
  std::lock_guard<std::mutex> g(c.mu);
  int st = ensure_device(c);
  if (st != SLOS_OK) {
    for (int k = 0; k < n; ++k) outs[k].status = st;
    return set_err(st, c.why);
  }
  if (!p->device_ok || p->L > kMaxTiers) {
    for (int k = 0; k < n; ++k) outs[k].status = SLOS_ERR_RANGE;
    return set_err(SLOS_ERR_RANGE, "planner not representable on device");
  }
  std::vector<int> todo(n), grow(n, 0);
  for (int k = 0; k < n; ++k) todo[k] = k;
  for (int round = 0; round < 8 && !todo.empty(); ++round) {
    const int m = (int)todo.size();
    int64_t TM = 0, TB = 0, TO = 0, TW = 0;
    std::vector<GapQueryDev> qd(m);
    for (int x = 0; x < m; ++x) {
      const slos_gap_query& q = qs[todo[x]];
      GapQueryDev& d = qd[x];
      std::memset(&d, 0, sizeof d);
      d.gap_s = q.gap_s;
      d.horizon = q.due_horizon_s;
      for (int l = 0; l < kMaxTiers; ++l) d.counts[l] = l < p->L ? q.counts_per_tier[l] : 0;
      d.mode = q.mode;
      d.n_exact = q.mode == SLOS_GAP_PREFILL_BUDGET ? 0 : q.n_exact;
      d.off_exact = TM;
      TM += d.n_exact;
      const double span = std::max({q.gap_s, q.due_horizon_s, 0.0});
      const int64_t S = (int64_t)std::ceil(span / p->tpot[0]) + 8;
      const int64_t gg = (int64_t)1 << (2 * grow[todo[x]]);
      d.cap_batch = (S + 8) * gg;
      d.cap_owner = (int64_t)(d.n_exact + 1) * d.cap_batch;
      d.off_out_batch = TB;
      d.off_out_owner = TO;
      TB += d.cap_batch;
      TO += d.cap_owner;
      d.cap_work = ((S + 2) * (d.n_exact + 2) * 4 + S * 128 + (int64_t)d.n_exact * 96 +
                    d.cap_batch * (int64_t)sizeof(GapBatchOut) + (1 << 16)) * gg;
      d.off_work = TW;
      TW += (d.cap_work + 255) & ~(int64_t)255;
    }
    Blob b;
    const size_t o_pl = b.add<PlannerDev>(1), o_q = b.add<GapQueryDev>(m), o_ph = b.add<double>(TM),
                 o_bl = b.add<int64_t>(TM), o_rm = b.add<int64_t>(TM), o_tr = b.add<int32_t>(TM),
                 o_ow = b.add<int32_t>(TM), in_bytes = b.bytes;
    const size_t o_ob = b.add<GapBatchOut>(TB), o_oo = b.add<int64_t>(2 * TO), o_wk = b.add<unsigned char>(TW),
                 o_out = b.add<GapOutDev>(m);
    cudaError_t e;
    if ((e = c.h_in.ensure(b.bytes)) != cudaSuccess || (e = c.d_in.ensure(b.bytes)) != cudaSuccess)
      return set_err(SLOS_ERR_CUDA, cudaGetErrorString(e));
    unsigned char* H = (unsigned char*)c.h_in.p;
    *(PlannerDev*)(H + o_pl) = p->dev;
    std::memcpy(H + o_q, qd.data(), sizeof(GapQueryDev) * m);
    double* ph = (double*)(H + o_ph);
    int64_t* bl = (int64_t*)(H + o_bl);
    int64_t* rm = (int64_t*)(H + o_rm);
    int32_t* tr = (int32_t*)(H + o_tr);
    int32_t* ow = (int32_t*)(H + o_ow);
    for (int x = 0; x < m; ++x) {
      const slos_gap_query& q = qs[todo[x]];
      for (int i = 0; i < qd[x].n_exact; ++i) {
        const int64_t o = qd[x].off_exact + i;
        ph[o] = q.exact[i].phase_s;
        bl[o] = q.exact[i].backlog;
        rm[o] = q.exact[i].remaining;
        tr[o] = q.exact[i].tier;
        ow[o] = q.exact[i].owner;
        if (q.exact[i].tier < 0 || q.exact[i].tier >= p->L) qd[x].mode = -1;
      }
    }
    unsigned char* D = (unsigned char*)c.d_in.p;
    cudaMemcpyAsync(D, H, in_bytes, cudaMemcpyHostToDevice, c.stream);
    GapParams gp;
    gp.planner = (const PlannerDev*)(D + o_pl);
    gp.q = (const GapQueryDev*)(D + o_q);
    gp.ph = (const double*)(D + o_ph);
    gp.bl = (const int64_t*)(D + o_bl);
    gp.rm = (const int64_t*)(D + o_rm);
    gp.tr = (const int32_t*)(D + o_tr);
    gp.ow = (const int32_t*)(D + o_ow);
    gp.ob = (GapBatchOut*)(D + o_ob);
    gp.oo = (int64_t*)(D + o_oo);
    gp.work = D + o_wk;
    gp.out = (GapOutDev*)(D + o_out);
    if ((e = launch_gap(gp, m, c.stream)) != cudaSuccess) return set_err(SLOS_ERR_CUDA, cudaGetErrorString(e));
    cudaMemcpyAsync(H + o_ob, D + o_ob, b.bytes - o_ob, cudaMemcpyDeviceToHost, c.stream);
    if ((e = cudaStreamSynchronize(c.stream)) != cudaSuccess) return set_err(SLOS_ERR_CUDA, cudaGetErrorString(e));
    const GapOutDev* ro = (const GapOutDev*)(H + o_out);
    const GapBatchOut* rb = (const GapBatchOut*)(H + o_ob);
    const int64_t* rown = (const int64_t*)(H + o_oo);
    std::vector<int> next;
    for (int x = 0; x < m; ++x) {
      const int k = todo[x];
      const GapOutDev& r = ro[x];
      slos_gap_result& o = outs[k];
      std::memset(&o, 0, sizeof o);
      if (r.status == SLOS_ERR_CAPACITY && grow[k] < 6) { ++grow[k]; next.push_back(k); continue; }
      o.status = r.status;
      if (r.status != SLOS_OK || !r.feasible) continue;
      o.feasible = 1;
      o.prefill_budget = r.budget;
      if (qs[k].mode == SLOS_GAP_PREFILL_BUDGET) continue;
      o.n_spec_lengths = r.n_spec;
      for (int l = 0; l < kMaxTiers; ++l) o.spec_lengths[l] = r.spec_lengths[l];
      const size_t bytes = sizeof(slos_gap_batch) * (size_t)r.n_batches + sizeof(int64_t) * 2 * (size_t)r.n_owner_pairs + 64;
      char* mem = (char*)std::calloc(1, bytes);
      slos_gap_batch* bs2 = (slos_gap_batch*)mem;
      int64_t* own = (int64_t*)(bs2 + r.n_batches);
      for (int64_t j = 0; j < r.n_batches; ++j) {
        const GapBatchOut& gb = rb[qd[x].off_out_batch + j];
        bs2[j].start_s = gb.start_s;
        bs2[j].end_s = gb.end_s;
        bs2[j].capacity_tokens = gb.capacity;
        bs2[j].spec_step = gb.spec_step;
        bs2[j].decode_tokens = gb.decode_tokens;
        bs2[j].prefill_budget = gb.prefill_budget;
        for (int l = 0; l < kMaxTiers; ++l) bs2[j].decode_per_tier[l] = gb.per_tier[l];
        bs2[j].first_owner = gb.first_owner;
        bs2[j].n_owners = gb.n_owner;
      }
      std::memcpy(own, rown + 2 * qd[x].off_out_owner, sizeof(int64_t) * 2 * (size_t)r.n_owner_pairs);
      o.n_batches = r.n_batches;
      o.batches = bs2;
      o.n_owner_pairs = r.n_owner_pairs;
      o.owner_tokens = own;
      o.owner_ = mem;
    }
    todo.swap(next);
  }
  for (int k : todo) outs[k].status = SLOS_ERR_CAPACITY;
  return SLOS_OK;
}

void slos_gap_result_free(slos_gap_result* r) {
  if (!r) return;
  std::free(r->owner_);
  std::memset(r, 0, sizeof *r);
}

static int small_call(slos_planner* p, int n, size_t in_bytes, const void* hin, size_t out_bytes,
                      void* hout, int kind, int64_t max_tokens) {
  Ctx& c = ctx();
  std::lock_guard<std::mutex> g(c.mu);
  int st = ensure_device(c);
  if (st != SLOS_OK) return set_err(st, c.why);
  Blob b;
  const size_t o_p = b.add<PlannerDev>(1), o_in = b.add<unsigned char>(in_bytes),
               o_out = b.add<unsigned char>(out_bytes);
  cudaError_t e;
  if ((e = c.d_small.ensure(b.bytes)) != cudaSuccess || (e = c.h_in.ensure(b.bytes)) != cudaSuccess)
    return set_err(SLOS_ERR_CUDA, cudaGetErrorString(e));
  unsigned char* H = (unsigned char*)c.h_in.p;
  unsigned char* D = (unsigned char*)c.d_small.p;
  *(PlannerDev*)(H + o_p) = p->dev;
  std::memcpy(H + o_in, hin, in_bytes);
  cudaMemcpyAsync(D, H, o_out, cudaMemcpyHostToDevice, c.stream);
  const PlannerDev* dP = (const PlannerDev*)(D + o_p);
  if (kind == 0) {  // time2bs: in = budgets[n] f64, spec[n] i64; out = res[n] i64, st[n] i32
    e = launch_time2bs(dP, n, (const double*)(D + o_in), (const int64_t*)(D + o_in + 8 * (size_t)n),
                       max_tokens, (int64_t*)(D + o_out), (int32_t*)(D + o_out + 8 * (size_t)n), c.stream);
  } else if (kind == 1) {  // predict
    e = launch_predict(dP, n, (const int64_t*)(D + o_in), (const int64_t*)(D + o_in + 8 * (size_t)n),
                       (double*)(D + o_out), (int32_t*)(D + o_out + 8 * (size_t)n), c.stream);
  } else {  // spec: in = counts[8], out = SpecSol
    e = launch_spec(dP, (const int64_t*)(D + o_in), D + o_out, c.stream);
  }
  if (e != cudaSuccess) return set_err(SLOS_ERR_CUDA, cudaGetErrorString(e));
  cudaMemcpyAsync(hout, D + o_out, out_bytes, cudaMemcpyDeviceToHost, c.stream);
  if ((e = cudaStreamSynchronize(c.stream)) != cudaSuccess) return set_err(SLOS_ERR_CUDA, cudaGetErrorString(e));
  return SLOS_OK;
}

int slos_time2bs_batch(slos_planner* p, int32_t n, const double* budget, const int64_t* spec,
                       int64_t max_tokens, int64_t* out, int32_t* status) {
  if (n <= 0) return SLOS_OK;
  std::vector<unsigned char> in(16 * (size_t)n), res(12 * (size_t)n);
  std::memcpy(in.data(), budget, 8 * (size_t)n);
  for (int k = 0; k < n; ++k) {
    const int64_t s = spec ? spec[k] : 0;
    std::memcpy(in.data() + 8 * (size_t)n + 8 * (size_t)k, &s, 8);
  }
  const int st = small_call(p, n, in.size(), in.data(), res.size(), res.data(), 0, max_tokens);
  if (st != SLOS_OK) {
    for (int k = 0; k < n; ++k) { out[k] = 0; status[k] = st; }
    return st;
  }
  std::memcpy(out, res.data(), 8 * (size_t)n);
  std::memcpy(status, res.data() + 8 * (size_t)n, 4 * (size_t)n);
  for (int k = 0; k < n; ++k)
    if (status[k] == SLOS_ERR_INFEASIBLE_BUDGET) set_err(status[k], "budget below single-token latency");
  return SLOS_OK;
}

int slos_predict_batch(slos_planner* p, int32_t n, const int64_t* tokens, const int64_t* spec, double* out) {
  if (n <= 0) return SLOS_OK;
  std::vector<unsigned char> in(16 * (size_t)n), res(12 * (size_t)n);
  std::memcpy(in.data(), tokens, 8 * (size_t)n);
  for (int k = 0; k < n; ++k) {
    const int64_t s = spec ? spec[k] : 0;
    std::memcpy(in.data() + 8 * (size_t)n + 8 * (size_t)k, &s, 8);
  }
  const int st = small_call(p, n, in.size(), in.data(), res.size(), res.data(), 1, 0);
  if (st != SLOS_OK) return st;
  std::memcpy(out, res.data(), 8 * (size_t)n);
  for (int k = 0; k < n; ++k) {
    int32_t s;
    std::memcpy(&s, res.data() + 8 * (size_t)n + 4 * (size_t)k, 4);
    if (s != SLOS_OK) return set_err(s, "predict needs nonnegative num_tokens and spec_step");
  }
  return SLOS_OK;
}

int slos_solve_spec_lengths(slos_planner* p, const int64_t* counts, int32_t n_tiers, double alpha,
                            int32_t max_len, slos_spec_plan* out) {
  std::memset(out, 0, sizeof *out);
  if (n_tiers != p->L) return set_err(SLOS_ERR_INVALID_PARAMETERS, "census width does not match tier count");
  if (alpha <= 0.0 || alpha > 1.0) return set_err(SLOS_ERR_INVALID_PARAMETERS, "alpha must be in (0, 1]");
  if (max_len < 1) return set_err(SLOS_ERR_INVALID_PARAMETERS, "spec_max_len must be >= 1");
  if (max_len > kMaxSpecLen || p->L > kMaxTiers) return set_err(SLOS_ERR_RANGE, "spec length / tiers");
  slos_planner tmp = *p;
  tmp.cfg.spec_alpha = alpha;
  tmp.cfg.spec_max_len = max_len;
  tmp.cfg.speculative = 1;
  fill_planner_dev(&tmp);
  int64_t c8[kMaxTiers] = {0};
  for (int l = 0; l < n_tiers; ++l) c8[l] = counts[l];
  std::vector<unsigned char> res(sizeof(SpecSolH) + 64);
  const int st = small_call(&tmp, 1, sizeof c8, c8, spec_sol_bytes(), res.data(), 2, 0);
  if (st != SLOS_OK) return st;
  SpecSolH sp;
  std::memcpy(&sp, res.data(), sizeof sp);
  if (sp.ok) {
    out->feasible = 1;
    for (int l = 0; l < kMaxTiers; ++l) out->lengths[l] = sp.lengths[l];
    out->batch_time_s = sp.bt;
    out->batch_capacity = sp.cap;
    out->decode_tokens = sp.decode;
    out->prefill_throughput = sp.tpt;
  }
  return SLOS_OK;
}


// ---- PerfModel::fit on the device (include/slos_fit.h) ----------------------
// The host checks the arguments (perf_model.cpp:134-140), forms the reference's
// initial regimes -- contiguous quantile bands of the (num_tokens, spec_step) order,
// the same std::sort call on the same input, hence the same permutation (:143-151)
// -- and orders the best terms at the end (:193-198); the iterations run in
// fit_kernel, one CTA per set.
int slos_perf_fit_batch(const slos_profile_sample* const* sets, const int32_t* n_samples, int32_t n_sets,
                        int32_t num_terms, int32_t max_iters, slos_perf_term* terms_out, int32_t* status) {
  g_err.clear();
  if (n_sets <= 0) return SLOS_OK;
  if (!sets || !n_samples || !terms_out || !status) return set_err(SLOS_ERR_INVALID_PARAMETERS, "null argument");
  if (num_terms < 1 || num_terms > SLOS_FIT_MAX_TERMS) {
    for (int k = 0; k < n_sets; ++k) status[k] = SLOS_ERR_INVALID_PARAMETERS;
    return set_err(SLOS_ERR_INVALID_PARAMETERS, "num_terms must be in [1, 32]");
  }
  Ctx& c = ctx();
  std::lock_guard<std::mutex> g(c.mu);
  int st = ensure_device(c);
  if (st != SLOS_OK) {
    for (int k = 0; k < n_sets; ++k) status[k] = st;
    return set_err(st, c.why);
  }
  const int T = num_terms;
  std::vector<FitSet> fs((size_t)n_sets);
  int64_t total = 0;
  for (int k = 0; k < n_sets; ++k) {
    fs[k].off = total;
    fs[k].n = std::max(0, n_samples[k]);
    fs[k].run = 0;
    total += fs[k].n;
  }
  std::vector<int64_t> nt((size_t)total), sp((size_t)total);
  std::vector<double> lat((size_t)total);
  std::vector<int32_t> assign((size_t)total);
  // per set (independent; the host worker pool takes them): checks, initial bands
  HostPool::get().run(n_sets, [&](int lo, int hi) {
  for (int k = lo; k < hi; ++k) {
    const int n = fs[k].n;
    const slos_profile_sample* x = sets[k];
    status[k] = SLOS_OK;
    if (n < 3 * T) { status[k] = SLOS_ERR_INSUFFICIENT_SAMPLES; continue; }  // "need at least 3 samples per term"
    {  // distinct num_tokens (the reference's std::set, :137-140)
      std::vector<int64_t> d((size_t)n);
      for (int i = 0; i < n; ++i) d[i] = x[i].num_tokens;
      std::sort(d.begin(), d.end());
      if ((int)(std::unique(d.begin(), d.end()) - d.begin()) < T) { status[k] = SLOS_ERR_DEGENERATE_SAMPLES; continue; }
    }
    std::vector<int> order((size_t)n);
    std::iota(order.begin(), order.end(), 0);
    std::sort(order.begin(), order.end(), [&](int a, int b) {
      if (x[a].num_tokens != x[b].num_tokens) return x[a].num_tokens < x[b].num_tokens;
      return x[a].spec_step < x[b].spec_step;
    });
    const int64_t o = fs[k].off;
    for (size_t r = 0; r < order.size(); ++r) assign[o + order[r]] = static_cast<int>(r * T / order.size());
    for (int i = 0; i < n; ++i) {
      nt[o + i] = x[i].num_tokens;
      sp[o + i] = x[i].spec_step;
      lat[o + i] = x[i].latency_s;
    }
    fs[k].run = 1;
  }
  });
  Blob b;
  const size_t o_set = b.add<FitSet>(n_sets), o_nt = b.add<int64_t>(total), o_ss = b.add<int64_t>(total),
               o_lat = b.add<double>(total), o_as = b.add<int32_t>(total), o_e2 = b.add<double>(total),
               o_nd = b.add<double>(total), o_sd = b.add<double>(total),
               o_out = b.add<double>((size_t)n_sets * T * 3), o_ok = b.add<int32_t>(n_sets);
  cudaError_t e;
  if ((e = c.d_fit.ensure(b.bytes)) != cudaSuccess || (e = c.h_fit.ensure(b.bytes)) != cudaSuccess)
    return set_err(SLOS_ERR_CUDA, cudaGetErrorString(e));
  unsigned char* D = (unsigned char*)c.d_fit.p;
  unsigned char* H = (unsigned char*)c.h_fit.p;  // pinned: inputs in, best terms out
  std::memcpy(H + o_set, fs.data(), sizeof(FitSet) * fs.size());
  if (total) {
    std::memcpy(H + o_nt, nt.data(), 8 * (size_t)total);
    std::memcpy(H + o_ss, sp.data(), 8 * (size_t)total);
    std::memcpy(H + o_lat, lat.data(), 8 * (size_t)total);
    std::memcpy(H + o_as, assign.data(), 4 * (size_t)total);
  }
  cudaMemcpyAsync(D, H, o_e2, cudaMemcpyHostToDevice, c.stream);
  cudaMemsetAsync(D + o_ok, 0, 4 * (size_t)n_sets, c.stream);
  FitParams prm;
  prm.sets = (const FitSet*)(D + o_set);
  prm.nt = (const int64_t*)(D + o_nt);
  prm.ss = (const int64_t*)(D + o_ss);
  prm.lat = (double*)(D + o_lat);
  prm.nd = (double*)(D + o_nd);
  prm.sd = (double*)(D + o_sd);
  // per sample in shared memory: num_tokens, spec_step, latency, residual (f64) and regime (i32)
  constexpr size_t kPerSample = 4 * sizeof(double) + sizeof(int32_t);
  int max_n = 0;
  for (const FitSet& f : fs) max_n = std::max(max_n, f.n);
  const size_t cap = std::min<size_t>(c.smem_optin, 200 * 1024) / kPerSample;
  prm.smem_samples = (int)std::min<size_t>((size_t)max_n, cap);
  const size_t fit_smem = (size_t)prm.smem_samples * kPerSample + 16;
  prm.assign = (int32_t*)(D + o_as);
  prm.e2 = (double*)(D + o_e2);
  prm.out = (double*)(D + o_out);
  prm.ok = (int32_t*)(D + o_ok);
  prm.T = T;
  prm.max_iters = max_iters;
  e = launch_fit(prm, n_sets, fit_smem, c.stream);
  if (e == cudaSuccess) {
    cudaMemcpyAsync(H + o_out, D + o_out, b.bytes - o_out, cudaMemcpyDeviceToHost, c.stream);
    e = cudaStreamSynchronize(c.stream);
  }
  if (e != cudaSuccess) return set_err(SLOS_ERR_CUDA, cudaGetErrorString(e));
  const double* out = (const double*)(H + o_out);
  const int32_t* ok = (const int32_t*)(H + o_ok);
  for (int k = 0; k < n_sets; ++k) {
    slos_perf_term* t = terms_out + (size_t)k * T;
    if (status[k] != SLOS_OK || !ok[k]) {
      // no iteration improved on +inf (NaN residuals): the reference's PerfModel
      // rejects the empty term list as invalid parameters (perf_model.cpp:97)
      if (status[k] == SLOS_OK) status[k] = SLOS_ERR_INVALID_PARAMETERS;
      for (int q = 0; q < T; ++q) t[q] = slos_perf_term{0.0, 0.0, 0.0};
      continue;
    }
    for (int q = 0; q < T; ++q) {
      const double* x = &out[((size_t)k * T + q) * 3];
      t[q] = slos_perf_term{x[0], x[1], x[2]};
    }
    std::sort(t, t + T, [](const slos_perf_term& a, const slos_perf_term& b) {
      if (a.k1 != b.k1) return a.k1 < b.k1;
      if (a.k2 != b.k2) return a.k2 < b.k2;
      return a.b < b.b;
    });
  }
  return SLOS_OK;
}
}  // extern "C"

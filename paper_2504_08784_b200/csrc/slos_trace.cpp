// Batched synthetic trace generation (include/slos_trace.h).
//
// One job = scale_scenario + generate_trace of the reference (metrics.cpp:214-221,
// workload.cpp:113-206). Jobs are independent: a pool of host threads takes them
// from an atomic counter, each job sampling into thread-local vectors that are
// copied once into one allocation owned by its slos_trace.
//
// Exactness. The reference draws from std::mt19937_64 through libstdc++'s
// distributions; the same engine and distribution objects are used here, created
// at the same points (a fresh normal_distribution per lognormal draw, so the polar
// method's spare value is never reused, workload.cpp:119; a fresh one per tool
// request's pair count, :186) and consumed in the same order (arrivals from
// seed ^ 0x9e3779b97f4a7c15, then lengths from `seed`; for a tool stage pair the
// delay draw precedes the prompt draw, :190-192). Scalar arithmetic keeps the
// reference's expressions term by term (built with -ffp-contract=off).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <random>
#include <thread>
#include <vector>

#include "../../include/slos_planner.h"
#include "../../include/slos_trace.h"

namespace {

constexpr int64_t kKvBlockTokens = 16;  // workload.hpp:49

struct Dist {
  double mean, std;
};

// workload.cpp:86-109 (+ SloConfig::validate :16-29), first failing check wins
int validate(const slos_scenario& s) {
  if (s.n_tiers <= 0 || !s.tpot_tiers_s || !s.ttft_slowdowns) return SLOS_ERR_INVALID_PARAMETERS;
  for (int i = 0; i < s.n_tiers; ++i) {
    if (s.tpot_tiers_s[i] <= 0) return SLOS_ERR_INVALID_PARAMETERS;
    if (i > 0 && s.tpot_tiers_s[i] < s.tpot_tiers_s[i - 1]) return SLOS_ERR_INVALID_PARAMETERS;
    if (s.ttft_slowdowns[i] < 1.0) return SLOS_ERR_INVALID_PARAMETERS;
  }
  if (s.tpot_window < 1) return SLOS_ERR_INVALID_PARAMETERS;
  if (s.rate_per_s <= 0) return SLOS_ERR_INVALID_DISTRIBUTION;
  if (s.process != SLOS_ARRIVAL_POISSON && s.process != SLOS_ARRIVAL_BURSTY) return SLOS_ERR_INVALID_PARAMETERS;
  if (s.process == SLOS_ARRIVAL_BURSTY && (s.on_multiplier < 1 || s.mean_on_s <= 0 || s.mean_off_s <= 0))
    return SLOS_ERR_INVALID_DISTRIBUTION;
  auto bad = [](double mean, double sd) { return mean < 1 || sd < 0; };
  if (bad(s.prompt_mean, s.prompt_std)) return SLOS_ERR_INVALID_DISTRIBUTION;
  if ((s.shape == SLOS_SHAPE_SINGLE || s.shape == SLOS_SHAPE_TOOL) && bad(s.output_mean, s.output_std))
    return SLOS_ERR_INVALID_DISTRIBUTION;
  if (s.shape == SLOS_SHAPE_REASONING) {
    if (bad(s.think_mean, s.think_std)) return SLOS_ERR_INVALID_DISTRIBUTION;
    if (bad(s.response_mean, s.response_std)) return SLOS_ERR_INVALID_DISTRIBUTION;
  }
  if (s.shape != SLOS_SHAPE_SINGLE && s.shape != SLOS_SHAPE_REASONING && s.shape != SLOS_SHAPE_TOOL)
    return SLOS_ERR_INVALID_PARAMETERS;
  if (s.shape == SLOS_SHAPE_TOOL && (s.tool_delay_min_s < 0 || s.tool_delay_max_s < s.tool_delay_min_s))
    return SLOS_ERR_INVALID_DISTRIBUTION;
  if (s.memory_overprovision < 1.0) return SLOS_ERR_INVALID_PARAMETERS;
  return SLOS_OK;
}

// workload.cpp:113-123
int64_t lognormal_tokens(const Dist& d, std::mt19937_64& rng) {
  if (d.std <= 0.0) return std::max<int64_t>(1, llround(d.mean));
  const double cv2 = (d.std * d.std) / (d.mean * d.mean);
  const double sigma2 = std::log1p(cv2);
  const double mu = std::log(d.mean) - 0.5 * sigma2;
  std::normal_distribution<double> norm(mu, std::sqrt(sigma2));
  const double v = std::exp(norm(rng));
  return std::max<int64_t>(1, llround(v));
}

// workload.cpp:125-157
void arrivals(const slos_scenario& s, double rate, double mean_on, uint64_t seed, double duration,
              std::vector<double>& out) {
  std::mt19937_64 rng(seed ^ 0x9e3779b97f4a7c15ULL);
  double t = 0.0;
  if (s.process == SLOS_ARRIVAL_POISSON) {
    std::exponential_distribution<double> gap(rate);
    for (t = gap(rng); t < duration; t += gap(rng)) out.push_back(t);
    return;
  }
  // alternating off / on phases; the pending gap is dropped at a phase flip
  std::exponential_distribution<double> on_len(1.0 / mean_on);
  std::exponential_distribution<double> off_len(1.0 / s.mean_off_s);
  std::uniform_real_distribution<double> uni(0.0, 1.0);
  bool on = false;
  double phase_end = off_len(rng);
  while (t < duration) {
    const double r = on ? rate * s.on_multiplier : rate;
    const double gap = -std::log(1.0 - uni(rng)) / r;
    if (t + gap >= phase_end) {
      t = phase_end;
      on = !on;
      phase_end = t + (on ? on_len(rng) : off_len(rng));
      continue;
    }
    t += gap;
    if (t < duration) out.push_back(t);
  }
}

struct Scratch {
  std::vector<double> arr;
  std::vector<slos_trace_request> req;
  std::vector<slos_trace_stage> st;
};

int run_job(const slos_trace_job& jb, Scratch& w) {
  if (!jb.scenario) return SLOS_ERR_INVALID_PARAMETERS;
  const slos_scenario& s = *jb.scenario;
  // scale_scenario (metrics.cpp:214-221)
  if (jb.rate_scale <= 0) return SLOS_ERR_INVALID_PARAMETERS;
  const double rate = s.rate_per_s * jb.rate_scale;
  const double mean_on = s.process == SLOS_ARRIVAL_BURSTY ? s.mean_on_s / jb.rate_scale : s.mean_on_s;
  slos_scenario sc = s;
  sc.rate_per_s = rate;
  sc.mean_on_s = mean_on;
  int st = validate(sc);
  if (st != SLOS_OK) return st;
  if (jb.duration_s <= 0) return SLOS_ERR_INVALID_PARAMETERS;
  w.arr.clear();
  w.req.clear();
  w.st.clear();
  arrivals(sc, rate, mean_on, jb.seed, jb.duration_s, w.arr);
  std::mt19937_64 rng(jb.seed);
  const Dist prompt{s.prompt_mean, s.prompt_std}, output{s.output_mean, s.output_std};
  const Dist think{s.think_mean, s.think_std}, response{s.response_mean, s.response_std};
  w.req.reserve(w.arr.size());
  for (size_t i = 0; i < w.arr.size(); ++i) {
    slos_trace_request r;
    r.arrival_s = w.arr[i];
    r.value = s.value;
    r.first_stage = (int32_t)w.st.size();
    auto stage = [&](int kind, int64_t tokens, int tier, double delay) {
      slos_trace_stage x;
      x.kind = kind;
      x.tokens = tokens;
      x.slo_tier = tier;
      x.external_delay_s = delay;
      w.st.push_back(x);
    };
    if (s.shape == SLOS_SHAPE_SINGLE) {
      stage(0, lognormal_tokens(prompt, rng), s.prefill_tier, 0.0);
      stage(1, lognormal_tokens(output, rng), s.decode_tier, 0.0);
    } else if (s.shape == SLOS_SHAPE_REASONING) {
      stage(0, lognormal_tokens(prompt, rng), s.prefill_tier, 0.0);
      stage(1, lognormal_tokens(think, rng), s.think_tier, 0.0);
      stage(1, lognormal_tokens(response, rng), s.response_tier, 0.0);
    } else {
      std::normal_distribution<double> pairs_dist(s.tool_pairs_mean, s.tool_pairs_std);
      const int pairs = std::max(1, static_cast<int>(llround(pairs_dist(rng))));
      std::uniform_real_distribution<double> delay(s.tool_delay_min_s, s.tool_delay_max_s);
      for (int p = 0; p < pairs; ++p) {
        const double d = p == 0 ? 0.0 : delay(rng);
        stage(0, lognormal_tokens(prompt, rng), s.prefill_tier, d);
        stage(1, lognormal_tokens(output, rng), s.decode_tier, 0.0);
      }
    }
    r.n_stages = (int32_t)(w.st.size() - (size_t)r.first_stage);
    // derive_memory_units (workload.cpp:69-73)
    int64_t total = 0;
    for (int k = 0; k < r.n_stages; ++k) total += w.st[(size_t)r.first_stage + k].tokens;
    const double tokens = static_cast<double>(total) * s.memory_overprovision;
    r.memory_units = static_cast<int64_t>(std::ceil(tokens / static_cast<double>(kKvBlockTokens)));
    // RequestSpec::validate (workload.cpp:51-67)
    if (r.arrival_s < 0 || r.value <= 0) return SLOS_ERR_INVARIANT;
    for (int k = 0; k < r.n_stages; ++k) {
      const slos_trace_stage& x = w.st[(size_t)r.first_stage + k];
      if (x.tokens < 1 || x.slo_tier < 0 || x.slo_tier >= s.n_tiers || x.external_delay_s < 0)
        return SLOS_ERR_INVARIANT;
    }
    w.req.push_back(r);
  }
  return SLOS_OK;
}

}  // namespace

extern "C" {

int slos_trace_batch(const slos_trace_job* jobs, int32_t n, int32_t threads, slos_trace* outs) {
  if (n < 0 || (n > 0 && (!jobs || !outs))) return SLOS_ERR_INVALID_PARAMETERS;
  for (int k = 0; k < n; ++k) std::memset(&outs[k], 0, sizeof(slos_trace));
  int T = threads > 0 ? threads : (int)std::max(1u, std::thread::hardware_concurrency());
  T = std::max(1, std::min(T, n));
  std::atomic<int> next{0};
  auto worker = [&] {
    Scratch w;
    for (;;) {
      const int k = next.fetch_add(1);
      if (k >= n) break;
      slos_trace& o = outs[k];
      o.status = run_job(jobs[k], w);
      if (o.status != SLOS_OK) continue;
      const size_t rb = sizeof(slos_trace_request) * w.req.size();
      const size_t sb = sizeof(slos_trace_stage) * w.st.size();
      unsigned char* mem = (unsigned char*)std::malloc(std::max<size_t>(1, rb + sb));
      if (!mem) { o.status = SLOS_ERR_ALLOC; continue; }
      // stages first: 8-byte aligned at the allocation's start for both records
      o.stages = (slos_trace_stage*)mem;
      o.requests = (slos_trace_request*)(mem + sb);
      if (sb) std::memcpy(o.stages, w.st.data(), sb);
      if (rb) std::memcpy(o.requests, w.req.data(), rb);
      o.n_requests = (int32_t)w.req.size();
      o.n_stages = (int64_t)w.st.size();
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < T; ++t) pool.emplace_back(worker);
  worker();
  for (auto& th : pool) th.join();
  return SLOS_OK;
}

void slos_trace_free(slos_trace* t) {
  if (!t) return;
  std::free(t->stages);  // one allocation: stages, then requests
  std::memset(t, 0, sizeof *t);
}

}  // extern "C"

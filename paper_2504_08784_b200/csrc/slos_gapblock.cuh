// Block-level full gap tiler: BatchPlanner::tile_gap / tile_gap_ar with the
// complete GapPlan (per-slot batches, per-owner decode tokens, per-tier canonical
// tokens, speculative lengths) -- batch_planner.cpp:152-406. Used by plan
// reconstruction (build_plan, dp_scheduler.cpp:196-354) and by the standalone
// slos_tile_gap_batch entry point (K1).
//
// Placement without materialising a sorted due list:
//   late dues fill slots first-fit in insertion order, so member m's late dues
//   occupy the global positions [P_m, P_m + l_m) of the cumulative capacity;
//   non-late dues form jit groups processed in slot order; thread 0 replays the
//   latest-fit stack over GROUP COUNTS, producing for every group its ordered
//   list of (slot, amount) segments. A single-segment group sends every one of
//   its dues to that slot, whatever their order. Only groups that spill over
//   several slots need their dues in (time, insertion) order: those few dues are
//   gathered and sorted (bitonic, block-wide) and dealt along the segments.
// Per-(slot, member) token counts are then emitted slot-major, owners ascending
// (the std::map order of batch_planner.cpp:258/306).
#pragma once

#include "slos_common.cuh"

namespace slos {

#ifndef SLOS_BT
#define SLOS_BT 512
#endif
constexpr int kBT = SLOS_BT;  // largest cooperating group of the build / gap kernels
constexpr int kBW = kBT / 32;  // BlockShared capacity: groups of up to kBT threads

struct MemBuf {  // exact census members (SoA), census order
  double* ph;
  int64_t* bl;
  int64_t* rm;
  int32_t* tr;
  int32_t* ow;
  int M;
};

struct GapBatchOut {
  double start_s, end_s;
  int64_t capacity, spec_step, decode_tokens, prefill_budget;
  int64_t per_tier[kMaxTiers];
  int32_t first_owner, n_owner;
};

struct GapPlanBuf {  // output of one tile_gap call
  GapBatchOut* b;
  int32_t cap_b;
  int32_t n_b;
  int64_t* own;   // (owner, tok) pairs
  int32_t cap_own;
  int32_t n_own;
  int32_t feasible;
  int32_t status;
  int64_t budget;
  int32_t n_spec;
  int32_t spec[kMaxTiers];
  int64_t need_b, need_own, need_work;
};

struct BlockShared {  // shared scratch of one cooperating group (a CTA or a warp)
  int64_t r64[kBW + 2];
  double rd[kBW + 2];
  int32_t r32[kBW + 2];
  int S;
  int flag;
  int flag2;
  int64_t v64a, v64b;
  double vd;
  SpecSol sp;
  int64_t mb[2][kBW][4];  // double-buffered per-warp totals of mscan (one barrier per call)
};

// Cooperative-group policies: the same engine runs on a whole CTA (BlockGrp,
// standalone gap queries) or on one warp (WarpGrp, plan reconstruction: one
// instance per warp, no CTA barriers).
template <int NT>
struct BlockGrpT {
  static constexpr int kSize = NT;
  static constexpr int kW = NT / 32;
  __device__ static int rank() { return threadIdx.x; }
  __device__ static void sync() { __syncthreads(); }
  __device__ static bool leader_warp() { return warp_id() == 0; }
  __device__ static int64_t sum64(BlockShared& sh, int64_t v) {
    v = warp_sum(v);
    __syncthreads();
    if (lane_id() == 0) sh.r64[warp_id()] = v;
    __syncthreads();
    int64_t t = 0;
    for (int w = 0; w < kW; ++w) t += sh.r64[w];
    __syncthreads();
    return t;
  }
  __device__ static int or_(BlockShared& sh, int v) {
    v = __reduce_or_sync(0xffffffffu, (unsigned)v);
    __syncthreads();
    if (lane_id() == 0) sh.r32[warp_id()] = v;
    __syncthreads();
    int t = 0;
    for (int w = 0; w < kW; ++w) t |= sh.r32[w];
    __syncthreads();
    return t;
  }
  __device__ static double max(BlockShared& sh, double v) {
    for (int o = 16; o; o >>= 1) { const double y = __shfl_xor_sync(0xffffffffu, v, o); v = dmax(v, y); }
    __syncthreads();
    if (lane_id() == 0) sh.rd[warp_id()] = v;
    __syncthreads();
    double t = sh.rd[0];
    for (int w = 1; w < kW; ++w) t = dmax(t, sh.rd[w]);
    __syncthreads();
    return t;
  }
  __device__ static double min(BlockShared& sh, double v) {
    for (int o = 16; o; o >>= 1) { const double y = __shfl_xor_sync(0xffffffffu, v, o); v = dmin(v, y); }
    __syncthreads();
    if (lane_id() == 0) sh.rd[warp_id()] = v;
    __syncthreads();
    double t = sh.rd[0];
    for (int w = 1; w < kW; ++w) t = dmin(t, sh.rd[w]);
    __syncthreads();
    return t;
  }
  // K simultaneous exclusive scans with ONE barrier: per-warp totals go to the
  // buffer `par` (alternating per call, so a buffer is rewritten only after every
  // thread has passed the barrier of the call in between, i.e. finished reading it).
  template <int K>
  __device__ static void mscan(BlockShared& sh, const int64_t* v, int64_t* ex, int64_t* tot, int& par) {
    int64_t inc[K];
#pragma unroll
    for (int k = 0; k < K; ++k) inc[k] = warp_incl_scan(v[k]);
    if (lane_id() == 31) {
#pragma unroll
      for (int k = 0; k < K; ++k) sh.mb[par][warp_id()][k] = inc[k];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; ++k) {
      int64_t base = 0, t = 0;
      for (int w = 0; w < kW; ++w) {
        const int64_t x = sh.mb[par][w][k];
        if (w < warp_id()) base += x;
        t += x;
      }
      ex[k] = base + inc[k] - v[k];
      tot[k] = t;
    }
    par ^= 1;
  }
  // exclusive scan (one value per thread); *tot = group total
  __device__ static int64_t excl(BlockShared& sh, int64_t v, int64_t* tot) {
    const int64_t inc = warp_incl_scan(v);
    __syncthreads();
    if (lane_id() == 31) sh.r64[warp_id()] = inc;
    __syncthreads();
    int64_t base = 0, t = 0;
    for (int w = 0; w < kW; ++w) {
      if (w < warp_id()) base += sh.r64[w];
      t += sh.r64[w];
    }
    __syncthreads();
    *tot = t;
    return base + inc - v;
  }
};

using BlockGrp = BlockGrpT<kBT>;

struct WarpGrp {
  static constexpr int kSize = 32;
  __device__ static int rank() { return lane_id(); }
  __device__ static void sync() { __syncwarp(); }
  __device__ static bool leader_warp() { return true; }
  __device__ static int64_t sum64(BlockShared&, int64_t v) { return warp_sum(v); }
  __device__ static int or_(BlockShared&, int v) { return (int)__reduce_or_sync(0xffffffffu, (unsigned)v); }
  __device__ static double max(BlockShared&, double v) {
    for (int o = 16; o; o >>= 1) { const double y = __shfl_xor_sync(0xffffffffu, v, o); v = dmax(v, y); }
    return v;
  }
  __device__ static double min(BlockShared&, double v) {
    for (int o = 16; o; o >>= 1) { const double y = __shfl_xor_sync(0xffffffffu, v, o); v = dmin(v, y); }
    return v;
  }
  __device__ static int64_t excl(BlockShared&, int64_t v, int64_t* tot) {
    const int64_t inc = warp_incl_scan(v);
    *tot = __shfl_sync(0xffffffffu, inc, 31);
    __syncwarp();
    return inc - v;
  }
  template <int K>
  __device__ static void mscan(BlockShared&, const int64_t* v, int64_t* ex, int64_t* tot, int&) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int64_t inc = warp_incl_scan(v[k]);
      tot[k] = __shfl_sync(0xffffffffu, inc, 31);
      ex[k] = inc - v[k];
    }
    __syncwarp();
  }
};

// Two-level bump allocator: a primary region (shared memory when the caller has
// one) and a secondary global-memory work area for whatever does not fit. Every
// thread of a group performs the same takes, so all agree on the placement.
struct Arena {
  unsigned char* base;   // primary
  int64_t cap;
  int64_t used;
  unsigned char* base2;  // secondary (global), may be null
  int64_t cap2;
  int64_t used2;
  __device__ void* take(int64_t bytes) {
    const int64_t o = (used + 15) & ~(int64_t)15;
    if (o + bytes <= cap || !base2) {
      used = o + bytes;
      return base + o;
    }
    const int64_t o2 = (used2 + 15) & ~(int64_t)15;
    used2 = o2 + bytes;
    return base2 + o2;
  }
  __device__ bool over() const { return used > cap || (base2 && used2 > cap2); }
  __device__ int64_t need() const { return 2 * ((base2 ? used2 : used) + 1024); }
};

// Multi-segment group due record, ordered by (time, insertion key).
struct MRec {
  double time;
  uint64_t key;   // exact: (m << 32 | k); canonical: (1<<63) | (l << 40) | t
  int32_t grp;
  int32_t who;    // member index, or -1-l for canonical tier l
  int64_t w;      // multiplicity (canonical: counts[l])
};

__device__ __forceinline__ bool mrec_less(const MRec& a, const MRec& b) {
  if (a.grp != b.grp) return a.grp < b.grp;
  if (a.time < b.time) return true;
  if (b.time < a.time) return false;
  return a.key < b.key;
}

// block bitonic sort over n records (n padded to pow2 with +inf sentinels)
template <class G>
__device__ inline void blk_sort_mrec(MRec* r, int n_pow2) {
  for (int k = 2; k <= n_pow2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = G::rank(); i < n_pow2; i += G::kSize) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const bool up = (i & k) == 0;
          MRec a = r[i], b = r[ixj];
          const bool sw = up ? mrec_less(b, a) : mrec_less(a, b);
          if (sw) { r[i] = b; r[ixj] = a; }
        }
      }
      G::sync();
    }
  }
}

// prefill_only (batch_planner.cpp:177-195), thread 0 writes batches.
__device__ __noinline__ int gap_prefill_only(const PlannerDev& P, double gap, double min_slot,
                                       GapPlanBuf& o) {
  double t = 0.0;
  const int64_t Cfull = imin(P.max_chunk, P.max_batch);  // see prefill_only_budget
  const double predC = predict(P, Cfull, 0);
  for (long guard = 0; gap - t >= min_slot - kTimeEps; ++guard) {
    int64_t size;
    if (time_le(predC, (gap - t) / P.margin1)) {
      size = Cfull;
    } else {
      size = plan_time2bs(P, gap - t, 0);
      if (size < 0) return SLOS_ERR_INFEASIBLE_BUDGET;
    }
    if (guard > 100000000L) return SLOS_ERR_INTERNAL_INCONSISTENCY;
    size = imin(size, P.max_chunk);
    const double dur = plan_predict(P, size, 0);
    if (o.n_b < o.cap_b) {
      GapBatchOut& b = o.b[o.n_b];
      b.start_s = t;
      b.end_s = t + dur;
      b.capacity = size;
      b.spec_step = 0;
      b.decode_tokens = 0;
      b.prefill_budget = size;
      for (int l = 0; l < kMaxTiers; ++l) b.per_tier[l] = 0;
      b.first_owner = o.n_own;
      b.n_owner = 0;
    }
    o.n_b++;
    o.budget += size;
    t += dur;
  }
  return 0;
}

// tile_gap_ar with full output. Block-wide; all threads must call. Returns in o
// (feasible/status). `E` holds the exact members; counts c[L] the canonical ones.
// owners_sorted: member owners strictly ascending (true for build_plan censuses).
template <class G>
__device__ inline void block_tile_gap_ar(const PlannerDev& P, BlockShared& sh, double gap,
                                         double dh, const int64_t* c, const MemBuf& E,
                                         bool owners_sorted, Arena ar, GapPlanBuf& o) {
  const int tid = G::rank();
  const int L = P.L;
  const int M = E.M;
  if (tid == 0) { o.n_b = 0; o.n_own = 0; o.budget = 0; o.feasible = 0; o.status = 0; o.n_spec = 0; }
  G::sync();
  const double horizon = dmax(gap, dh);
  if (gap <= kTimeEps) {  // :156-164
    int any = 0;
    for (int m = tid; m < M; m += G::kSize) {
      if (E.rm[m] <= 0) continue;
      if (E.bl[m] > 0) any = 1;
      if (horizon > kTimeEps && time_le(E.ph[m], horizon)) any = 1;
    }
    any = G::or_(sh, any);
    if (tid == 0) o.feasible = any ? 0 : 1;
    G::sync();
    return;
  }
  const double min_slot = plan_predict(P, 1, 0);
  unsigned cmask = 0;
  for (int l = 0; l < L; ++l) if (c[l] > 0) cmask |= 1u << l;
  int em = 0;
  for (int m = tid; m < M; m += G::kSize) if (E.rm[m] > 0) em |= 1 << E.tr[m];
  const unsigned present = (unsigned)G::or_(sh, em) | cmask;
  if (!present) {
    if (tid == 0) { o.status = gap_prefill_only(P, gap, min_slot, o); o.feasible = o.status == 0; }
    G::sync();
    return;
  }
  // per-member due counts (late l_m, non-late), spill not needed here
  int64_t* lcount = (int64_t*)ar.take(sizeof(int64_t) * (M + 1));
  int64_t* lpre = (int64_t*)ar.take(sizeof(int64_t) * (M + 1));
  if (ar.over()) {
    if (tid == 0) { o.status = SLOS_ERR_CAPACITY; o.need_work = ar.need(); }
    G::sync();
    return;
  }
  int64_t nd = 0;
  for (int m = tid; m < M; m += G::kSize) {
    int64_t late = 0, nl = 0;
    const int64_t rem = E.rm[m];
    if (rem > 0) {
      int64_t issued = E.bl[m] > 0 ? imin(E.bl[m], rem) : 0;
      late = issued;
      const double tpot = P.tpot[E.tr[m]];
      for (double d = dmax(E.ph[m], 0.0); time_le(d, horizon) && issued < rem; d += tpot, ++issued) {
        if (d <= kTimeEps) ++late; else ++nl;
      }
    }
    lcount[m] = late;
    nd += late + nl;
  }
  int q[kMaxTiers];
  for (int l = 0; l < L; ++l) {
    int n = 0;
    for (double d = P.tpot[l]; time_le(d, gap); d += P.tpot[l]) ++n;
    q[l] = n;
    nd += (tid == 0) ? c[l] * (int64_t)n : 0;
  }
  const int64_t D = G::sum64(sh, nd);
  if (D == 0) {  // :223
    if (tid == 0) { o.status = gap_prefill_only(P, gap, min_slot, o); o.feasible = o.status == 0; }
    G::sync();
    return;
  }
  const double t0 = P.tpot[__ffs(present) - 1];
  if (min_slot > t0 + kTimeEps) return;  // :231 (feasible = 0)
  // t0_first (:234-239): ordered scan by warp 0
  if (G::leader_warp()) {
    double cur = t0;
    for (int base = 0; base < M; base += 32) {
      const int m = base + lane_id();
      const bool ok = m < M && E.rm[m] > 0 && E.ph[m] > kTimeEps;
      const double ph = ok ? E.ph[m] : 0.0;
      unsigned above = 0xffffffffu;
      for (;;) {
        const unsigned qq = __ballot_sync(0xffffffffu, ok && ph < cur - kTimeEps) & above;
        if (!qq) break;
        const int f = __ffs(qq) - 1;
        cur = dmax(__shfl_sync(0xffffffffu, ph, f), min_slot);
        above = (f == 31) ? 0u : (0xffffffffu << (f + 1));
      }
    }
    if (lane_id() == 0) sh.vd = cur;
  }
  G::sync();
  const double t0_first = sh.vd;
  // slot ends (thread 0): count first, then fill
  if (tid == 0) {
    int S = 0;
    double last = 0.0;
    for (double e = t0_first; time_le(e, gap); e += t0) { last = e; ++S; }
    if (S == 0) { if (time_le(min_slot, gap)) ++S; }
    else if (gap - last >= min_slot - kTimeEps) ++S;
    sh.S = S;
  }
  G::sync();
  const int S = sh.S;
  if (S == 0) return;  // :248
  double* ends = (double*)ar.take(sizeof(double) * S);
  int64_t* cap = (int64_t*)ar.take(sizeof(int64_t) * S);
  int64_t* fr = (int64_t*)ar.take(sizeof(int64_t) * S);     // free capacity (evolving)
  int64_t* ng = (int64_t*)ar.take(sizeof(int64_t) * S);     // group due counts
  int32_t* seg0 = (int32_t*)ar.take(sizeof(int32_t) * (S + 1));
  int32_t* sslot = (int32_t*)ar.take(sizeof(int32_t) * (2 * S + 2));
  int64_t* samt = (int64_t*)ar.take(sizeof(int64_t) * (2 * S + 2));
  int32_t* tok = (int32_t*)ar.take(sizeof(int32_t) * (int64_t)S * (M + 1));
  int64_t* ptier = (int64_t*)ar.take(sizeof(int64_t) * (int64_t)S * L);
  if (ar.over()) {
    if (tid == 0) { o.status = SLOS_ERR_CAPACITY; o.need_work = ar.need(); }
    G::sync();
    return;
  }
  if (tid == 0) {
    int s = 0;
    double last = 0.0;
    for (double e = t0_first; time_le(e, gap); e += t0) { ends[s++] = e; last = e; }
    if (s == 0) { if (time_le(min_slot, gap)) ends[s++] = gap; }
    else if (gap - last >= min_slot - kTimeEps) ends[s++] = gap;
  }
  G::sync();
  int cerr = 0;
  for (int s = tid; s < S; s += G::kSize) {  // :250-255
    const double dur = ends[s] - (s == 0 ? 0.0 : ends[s - 1]);
    const int64_t cc = plan_time2bs(P, dur, 0);
    if (cc < 0) cerr = 1;
    cap[s] = imin(cc, P.max_batch);
    ng[s] = 0;
  }
  for (int64_t x = tid; x < (int64_t)S * (M + 1); x += G::kSize) tok[x] = 0;
  for (int64_t x = tid; x < (int64_t)S * L; x += G::kSize) ptier[x] = 0;
  cerr = G::or_(sh, cerr);
  if (cerr) {
    if (tid == 0) o.status = SLOS_ERR_INFEASIBLE_BUDGET;
    G::sync();
    return;
  }
  // jit histogram of non-late dues (exact + canonical)
  int fail = 0;
  for (int m = tid; m < M; m += G::kSize) {
    const int64_t rem = E.rm[m];
    if (rem <= 0) continue;
    int64_t issued = E.bl[m] > 0 ? imin(E.bl[m], rem) : 0;
    const double tpot = P.tpot[E.tr[m]];
    for (double d = dmax(E.ph[m], 0.0); time_le(d, horizon) && issued < rem; d += tpot, ++issued) {
      if (d <= kTimeEps) continue;
      const int jit = jit_search(ends, S, d);
      if (jit < 0) fail = 1; else atomicAdd((unsigned long long*)&ng[jit], 1ull);
    }
  }
  if (tid < L && c[tid] > 0) {
    for (double d = P.tpot[tid]; time_le(d, gap); d += P.tpot[tid]) {
      const int jit = jit_search(ends, S, d);
      if (jit < 0) fail = 1; else atomicAdd((unsigned long long*)&ng[jit], (unsigned long long)c[tid]);
    }
  }
  // late prefix over members (insertion order)
  {
    int64_t carry = 0;
    for (int base = 0; base < M; base += G::kSize) {
      const int m = base + tid;
      int64_t tot;
      const int64_t ex = G::excl(sh, m < M ? lcount[m] : 0, &tot);
      if (m < M) lpre[m] = carry + ex;
      carry += tot;
    }
    if (tid == 0) sh.v64a = carry;
  }
  fail = G::or_(sh, fail);
  if (fail) return;  // a non-late due precedes every slot end
  // latest-fit stack over groups (thread 0)
  if (tid == 0) {
    const int64_t Lt = sh.v64a;
    int64_t left = Lt;
    for (int s = 0; s < S; ++s) {  // late dues: first-fit
      const int64_t u = imin(left, cap[s]);
      fr[s] = cap[s] - u;
      left -= u;
    }
    int ok = left == 0;
    int nseg = 0;
    int top = -1;  // stack via "previous free slot" search
    (void)top;
    if (ok) {
      for (int s = 0; s < S && ok; ++s) {
        seg0[s] = nseg;
        int64_t need = ng[s];
        int t = s;
        while (need > 0) {
          while (t >= 0 && fr[t] == 0) --t;
          if (t < 0) { ok = 0; break; }
          const int64_t take = imin(need, fr[t]);
          sslot[nseg] = t;
          samt[nseg] = take;
          ++nseg;
          fr[t] -= take;
          need -= take;
          if (nseg >= 2 * S + 2) { ok = 0; sh.flag2 = 1; break; }
        }
      }
      seg0[S] = nseg;
    }
    sh.flag = ok;
  }
  G::sync();
  if (!sh.flag) return;
  // late tokens: member m's late dues occupy [lpre, lpre + l) of the cumulative cap
  for (int m = tid; m < M; m += G::kSize) {
    int64_t a = lpre[m], n = lcount[m];
    int64_t before = 0;
    for (int s = 0; s < S && n > 0; ++s) {
      const int64_t lo = before, hi = before + cap[s];
      if (a < hi) {
        const int64_t take = imin(n, hi - a);
        tok[(int64_t)s * (M + 1) + m] += (int32_t)take;
        a += take;
        n -= take;
      }
      before = hi;
      (void)lo;
    }
  }
  // non-late tokens: single-segment groups direct; multi-segment groups gathered
  int64_t nmulti = 0;
  for (int m = tid; m < M; m += G::kSize) {
    const int64_t rem = E.rm[m];
    if (rem <= 0) continue;
    int64_t issued = E.bl[m] > 0 ? imin(E.bl[m], rem) : 0;
    const double tpot = P.tpot[E.tr[m]];
    for (double d = dmax(E.ph[m], 0.0); time_le(d, horizon) && issued < rem; d += tpot, ++issued) {
      if (d <= kTimeEps) continue;
      const int g = jit_search(ends, S, d);
      if (seg0[g + 1] - seg0[g] == 1) tok[(int64_t)sslot[seg0[g]] * (M + 1) + m] += 1;
      else ++nmulti;
    }
  }
  if (tid < L && c[tid] > 0) {
    for (double d = P.tpot[tid]; time_le(d, gap); d += P.tpot[tid]) {
      const int g = jit_search(ends, S, d);
      if (seg0[g + 1] - seg0[g] == 1) ptier[(int64_t)sslot[seg0[g]] * L + tid] += c[tid];
      else ++nmulti;
    }
  }
  nmulti = G::sum64(sh, nmulti);
  if (nmulti > 0) {
    int np2 = 1;
    while (np2 < nmulti) np2 <<= 1;
    MRec* rec = (MRec*)ar.take(sizeof(MRec) * np2);
    if (ar.over()) {
      if (tid == 0) { o.status = SLOS_ERR_CAPACITY; o.need_work = ar.need(); }
      G::sync();
      return;
    }
    if (tid == 0) sh.v64b = 0;
    G::sync();
    for (int m = tid; m < M; m += G::kSize) {
      const int64_t rem = E.rm[m];
      if (rem <= 0) continue;
      int64_t issued = E.bl[m] > 0 ? imin(E.bl[m], rem) : 0;
      const int64_t k0 = issued;
      const double tpot = P.tpot[E.tr[m]];
      for (double d = dmax(E.ph[m], 0.0); time_le(d, horizon) && issued < rem; d += tpot, ++issued) {
        if (d <= kTimeEps) continue;
        const int g = jit_search(ends, S, d);
        if (seg0[g + 1] - seg0[g] == 1) continue;
        const int64_t at = atomicAdd((unsigned long long*)&sh.v64b, 1ull);
        MRec r;
        r.time = d; r.key = ((uint64_t)m << 32) | (uint64_t)(issued - k0); r.grp = g; r.who = m; r.w = 1;
        rec[at] = r;
      }
    }
    if (tid < L && c[tid] > 0) {
      int t = 0;
      for (double d = P.tpot[tid]; time_le(d, gap); d += P.tpot[tid], ++t) {
        const int g = jit_search(ends, S, d);
        if (seg0[g + 1] - seg0[g] == 1) continue;
        const int64_t at = atomicAdd((unsigned long long*)&sh.v64b, 1ull);
        MRec r;
        r.time = d; r.key = (1ull << 63) | ((uint64_t)tid << 40) | (uint64_t)t; r.grp = g; r.who = -1 - tid;
        r.w = c[tid];
        rec[at] = r;
      }
    }
    G::sync();
    for (int64_t x = nmulti + tid; x < np2; x += G::kSize) {
      MRec r;
      r.time = INFINITY; r.key = ~0ull; r.grp = 0x7fffffff; r.who = 0; r.w = 0;
      rec[x] = r;
    }
    G::sync();
    blk_sort_mrec<G>(rec, np2);
    if (tid == 0) {  // deal sorted dues along each group's segments
      int64_t x = 0;
      while (x < nmulti) {
        const int g = rec[x].grp;
        int sg = seg0[g];
        int64_t room = samt[sg];
        for (; x < nmulti && rec[x].grp == g; ++x) {
          int64_t w = rec[x].w;
          while (w > 0) {
            while (room == 0) { ++sg; room = samt[sg]; }
            const int64_t take = imin(w, room);
            const int s = sslot[sg];
            if (rec[x].who >= 0) tok[(int64_t)s * (M + 1) + rec[x].who] += (int32_t)take;
            else ptier[(int64_t)s * L + (-1 - rec[x].who)] += take;
            room -= take;
            w -= take;
          }
        }
      }
    }
  }
  G::sync();
  // emission: batches slot by slot; owners in member order (ascending owner)
  if (tid == 0) { o.n_b = S; }
  int64_t budget = 0;
  if (owners_sorted) {
    // constant number of barriers: per-slot nonzero counts -> offsets -> scatter
    int32_t* scnt = (int32_t*)ar.take(sizeof(int32_t) * (S + 1));
    int32_t* soff = (int32_t*)ar.take(sizeof(int32_t) * (S + 1));
    if (ar.over()) {
      if (tid == 0) { o.status = SLOS_ERR_CAPACITY; o.need_work = ar.need(); }
      G::sync();
      return;
    }
    const int nw = G::kSize / 32, wr = tid / 32, lane = lane_id();
    for (int s = wr; s < S; s += nw) {
      const int32_t* row = tok + (int64_t)s * (M + 1);
      int cnt = 0;
      for (int base = 0; base < M; base += 32) {
        const int m = base + lane;
        cnt += __popc(__ballot_sync(0xffffffffu, m < M && row[m] > 0));
      }
      if (lane == 0) scnt[s] = cnt;
    }
    G::sync();
    if (wr == 0) {
      int carry = 0;
      for (int base = 0; base < S; base += 32) {
        const int s = base + lane;
        const int x = s < S ? scnt[s] : 0;
        const int inc = warp_incl_scan(x);
        if (s < S) soff[s] = carry + inc - x;
        carry += __shfl_sync(0xffffffffu, inc, 31);
      }
      if (lane == 0) soff[S] = carry;
    }
    G::sync();
    const int base_own = o.n_own;
    for (int s = wr; s < S; s += nw) {
      const int32_t* row = tok + (int64_t)s * (M + 1);
      int carry = 0;
      for (int base = 0; base < M; base += 32) {
        const int m = base + lane;
        const bool has = m < M && row[m] > 0;
        const unsigned msk = __ballot_sync(0xffffffffu, has);
        if (has) {
          const int64_t at = base_own + soff[s] + carry + __popc(msk & ((1u << lane) - 1));
          if (at < o.cap_own) { o.own[2 * at] = E.ow[m]; o.own[2 * at + 1] = row[m]; }
        }
        carry += __popc(msk);
      }
      if (lane == 0 && s < o.cap_b) {
        GapBatchOut& bt = o.b[s];
        bt.start_s = s == 0 ? 0.0 : ends[s - 1];
        bt.end_s = ends[s];
        bt.capacity = cap[s];
        bt.spec_step = 0;
        bt.decode_tokens = cap[s] - fr[s];
        bt.prefill_budget = imin(fr[s], P.max_chunk);
        for (int l = 0; l < kMaxTiers; ++l) bt.per_tier[l] = l < L ? ptier[(int64_t)s * L + l] : 0;
        bt.first_owner = base_own + soff[s];
        bt.n_owner = scnt[s];
      }
    }
    for (int s = tid; s < S; s += G::kSize) budget += imin(fr[s], P.max_chunk);
    budget = G::sum64(sh, budget);
    G::sync();
    if (tid == 0) { o.n_own = base_own + soff[S]; o.budget = budget; o.feasible = 1; }
    G::sync();
    return;
  }
  for (int s = 0; s < S; ++s) {
    int32_t* row = tok + (int64_t)s * (M + 1);
    const int base_own = o.n_own;
    int64_t carry = 0;
    for (int base = 0; base < M; base += G::kSize) {
      const int m = base + tid;
      const int has = (m < M && row[m] > 0) ? 1 : 0;
      int64_t tot;
      const int64_t ex = G::excl(sh, has, &tot);
      if (has) {
        const int64_t at = base_own + carry + ex;
        if (at < o.cap_own) { o.own[2 * at] = E.ow[m]; o.own[2 * at + 1] = row[m]; }
      }
      carry += tot;
    }
    G::sync();
    if (tid == 0) {
      int n_here = (int)carry;
      if (base_own + n_here <= o.cap_own) {  // std::map order + merge (owners may repeat)
        int64_t* pr = o.own + 2 * base_own;
        for (int a2 = 1; a2 < n_here; ++a2) {
          const int64_t ko = pr[2 * a2], kt = pr[2 * a2 + 1];
          int b2 = a2 - 1;
          while (b2 >= 0 && pr[2 * b2] > ko) { pr[2 * (b2 + 1)] = pr[2 * b2]; pr[2 * (b2 + 1) + 1] = pr[2 * b2 + 1]; --b2; }
          pr[2 * (b2 + 1)] = ko; pr[2 * (b2 + 1) + 1] = kt;
        }
        int w = 0;
        for (int a2 = 0; a2 < n_here; ++a2) {
          if (w > 0 && pr[2 * (w - 1)] == pr[2 * a2]) pr[2 * (w - 1) + 1] += pr[2 * a2 + 1];
          else { pr[2 * w] = pr[2 * a2]; pr[2 * w + 1] = pr[2 * a2 + 1]; ++w; }
        }
        n_here = w;
      }
      if (s < o.cap_b) {
        GapBatchOut& bt = o.b[s];
        bt.start_s = s == 0 ? 0.0 : ends[s - 1];
        bt.end_s = ends[s];
        bt.capacity = cap[s];
        bt.spec_step = 0;
        bt.decode_tokens = cap[s] - fr[s];
        bt.prefill_budget = imin(fr[s], P.max_chunk);
        for (int l = 0; l < kMaxTiers; ++l) bt.per_tier[l] = l < L ? ptier[(int64_t)s * L + l] : 0;
        bt.first_owner = base_own;
        bt.n_owner = n_here;
      }
      budget += imin(fr[s], P.max_chunk);
      o.n_own = base_own + n_here;
    }
    G::sync();
  }
  if (tid == 0) { o.budget = budget; o.feasible = 1; }
  G::sync();
}

// tile_gap (batch_planner.cpp:315-406) with full output. `Ebuf` must hold the
// exact members; `merged_all` are census.merged_counts (exact members of every
// remaining, plus canonical).
template <class G>
__device__ inline void block_tile_gap(const PlannerDev& P, BlockShared& sh, double gap, double dh,
                                      const int64_t* c, const MemBuf& E, bool owners_sorted,
                                      Arena ar, GapPlanBuf& o, GapPlanBuf& tmp) {
  const int tid = G::rank();
  const int L = P.L;
  block_tile_gap_ar<G>(P, sh, gap, dh, c, E, owners_sorted, ar, o);
  if (o.status) return;
  if (!P.speculative) return;
  unsigned cmask = 0;
  for (int l = 0; l < L; ++l) if (c[l] > 0) cmask |= 1u << l;
  if (E.M == 0 && cmask == 0) return;  // census.empty()
  // spec_serviceable (:320-334)
  int bad = 0;
  int64_t per[kMaxTiers];
  for (int l = 0; l < kMaxTiers; ++l) per[l] = 0;
  double minph = INFINITY;
  for (int m = tid; m < E.M; m += G::kSize) {
    per[E.tr[m]] += 1;
    if (E.bl[m] > 0) bad = 1;
    const int64_t rem = E.rm[m];
    if (rem > 0) minph = dmin(minph, E.ph[m]);
    if (dh > gap + kTimeEps && rem > 0) {
      const double tpot = P.tpot[E.tr[m]];
      int64_t issued = imin(E.bl[m], rem);
      for (double d = dmax(E.ph[m], 0.0); time_le(d, dh) && issued < rem; d += tpot, ++issued)
        if (!time_le(d, gap)) { bad = 1; break; }
    }
  }
  bad = G::or_(sh, bad);
  int64_t merged[kMaxTiers];
  for (int l = 0; l < L; ++l) merged[l] = c[l] + G::sum64(sh, per[l]);
  minph = G::min(sh, minph);
  if (bad) return;
  if (tid == 0) sh.sp = solve_spec(P, merged);
  G::sync();
  const SpecSol sp = sh.sp;
  if (!sp.ok) return;
  if (minph < sp.bt - kTimeEps) return;  // (:341-346) over members with remaining > 0
  const int full = (int)floor(gap / sp.bt + kTimeEps);
  if (full == 0) return;
  // spec batches budget (closed form per member)
  int64_t spec_budget = 0;
  {
    int64_t canon = 0;
    for (int l = 0; l < L; ++l) canon += c[l] * (int64_t)sp.lengths[l];
    int64_t* kh = (int64_t*)ar.take(sizeof(int64_t) * (full + 2));
    if (ar.over()) {
      if (tid == 0) { o.status = SLOS_ERR_CAPACITY; o.need_work = ar.need(); }
      G::sync();
      return;
    }
    for (int k = tid; k <= full + 1; k += G::kSize) kh[k] = 0;
    G::sync();
    for (int m = tid; m < E.M; m += G::kSize) {
      const int64_t rem = E.rm[m];
      if (rem <= 0) continue;
      const int64_t sl = sp.lengths[E.tr[m]];
      const int64_t q = rem / sl, r = rem % sl;
      atomicAdd((unsigned long long*)&kh[0], (unsigned long long)sl);
      if (q < full) {
        atomicAdd((unsigned long long*)&kh[q], (unsigned long long)(r - sl));
        atomicAdd((unsigned long long*)&kh[q + 1], (unsigned long long)(-r));
      }
    }
    G::sync();
    if (tid == 0) {
      int64_t e = 0;
      for (int k = 0; k < full; ++k) {
        e += kh[k];
        spec_budget += imax(0, imin(sp.cap - (canon + e), P.max_chunk));
      }
      sh.v64a = spec_budget;
    }
    G::sync();
    spec_budget = sh.v64a;
  }
  const double used = full * sp.bt;
  int64_t zero[kMaxTiers];
  for (int l = 0; l < kMaxTiers; ++l) zero[l] = 0;
  (void)zero;
  bool has_tail = false;
  if (gap - used > kTimeEps) {
    MemBuf none = E;
    none.M = 0;
    block_tile_gap_ar<G>(P, sh, gap - used, 0.0, merged, none, true, ar, tmp);
    if (tmp.status) { if (tid == 0) { o.status = tmp.status; o.need_work = tmp.need_work; } G::sync(); return; }
    if (!tmp.feasible) return;  // keep ar
    spec_budget += tmp.budget;
    has_tail = true;
  }
  if (o.feasible && o.budget >= spec_budget) return;  // :404
  // materialise the speculative plan into o (:353-402)
  if (tid == 0) {
    o.n_b = 0;
    o.n_own = 0;
    o.budget = spec_budget;
    o.feasible = 1;
    o.n_spec = L;
    for (int l = 0; l < kMaxTiers; ++l) o.spec[l] = l < L ? sp.lengths[l] : 0;
  }
  G::sync();
  // per batch k: owners in census order with n = min(left, sl) > 0
  for (int k = 0; k < full; ++k) {
    const int base_own = o.n_own;
    int64_t carry = 0, dec_ex = 0, step = 0;
    for (int base = 0; base < E.M; base += G::kSize) {
      const int m = base + tid;
      int64_t n = 0, sl = 0;
      if (m < E.M) {
        sl = sp.lengths[E.tr[m]];
        const int64_t left = imax(0, E.rm[m] - (int64_t)k * sl);
        n = imin(left, sl);
      }
      const int has = n > 0;
      int64_t tot;
      const int64_t ex = G::excl(sh, has, &tot);
      if (has) {
        const int64_t at = base_own + carry + ex;
        if (at < o.cap_own) { o.own[2 * at] = E.ow[m]; o.own[2 * at + 1] = n; }
        dec_ex += n;
        step = imax(step, sl);
      }
      carry += tot;
    }
    dec_ex = G::sum64(sh, dec_ex);
    for (int o2 = 16; o2; o2 >>= 1) step = imax(step, __shfl_xor_sync(0xffffffffu, step, o2));
    G::sync();
    if (lane_id() == 0) sh.r64[G::kSize == 32 ? 0 : warp_id()] = step;
    G::sync();
    if (tid == 0) {
      int64_t st = 0;
      for (int w = 0; w < (G::kSize + 31) / 32; ++w) st = imax(st, sh.r64[w]);
      int64_t decode = 0;
      GapBatchOut b;
      b.start_s = k * sp.bt;
      b.end_s = (k + 1) * sp.bt;
      b.capacity = sp.cap;
      for (int l = 0; l < kMaxTiers; ++l) {
        b.per_tier[l] = l < L ? c[l] * (int64_t)sp.lengths[l] : 0;
        decode += b.per_tier[l];
      }
      decode += dec_ex;
      for (int l = 0; l < L; ++l) if (b.per_tier[l] > 0) st = imax(st, sp.lengths[l]);
      b.spec_step = st;
      b.decode_tokens = decode;
      b.prefill_budget = imax(0, imin(sp.cap - decode, P.max_chunk));
      b.first_owner = base_own;
      b.n_owner = (int32_t)carry;
      if (o.n_b < o.cap_b) o.b[o.n_b] = b;
      o.n_b++;
      o.n_own = base_own + (int32_t)carry;
    }
    G::sync();
  }
  if (has_tail && tid == 0) {
    for (int k = 0; k < tmp.n_b; ++k) {
      GapBatchOut b = tmp.b[k];
      b.start_s += used;
      b.end_s += used;
      b.first_owner = o.n_own;
      b.n_owner = 0;
      if (o.n_b < o.cap_b) o.b[o.n_b] = b;
      o.n_b++;
    }
  }
  G::sync();
}

}  // namespace slos

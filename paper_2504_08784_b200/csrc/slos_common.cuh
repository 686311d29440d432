// Device arithmetic shared by every kernel. Bit-exactness rules (SURVEY.md §7 hard
// part 1): compiled with -fmad=false and IEEE division/sqrt (nvcc defaults for
// fp64), no fast-math; every expression keeps the reference's evaluation order.
#pragma once

#include <stdint.h>

#include "slos_dev.h"
#include "../../include/slos_planner.h"

namespace slos {

__device__ __forceinline__ bool time_le(double a, double b) { return a <= b + kTimeEps; }  // common.hpp:31
__device__ __forceinline__ bool time_lt(double a, double b) { return a < b - kTimeEps; }   // common.hpp:32
// std::max / std::min: first argument on ties.
__device__ __forceinline__ double dmax(double a, double b) { return (a < b) ? b : a; }
__device__ __forceinline__ double dmin(double a, double b) { return (b < a) ? b : a; }
__device__ __forceinline__ int64_t imax(int64_t a, int64_t b) { return (a < b) ? b : a; }
__device__ __forceinline__ int64_t imin(int64_t a, int64_t b) { return (b < a) ? b : a; }

// PerfModel::predict perf_model.cpp:106-114 (term_value :92-94).
// Code size matters here: predict is inlined at hundreds of sites of the
// reconstruction engine, whose warp form (one instance per warp) stalled on
// instruction fetch; the loop stays rolled.
__device__ __forceinline__ double predict(const PlannerDev& P, int64_t n, int64_t s) {
  double best = 0.0;
#pragma unroll 1
  for (int t = 0; t < P.n_terms; ++t) {
    const double v = P.k1[t] * (double)n + P.k2[t] * (double)s + P.b[t];
    best = dmax(best, v);
  }
  return best;
}

// PerfModel::time2bs perf_model.cpp:116-130; -1 == throw "infeasible-budget".
__device__ __forceinline__ int64_t time2bs(const PlannerDev& P, double budget, int64_t s,
                                           int64_t max_tokens) {
  if (!time_le(predict(P, 1, s), budget)) return -1;
  // With every k1 >= 0, predict(n, s) is non-decreasing in n (each rounded term
  // k1*n + k2*s + b is, and so is their max), so the reference's binary search
  // returns the largest n in [1, max_tokens] with time_le(predict(n), budget).
  // Start from the real-valued solution of each term and step to that boundary
  // with the exact predicate; a guess more than a few steps off (never seen)
  // falls through to the binary search itself.
  bool mono = true;
  int64_t n = max_tokens;
  for (int t = 0; t < P.n_terms; ++t) {
    if (P.k1[t] < 0.0) { mono = false; break; }
    if (P.k1[t] > 0.0) {
      const double r = (budget + kTimeEps - P.k2[t] * (double)s - P.b[t]) / P.k1[t];
      const int64_t g = r < 1.0 ? 1 : (r >= (double)max_tokens ? max_tokens : (int64_t)r);
      n = imin(n, g);
    }
  }
  if (mono) {
    int steps = 0;
    while (n < max_tokens && time_le(predict(P, n + 1, s), budget) && ++steps < 8) ++n;
    while (n > 1 && !time_le(predict(P, n, s), budget) && ++steps < 8) --n;
    if (steps < 8) return n;
  }
  int64_t lo = 1, hi = max_tokens;
  while (lo < hi) {
    const int64_t mid = lo + (hi - lo + 1) / 2;
    if (time_le(predict(P, mid, s), budget)) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// BatchPlanner::plan_predict / plan_time2bs / quantize_gap batch_planner.cpp:125-139.
__device__ __forceinline__ double plan_predict(const PlannerDev& P, int64_t n, int64_t s) {
  return predict(P, n, s) * P.margin1;
}
__device__ __forceinline__ int64_t plan_time2bs(const PlannerDev& P, double budget, int64_t s) {
  return time2bs(P, budget / P.margin1, s, P.max_batch);
}
__device__ __forceinline__ double quantize_gap(double g) {
  if (g <= 0) return 0.0;
  return floor(g * 1000.0 + 1e-6) / 1000.0;
}

// members_at dp_scheduler.cpp:55-91 for one running decoder. valid=false when the
// member drops out (remaining exhausted by the pull window, :74-75).
struct Member {
  double phase;
  int64_t backlog;
  int64_t rem;
  int32_t tier;
  bool valid;
};

__device__ __forceinline__ Member member_at(const PlannerDev& P, double next, int64_t backlog0,
                                            int64_t rem0, int32_t tier, double now, double at,
                                            double pull) {
  Member m;
  const double tpot = P.tpot[tier];
  int64_t remaining = rem0;
  int64_t backlog = imin(backlog0, remaining);
  m.tier = tier;
  m.valid = true;
  if (at > now + kTimeEps) {
    int64_t served = backlog;
    backlog = 0;
    if (time_le(next, at + pull)) {
      const int64_t k = (int64_t)floor((at + pull - next) / tpot + kTimeEps) + 1;
      served += k;
      next += (double)k * tpot;
    }
    remaining -= imin(served, remaining);
    if (remaining <= 0) {
      m.valid = false;
      m.phase = 0.0;
      m.backlog = 0;
      m.rem = 0;
      return m;
    }
  } else {
    while (backlog < remaining && time_lt(next - at, pull)) {
      backlog += 1;
      next += tpot;
    }
  }
  m.phase = dmax(next - at, 0.0);
  m.backlog = backlog;
  m.rem = remaining;
  return m;
}

// The reference's jit binary search over slot ends (batch_planner.cpp:272-284).
__device__ __forceinline__ int jit_search(const double* ends, int S, double t) {
  int jit = -1, lo = 0, hi = S - 1;
  while (lo <= hi) {
    const int mid = (lo + hi) / 2;
    if (time_le(ends[mid], t)) { jit = mid; lo = mid + 1; } else { hi = mid - 1; }
  }
  return jit;
}

// pack_add / pack_get dp_scheduler.cpp:28-29.
__device__ __forceinline__ uint64_t pack_add(uint64_t c, int tier) { return c + ((uint64_t)1 << (8 * tier)); }
__device__ __forceinline__ int64_t pack_get(uint64_t c, int tier) { return (int64_t)((c >> (8 * tier)) & 0xff); }

// ---- warp primitives ------------------------------------------------------
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ int warp_id() { return threadIdx.x >> 5; }

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
template <typename T>
__device__ __forceinline__ T warp_min(T v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) { T y = __shfl_xor_sync(0xffffffffu, v, o); v = (y < v) ? y : v; }
  return v;
}
template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
  const int l = lane_id();
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T y = __shfl_up_sync(0xffffffffu, v, o);
    if (l >= o) v += y;
  }
  return v;
}
__device__ __forceinline__ int warp_or(int v) { return __reduce_or_sync(0xffffffffu, (unsigned)v); }

// ---- expected_accepted table lookup & spec solver --------------------------

struct SpecSol {
  bool ok;
  int lengths[kMaxTiers];
  double bt;       // batch_time_s
  int64_t cap;     // batch_capacity
  int64_t decode;  // decode_tokens
  double tpt;      // prefill_throughput
};

// min_len_covering batch_planner.cpp:42-47 with expected_accepted from P.acc.
__device__ __forceinline__ int min_len_covering(const PlannerDev& P, double tpot, double target) {
  for (int sl = 1; sl <= P.spec_max_len; ++sl)
    if (tpot * P.acc[sl] >= target - kTimeEps) return sl;
  return 0;
}

// solve_spec_lengths batch_planner.cpp:51-115 (sequential, one thread).
__device__ __noinline__ SpecSol solve_spec(const PlannerDev& P, const int64_t* counts) {
  SpecSol best;
  best.ok = false;
  const int L = P.L;
  const double margin = P.margin1;
  for (int bind = 0; bind < L; ++bind) {
    if (counts[bind] <= 0) continue;
    for (int sl_bind = 1; sl_bind <= P.spec_max_len; ++sl_bind) {
      const double t_batch = P.tpot[bind] * P.acc[sl_bind];
      int lens[kMaxTiers];
      for (int l = 0; l < L; ++l) lens[l] = 0;
      lens[bind] = sl_bind;
      bool ok = true;
      for (int l = 0; l < L; ++l) {
        if (counts[l] <= 0 || l == bind) continue;
        const int sl = min_len_covering(P, P.tpot[l], t_batch);
        if (sl == 0) { ok = false; break; }
        lens[l] = sl;
      }
      if (!ok) continue;
      int64_t spec_step = 0, decode = 0;
      for (int l = 0; l < L; ++l) {
        if (counts[l] <= 0) continue;
        spec_step = imax(spec_step, lens[l]);
        decode += counts[l] * lens[l];
      }
      if (!time_le(predict(P, 1, spec_step) * margin, t_batch)) continue;
      int64_t lo = 1, hi = P.max_batch;
      while (lo < hi) {
        const int64_t mid = lo + (hi - lo + 1) / 2;
        if (time_le(predict(P, mid, spec_step) * margin, t_batch)) lo = mid; else hi = mid - 1;
      }
      const int64_t cap = lo;
      if (cap < decode) continue;
      const int64_t budget = imin(cap - decode, P.max_chunk);
      const double tpt = (double)budget / t_batch;
      bool better = !best.ok || tpt > best.tpt + 1e-12;
      if (!better && fabs(tpt - best.tpt) <= 1e-12) {
        if (t_batch < best.bt - kTimeEps) better = true;
        else if (fabs(t_batch - best.bt) <= kTimeEps) {
          for (int l = 0; l < L; ++l) {  // std::vector<int> operator<
            if (lens[l] < best.lengths[l]) { better = true; break; }
            if (best.lengths[l] < lens[l]) break;
          }
        }
      }
      if (better) {
        best.ok = true;
        for (int l = 0; l < kMaxTiers; ++l) best.lengths[l] = l < L ? lens[l] : 0;
        best.bt = t_batch;
        best.cap = cap;
        best.decode = decode;
        best.tpt = tpt;
      }
    }
  }
  return best;
}

// Cooperative copy of a header struct (planner, instance) into shared memory:
// nt threads, 8-byte words (one thread copying ~1 KB serialises ~100 loads).
template <class T>
__device__ __forceinline__ void block_copy_struct(T& dst, const T& src, int tid, int nt) {
  static_assert(sizeof(T) % 8 == 0, "8-byte words");
  const uint64_t* s = (const uint64_t*)&src;
  uint64_t* d = (uint64_t*)&dst;
  for (int k = tid; k < (int)(sizeof(T) / 8); k += nt) d[k] = s[k];
}

}  // namespace slos

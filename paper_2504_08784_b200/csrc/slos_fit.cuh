// PerfModel::fit on the device (include/slos_fit.h): one CTA per
// profile set runs the reference's regime iteration (perf_model.cpp:132-201).
//
// Per iteration: (A) each regime's first member and whether its num_tokens /
// spec_step vary (nonneg_least_squares :21-25); (B) one warp per non-empty regime
// refits it -- every entry of the normal equations is one lane accumulating over
// the regime's samples in index order (the reference's summation order, so the
// same bits), lane 0 eliminates with the reference's partial pivoting and drops
// the most negative coefficient, at most 4 passes (:33-89); (C) threads over
// samples take the argmax term with the reference's tie rule (:163-172) and the
// squared residuals; (D) one thread sums the residuals in index order and keeps
// the best iteration (:182-185). Built with -fmad=false like every kernel here.
#pragma once

#include <climits>

#include "slos_common.cuh"

namespace slos {

constexpr int kFitThreads = 256;
constexpr int kFitMaxTerms = 32;

// term_value perf_model.cpp:92-94
__device__ __forceinline__ double fit_term(double k1, double k2, double b, double n, double s) {
  return k1 * n + k2 * s + b;
}

__global__ void __launch_bounds__(kFitThreads) fit_kernel(FitParams prm) {
  const FitSet S = prm.sets[blockIdx.x];
  if (!S.run) return;
  const int n = S.n, T = prm.T;
  // the set's samples as doubles (the reference converts each use, :28-31, exactly),
  // staged in shared memory when they fit (prm.smem_samples), else read from HBM
  extern __shared__ __align__(16) unsigned char fsm[];
  const bool staged = n <= prm.smem_samples;
  double* nd = staged ? (double*)fsm : prm.nd + S.off;
  double* sd = staged ? nd + n : prm.sd + S.off;
  double* lat = staged ? sd + n : prm.lat + S.off;
  double* e2 = staged ? lat + n : prm.e2 + S.off;
  int32_t* assign = staged ? (int32_t*)(e2 + n) : prm.assign + S.off;
  const int64_t* nt = prm.nt + S.off;
  const int64_t* ss = prm.ss + S.off;
  for (int i = threadIdx.x; i < n; i += kFitThreads) {
    nd[i] = (double)nt[i];
    sd[i] = (double)ss[i];
    if (staged) {
      lat[i] = prm.lat[S.off + i];
      assign[i] = prm.assign[S.off + i];
    }
  }
  __syncthreads();
  __shared__ double tk1[kFitMaxTerms], tk2[kFitMaxTerms], tb[kFitMaxTerms];
  __shared__ double bk1[kFitMaxTerms], bk2[kFitMaxTerms], bb[kFitMaxTerms];
  __shared__ int first[kFitMaxTerms], uk1[kFitMaxTerms], uk2[kFitMaxTerms];
  __shared__ double s_best;
  __shared__ int s_have;
  const int tid = threadIdx.x, lane = lane_id(), w = warp_id();
  constexpr int NW = kFitThreads / 32;
  if (tid < T) { tk1[tid] = 0.0; tk2[tid] = 0.0; tb[tid] = 0.0; }
  if (tid == 0) { s_best = INFINITY; s_have = 0; }
  for (int iter = 0; iter < prm.max_iters; ++iter) {
    // (A) regimes: first member, varying columns
    if (tid < T) { first[tid] = INT_MAX; uk1[tid] = 0; uk2[tid] = 0; }
    __syncthreads();
    for (int i = tid; i < n; i += kFitThreads) atomicMin(&first[assign[i]], i);
    __syncthreads();
    for (int i = tid; i < n; i += kFitThreads) {
      const int g = assign[i], f = first[g];
      if (nt[i] != nt[f]) uk1[g] = 1;  // int64 compares, like the reference
      if (ss[i] != ss[f]) uk2[g] = 1;
    }
    __syncthreads();
    // (B) nonneg_least_squares per non-empty regime, one warp each
    for (int g = w; g < T; g += NW) {
      if (first[g] == INT_MAX) continue;
      bool act[3] = {uk1[g] != 0, uk2[g] != 0, true};
      double coef[3] = {0.0, 0.0, 0.0};
      for (int pass = 0; pass < 4; ++pass) {
        int cols[3], k = 0;
        for (int c = 0; c < 3; ++c)
          if (act[c]) cols[k++] = c;
        // normal equations A x = y on the active columns: lane e = entry (r, c) of
        // the k x (k+1) augmented matrix, summed in sample order
        double acc = 0.0;
        if (lane < k * (k + 1)) {
          const int r = lane / (k + 1), c = lane % (k + 1);
          const int cr = cols[r], cc = c < k ? cols[c] : -1;
          const double* xa = cr == 0 ? nd : (cr == 1 ? sd : nullptr);
          const double* ya = cc == 0 ? nd : (cc == 1 ? sd : (cc == 2 ? nullptr : lat));
#pragma unroll 4
          for (int i = 0; i < n; ++i) {
            if (assign[i] != g) continue;
            const double xr = xa ? xa[i] : 1.0;
            acc += xr * (ya ? ya[i] : 1.0);
          }
        }
        double a[3][4];
        for (int e = 0; e < 12; ++e) {
          const double v = __shfl_sync(0xffffffffu, acc, e);
          if (e < k * (k + 1)) a[e / (k + 1)][e % (k + 1)] = v;
        }
        int worst = -1;
        if (lane == 0) {
          // Gaussian elimination with partial pivoting (perf_model.cpp:52-68)
          for (int r = 0; r < k; ++r) {
            int piv = r;
            for (int r2 = r + 1; r2 < k; ++r2)
              if (fabs(a[r2][r]) > fabs(a[piv][r])) piv = r2;
            if (piv != r)
              for (int c = 0; c <= k; ++c) { const double t = a[r][c]; a[r][c] = a[piv][c]; a[piv][c] = t; }
            if (fabs(a[r][r]) < 1e-30) {
              a[r][r] = 1.0;
              a[r][k] = 0.0;
              for (int c = 0; c < k; ++c)
                if (c != r) a[r][c] = 0.0;
            }
            for (int r2 = 0; r2 < k; ++r2) {
              if (r2 == r) continue;
              const double f = a[r2][r] / a[r][r];
              for (int c = r; c <= k; ++c) a[r2][c] -= f * a[r][c];
            }
          }
          coef[0] = coef[1] = coef[2] = 0.0;
          for (int r = 0; r < k; ++r) coef[cols[r]] = a[r][k] / a[r][r];
          double worst_v = -1e-12;
          for (int c = 0; c < 3; ++c)
            if (act[c] && coef[c] < worst_v) { worst = c; worst_v = coef[c]; }
        }
        worst = __shfl_sync(0xffffffffu, worst, 0);
        for (int c = 0; c < 3; ++c) coef[c] = __shfl_sync(0xffffffffu, coef[c], 0);
        if (worst < 0) break;
        act[worst] = false;
        if (worst == 2) {  // the intercept column stays; a negative intercept clamps to zero
          coef[2] = 0.0;
          break;
        }
      }
      if (lane == 0) {  // std::max(coef, 0.0)
        tk1[g] = dmax(coef[0], 0.0);
        tk2[g] = dmax(coef[1], 0.0);
        tb[g] = dmax(coef[2], 0.0);
      }
    }
    __syncthreads();
    // (C) argmax regime of every sample (ties prefer the smaller intercept)
    int changed = 0;
    for (int i = tid; i < n; i += kFitThreads) {
      const double ni = nd[i], si = sd[i];
      int arg = 0;
      double v = fit_term(tk1[0], tk2[0], tb[0], ni, si);
      for (int g = 1; g < T; ++g) {
        const double vg = fit_term(tk1[g], tk2[g], tb[g], ni, si);
        if (vg > v + 1e-15 || (fabs(vg - v) <= 1e-15 && tb[g] < tb[arg])) {
          v = vg;
          arg = g;
        }
      }
      const double e = v - lat[i];
      e2[i] = e * e;
      if (arg != assign[i]) {
        assign[i] = arg;
        changed = 1;
      }
    }
    changed = __syncthreads_or(changed);
    // (D) sse in sample order; keep the best iteration
    if (tid == 0) {
      double sse = 0.0;
      for (int i = 0; i < n; ++i) sse += e2[i];
      if (sse < s_best) {
        s_best = sse;
        s_have = 1;
        for (int g = 0; g < T; ++g) { bk1[g] = tk1[g]; bk2[g] = tk2[g]; bb[g] = tb[g]; }
      }
    }
    __syncthreads();
    if (!changed) break;
  }
  if (tid < T && s_have) {
    double* o = prm.out + ((size_t)blockIdx.x * T + tid) * 3;
    o[0] = bk1[tid];
    o[1] = bk2[tid];
    o[2] = bb[tid];
  }
  if (tid == 0) prm.ok[blockIdx.x] = s_have;
}

}  // namespace slos

// sm_100a kernels of the batched multi-SLO planner and their launchers.
// Compiled with: -gencode arch=compute_100a,code=sm_100a -fmad=false -lineinfo -O3
// (-fmad=false is part of the bit-exactness contract, see slos_common.cuh).
#include <cuda_runtime.h>

#include <algorithm>

#include "slos_build.cuh"
#include "slos_dp.cuh"
#include "slos_fit.cuh"
#include "slos_launch.h"

namespace slos {

// Pack each instance's batches / entries / admitted+declined ids densely so the
// host copies exactly the bytes of the results (one D2H).
__global__ void __launch_bounds__(256) compact_kernel(CompactParams p) {
  const int x = blockIdx.x;
  const int k = p.vlist ? p.vlist[x] : x;
  const InstDev& I = p.inst[k];
  const OutHdr& o = p.out[k];
  if (o.status != 0) return;
  const int64_t nb = o.n_batches, ne = o.n_entries;
  slos_batch* db = (slos_batch*)(p.dst + p.boff[x]);
  slos_entry* de = (slos_entry*)(p.dst + p.eoff[x]);
  int32_t* di = (int32_t*)(p.dst + p.ioff[x]);
  for (int64_t y = threadIdx.x; y < nb; y += blockDim.x) db[y] = p.batches[I.off_batch + y];
  // entries: 8 B each, copied as 8-byte words
  const uint2* se = (const uint2*)(p.entries + I.off_entry);
  uint2* dw = (uint2*)de;
  for (int64_t y = threadIdx.x; y < ne; y += blockDim.x) dw[y] = se[y];
  const int32_t* ids = p.ids + I.off_ids;
  for (int y = threadIdx.x; y < o.n_admitted; y += blockDim.x) di[y] = ids[y];
  for (int y = threadIdx.x; y < o.n_declined; y += blockDim.x) di[o.n_admitted + y] = ids[I.n_pending + y];
}

// dynamic shared memory of dp_kernel (must mirror the carve-up in dp_kernel)
size_t dp_smem_bytes(int max_N, int max_dec_staged, int Sc, int L, int Tsm, size_t* overlay, int dtab, int kind) {
  const int nwarps = kind == 1 ? kDpSmallThreads / 32 : (kind == 2 ? kDpBigThreads / 32 : kDpWarps);
  const size_t N = (size_t)max_N;
  size_t b = 5 * ((8 * (N + 1) + 15) & ~(size_t)15) + 3 * ((4 * (N + 1) + 15) & ~(size_t)15) + 16;  // chain (TMA)
  b += (size_t)max_dec_staged * 28 + 16;                              // decoders
  b += 8 * (size_t)Sc * nwarps + 16;                                  // placement temporaries
  const size_t ov = (size_t)76 * (size_t)Tsm;
  *overlay = ov;
  b += ov + 16;                                                       // candidate states
  b += (size_t)20 * (size_t)Tsm;                                      // kept candidate arrays
  b += 4 * (size_t)dtab;                                              // direct bucket table
  (void)L;
  return b + 64;
}

size_t dp_group_hdr_bytes() { return (sizeof(GroupHdr) + 15) & ~(size_t)15; }

size_t dp_group_eval_bytes(int Sc, int L) { return group_var_eval_bytes(Sc, L); }

size_t dp_anchor_stride(int R, int Sc, int L, int N) { return anchor_stride_bytes(R, Sc, L, N);
}

size_t dp_group_stride(int Sc, int L) { return group_var_stride(Sc, L); }

size_t dp_warp_scr_stride(int Sc, int L) {
  const size_t s = (size_t)Sc * (8 + 8 + 4 + 4 * L + 8 + 8 + 8 + 4 * L) + (size_t)(Sc + 2) * 8 + 64;
  return (s + 127) & ~(size_t)127;
}

size_t anchor_smem_bytes(int max_N, int Sc, int L, size_t* scr) {
  const size_t N = (size_t)max_N, S = (size_t)Sc;
  // due pass: grid copy, per-group gap/horizon/Sp/lo/hi/accumulators, cell histogram,
  // list offsets and a list area of 8 entries per group plus one per cell
  const size_t b = 8 * S + N * (8 + 8 + 4 * 3 + 4 * 5) + 4 * (S + 1) + 4 * (S + 2) + 4 * (8 * N + S) + 64;
  *scr = b;
  return sizeof(double) * (size_t)L * S + b;
}

cudaError_t launch_anchor(const DpParams& prm, int grid, size_t smem, cudaStream_t s, bool big) {
  if (grid <= 0) return cudaSuccess;
  if (big) {
    cudaError_t e = cudaFuncSetAttribute(anchor_kernel_big, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    anchor_kernel_big<<<grid, kAnchorBigThreads, smem, s>>>(prm);
    return cudaGetLastError();
  }
  cudaError_t e = cudaFuncSetAttribute(anchor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  anchor_kernel<<<grid, kAnchorThreads, smem, s>>>(prm);
  return cudaGetLastError();
}

cudaError_t launch_group(const DpParams& prm, int n_atask, int max_N, cudaStream_t s) {
  if (n_atask <= 0 || max_N <= 0) return cudaSuccess;
  const dim3 grid((unsigned)n_atask, (unsigned)((max_N + kGroupWarps - 1) / kGroupWarps));
  group_kernel<<<grid, 32 * kGroupWarps, 0, s>>>(prm);
  return cudaGetLastError();
}

cudaError_t launch_dp(const DpParams& prm, int grid, size_t smem, cudaStream_t s, int kind) {
  if (grid <= 0) return cudaSuccess;
  if (kind == 2) {
    cudaError_t e = cudaFuncSetAttribute(dp_kernel_big, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dp_kernel_big<<<grid, kDpBigThreads, smem, s>>>(prm);
    return cudaGetLastError();
  }
  if (kind == 1) {
    cudaError_t e = cudaFuncSetAttribute(dp_kernel_small, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dp_kernel_small<<<grid, kDpSmallThreads, smem, s>>>(prm);
    return cudaGetLastError();
  }
  cudaError_t e = cudaFuncSetAttribute(dp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dp_kernel<<<grid, kDpThreads, smem, s>>>(prm);
  return cudaGetLastError();
}

cudaError_t launch_build(const BuildParams& prm, int n_small, int n_large, int n_big, int n_huge, cudaStream_t s) {
  cudaError_t e;
  if (n_small > 0) {
    if ((e = cudaFuncSetAttribute(build_kernel_warp, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)prm.smem_warp)) != cudaSuccess)
      return e;
    build_kernel_warp<<<(n_small + kBuildWarps - 1) / kBuildWarps, 32 * kBuildWarps, prm.smem_warp, s>>>(prm);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  if (n_large > 0) {
    if ((e = cudaFuncSetAttribute(build_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)prm.smem_bytes)) != cudaSuccess)
      return e;
    build_kernel<<<n_large, kBuildThreads, prm.smem_bytes, s>>>(prm);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  if (n_big > 0) {
    if ((e = cudaFuncSetAttribute(build_kernel_big, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)prm.smem_big)) != cudaSuccess)
      return e;
    build_kernel_big<<<n_big, SLOS_BUILD_BIG_THREADS, prm.smem_big, s>>>(prm);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  if (n_huge > 0) {
    if ((e = cudaFuncSetAttribute(build_kernel_huge, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)prm.smem_big)) != cudaSuccess)
      return e;
    build_kernel_huge<<<n_huge, SLOS_BUILD_HUGE_THREADS, prm.smem_big, s>>>(prm);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_compact(const CompactParams& prm, int grid, cudaStream_t s) {
  if (grid <= 0) return cudaSuccess;
  compact_kernel<<<grid, 256, 0, s>>>(prm);
  return cudaGetLastError();
}

cudaError_t launch_gap(const GapParams& prm, int grid, cudaStream_t s) {
  if (grid <= 0) return cudaSuccess;
  gap_kernel<<<grid, kBT, 0, s>>>(prm);
  return cudaGetLastError();
}

cudaError_t launch_time2bs(const PlannerDev* P, int n, const double* b, const int64_t* sp,
                           int64_t max_tokens, int64_t* out, int32_t* st, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  time2bs_kernel<<<(n + 255) / 256, 256, 0, s>>>(P, n, b, sp, max_tokens, out, st);
  return cudaGetLastError();
}

cudaError_t launch_predict(const PlannerDev* P, int n, const int64_t* t, const int64_t* sp,
                           double* out, int32_t* st, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  predict_kernel<<<(n + 255) / 256, 256, 0, s>>>(P, n, t, sp, out, st);
  return cudaGetLastError();
}

__global__ void spec_kernel(const PlannerDev* P, const int64_t* counts, SpecSol* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) *out = solve_spec(*P, counts);
}

cudaError_t launch_spec(const PlannerDev* P, const int64_t* counts, void* out, cudaStream_t s) {
  spec_kernel<<<1, 32, 0, s>>>(P, counts, (SpecSol*)out);
  return cudaGetLastError();
}

size_t spec_sol_bytes() { return sizeof(SpecSol); }

cudaError_t launch_fit(const FitParams& prm, int n_sets, size_t smem, cudaStream_t s) {
  if (n_sets <= 0) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(fit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  fit_kernel<<<n_sets, kFitThreads, smem, s>>>(prm);
  return cudaGetLastError();
}

__global__ void records_kernel(const OutHdr* out, const int32_t* map, int nv, slos_record* rec) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nv) return;
  const OutHdr& h = out[v];
  slos_record r;
  r.status = h.status;
  r.running_set_infeasible = h.infeasible;
  r.n_admitted = h.n_admitted;
  r.n_declined = h.n_declined;
  r.admitted_value = h.value;
  r.n_batches = h.n_batches;
  r.n_entries = h.n_entries;
  r.exact_until_s = h.exact_until;
  r.counters.transitions = h.ctr[0];
  r.counters.gap_evals = h.ctr[1];
  r.counters.dues = h.ctr[2];
  r.counters.slots = h.ctr[3];
  r.counters.states = h.ctr[4];
  rec[map[v]] = r;
}

cudaError_t launch_records(const OutHdr* out, const int32_t* map, int nv, slos_record* rec, cudaStream_t s) {
  if (nv <= 0) return cudaSuccess;
  records_kernel<<<(nv + 127) / 128, 128, 0, s>>>(out, map, nv, rec);
  return cudaGetLastError();
}

}  // namespace slos

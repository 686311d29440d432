// Host-visible launch interface of slos_kernels.cu (C++; used by slos_host.cpp).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>

#include "slos_dev.h"

namespace slos {

struct DpParams;
struct BuildParams;
struct GapParams;

struct CompactParams {
  const InstDev* inst;
  const OutHdr* out;
  const slos_batch* batches;
  const slos_entry* entries;
  const int32_t* ids;
  const int32_t* vlist;  // position -> instance (nullptr: identity)
  const int64_t* boff;  // byte offsets into dst, per position
  const int64_t* eoff;
  const int64_t* ioff;
  unsigned char* dst;
};

// kind: 0 dp_kernel, 1 dp_kernel_small, 2 dp_kernel_big
size_t dp_smem_bytes(int max_N, int max_dec_staged, int Sc, int L, int Tsm, size_t* overlay, int dtab,
                     int kind = 0);
constexpr int kDpMaxWarpsHost = 16;  // warps of the widest DP kernel (dp_kernel_big)
constexpr int kDpSmallMaxChainHost = 16;  // dp_kernel_small: chain items (kDpSmallMaxChain)
size_t dp_group_hdr_bytes();
size_t dp_group_eval_bytes(int Sc, int L);
size_t dp_group_stride(int Sc, int L);
size_t dp_anchor_stride(int R, int Sc, int L, int N);
size_t dp_warp_scr_stride(int Sc, int L);
cudaError_t launch_dp(const DpParams& prm, int grid, size_t smem, cudaStream_t s, int kind = 0);
size_t anchor_smem_bytes(int max_N, int Sc, int L, size_t* scr);
cudaError_t launch_anchor(const DpParams& prm, int grid, size_t smem, cudaStream_t s, bool big = false);
cudaError_t launch_group(const DpParams& prm, int n_atask, int max_N, cudaStream_t s);
cudaError_t launch_build(const BuildParams& prm, int n_small, int n_large, int n_big, int n_huge, cudaStream_t s);
cudaError_t launch_compact(const CompactParams& prm, int grid, cudaStream_t s);
cudaError_t launch_gap(const GapParams& prm, int grid, cudaStream_t s);
cudaError_t launch_time2bs(const PlannerDev* P, int n, const double* b, const int64_t* sp,
                           int64_t max_tokens, int64_t* out, int32_t* st, cudaStream_t s);
cudaError_t launch_predict(const PlannerDev* P, int n, const int64_t* t, const int64_t* sp,
                           double* out, int32_t* st, cudaStream_t s);
cudaError_t launch_spec(const PlannerDev* P, const int64_t* counts, void* out, cudaStream_t s);
size_t spec_sol_bytes();
cudaError_t launch_fit(const FitParams& prm, int n_sets, size_t smem, cudaStream_t s);
cudaError_t launch_records(const OutHdr* out, const int32_t* map, int nv, slos_record* rec, cudaStream_t s);

}  // namespace slos

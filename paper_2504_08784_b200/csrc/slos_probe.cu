// Shared-memory bandwidth probe (measurement tool, not part of the planner ABI).
//
// The DP stage's roofline is stated against the shared-memory
// pipe. Its nominal figure (148 SM x 128 B/clk x f_SM) is a formula; this probe
// measures what the pipe actually delivers on the box: every CTA streams 16-byte
// conflict-free loads (LDS.128) out of a 16 KB shared buffer, 8 CTAs of 256 threads
// per SM on all SMs, timed with CUDA events, with the SM clock measured in the same
// launch (the longest CTA's clock64 delta / elapsed time). bench.py reads it once per run.
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

constexpr int kThreads = 256;
constexpr int kWords = 1024;  // uint4 words = 16 KB per CTA (8 CTAs fit an SM)

__global__ void __launch_bounds__(kThreads) smem_read_kernel(int iters, uint4* sink, long long* cycles) {
  __shared__ uint4 buf[kWords];
  for (int i = threadIdx.x; i < kWords; i += kThreads)
    buf[i] = make_uint4(i, i * 3u, i * 5u, i * 7u);
  __syncthreads();
  const long long t0 = clock64();
  uint4 acc = make_uint4(0, 0, 0, 0);
  int idx = threadIdx.x;
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {  // 4 distinct words per thread per iteration
      const uint4 v = buf[(idx + k * kThreads) & (kWords - 1)];
      acc.x ^= v.x;
      acc.y += v.y;
      acc.z ^= v.z;
      acc.w += v.w;
    }
    idx = (idx + 37) & (kWords - 1);
  }
  const long long t1 = clock64();
  if (acc.x == 0x12345678u && acc.y == 1u) sink[blockIdx.x] = acc;  // keep the loads
  if (threadIdx.x == 0) atomicMax((unsigned long long*)cycles, (unsigned long long)(t1 - t0));
}

}  // namespace

extern "C" int slos_probe_smem(int iters, double* gbs, double* sm_mhz) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = sms * 8;
  uint4* sink = nullptr;
  long long* cyc = nullptr;
  if (cudaMalloc(&sink, sizeof(uint4) * grid) != cudaSuccess) return 1;
  if (cudaMalloc(&cyc, sizeof(long long)) != cudaSuccess) return 1;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  smem_read_kernel<<<grid, kThreads>>>(iters / 8, sink, cyc);  // warm-up
  cudaMemset(cyc, 0, sizeof(long long));
  cudaEventRecord(a);
  smem_read_kernel<<<grid, kThreads>>>(iters, sink, cyc);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0.0f;
  cudaEventElapsedTime(&ms, a, b);
  long long c = 0;
  cudaMemcpy(&c, cyc, sizeof c, cudaMemcpyDeviceToHost);
  const double bytes = (double)grid * kThreads * (double)iters * 4.0 * sizeof(uint4);
  *gbs = bytes / (ms * 1e-3) / 1e9;
  *sm_mhz = (double)c / (ms * 1e-3) / 1e6;  // the longest CTA's loop ~ the whole launch (one wave)
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(sink);
  cudaFree(cyc);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

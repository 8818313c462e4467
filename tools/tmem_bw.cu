// tmem_bw.cu - microbenchmark: tcgen05.ld (32x32b.x32) throughput per SM as a
// function of the number of warps loading (development tool, not product).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_bw tmem_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2402_15106_b200/csrc/tc.cuh"
using namespace dsmpnn;

__global__ void __launch_bounds__(512, 1) tmem_bw_kernel(int nwarps, int iters, unsigned long long *cycles, uint32_t *sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tc::tmem_alloc<512>(&slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = slot;
  uint32_t acc = 0;
  __syncthreads();
  const unsigned long long t0 = clock64();
  if (warp < nwarps) {
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t col0 = (uint32_t)((warp >> 2) * 64) & 511u;
    for (int i = 0; i < iters; ++i) {
      uint32_t v[32], w[32];
      tc::tmem_ld32(tmem + lane_off + ((col0 + (i & 3) * 128) & 511u), v);
      tc::tmem_ld32(tmem + lane_off + ((col0 + 32 + (i & 3) * 128) & 511u), w);
      tc::tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 32; ++j) acc += v[j] ^ w[j];
    }
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * 512 + threadIdx.x] = acc;
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tmem);
}

int main() {
  unsigned long long *cyc;
  uint32_t *sink;
  cudaMalloc(&cyc, 148 * sizeof(unsigned long long));
  cudaMalloc(&sink, 148 * 512 * 4);
  const int iters = 4096;
  for (int nw : {1, 2, 4, 8, 16}) {
    tmem_bw_kernel<<<148, 512>>>(nw, iters, cyc, sink);
    cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    const double bytes = (double)nw * iters * 2 * 32 * 32 * 4;  // per SM
    printf("warps %2d: %8llu cycles, %.1f bytes/cycle/SM  (%s)\n", nw, h[0], bytes / h[0],
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}

// mma_rate.cu - cycles per tcgen05.mma (bf16, cta_group::1) for the shapes of
// the fused edge kernels: SS vs TS (A in TMEM), N = 64 / 128 / 256, K-major vs
// MN-major B, one accumulator (dependent chain) vs 4 alternating.  Operand
// contents are irrelevant (timing only).  Development tool:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/mma_rate.cu -o tools/mma_rate && tools/mma_rate
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "../paper_2402_15106_b200/csrc/tc.cuh"
using namespace dsmpnn;

__global__ void rate_kernel(unsigned long long *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int t = threadIdx.x, warp = t >> 5;
  if (warp == 0) tc::tmem_alloc<512>(&slot);
  if (t == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
  for (int q = t; q < (96 * 1024) / 16; q += blockDim.x) reinterpret_cast<uint4 *>(sm)[q] = make_uint4(0x3F803F80u, 0, 0, 0);
  tc::fence_async_shared();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = slot;
  uint32_t ph = 0;
  if (t == 0) {
    const uint32_t a = tc::smem_u32(sm), b = a + 32768;
    int o = 0;
    // cases: (N, ts, b_mn, nacc)
    const int Ns[] = {64, 128, 256};
    for (int ci = 0; ci < 3; ++ci)
      for (int ts = 0; ts < 2; ++ts)
        for (int bmn = 0; bmn < 2; ++bmn)
          for (int nacc = 1; nacc <= 4; nacc *= 4) {
            const int N = Ns[ci];
            if (N * nacc > 256) continue;
            const uint32_t id = tc::idesc_bf16(128, N, false, bmn != 0);
            for (int rep = 0; rep < 2; ++rep) {
              const unsigned long long t0 = clock64();
              for (int i = 0; i < 64; ++i) {
                const uint32_t d = tmem + (uint32_t)((i % nacc) * N);
                const uint64_t bd = bmn ? tc::sdesc(b + (i & 3) * 2048, 8192, 1024, tc::kSw128)
                                        : tc::sdesc(b + (i & 3) * 32, 16, 1024, tc::kSw128);
                if (ts)
                  tc::mma_bf16_ts(d, tmem + 256 + (i & 3) * 8, bd, id, i >= nacc ? 1u : 0u);
                else
                  tc::mma_bf16_ss(d, tc::sdesc(a + (i & 3) * 32, 16, 1024, tc::kSw128), bd, id, i >= nacc ? 1u : 0u);
              }
              tc::mma_commit(&bar);
              tc::mbar_wait(&bar, ph);
              ph ^= 1;
              const unsigned long long t1 = clock64();
              if (rep == 1) {
                out[o * 5 + 0] = N; out[o * 5 + 1] = ts; out[o * 5 + 2] = bmn; out[o * 5 + 3] = nacc;
                out[o * 5 + 4] = (t1 - t0) / 64;
                ++o;
              }
            }
          }
    // unrolled: 16 MMAs per group with compile-time descriptors (as the kernels issue them)
    {
      const uint32_t id64 = tc::idesc_bf16(128, 64, false, false), id128 = tc::idesc_bf16(128, 128, false, false),
                     id256 = tc::idesc_bf16(128, 256, false, false);
      const uint32_t ids[3] = {id64, id128, id256};
      for (int ci = 0; ci < 3; ++ci)
        for (int ts = 0; ts < 2; ++ts)
          for (int rep = 0; rep < 2; ++rep) {
            const uint32_t id = ids[ci];
            const unsigned long long t0 = clock64();
#pragma unroll 1
            for (int it = 0; it < 4; ++it) {
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                const uint64_t bd = tc::sdesc(b + (i & 3) * 32, 16, 1024, tc::kSw128);
                if (ts)
                  tc::mma_bf16_ts(tmem, tmem + 256 + (i & 3) * 8, bd, id, (it | i) ? 1u : 0u);
                else
                  tc::mma_bf16_ss(tmem, tc::sdesc(a + (i & 3) * 32, 16, 1024, tc::kSw128), bd, id, (it | i) ? 1u : 0u);
              }
            }
            tc::mma_commit(&bar);
            tc::mbar_wait(&bar, ph);
            ph ^= 1;
            const unsigned long long t1 = clock64();
            if (rep == 1) {
              out[o * 5 + 0] = 64 << ci; out[o * 5 + 1] = ts; out[o * 5 + 2] = 9; out[o * 5 + 3] = 1;
              out[o * 5 + 4] = (t1 - t0) / 64;
              ++o;
            }
          }
    }
    out[255] = o;
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tmem);
}

int main() {
  unsigned long long *d, h[256];
  cudaMalloc(&d, sizeof(h));
  cudaMemset(d, 0, sizeof(h));
  cudaFuncSetAttribute(rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  rate_kernel<<<1, 128, 96 * 1024>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("M=128 K=16 bf16: cycles per MMA (64 issued, floor = N/2)\n   N  A      B       acc  cyc\n");
  for (int i = 0; i < (int)h[255]; ++i)
    printf("%4llu  %s  %s  %4llu  %4llu\n", h[i * 5], h[i * 5 + 1] ? "tmem" : "smem", h[i * 5 + 2] == 9 ? "unroll" : h[i * 5 + 2] ? "MN-maj" : "K-maj ",
           h[i * 5 + 3], h[i * 5 + 4]);
  return 0;
}

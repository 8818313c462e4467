// ts_test.cu - checks the tcgen05 "A in TMEM" operand layout of tc::mma_bf16_ts /
// tc::tmem_st32 (tc.cuh): A[m][k] (bf16) at TMEM lane m, column k/2, low half for even k
// (tcgen05.st.32x32b from the thread owning lane m).  Development tool.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "../paper_2402_15106_b200/csrc/tc.cuh"
using namespace dsmpnn;

// D[128 x 64] = A[128 x 64] B^T, B stored [64 n][64 k] K-major SW128
__global__ void ts_kernel(const __nv_bfloat16 *A, const __nv_bfloat16 *B, float *D) {
  __shared__ __align__(1024) uint8_t sB[8192];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int t = threadIdx.x, warp = t >> 5;
  if (warp == 0) tc::tmem_alloc<128>(&slot);
  if (t == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
  for (int q = t; q < 64 * 8; q += 128) {
    const int n = q / 8, c = q % 8;
    *reinterpret_cast<uint4 *>(sB + tc::sw128_off(n, c)) = reinterpret_cast<const uint4 *>(B)[q];
  }
  tc::fence_async_shared();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = slot;
  // A row m = t -> TMEM lane t, columns 64 .. 64 + 31
  {
    uint32_t r[32];
    for (int j = 0; j < 32; ++j) {
      __nv_bfloat162 h;
      h.x = A[t * 64 + 2 * j];
      h.y = A[t * 64 + 2 * j + 1];
      r[j] = *reinterpret_cast<uint32_t *>(&h);
    }
    tc::tmem_st32(tmem + ((uint32_t)(warp * 32) << 16) + 64, r);
    tc::tmem_st_wait();
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (t == 0) {
    constexpr uint32_t id = tc::idesc_bf16(128, 64, false, false);
    for (int kk = 0; kk < 4; ++kk) {
      const uint64_t bd = tc::sdesc(tc::smem_u32(sB) + kk * 32, 16, 1024, tc::kSw128);
      tc::mma_bf16_ts(tmem, tmem + 64 + kk * 8, bd, id, kk > 0 ? 1u : 0u);
    }
    tc::mma_commit(&bar);
  }
  tc::mbar_wait(&bar, 0);
  tc::tc_fence_after();
  uint32_t v[32], w[32];
  tc::tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16), v);
  tc::tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + 32, w);
  tc::tmem_ld_wait();
  for (int j = 0; j < 32; ++j) { D[t * 64 + j] = __uint_as_float(v[j]); D[t * 64 + 32 + j] = __uint_as_float(w[j]); }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<128>(tmem);
}

int main() {
  const int M = 128, N = 64, K = 64;
  __nv_bfloat16 *hA = (__nv_bfloat16 *)malloc(M * K * 2), *hB = (__nv_bfloat16 *)malloc(N * K * 2);
  float *hD = (float *)malloc(M * N * 4);
  srand(1);
  for (int i = 0; i < M * K; ++i) hA[i] = __float2bfloat16((rand() % 17 - 8) / 8.0f);
  for (int i = 0; i < N * K; ++i) hB[i] = __float2bfloat16((rand() % 13 - 6) / 4.0f);
  __nv_bfloat16 *dA, *dB; float *dD;
  cudaMalloc(&dA, M * K * 2); cudaMalloc(&dB, N * K * 2); cudaMalloc(&dD, M * N * 4);
  cudaMemcpy(dA, hA, M * K * 2, cudaMemcpyHostToDevice); cudaMemcpy(dB, hB, N * K * 2, cudaMemcpyHostToDevice);
  ts_kernel<<<1, 128>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(hD, dD, M * N * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += (double)__bfloat162float(hA[m * K + k]) * __bfloat162float(hB[n * K + k]);
      maxerr = fmax(maxerr, fabs(s - hD[m * N + n]));
    }
  printf("ts_test: %s, max abs err %g (D[0]=%g)\n", cudaGetErrorString(e), maxerr, hD[0]);
  return maxerr < 1e-3 ? 0 : 1;
}

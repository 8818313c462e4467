// tgemm.cuh - generic bf16 tcgen05 GEMM (TMA -> SMEM ring -> tcgen05.mma ->
// TMEM -> fp32 epilogue) used by the BF16 layer for its dense contractions.
#pragma once
#include "common.cuh"

namespace dsmpnn {

// Operand description: a bf16 row-major matrix in global memory.
//   A is M x K: K-major if stored [M][K] (a_mn_major = false) or M-major if
//   stored [K][M] (a_mn_major = true).  B is K x N: K-major if stored [N][K],
//   N-major if stored [K][N].  ld = elements between consecutive stored rows.
struct TgemmArgs {
  int64_t M, N, K;
  const void *A;
  int64_t lda;
  bool a_mn_major;
  const void *B;
  int64_t ldb;
  bool b_mn_major;
  float *C;          // fp32 output [M x N] with row stride ldc (or split-K partials)
  int64_t ldc;
  int splits;        // split-K count; > 1 writes partial z at C + z * split_stride
  int64_t split_stride;
  int accumulate;    // 1: C += result (only when splits == 1)
};

// C = A * B (+ C).  N-tile = min(N rounded up to 16, 256) per CTA.
dsmpnn_status tgemm(const TgemmArgs &a, cudaStream_t s);

// sum_z partial[z] (fixed order) -> C (+= if accumulate)
dsmpnn_status splitk_sum(const float *partial, int splits, int64_t split_stride, int64_t M, int64_t N, int64_t ld,
                         float *C, int64_t ldc, int accumulate, cudaStream_t s);

}  // namespace dsmpnn

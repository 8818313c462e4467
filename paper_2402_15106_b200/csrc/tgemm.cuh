// tgemm.cuh - generic bf16 tcgen05 GEMM (TMA -> SMEM ring -> tcgen05.mma ->
// TMEM -> fp32 epilogue) used by the BF16 layer for its dense contractions.
#pragma once
#include "common.cuh"
#include <cuda.h>
#include <cuda_bf16.h>

namespace dsmpnn {

// Operand description: a bf16 row-major matrix in global memory.
//   A is M x K: K-major if stored [M][K] (a_mn_major = false) or M-major if
//   stored [K][M] (a_mn_major = true).  B is K x N: K-major if stored [N][K],
//   N-major if stored [K][N].  ld = elements between consecutive stored rows.
constexpr int kColsumRows = 148 * 2 * 4;

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
  // optional bf16 epilogue (splits == 1): if out16 != null the tile is written
  // as bf16 to out16[m*ld16 + n] instead of C, after
  //   x *= row_scale[m]             (row_scale != null)
  //   x  = mask16[m*ldmask + n] > 0 ? x : 0   (mask16 != null)
  // and column sums of the written values, per CTA and epilogue warp, go to
  //   colsum_part[(cta*4 + warp) * N + n]   (colsum_part != null, N <= 256;
  //   the caller zero-fills kColsumRows x N and sums all rows)
  __nv_bfloat16 *out16 = nullptr;
  int64_t ld16 = 0;
  const float *row_scale = nullptr;
  const __nv_bfloat16 *mask16 = nullptr;
  int64_t ldmask = 0;
  float *colsum_part = nullptr;
  // keep the whole B in SMEM across tiles (bf16 epilogue, N <= 256, K <= 256,
  // no split-K): only A streams (B5's W2)
  bool b_resident = false;
};

// 2-D bf16 TMA descriptor: `inner` contiguous elements, `outer` rows of `ld`
// elements, box {box_inner, box_outer}; swizzle = box row bytes (32/64/128).
dsmpnn_status make_tmap_bf16(CUtensorMap *m, const void *base, int64_t inner, int64_t outer, int64_t ld,
                             int box_inner, int box_outer);

// C = A * B (+ C).  N-tile = min(N rounded up to 16, 256) per CTA.
dsmpnn_status tgemm(const TgemmArgs &a, cudaStream_t s);

// sum_z partial[z] (fixed order) -> C (+= if accumulate)
dsmpnn_status splitk_sum(const float *partial, int splits, int64_t split_stride, int64_t M, int64_t N, int64_t ld,
                         float *C, int64_t ldc, int accumulate, cudaStream_t s);

}  // namespace dsmpnn

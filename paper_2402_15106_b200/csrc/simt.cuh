// simt.cuh - fp32 SIMT building blocks of the F32 mode (reading R18: fp32
// FFMA, no TF32): a strided tiled GEMM with bias/ReLU epilogue and
// deterministic split-K, and a deterministic column sum.
#pragma once
#include "common.cuh"

namespace dsmpnn {

struct SgemmArgs {
  int64_t M, N, K;
  const float *A;
  int64_t sam, sak;  // A(m,k) = A[m*sam + k*sak]
  const float *B;
  int64_t sbk, sbn;  // B(k,n) = B[k*sbk + n*sbn]
  float *C;
  int64_t ldc;       // C(m,n) = C[m*ldc + n]
  const float *bias; // [N] or null
  int relu;          // apply ReLU after bias
  int beta;          // 1: C += result, 0: C = result
  float alpha;       // result = alpha * A.B (before bias)
};

// C = act(alpha*A.B + bias) (+ C).  With split-K (splits > 1) the partial
// products go to `partial` [splits x M x N] and are summed in split order.
dsmpnn_status sgemm(const SgemmArgs &a, int splits, float *partial, cudaStream_t s);

// out[n] (+)= sum_{m<M} A[m*lda + n] in a fixed order (deterministic)
dsmpnn_status colsum(const float *A, int64_t M, int64_t N, int64_t lda, float *out, int accumulate, cudaStream_t s);
// same result semantics, two-level (row chunks -> partials -> sum in chunk
// order) when M is large; ws must hold kColsumChunks * N floats
constexpr int kColsumChunks = 128;
dsmpnn_status colsum_ws(const float *A, int64_t M, int64_t N, int64_t lda, float *out, int accumulate, float *ws,
                        cudaStream_t s);

}  // namespace dsmpnn

// layer_bf16_common.cuh - shared pieces of the BF16 layer kernels: packed
// weight layout and SMEM operand layouts (the tile walker is in edge_fwd2.cuh).
#pragma once
#include <cuda_bf16.h>

#include "common.cuh"
#include "tc.cuh"

namespace dsmpnn {

constexpr int KH = 256;  // kappa hidden width of the BF16 kernels; k < KH runs zero-padded to KH
                         // (pack_bf16_kernel: the padded units are exact zeros, layer_bf16_bwd.cu
                         // returns the gradients of the k real units)
// columns of the 16-wide padded edge tile / packed W1 that carry the first
// kappa layer's bias as three bf16 terms (layer_bf16.cu pack_bf16_kernel):
// d_e <= 13 in BF16 mode
constexpr int kBiasCol0 = 13;

static inline int64_t kpad_of(const dsmpnn_layer_desc &d) {
  int64_t kp = (int64_t)(KH + 2) * d.d_in;
  return (kp + 63) / 64 * 64;
}

// ---------------------------------------------------------- packed weights
struct Packed {
  __nv_bfloat16 *W1;   // [KH x 16]   zero-padded d_e
  __nv_bfloat16 *W2;   // [KH x KH]
  __nv_bfloat16 *ThT;  // [D x Kpad]  Theta~_aug^T  (K-major B of the node GEMM)
  __nv_bfloat16 *Th;   // [Kpad x D]  Theta~_aug    (K-major B of the dS GEMM)
  float *b1, *b2;      // [KH] the kappa biases, zero-padded (the kernels' copies)
};
static inline Packed carve_packed(const dsmpnn_layer_desc &d, void *base) {
  Carver c(base, SIZE_MAX);
  Packed p;
  int64_t kp = kpad_of(d);
  p.W1 = c.take<__nv_bfloat16>((int64_t)KH * 16);
  p.W2 = c.take<__nv_bfloat16>((int64_t)KH * KH);
  p.ThT = c.take<__nv_bfloat16>((int64_t)d.d_out * kp);
  p.Th = c.take<__nv_bfloat16>(kp * d.d_out);
  p.b1 = c.take<float>(KH);
  p.b2 = c.take<float>(KH);
  return p;
}

// ------------------------------------------------------------- SMEM layouts
// interleaved (no swizzle) K-major K=16 operand: row r, 16-byte chunk u
__device__ __forceinline__ uint32_t il_off(uint32_t r, uint32_t u) { return (r >> 3) * 256u + u * 128u + (r & 7u) * 16u; }
__device__ __forceinline__ uint32_t sw64_off(uint32_t r, uint32_t c) { return r * 64u + ((c ^ ((r >> 1) & 3u)) << 4); }

template <int D>
__device__ __forceinline__ uint32_t v_off(uint32_t s, uint32_t c) {
  return D == 64 ? tc::sw128_off(s, c) : sw64_off(s, c);
}

}  // namespace dsmpnn

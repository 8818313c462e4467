// layer_bf16_common.cuh - shared pieces of the BF16 layer kernels: packed
// weight layout, the 128-slot edge tile walker and SMEM operand layouts.
#pragma once
#include <cuda_bf16.h>

#include "common.cuh"
#include "tc.cuh"

namespace dsmpnn {

constexpr int KH = 256;  // kappa hidden width supported by the BF16 kernels

static inline int64_t kpad_of(const dsmpnn_layer_desc &d) {
  int64_t kp = (int64_t)(d.k + 2) * d.d_in;
  return (kp + 63) / 64 * 64;
}

// ---------------------------------------------------------- packed weights
struct Packed {
  __nv_bfloat16 *W1;   // [KH x 16]   zero-padded d_e
  __nv_bfloat16 *W2;   // [KH x KH]
  __nv_bfloat16 *ThT;  // [D x Kpad]  Theta~_aug^T  (K-major B of the node GEMM)
  __nv_bfloat16 *Th;   // [Kpad x D]  Theta~_aug    (K-major B of the dS GEMM)
};
static inline Packed carve_packed(const dsmpnn_layer_desc &d, void *base) {
  Carver c(base, SIZE_MAX);
  Packed p;
  int64_t kp = kpad_of(d);
  p.W1 = c.take<__nv_bfloat16>((int64_t)d.k * 16);
  p.W2 = c.take<__nv_bfloat16>((int64_t)d.k * d.k);
  p.ThT = c.take<__nv_bfloat16>((int64_t)d.d_out * kp);
  p.Th = c.take<__nv_bfloat16>(kp * d.d_out);
  return p;
}

// ------------------------------------------------------------- edge kernel
struct Seg {
  int64_t node;
  int32_t slot0, nslots;  // slots [slot0, slot0 + nslots), multiple of 16
  int32_t deg;
  int32_t start;          // 1: first segment of the node (no accumulation)
  int32_t complete;       // 1: last segment of the node
  int32_t tslot;          // TMEM S slot
};
constexpr int kMaxSeg = 8;

template <int D>
struct EF {
  static constexpr int W2_BYTES = KH * KH * 2;          // 131072
  static constexpr int AH_BYTES = 128 * KH * 2;         // 65536
  static constexpr int V_BYTES = 128 * D * 2;           // 16384 / 8192
  static constexpr int W1_BYTES = KH * 32;              // 8192
  static constexpr int E_BYTES = 128 * 32;              // 4096
  static constexpr int OFF_W2 = 0;
  static constexpr int OFF_AH = OFF_W2 + W2_BYTES;
  static constexpr int OFF_V = OFF_AH + AH_BYTES;
  static constexpr int OFF_W1 = OFF_V + V_BYTES;
  static constexpr int OFF_E = OFF_W1 + W1_BYTES;
  static constexpr int OFF_MISC = OFF_E + E_BYTES;
  static constexpr int SMEM = OFF_MISC + 1024 + 1024;   // misc + alignment slack
  static constexpr uint32_t TMEM_COLS = 512;
  static constexpr int NSLOT = (512 - KH) / (2 * D);    // TMEM S slots: 2 (D=64) or 4 (D=32)
};

struct EdgeMisc {
  int32_t slot_edge[128];   // edge id per slot, -1 = padding
  Seg seg[kMaxSeg];
  int32_t nseg;
  int32_t more;             // 1 if this tile has slots
  int64_t cur_row;          // walker state
  int32_t cur_off;
  int32_t node_ctr;
  int64_t row_end;
  uint64_t bar;             // MMA completion barrier
  uint32_t tmem;
};

// interleaved (no swizzle) K-major K=16 operand: row r, 16-byte chunk u
__device__ __forceinline__ uint32_t il_off(uint32_t r, uint32_t u) { return (r >> 3) * 256u + u * 128u + (r & 7u) * 16u; }
__device__ __forceinline__ uint32_t sw64_off(uint32_t r, uint32_t c) { return r * 64u + ((c ^ ((r >> 1) & 3u)) << 4); }

template <int D>
__device__ __forceinline__ uint32_t v_off(uint32_t s, uint32_t c) {
  return D == 64 ? tc::sw128_off(s, c) : sw64_off(s, c);
}

// build the next tile: segments of whole 16-slot blocks, rows padded to 16
__device__ __forceinline__ void build_tile(EdgeMisc *m, const int64_t *__restrict__ row_ptr) {
  int used = 0, ns = 0;
  for (int s = 0; s < 128; ++s) m->slot_edge[s] = -1;
  while (used < 128 && m->cur_row < m->row_end && ns < kMaxSeg) {
    int64_t i = m->cur_row;
    int64_t p0 = row_ptr[i];
    int deg = (int)(row_ptr[i + 1] - p0);
    if (deg == 0) {
      m->cur_row++;
      continue;
    }
    int padded = (deg + 15) & ~15;
    int off = m->cur_off;
    int take = padded - off;
    if (take > 128 - used) take = 128 - used;
    Seg &g = m->seg[ns++];
    g.node = i;
    g.slot0 = used;
    g.nslots = take;
    g.deg = deg;
    g.start = off == 0;
    if (off == 0) m->node_ctr++;
    g.tslot = (m->node_ctr - 1) & 1;  // two TMEM S slots: the open row and the next one
    for (int q = 0; q < take; ++q) {
      int eidx = off + q;
      m->slot_edge[used + q] = eidx < deg ? (int32_t)(p0 + eidx) : -1;
    }
    off += take;
    used += take;
    g.complete = off >= padded;
    if (g.complete) {
      m->cur_row++;
      m->cur_off = 0;
    } else {
      m->cur_off = off;
    }
  }
  m->nseg = ns;
  m->more = used > 0;
}


}  // namespace dsmpnn

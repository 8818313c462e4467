// layer_bf16_bwd.cu - BF16 backward of the edge-conditioned convolution
// (Alg. 1 :417 "Backprop", reading R16 detach), tcgen05 (sm_100a).
//
// With ghat = G * sigma'(pre), S~_aug and the packed Theta~_aug of the forward:
//   B0  ghat (fp32 + bf16 copy), db += colsum(ghat), root term of dv
//   B1  dTheta~_aug = S~_aug^T ghat              (tgemm, M-major A, N-major B)
//       -> dW3, db3, dW_root
//   B2  dS_i = (ghat_i Theta~^T) / deg_i          (tgemm, bf16 epilogue, row scale)
//   B3  edge kernel per 128-slot tile: recompute a1, h (W1 resident, W2
//       streamed by TMA), then per row  dH^T = dS_i V^T  and  U = H dS_i
//       (tcgen05), dz2 = dH * [h > 0] -> global, u_p = U + dS_i[k] -> global,
//       a1 -> global (only for the unfused B4/B5), per-CTA db2 partial sums.
//   Without the edge-attribute gradient (the hot path):
//   B4' dW2 += dz2^T a1, a1 recomputed from e     (dw2.cuh)
//   B56 dz1 = (dz2 W2) * [a1 > 0] on chip; dW1 += dz1^T e, db1 (dz1w1.cuh)
//   With it (training with edge refresh, f1):
//   B4  dW2 += dz2^T a1                           (tgemm, split-K over edges)
//   B5  dz1 = (dz2 W2) * [a1 > 0]                  (tgemm, bf16 + mask epilogue,
//                                                   column sums -> db1)
//   B6  dW1 += dz1^T e ; de = dz1 W1              (tgemm)
//   B7  dv[j] += sum_{p: col(p)=j} u_p            (deterministic CSC scatter)
#include <cuda.h>
#include <cstdlib>

#include "layer_bf16.cuh"
#include "layer_bf16_common.cuh"
#include "simt.cuh"
#include "tc.cuh"
#include "tgemm.cuh"
#include "edge_bwd2.cuh"
#include "edge_bwd3.cuh"
#include "edge_bwd4.cuh"
#include "dz1w1.cuh"
#include "dw2.cuh"

namespace dsmpnn {

// ------------------------------------------------------------- B0 kernels
// B0 in one pass over 32-row blocks: ghat = G * sigma'(pre) (fp32 + bf16
// copy), 1/deg, the block's column sums of ghat (-> db, summed over blocks in
// block order by colsum), and the root term of dv: dv += ghat W_root (dense)
// or dv += ghat (identity).  W_root is [D x D] with dv[m][n] += sum_c ghat[m][c] W_root[c][n].
template <int D>
__global__ void __launch_bounds__(256) b0_bf16_kernel(const float *__restrict__ G, const float *__restrict__ pre,
                                                      const int64_t *__restrict__ row_ptr, int64_t rb, int64_t re,
                                                      int act, int root, const float *__restrict__ Wr,
                                                      float *__restrict__ gh, __nv_bfloat16 *__restrict__ gh16,
                                                      float *__restrict__ inv_deg, float *__restrict__ cs_part,
                                                      float *__restrict__ dv) {
  pdl_wait();
  pdl_trigger();
  __shared__ float sg[32][D + 1];
  __shared__ __align__(16) float sw[D][D];
  const int t = threadIdx.x;
  const int64_t r0 = rb + (int64_t)blockIdx.x * 32;
  const bool dense = root == DSMPNN_ROOT_DENSE && dv != nullptr;
  // thread = (row rr, group of D / 8 consecutive columns) for the root term:
  // its dv entries are loaded first, so the read-modify-write at the end
  // does not wait on them
  constexpr int NC = D / 8;
  const int rr = t >> 3, n0 = (t & 7) * NC;
  const bool mine = dv != nullptr && root != DSMPNN_ROOT_NONE && r0 + rr < re;
  float4 dvv[NC / 4];
  if (mine) {
#pragma unroll
    for (int j = 0; j < NC / 4; ++j) dvv[j] = reinterpret_cast<const float4 *>(dv + (r0 + rr) * D + n0)[j];
  }
  if (dense)
    for (int i = t; i < D * D / 4; i += 256) reinterpret_cast<float4 *>(&sw[0][0])[i] = reinterpret_cast<const float4 *>(Wr)[i];
  for (int i = t; i < 32 * D / 4; i += 256) {  // four consecutive columns per thread
    const int r = (i * 4) / D, c = (i * 4) % D;
    const int64_t row = r0 + r;
    float4 g = make_float4(0.f, 0.f, 0.f, 0.f);
    if (row < re) {
      const int64_t idx = row * D + c;
      g = *reinterpret_cast<const float4 *>(G + idx);
      if (act == DSMPNN_ACT_RELU) {
        const float4 p = *reinterpret_cast<const float4 *>(pre + idx);
        g.x = p.x > 0.f ? g.x : 0.f;
        g.y = p.y > 0.f ? g.y : 0.f;
        g.z = p.z > 0.f ? g.z : 0.f;
        g.w = p.w > 0.f ? g.w : 0.f;
      }
      *reinterpret_cast<float4 *>(gh + idx) = g;
      *reinterpret_cast<uint2 *>(gh16 + idx) = make_uint2(tc::pack_bf16(g.x, g.y), tc::pack_bf16(g.z, g.w));
    }
    sg[r][c] = g.x;
    sg[r][c + 1] = g.y;
    sg[r][c + 2] = g.z;
    sg[r][c + 3] = g.w;
  }
  if (t < 32 && r0 + t < re) {
    const int64_t i = r0 + t;
    const int64_t deg = row_ptr[i + 1] - row_ptr[i];
    inv_deg[i] = deg > 0 ? 1.0f / (float)deg : 0.f;
  }
  __syncthreads();
  if (t < D) {
    float cs = 0.f;
#pragma unroll 8
    for (int r = 0; r < 32; ++r) cs += sg[r][t];
    cs_part[(int64_t)blockIdx.x * D + t] = cs;
  }
  if (!mine) return;
  float acc[NC];
  if (dense) {
#pragma unroll
    for (int j = 0; j < NC; ++j) acc[j] = 0.f;
#pragma unroll 4
    for (int c = 0; c < D; ++c) {
      const float g = sg[rr][c];
#pragma unroll
      for (int j = 0; j < NC; j += 4) {
        const float4 w4 = *reinterpret_cast<const float4 *>(&sw[c][n0 + j]);
        acc[j] += g * w4.x;
        acc[j + 1] += g * w4.y;
        acc[j + 2] += g * w4.z;
        acc[j + 3] += g * w4.w;
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < NC; ++j) acc[j] = sg[rr][n0 + j];
  }
  float4 *o = reinterpret_cast<float4 *>(dv + (r0 + rr) * D + n0);
#pragma unroll
  for (int j = 0; j < NC / 4; ++j) {
    float4 x = dvv[j];
    x.x += acc[4 * j];
    x.y += acc[4 * j + 1];
    x.z += acc[4 * j + 2];
    x.w += acc[4 * j + 3];
    o[j] = x;
  }
}

// dW3[c*D+o, kap] += dT[c*k+kap, o]  (the [c][kappa] block of S~_aug's K
// order): 32 x 32 tiles transposed through shared memory so both the dT reads
// and the dW3 read-modify-writes are coalesced.  grid = (k/32, D/32, D)
__global__ void unpack_dw3_kernel(const float *__restrict__ dT, int k, int D, float *__restrict__ dW3) {
  pdl_wait();
  pdl_trigger();
  __shared__ float t[32][33];
  const int kap0 = blockIdx.x * 32, o0 = blockIdx.y * 32, c = blockIdx.z;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 256 threads: 8 rows per pass
  for (int r = ty; r < 32; r += 8) t[r][tx] = dT[((int64_t)c * k + kap0 + r) * D + o0 + tx];
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    float *w = dW3 + ((int64_t)c * D + o0 + r) * k + kap0 + tx;
    *w += t[tx][r];
  }
}

// db3[c*D+o] += dT[k*D+c, o]; dW_root[o, c] += dT[(k+1)*D+c, o]
__global__ void unpack_bias_root_kernel(const float *__restrict__ dT, int k, int D, float *__restrict__ db3,
                                        float *__restrict__ dWr) {
  pdl_wait();
  pdl_trigger();
  const int64_t total = (int64_t)D * D;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int a = (int)(t / D), b = (int)(t - (int64_t)a * D);
    if (db3) db3[t] += dT[((int64_t)k * D) * D + t];                       // c = a, o = b
    if (dWr) dWr[(int64_t)b * D + a] += dT[((int64_t)(k + 1) * D) * D + t];  // c = a, o = b
  }
}

// dst[r * ld_dst + c] += src[r * ld_src + c] for r < rows, c < cols: the k
// real units of a KH-wide gradient (k < KH, zero-padded kappa MLP)
__global__ void add_block_kernel(const float *__restrict__ src, int64_t ld_src, float *__restrict__ dst,
                                 int64_t ld_dst, int64_t rows, int64_t cols) {
  const int64_t total = rows * cols;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / cols, c = t - r * cols;
    dst[r * ld_dst + c] += src[r * ld_src + c];
  }
}

// dW1[r, c] += full[r, c] for c < d_e (full is [k x 16]); same for de rows
__global__ void add_cols_kernel(const float *__restrict__ full, int64_t rows, int ld_full, int ncols,
                                float *__restrict__ dst, int accumulate) {
  int64_t total = rows * ncols;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = t / ncols;
    int c = (int)(t - r * ncols);
    float x = full[r * ld_full + c];
    dst[t] = accumulate ? dst[t] + x : x;
  }
}

// ---------------------------------------------------------- B3 edge kernel
// edge_bwd2.cuh (warp-specialised, pipelined)

// ------------------------------------------------------------ workspace
struct BBwd {
  float *gh;               // [n_dst x D]
  __nv_bfloat16 *gh16;     // [n_dst x D]
  float *inv_deg;          // [n_dst]
  float *dT;               // [kp x D]
  __nv_bfloat16 *dS;       // [n_dst x (k+1) x D]
  __nv_bfloat16 *A1;       // [E x k]
  __nv_bfloat16 *dZ2;      // [E x k]
  __nv_bfloat16 *dZ1;      // [E x k]
  __nv_bfloat16 *U;        // [E x D] (bf16)
  float *part;             // split-K partials (max over users)
  float *db2_part;         // [kNumSMs x k]
  float *db1_part;         // [kColsumRows x k]
  float *cs_ws;            // colsum partials [kColsumChunks x max(D, k)]
  float *dW1f;             // [k x 16]
  float *de16;             // [E x 16]
  float *w1_part;          // [kNumSMs/2 x KH x 16] fused B5+B6 per-pair dW1
  float *b1_part;          // [kNumSMs/2 x 2 x KH]  fused B5+B6 per-pair db1
  float *w2_part;          // [kNumSMs/2 x KH x KH] B4 (dw2.cuh) per-pair dW2
  float *b0_part;          // [ceil(n_dst/32) x D] B0 per-block column sums of ghat
  int32_t *upos;           // [E] CSC position of every edge (U rows in CSC order for the B7 stream)
  // k < KH: the KH-wide W1, b1, W2, b2, W3 gradients (contiguous, zeroed per call)
  float *gW1 = nullptr, *gb1 = nullptr, *gW2 = nullptr, *gb2 = nullptr, *gW3 = nullptr;
  char *gpad_end = nullptr;
};
constexpr int kSplitsW = 64;
static BBwd carve_bf16_bwd(Carver &c, const dsmpnn_layer_desc &d, int64_t n_dst, int64_t E) {
  BBwd b;
  const int D = d.d_in;
  int64_t kp = (int64_t)(KH + 2) * D;
  kp = (kp + 63) / 64 * 64;
  b.gh = c.take<float>(n_dst * D);
  b.gh16 = c.take<__nv_bfloat16>(n_dst * D);
  b.inv_deg = c.take<float>(n_dst);
  b.dT = c.take<float>(kp * D);
  b.dS = c.take<__nv_bfloat16>(n_dst * (int64_t)(KH + 1) * D);
  b.A1 = c.take<__nv_bfloat16>(E * KH);
  b.dZ2 = c.take<__nv_bfloat16>(E * KH);
  b.dZ1 = c.take<__nv_bfloat16>(E * KH);
  b.U = c.take<__nv_bfloat16>(E * D);
  b.part = c.take<float>((int64_t)kSplitsW * KH * KH);
  b.db2_part = c.take<float>((int64_t)kNumSMs * KH);
  b.db1_part = c.take<float>((int64_t)kColsumRows * KH);
  b.cs_ws = c.take<float>((int64_t)kColsumChunks * std::max(KH, d.d_in));
  b.dW1f = c.take<float>((int64_t)KH * 16);
  b.de16 = c.take<float>(E * 16);
  b.w1_part = c.take<float>((int64_t)(kNumSMs / 2) * KH * 16);
  b.b1_part = c.take<float>((int64_t)kNumSMs * KH);
  b.w2_part = c.take<float>((int64_t)(kNumSMs / 2 + kDw2Groups) * KH * KH);
  b.b0_part = c.take<float>(ceil_div(std::max<int64_t>(n_dst, 1), 32) * D);
  b.upos = c.take<int32_t>(std::max<int64_t>(E, 1));
  if (d.k < KH) {  // KH-wide gradients of the kappa MLP (k real units added to the caller's at the end)
    b.gW1 = c.take<float>((int64_t)KH * d.d_e);
    b.gb1 = c.take<float>(KH);
    b.gW2 = c.take<float>((int64_t)KH * KH);
    b.gb2 = c.take<float>(KH);
    b.gW3 = c.take<float>((int64_t)d.d_in * d.d_out * KH);
    b.gpad_end = c.take<char>(0);
  }
  return b;
}

size_t bf16_bwd_ws_bytes(const dsmpnn_layer_desc &d, int64_t n_dst, int64_t n_loc, int64_t E) {
  Carver c(nullptr, 0);
  carve_bf16_bwd(c, d, n_dst, E);
  return c.used();
}

static int grid_of(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), 148 * 8)); }

// forward workspace layout (must match layer_bf16.cu)
struct BFwdView {
  const __nv_bfloat16 *S;
  const float *pre;
};
static BFwdView view_fwd(const dsmpnn_layer_desc &d, const void *ws, int64_t n_dst) {
  Carver c(const_cast<void *>(ws), SIZE_MAX);
  BFwdView f;
  f.S = c.take<__nv_bfloat16>(n_dst * kpad_of(d));
  f.pre = c.take<float>(n_dst * d.d_out);
  return f;
}

// dv[j] += sum over the CSC list of j of u_p (p in [eb, ee)).  One warp per
// node: the list's edge ids are read 32 at a time (one coalesced load) and
// handed out by shuffles; lane = (edge sub-slot, 16-byte channel chunk), so
// every U row gather of a batch is in flight at once.  Sub-slot sums combine
// by a butterfly: the summation order is fixed.
template <int D>
__global__ void scatter_csc_bf16_kernel(const __nv_bfloat16 *__restrict__ U, const int32_t *__restrict__ perm,
                                        const int64_t *__restrict__ cptr, int64_t n_loc, int64_t eb, int64_t ee,
                                        float *__restrict__ dv) {
  constexpr int LPR = D / 8, EPI = 32 / LPR, UNR = 32 / EPI;
  const int lane = threadIdx.x & 31, cl = lane % LPR, sub = lane / LPR;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; j < n_loc; j += nw) {
    const int64_t q0 = cptr[j], q1 = cptr[j + 1];
    float acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = 0.f;
    bool any = false;
    for (int64_t qb = q0; qb < q1; qb += 32) {
      const int32_t pl = qb + lane < q1 ? __ldg(perm + qb + lane) : -1;
      const int nb = (int)(q1 - qb < 32 ? q1 - qb : 32);
      uint4 x[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const int q = u * EPI + sub;
        const int64_t pe = __shfl_sync(0xffffffffu, pl, q);
        const bool ok = q < nb && pe >= eb && pe < ee;
        any |= ok;
        x[u] = ok ? __ldg(reinterpret_cast<const uint4 *>(U + pe * D) + cl) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&x[u]);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 f = __bfloat1622float2(h[i]);
          acc[2 * i] += f.x;
          acc[2 * i + 1] += f.y;
        }
      }
    }
#pragma unroll
    for (int off = LPR; off < 32; off <<= 1) {
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], off);
    }
    any = __any_sync(0xffffffffu, any);
    if (any && sub == 0) {
      float4 *o = reinterpret_cast<float4 *>(dv + j * D + cl * 8);
      float4 a0 = o[0], a1 = o[1];
      a0.x += acc[0]; a0.y += acc[1]; a0.z += acc[2]; a0.w += acc[3];
      a1.x += acc[4]; a1.y += acc[5]; a1.z += acc[6]; a1.w += acc[7];
      o[0] = a0;
      o[1] = a1;
    }
  }
}

// upos[perm[q]] = q: the CSC position of every edge
__global__ void csc_inverse_kernel(const int32_t *__restrict__ perm, int64_t n, int32_t *__restrict__ upos) {
  pdl_wait();
  pdl_trigger();
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
    upos[perm[q]] = (int32_t)q;
}

// B7 with U already in CSC order (edge_bwd4 wrote u_p to row upos[p]):
// dv[j] += sum of U rows cptr[j] .. cptr[j+1] (edges outside [eb, ee) skipped
// through perm unless the range is the whole graph).  One warp per node;
// lane = (row sub-slot, 16-byte chunk), consecutive rows: every warp load is
// one contiguous 512-byte (D = 64) block.  Sub-slot sums combine by a
// butterfly: the summation order is fixed.
template <int D>
__global__ void scatter_sorted_bf16_kernel(const __nv_bfloat16 *__restrict__ U, const int32_t *__restrict__ perm,
                                           const int64_t *__restrict__ cptr, int64_t n_loc, int64_t eb, int64_t ee,
                                           int full, float *__restrict__ dv) {
  pdl_wait();
  pdl_trigger();
  constexpr int LPR = D / 8, RPI = 32 / LPR, UNR = 4;
  const int lane = threadIdx.x & 31, cl = lane % LPR, sub = lane / LPR;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; j < n_loc; j += nw) {
    const int64_t q0 = cptr[j], q1 = cptr[j + 1];
    float acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = 0.f;
    bool any = false;
    for (int64_t qb = q0; qb < q1; qb += RPI * UNR) {
      uint4 x[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const int64_t q = qb + u * RPI + sub;
        bool ok = q < q1;
        if (ok && !full) {
          const int32_t pe = __ldg(perm + q);
          ok = pe >= eb && pe < ee;
        }
        any |= ok;
        x[u] = ok ? __ldg(reinterpret_cast<const uint4 *>(U + q * D) + cl) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&x[u]);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 f = __bfloat1622float2(h[i]);
          acc[2 * i] += f.x;
          acc[2 * i + 1] += f.y;
        }
      }
    }
#pragma unroll
    for (int off = LPR; off < 32; off <<= 1) {
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], off);
    }
    any = __any_sync(0xffffffffu, any);
    if (any && sub == 0) {
      float4 *o = reinterpret_cast<float4 *>(dv + j * D + cl * 8);
      float4 a0 = o[0], a1 = o[1];
      a0.x += acc[0]; a0.y += acc[1]; a0.z += acc[2]; a0.w += acc[3];
      a1.x += acc[4]; a1.y += acc[5]; a1.z += acc[6]; a1.w += acc[7];
      o[0] = a0;
      o[1] = a1;
    }
  }
}

template <int D>
static dsmpnn_status launch_edge_bwd(const dsmpnn_layer_desc &d, const Packed &pw, const __nv_bfloat16 *e,
                                     const __nv_bfloat16 *v, const int64_t *row_ptr, const int32_t *col, int64_t n_dst,
                                     int64_t rb, int64_t re, int64_t eb, int64_t ee, const float *b1, const float *b2,
                                     const BBwd &b, bool write_a1, const int32_t *upos, bool *u_sorted, int *grid_out,
                                     cudaStream_t s) {
  CUtensorMap tW2, tDS;
  DS_TRY(make_tmap_bf16(&tW2, pw.W2, KH, KH, KH, 64, KH));
  DS_TRY(make_tmap_bf16(&tDS, b.dS, D, n_dst * (int64_t)(KH + 1), D, D, KH));
  int64_t tiles = (ee - eb + 127) / 128 + 1;
  int grid = (int)std::max<int64_t>(1, std::min<int64_t>(kNumSMs, tiles));
  *grid_out = grid;
  ProbeScope probe(DSMPNN_PROBE_BF16_EDGE_BWD, s);
  // edge_bwd4 (a1 / h in TMEM, W2 resident, dz2 through the TMA engine) unless
  // A1 is wanted (the unfused backward with the edge-attribute gradient: edge_bwd2);
  // DSMPNN_EDGE_BWD=2 / 3 select the earlier designs for A/B timing
  static const int ver = getenv("DSMPNN_EDGE_BWD") ? atoi(getenv("DSMPNN_EDGE_BWD")) : 4;
  if (!write_a1 && ver == 4) {
    auto kern = edge_bwd4_kernel<D>;
    DS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, EB4<D>::SMEM));
#ifdef DSMPNN_TIMELINE
    static unsigned long long *dbg4 = nullptr;
    if (!dbg4) {
      cudaMalloc(&dbg4, 32 * 32 * 8);
      cudaMemcpyToSymbol(g_tlb4, &dbg4, sizeof(dbg4));
    }
    cudaMemsetAsync(dbg4, 0, 32 * 32 * 8, s);
#endif
    DS_CUDA(launch_pdl(kern, grid, 512, EB4<D>::SMEM, s, tW2, tDS, e, v, row_ptr, col, rb, re, eb, ee, pw, b2, b.dS, b.dZ2, b.U,
                                         upos, b.db2_part));
    *u_sorted = upos != nullptr;
#ifdef DSMPNN_TIMELINE
    dump_timeline("edge_bwd4", dbg4, 24, s);
#endif
  } else if (write_a1 || ver == 2) {
    auto kern = edge_bwd2_kernel<D>;
    DS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, EB2<D>::SMEM));
    kern<<<grid, 512, EB2<D>::SMEM, s>>>(tW2, tDS, e, v, row_ptr, col, rb, re, eb, ee, pw, b1, b2, b.dS,
                                         write_a1 ? b.A1 : nullptr, b.dZ2, b.U, b.db2_part);
  } else {
    auto kern = edge_bwd3_kernel<D>;
    DS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, EB3<D>::SMEM));
#ifdef DSMPNN_TIMELINE
    static unsigned long long *dbg = nullptr;
    if (!dbg) {
      cudaMalloc(&dbg, 32 * 32 * 8);
      cudaMemcpyToSymbol(g_tlb3, &dbg, sizeof(dbg));
    }
    cudaMemsetAsync(dbg, 0, 32 * 32 * 8, s);
#endif
    kern<<<grid, 512, EB3<D>::SMEM, s>>>(tW2, tDS, e, v, row_ptr, col, rb, re, eb, ee, pw, b2, b.dS, b.dZ2, b.U,
                                         b.db2_part);
#ifdef DSMPNN_TIMELINE
    dump_timeline("edge_bwd3", dbg, 30, s);
#endif
  }
  DS_LAUNCH_CHECK();
  return DSMPNN_OK;
}

// B5 + B6 fused (dz1w1.cuh): dW1 += dz1^T e, db1 += colsum(dz1) with
// dz1 = (dz2 W2) * [a1 > 0] kept on chip
static dsmpnn_status launch_dz1w1(const Packed &pw, const __nv_bfloat16 *dZ2, const __nv_bfloat16 *e, int64_t nE,
                                  const float *b1, float *part_w, float *part_b, int d_e, float *gW1, float *gb1,
                                  cudaStream_t s) {
  if (nE <= 0 || (!gW1 && !gb1)) return DSMPNN_OK;
  CUtensorMap tW2, tW1, tDZ, tE;
  DS_TRY(make_tmap_bf16(&tW2, pw.W2, KH, KH, KH, 64, 64));
  DS_TRY(make_tmap_bf16(&tW1, pw.W1, 16, KH, 16, 16, 128));
  DS_TRY(make_tmap_bf16(&tDZ, dZ2, KH, nE, KH, 64, 128));
  DS_TRY(make_tmap_bf16(&tE, e, 16, nE, 16, 16, 128));
  // set on every launch: the attribute belongs to the current device's context
  DS_CUDA(cudaFuncSetAttribute(dz1w1_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, DZ1C::SMEM));
  const int npairs = (int)std::max<int64_t>(1, std::min<int64_t>(kNumSMs / 2, ceil_div(nE, 128)));
  {
    ProbeScope probe(DSMPNN_PROBE_BF16_DZ1W1, s);
    DS_CUDA(launch_pdl(dz1w1_kernel, 2 * npairs, DZ1C::THREADS, DZ1C::SMEM, s, tW2, tW1, tDZ, tE, nE, b1, part_w, part_b));
    DS_LAUNCH_CHECK();
  }
  const int n = KH * (d_e + 1) * 32;
  DS_CUDA(launch_pdl(dz1w1_reduce_kernel, (n + 255) / 256, 256, 0, s, part_w, part_b, npairs, d_e, gW1, gb1));
  DS_LAUNCH_CHECK();
  return DSMPNN_OK;
}

// B4 with a1 recomputed from e (dw2.cuh): gW2 += dz2^T a1
static dsmpnn_status launch_dw2(const Packed &pw, const __nv_bfloat16 *dZ2, const __nv_bfloat16 *e, int64_t nE,
                                const float *b1, float *part, float *gW2, cudaStream_t s) {
  if (nE <= 0) return DSMPNN_OK;
  CUtensorMap tW1, tDZ, tE;
  DS_TRY(make_tmap_bf16(&tW1, pw.W1, 16, KH, 16, 16, 128));
  DS_TRY(make_tmap_bf16(&tDZ, dZ2, KH, nE, KH, 64, 128));
  DS_TRY(make_tmap_bf16(&tE, e, 16, nE, 16, 16, 128));
  // set on every launch: the attribute belongs to the current device's context
  DS_CUDA(cudaFuncSetAttribute(dw2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, DW2C::SMEM));
  const int npairs = (int)std::max<int64_t>(1, std::min<int64_t>(kNumSMs / 2, ceil_div(nE, 128)));
  {
    ProbeScope probe(DSMPNN_PROBE_BF16_DW2, s);
    DS_CUDA(launch_pdl(dw2_kernel, 2 * npairs, DW2C::THREADS, DW2C::SMEM, s, tW1, tDZ, tE, nE, b1, part));
    DS_LAUNCH_CHECK();
  }
  float4 *tmp = reinterpret_cast<float4 *>(part + (int64_t)(kNumSMs / 2) * KH * KH);
  DS_CUDA(launch_pdl(dw2_reduce1_kernel, dim3(KH * KH / 4 / 256, kDw2Groups), 256, 0, s, reinterpret_cast<const float4 *>(part),
                                                                         npairs, tmp));
  DS_LAUNCH_CHECK();
  DS_CUDA(launch_pdl(dw2_reduce2_kernel, KH * KH / 4 / 256, 256, 0, s, tmp, reinterpret_cast<float4 *>(gW2)));
  DS_LAUNCH_CHECK();
  return DSMPNN_OK;
}

dsmpnn_status bf16_bwd(const dsmpnn_layer_desc &d, const dsmpnn_weights &w, const __nv_bfloat16 *v,
                       const __nv_bfloat16 *e, const int64_t *row_ptr, const int32_t *col, const int32_t *perm,
                       const int64_t *cptr, int64_t n_dst, int64_t n_loc, int64_t E, int64_t rb, int64_t re,
                       int64_t eb, int64_t ee, const float *G, float *dv, float *de, const dsmpnn_grads &gr,
                       const void *ws, void *bws, size_t bws_bytes, cudaStream_t s) {
  Carver c(bws, bws_bytes);
  BBwd b = carve_bf16_bwd(c, d, n_dst, E);
  DS_CHECK_ARG(c.ok(), DSMPNN_ERR_CAPACITY, "layer_bwd: bwd workspace too small");
  BFwdView f = view_fwd(d, ws, n_dst);
  Packed pw = carve_packed(d, const_cast<void *>(w.packed));
  const int D = d.d_in, k = KH;  // k < KH: the padded units run too (their gradients are dropped below)
  const bool padk = d.k < KH;
  dsmpnn_grads g = gr;
  if (padk) {
    DS_CUDA(cudaMemsetAsync(b.gW1, 0, (size_t)(b.gpad_end - reinterpret_cast<char *>(b.gW1)), s));
    g.W1 = gr.W1 ? b.gW1 : nullptr;
    g.b1 = gr.b1 ? b.gb1 : nullptr;
    g.W2 = gr.W2 ? b.gW2 : nullptr;
    g.b2 = gr.b2 ? b.gb2 : nullptr;
    g.W3 = gr.W3 ? b.gW3 : nullptr;
  }
  auto unpad = [&]() -> dsmpnn_status {
    if (!padk) return DSMPNN_OK;
    const int64_t kr = d.k, DD = (int64_t)d.d_in * d.d_out;
    struct { const float *src; float *dst; int64_t ld_src, ld_dst, rows, cols; } parts[5] = {
        {b.gW1, gr.W1, d.d_e, d.d_e, kr, d.d_e}, {b.gb1, gr.b1, KH, kr, 1, kr}, {b.gW2, gr.W2, KH, kr, kr, kr},
        {b.gb2, gr.b2, KH, kr, 1, kr}, {b.gW3, gr.W3, KH, kr, DD, kr}};
    for (auto &q : parts) {
      if (!q.dst) continue;
      add_block_kernel<<<grid_of(q.rows * q.cols), 256, 0, s>>>(q.src, q.ld_src, q.dst, q.ld_dst, q.rows, q.cols);
      DS_LAUNCH_CHECK();
    }
    return DSMPNN_OK;
  };
  const int64_t kp = kpad_of(d);
  const int64_t nR = re - rb, nE = ee - eb;
  if (nR <= 0) return unpad();

  // B0
  {
    const int nblk = (int)ceil_div(nR, 32);
    if (D == 64)
      DS_CUDA(launch_pdl(b0_bf16_kernel<64>, nblk, 256, 0, s, G, f.pre, row_ptr, rb, re, d.act, d.root, w.W_root, b.gh, b.gh16,
                                              b.inv_deg, b.b0_part, dv));
    else
      DS_CUDA(launch_pdl(b0_bf16_kernel<32>, nblk, 256, 0, s, G, f.pre, row_ptr, rb, re, d.act, d.root, w.W_root, b.gh, b.gh16,
                                              b.inv_deg, b.b0_part, dv));
    DS_LAUNCH_CHECK();
    if (g.b) DS_TRY(colsum(b.b0_part, nblk, D, D, g.b, 1, s));
  }
  // B1: dTheta~_aug [kp x D] = S~_aug^T ghat  (K = rows)
  if (g.W3 || g.b3 || g.W_root) {
    TgemmArgs a{kp, D, nR, f.S + rb * kp, kp, true, b.gh16 + rb * D, D, true, b.dT, D, 1, 0, 0};
    DS_TRY(tgemm(a, s));
    if (g.W3) {
      DS_CUDA(launch_pdl(unpack_dw3_kernel, dim3(k / 32, D / 32, D), 256, 0, s, b.dT, k, D, g.W3));
      DS_LAUNCH_CHECK();
    }
    DS_CUDA(launch_pdl(unpack_bias_root_kernel, grid_of((int64_t)D * D), 256, 0, s, 
        b.dT, k, D, g.b3, d.root == DSMPNN_ROOT_DENSE ? g.W_root : nullptr));
    DS_LAUNCH_CHECK();
  }
  if (nE <= 0) return unpad();
  // B2: dS_i = (ghat_i Theta~^T) / deg_i   -> bf16 [n_dst x (k+1)*D]
  {
    TgemmArgs a{nR, (int64_t)(k + 1) * D, D, b.gh16 + rb * D, D, false, pw.Th, D, false, nullptr, 0, 1, 0, 0};
    a.out16 = b.dS + rb * (int64_t)(k + 1) * D;
    a.ld16 = (int64_t)(k + 1) * D;
    a.row_scale = b.inv_deg + rb;
    DS_TRY(tgemm(a, s));
  }
  // Without the edge-attribute gradient (which needs dz1 in HBM) the
  // kappa_phi weight gradients recompute a1 from e instead of reading A1:
  // B4 -> dw2.cuh, B5 + B6 -> dz1w1.cuh (dz1 stays on chip)
  const bool fused = !de && k == KH && d.d_e <= 16;
  // B3: edge kernel
  int grid = 1;
  // U rows in CSC order (edge_bwd4 only) so that B7 streams them
  const int32_t *upos = nullptr;
  if (dv && fused && E > 0) {
    DS_CUDA(launch_pdl(csc_inverse_kernel, grid_of(E), 256, 0, s, perm, E, b.upos));
    DS_LAUNCH_CHECK();
    upos = b.upos;
  }
  bool u_sorted = false;
  if (D == 64)
    DS_TRY(launch_edge_bwd<64>(d, pw, e, v, row_ptr, col, n_dst, rb, re, eb, ee, pw.b1, pw.b2, b, !fused, upos,
                               &u_sorted, &grid, s));
  else
    DS_TRY(launch_edge_bwd<32>(d, pw, e, v, row_ptr, col, n_dst, rb, re, eb, ee, pw.b1, pw.b2, b, !fused, upos,
                               &u_sorted, &grid, s));
  DS_TRY(colsum(b.db2_part, grid, k, k, g.b2, 1, s));
  // B4: dW2 += dz2^T a1   (M = k, N = k, K = edges)
  if (g.W2 && fused) {
    DS_TRY(launch_dw2(pw, b.dZ2 + eb * k, e + eb * 16, nE, pw.b1, b.w2_part, g.W2, s));
  } else if (g.W2) {
    int splits = (int)std::max<int64_t>(1, std::min<int64_t>(kSplitsW, nE / 512));
    TgemmArgs a{k, k, nE, b.dZ2 + eb * k, k, true, b.A1 + eb * k, k, true, b.part, k, splits, (int64_t)k * k, 0};
    DS_TRY(tgemm(a, s));
    int64_t nkb = (nE + 63) / 64;
    int kbps = (int)std::max<int64_t>(1, ceil_div(nkb, splits));
    int real = (int)std::max<int64_t>(1, ceil_div(nkb, kbps));
    DS_TRY(splitk_sum(b.part, real, (int64_t)k * k, k, k, k, g.W2, k, 1, s));
  }
  if (fused) {
    DS_TRY(launch_dz1w1(pw, b.dZ2 + eb * k, e + eb * 16, nE, pw.b1, b.w1_part, b.b1_part, d.d_e, g.W1, g.b1, s));
  } else {
    // B5: dz1 = (dz2 W2) * [a1 > 0]  (bf16), column sums -> db1
    {
      TgemmArgs a{nE, k, k, b.dZ2 + eb * k, k, false, pw.W2, k, true, nullptr, 0, 1, 0, 0};
      a.out16 = b.dZ1 + eb * k;
      a.ld16 = k;
      a.mask16 = b.A1 + eb * k;
      a.ldmask = k;
      a.colsum_part = b.db1_part;
      a.b_resident = true;
      DS_CUDA(cudaMemsetAsync(b.db1_part, 0, (size_t)kColsumRows * k * sizeof(float), s));
      DS_TRY(tgemm(a, s));
      DS_TRY(colsum_ws(b.db1_part, kColsumRows, k, k, g.b1, 1, b.cs_ws, s));
    }
    // B6: dW1 += dz1^T e ;  de = dz1 W1
    if (g.W1) {
      int splits = (int)std::max<int64_t>(1, std::min<int64_t>(kSplitsW, nE / 512));
      TgemmArgs a{k, 16, nE, b.dZ1 + eb * k, k, true, e + eb * 16, 16, true, b.part, 16, splits, (int64_t)k * 16, 0};
      DS_TRY(tgemm(a, s));
      int64_t nkb = (nE + 63) / 64;
      int kbps = (int)std::max<int64_t>(1, ceil_div(nkb, splits));
      int real = (int)std::max<int64_t>(1, ceil_div(nkb, kbps));
      DS_TRY(splitk_sum(b.part, real, (int64_t)k * 16, k, 16, 16, b.dW1f, 16, 0, s));
      add_cols_kernel<<<grid_of((int64_t)k * d.d_e), 256, 0, s>>>(b.dW1f, k, 16, d.d_e, g.W1, 1);
      DS_LAUNCH_CHECK();
    }
    if (de) {
      TgemmArgs a{nE, 16, k, b.dZ1 + eb * k, k, false, pw.W1, 16, true, b.de16, 16, 1, 0, 0};
      DS_TRY(tgemm(a, s));
      add_cols_kernel<<<grid_of(nE * d.d_e), 256, 0, s>>>(b.de16, nE, 16, d.d_e, de + eb * d.d_e, 0);
      DS_LAUNCH_CHECK();
    }
  }
  // B7: dv[j] += sum of u_p over edges with source j (CSC order)
  if (dv) {
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n_loc, 8), 148 * 16));
    const int full = eb == 0 && ee == E;
    if (u_sorted) {
      if (D == 64) DS_CUDA(launch_pdl(scatter_sorted_bf16_kernel<64>, blocks, 256, 0, s, b.U, perm, cptr, n_loc, eb, ee, full, dv));
      else DS_CUDA(launch_pdl(scatter_sorted_bf16_kernel<32>, blocks, 256, 0, s, b.U, perm, cptr, n_loc, eb, ee, full, dv));
    } else if (D == 64) {
      scatter_csc_bf16_kernel<64><<<blocks, 256, 0, s>>>(b.U, perm, cptr, n_loc, eb, ee, dv);
    } else {
      scatter_csc_bf16_kernel<32><<<blocks, 256, 0, s>>>(b.U, perm, cptr, n_loc, eb, ee, dv);
    }
    DS_LAUNCH_CHECK();
  }
  return unpad();
}

}  // namespace dsmpnn

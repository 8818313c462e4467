// layer_bf16.cu - BF16 mode of the edge-conditioned convolution on the
// tcgen05 tensor cores (sm_100a).  Formulation: DESIGN.md §6 ("aggregate
// first", see layer.cu).  Widths supported: k <= 256 (k < 256 zero-padded
// to 256: same results, the k = 256 cost), d_in = d_out = D in {32, 64},
// d_e <= 13 (zero-padded to 16; columns 13..15 carry the bias b1).
//
// Forward of rows [rb, re):
//   1. fill kernel   : S~_aug[i][k*D + c] = mean_p v_j[c]  (the h~ = 1 row),
//                      S~_aug[i][(k+1)*D + c] = v_i[c]      (root operand),
//                      zero S~ rows of isolated nodes.
//   2. edge kernel   : edge_fwd2.cuh, per 128-slot tile (each row padded to a
//                      multiple of 16 slots): a1 = relu(E W1^T + b1),
//                      h = relu(a1 W2^T + b2) as two tcgen05 GEMMs (W1, W2
//                      resident in SMEM, D in TMEM), then S_i = H_i^T V_i per
//                      row (A = H^T read MN-major from the same SMEM tile,
//                      B = gathered v rows), scaled by 1/deg_i ->
//                      S~_aug[i][c*k + kap] (bf16).  K_p is never formed.
//   3. node GEMM     : [S~_aug] . [Theta~ ; W_root^T] on tcgen05 (split-K),
//   4. node epilogue : + b (+ v_i), sigma, out (fp32), out_lowp (bf16), pre.
#include <cuda.h>
#include <cstdlib>

#include "layer_bf16.cuh"
#include "layer_bf16_common.cuh"
#include "edge_fwd2.cuh"
#include "edge_fwd3.cuh"
#include "simt.cuh"
#include "tc.cuh"
#include "tgemm.cuh"

namespace dsmpnn {

// W1 packed [KH x 16]: columns 0..d_e-1 the weights, columns 13, 14, 15 the
// bias b1 split into three bf16 terms (their fp32 sum is b1 to ~2^-24
// relative: the MMA's fp32 accumulation adds it like an fp32 bias add), the
// rest zero.  The fused edge kernels set e columns 13..15 to 1 in their SMEM
// copy of the edge tile, so z1 = E W1^T already holds + b1 (edge_fwd3.cuh,
// edge_bwd3.cuh); every other reader of W1 sees zeros there and adds b1 itself.
// k < KH: units k..KH-1 get zero weights and biases (W1 rows, W2 rows and
// columns, Theta~ rows), so their a1 and h are exactly 0 and they add exact
// zeros to every product: the results are those of the width-k MLP.
__global__ void pack_bf16_kernel(const float *__restrict__ W1, const float *__restrict__ b1,
                                 const float *__restrict__ W2, const float *__restrict__ b2,
                                 const float *__restrict__ W3, const float *__restrict__ b3,
                                 const float *__restrict__ Wr, int root_dense, int k, int de, int di, int dout,
                                 int64_t kp, Packed p) {
  int64_t n1 = (int64_t)KH * 16, n2 = (int64_t)KH * KH, n3 = kp * dout;
  int64_t total = n1 + n2 + n3 + 2 * KH;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    if (t < n1) {
      int r = (int)(t / 16), c = (int)(t % 16);
      float w = (r < k && c < de) ? W1[(int64_t)r * de + c] : 0.f;
      if (c >= kBiasCol0) {  // b1 = t0 + t1 + t2, each a bf16 value (t2 absorbs the rest to ~2^-24 |b1|)
        const float bb = r < k ? b1[r] : 0.f;
        const float t0 = __bfloat162float(__float2bfloat16_rn(bb));
        const float t1 = __bfloat162float(__float2bfloat16_rn(bb - t0));
        w = c == kBiasCol0 ? t0 : c == kBiasCol0 + 1 ? t1 : bb - t0 - t1;
      }
      p.W1[t] = __float2bfloat16_rn(w);
    } else if (t < n1 + n2) {
      const int64_t u = t - n1;
      const int r = (int)(u / KH), c = (int)(u % KH);
      p.W2[u] = __float2bfloat16_rn((r < k && c < k) ? W2[(int64_t)r * k + c] : 0.f);
    } else if (t < n1 + n2 + n3) {
      int64_t u = t - n1 - n2;
      int64_t row = u / dout;  // Theta~_aug row
      int o = (int)(u - row * dout);
      int kap = (int)(row / di), c = (int)(row - (int64_t)kap * di);
      float val = 0.f;
      if (kap < k) val = W3[((int64_t)c * dout + o) * k + kap];
      else if (kap == KH) val = b3[(int64_t)c * dout + o];
      else if (kap == KH + 1 && root_dense) val = Wr[(int64_t)o * di + c];
      __nv_bfloat16 bv = __float2bfloat16_rn(val);
      p.Th[row * dout + o] = bv;
      // the forward S~ rows store the kappa < KH block as [c][kappa]: K index
      // c*KH + kappa (edge kernel EPI_B); the bias and root blocks keep KH*d_in + c
      const int64_t kk = kap < KH ? (int64_t)c * KH + kap : row;
      p.ThT[(int64_t)o * kp + kk] = bv;
    } else {
      const int u = (int)(t - n1 - n2 - n3);
      if (u < KH) p.b1[u] = u < k ? b1[u] : 0.f;
      else p.b2[u - KH] = u - KH < k ? b2[u - KH] : 0.f;
    }
  }
}

dsmpnn_status bf16_check_desc(const dsmpnn_layer_desc &d) {
  DS_CHECK_ARG(d.k >= 1 && d.k <= KH, DSMPNN_ERR_UNSUPPORTED, "layer BF16: 1 <= k <= %d (got %d)", KH, d.k);
  DS_CHECK_ARG(d.d_in == d.d_out && (d.d_in == 32 || d.d_in == 64), DSMPNN_ERR_UNSUPPORTED,
               "layer BF16: d_in = d_out in {32, 64} (got %d, %d)", d.d_in, d.d_out);
  DS_CHECK_ARG(d.d_e <= kBiasCol0, DSMPNN_ERR_SHAPE,
               "layer BF16: d_e <= %d (got %d; columns 13..15 of the padded edge tile carry the kappa bias)",
               kBiasCol0, d.d_e);
  return DSMPNN_OK;
}

size_t bf16_packed_bytes(const dsmpnn_layer_desc &d) {
  Carver c(nullptr, 0);
  int64_t kp = kpad_of(d);
  c.take<__nv_bfloat16>((int64_t)KH * 16);
  c.take<__nv_bfloat16>((int64_t)KH * KH);
  c.take<__nv_bfloat16>((int64_t)d.d_out * kp);
  c.take<__nv_bfloat16>(kp * d.d_out);
  c.take<float>(KH);
  c.take<float>(KH);
  return c.used();
}

dsmpnn_status bf16_pack(const dsmpnn_layer_desc &d, const dsmpnn_weights &w, void *packed, cudaStream_t s) {
  DS_CHECK_ARG(d.root != DSMPNN_ROOT_DENSE || w.W_root, DSMPNN_ERR_INVALID_ARG, "pack: W_root is NULL");
  Packed p = carve_packed(d, packed);
  int64_t kp = kpad_of(d);
  DS_CUDA(cudaMemsetAsync(p.ThT, 0, (size_t)d.d_out * kp * 2, s));
  DS_CHECK_ARG(w.W1 && w.b1 && w.W2 && w.b2 && w.W3 && w.b3, DSMPNN_ERR_INVALID_ARG, "pack: a kappa weight is NULL");
  int64_t total = (int64_t)KH * 16 + (int64_t)KH * KH + kp * d.d_out + 2 * KH;
  pack_bf16_kernel<<<(int)std::min<int64_t>(ceil_div(total, 256), 148 * 8), 256, 0, s>>>(
      w.W1, w.b1, w.W2, w.b2, w.W3, w.b3, w.W_root, d.root == DSMPNN_ROOT_DENSE, d.k, d.d_e, d.d_in, d.d_out, kp,
      p);
  DS_LAUNCH_CHECK();
  return DSMPNN_OK;
}

// ------------------------------------------------------------- fill kernel
// one warp per row: bias row (mean of v_j), root operand copy, zero rows w/o edges
template <int D>
__global__ void s_fill_kernel(const __nv_bfloat16 *__restrict__ v, const int64_t *__restrict__ row_ptr,
                              const int32_t *__restrict__ col, int64_t rb, int64_t re, int64_t kp,
                              __nv_bfloat16 *__restrict__ S) {
  pdl_wait();
  pdl_trigger();
  // warp per row; lane = (edge sub-slot, 16-byte column chunk): D / 8 lanes
  // cover one v row, so a warp instruction gathers 32 / (D / 8) rows and
  // UNR instructions are in flight; sub-slot sums combine by a butterfly
  // (fixed order)
  constexpr int LPR = D / 8, EPI = 32 / LPR, UNR = 32 / EPI;  // one batch of 32 edges in flight
  const int lane = threadIdx.x & 31, cl = lane % LPR, sub = lane / LPR;
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = rb + warp; i < re; i += nw) {
    const int64_t p0 = row_ptr[i], p1 = row_ptr[i + 1];
    const int deg = (int)(p1 - p0);
    __nv_bfloat16 *Si = S + i * kp;
    float acc[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = 0.f;
    for (int64_t pb = p0; pb < p1; pb += 32) {
      // 32 column indices per coalesced load, handed out by shuffles, so the
      // row gathers of a batch are independent of each other
      const int32_t jl = pb + lane < p1 ? __ldg(col + pb + lane) : 0;
      const int nb = (int)(p1 - pb < 32 ? p1 - pb : 32);
#pragma unroll
      for (int q0 = 0; q0 < 32; q0 += EPI * UNR) {
        uint4 x[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          const int q = q0 + u * EPI + sub;
          const int32_t j = __shfl_sync(0xffffffffu, jl, q & 31);
          x[u] = q < nb ? __ldg(reinterpret_cast<const uint4 *>(v + (int64_t)j * D) + cl) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&x[u]);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float2 f = __bfloat1622float2(h[q]);
            acc[2 * q] += f.x;
            acc[2 * q + 1] += f.y;
          }
        }
      }
    }
#pragma unroll
    for (int off = LPR; off < 32; off <<= 1)
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], off);
    const float inv = deg > 0 ? 1.0f / (float)deg : 0.f;
    if (sub == 0) {
      reinterpret_cast<uint4 *>(Si + (int64_t)KH * D)[cl] =
          make_uint4(tc::pack_bf16(acc[0] * inv, acc[1] * inv), tc::pack_bf16(acc[2] * inv, acc[3] * inv),
                     tc::pack_bf16(acc[4] * inv, acc[5] * inv), tc::pack_bf16(acc[6] * inv, acc[7] * inv));
    } else if (sub == 1) {
      reinterpret_cast<uint4 *>(Si + (int64_t)(KH + 1) * D)[cl] = reinterpret_cast<const uint4 *>(v + i * D)[cl];
    }
    for (int64_t t = (int64_t)(KH + 2) * D + lane; t < kp; t += 32) Si[t] = __float2bfloat16_rn(0.f);
    if (deg == 0)
      for (int64_t t = lane; t < (int64_t)KH * D; t += 32) Si[t] = __float2bfloat16_rn(0.f);
  }
}


// ------------------------------------------------------- node epilogue
// pre = sum_z partial[z] + b (+ v_i for IDENTITY); out = sigma(pre)
__global__ void node_epi_bf16_kernel(const float *__restrict__ part, int splits, int64_t split_stride, int64_t rb,
                                     int64_t re, int D, const float *__restrict__ b,
                                     const __nv_bfloat16 *__restrict__ v, int root, int act, float *__restrict__ pre,
                                     float *__restrict__ out, __nv_bfloat16 *__restrict__ out_lowp) {
  pdl_wait();
  pdl_trigger();
  int64_t total = (re - rb) * D;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    float x = 0.f;
    for (int z = 0; z < splits; ++z) x += part[z * split_stride + t];
    int64_t idx = rb * D + t;
    int o = (int)(t % D);
    x += b[o];
    if (root == DSMPNN_ROOT_IDENTITY) x += __bfloat162float(v[idx]);
    pre[idx] = x;
    float y = act == DSMPNN_ACT_RELU ? fmaxf(x, 0.f) : x;
    out[idx] = y;
    if (out_lowp) out_lowp[idx] = __float2bfloat16_rn(y);
  }
}

// ------------------------------------------------------------ workspace
struct BFwd {
  __nv_bfloat16 *S;  // [n_dst x kp]
  float *pre;        // [n_dst x D]
  float *part;       // [kMaxSplitsFwd x n_dst x D]
};
constexpr int kMaxSplitsFwd = 16;
// split-K count of the node GEMM: the persistent tgemm runs ceil(T / 148)
// rounds of T = m-tiles x splits tiles, so pick the split count in [4, 16]
// whose last round is fullest (fewest idle SMs), ties to fewer splits
static int node_gemm_splits(int64_t nR, int64_t kp, int *real_out) {
  const int64_t mt = ceil_div(nR, 128), nkb = ceil_div(kp, 64);
  // enough row tiles to occupy most SMs: one CTA streams a tile's whole K
  // (no partial sums to write and re-read; the S~ stream runs at the rate of
  // the B1 GEMM, which has the same shape transposed)
  static const int64_t min_tiles = [] {
    const char *e = getenv("DSMPNN_NODE_GEMM_NOSPLIT_TILES");
    return e ? atoll(e) : (int64_t)(kNumSMs * 3 / 4);
  }();
  if (mt >= min_tiles) {
    *real_out = 1;
    return 1;
  }
  int best = 4, best_real = 4;
  double best_eff = -1.0;
  for (int sp = 4; sp <= kMaxSplitsFwd; ++sp) {
    const int64_t kbps = ceil_div(nkb, sp), real = ceil_div(nkb, kbps), T = mt * real;
    const double eff = (double)T / (double)(kNumSMs * ceil_div(T, kNumSMs));
    if (eff > best_eff + 1e-9) {
      best_eff = eff;
      best = sp;
      best_real = (int)real;
    }
  }
  *real_out = best_real;
  return best;
}
static BFwd carve_bf16_fwd(Carver &c, const dsmpnn_layer_desc &d, int64_t n_dst) {
  BFwd f;
  f.S = c.take<__nv_bfloat16>(n_dst * kpad_of(d));
  f.pre = c.take<float>(n_dst * d.d_out);
  f.part = c.take<float>((int64_t)kMaxSplitsFwd * n_dst * d.d_out);
  return f;
}

size_t bf16_fwd_ws_bytes(const dsmpnn_layer_desc &d, int64_t n_dst, int64_t E) {
  Carver c(nullptr, 0);
  carve_bf16_fwd(c, d, n_dst);
  return c.used();
}

template <int D>
static dsmpnn_status launch_edge_fwd(const __nv_bfloat16 *e, const __nv_bfloat16 *v, const int64_t *row_ptr,
                                     const int32_t *col, int64_t rb, int64_t re, int64_t eb, int64_t ee,
                                     const Packed &pw, const float *b1, const float *b2, __nv_bfloat16 *S,
                                     int64_t kp, cudaStream_t s) {
  CUtensorMap tW2;
  DS_TRY(make_tmap_bf16(&tW2, pw.W2, KH, KH, KH, 64, KH));
  int64_t tiles = (ee - eb + 127) / 128 + 1;
  int grid = (int)std::max<int64_t>(1, std::min<int64_t>(kNumSMs, tiles));
  ProbeScope probe(DSMPNN_PROBE_BF16_EDGE_FWD, s);
  // DSMPNN_EDGE_FWD=2 selects the previous design (h through SMEM) for A/B timing
  static const bool v2 = getenv("DSMPNN_EDGE_FWD") && atoi(getenv("DSMPNN_EDGE_FWD")) == 2;
  if (v2) {
    auto kern = edge_fwd2_kernel<D>;
    DS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, EF2<D>::SMEM));
    kern<<<grid, 512, EF2<D>::SMEM, s>>>(tW2, e, v, row_ptr, rb, re, eb, ee, pw, b1, b2, S, kp, col);
  } else {
    auto kern = edge_fwd3_kernel<D>;
    DS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, EF3<D>::SMEM));
#ifdef DSMPNN_TIMELINE
    static unsigned long long *dbg = nullptr;
    if (!dbg) {
      cudaMalloc(&dbg, 32 * 32 * 8);
      cudaMemcpyToSymbol(g_tl3, &dbg, sizeof(dbg));
    }
    cudaMemsetAsync(dbg, 0, 32 * 32 * 8, s);
#endif
    DS_CUDA(launch_pdl(kern, grid, 512, EF3<D>::SMEM, s, tW2, e, v, row_ptr, rb, re, eb, ee, pw, b1, b2, S, kp, col));
#ifdef DSMPNN_TIMELINE
    dump_timeline("edge_fwd3", dbg, 29, s);
#endif
  }
  DS_LAUNCH_CHECK();
  return DSMPNN_OK;
}

dsmpnn_status bf16_fwd(const dsmpnn_layer_desc &d, const dsmpnn_weights &w, const __nv_bfloat16 *v,
                       const __nv_bfloat16 *e, const int64_t *row_ptr, const int32_t *col, int64_t n_dst, int64_t E,
                       int64_t rb, int64_t re, int64_t eb, int64_t ee, float *out, __nv_bfloat16 *out_lowp, void *ws,
                       size_t ws_bytes, cudaStream_t s) {
  Carver c(ws, ws_bytes);
  BFwd f = carve_bf16_fwd(c, d, n_dst);
  DS_CHECK_ARG(c.ok(), DSMPNN_ERR_CAPACITY, "layer_fwd: workspace too small");
  Packed pw = carve_packed(d, const_cast<void *>(w.packed));
  const int D = d.d_in;
  const int64_t kp = kpad_of(d);
  const int64_t nR = re - rb;
  // 1. bias row, root operand, isolated rows
  {
    int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(nR * 32, 256), 148 * 8));
    if (D == 64) DS_CUDA(launch_pdl(s_fill_kernel<64>, blocks, 256, 0, s, v, row_ptr, col, rb, re, kp, f.S));
    else DS_CUDA(launch_pdl(s_fill_kernel<32>, blocks, 256, 0, s, v, row_ptr, col, rb, re, kp, f.S));
    DS_LAUNCH_CHECK();
  }
  // 2. fused kappa MLP + S formation
  if (ee > eb) {
    if (D == 64) DS_TRY(launch_edge_fwd<64>(e, v, row_ptr, col, rb, re, eb, ee, pw, pw.b1, pw.b2, f.S, kp, s));
    else DS_TRY(launch_edge_fwd<32>(e, v, row_ptr, col, rb, re, eb, ee, pw, pw.b1, pw.b2, f.S, kp, s));
  }
  // 3. node GEMM [S~_aug] . [Theta~_aug]  (split-K partials)
  int real = 1;
  const int splits = node_gemm_splits(nR, kp, &real);
  {
    ProbeScope probe(DSMPNN_PROBE_BF16_NODE_GEMM, s);
    TgemmArgs a{nR, D, kp, f.S + rb * kp, kp, false, pw.ThT, kp, false, f.part, D, splits, nR * D, 0};
    DS_TRY(tgemm(a, s));
  }
  DS_CUDA(launch_pdl(node_epi_bf16_kernel, (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(nR * D, 256), 148 * 8)), 256, 0, s, 
      f.part, real, nR * D, rb, re, D, w.b, v, d.root, d.act, f.pre, out, out_lowp));
  DS_LAUNCH_CHECK();
  return DSMPNN_OK;
}

}  // namespace dsmpnn

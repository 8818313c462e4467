// layer.cu - a4/a5/a7: the edge-conditioned convolution, Eq. (1)
// (eq. (ii) :40; Alg. 1 :407-409 residual; readings R1-R5, R18).
//
// Formulation ("aggregate first"): with h~_p = [h_p; 1] and the
// packed last kappa layer Theta~[kap*d_in + c, o] = W3[c*d_out + o, kap]
// (Theta~[k*d_in + c, o] = b3[c*d_out + o]),
//     mean_p K_p^T v_j = vec(S_i) . Theta~,   S_i = (1/deg_i) sum_p h~_p (x) v_j
// so K_p (d_in x d_out per edge) is never formed and the large contraction
// runs once per destination row instead of once per edge.
//
// This file holds the API entry points, the fp32 (F32 mode) kernels and the
// shared node-level epilogues.  The bf16 tcgen05 kernels live in
// layer_bf16.cu.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "layer_bf16.cuh"
#include "simt.cuh"

namespace dsmpnn {

// ------------------------------------------------------------- packing ----
// Theta~ fp32 [(k+1)*d_in x d_out]
__global__ void pack_theta_f32_kernel(const float *__restrict__ W3, const float *__restrict__ b3, int k, int di,
                                      int dout, float *__restrict__ T) {
  int64_t total = (int64_t)(k + 1) * di * dout;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t row = t / dout;
    int o = (int)(t - row * dout);
    int kap = (int)(row / di), c = (int)(row - (int64_t)kap * di);
    T[t] = kap < k ? W3[((int64_t)c * dout + o) * k + kap] : b3[(int64_t)c * dout + o];
  }
}

// dW3[c*d_out+o, kap] += dT[kap*d_in + c, o];  db3[c*d_out+o] += dT[k*d_in + c, o]
__global__ void unpack_dtheta_kernel(const float *__restrict__ dT, int k, int di, int dout, float *__restrict__ dW3,
                                     float *__restrict__ db3) {
  int64_t total = (int64_t)(k + 1) * di * dout;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t row = t / dout;
    int o = (int)(t - row * dout);
    int kap = (int)(row / di), c = (int)(row - (int64_t)kap * di);
    if (kap < k) { if (dW3) dW3[((int64_t)c * dout + o) * k + kap] += dT[t]; }
    else if (db3) db3[(int64_t)c * dout + o] += dT[t];
  }
}

// ------------------------------------------------------- F32 node kernels --
// S~_i[kap*d_in + c] = (1/deg_i) sum_p h~_p[kap] v_j[c]   (rows [rb, re));
// edges are staged 128 at a time, partial sums kept in the output row.
constexpr int kEdgeChunk = 128;
__global__ void s_form_f32_kernel(const float *__restrict__ H, const float *__restrict__ v,
                                  const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col, int64_t rb,
                                  int k, int di, float *__restrict__ S) {
  extern __shared__ float sv[];  // [kEdgeChunk x di]
  int64_t i = rb + blockIdx.x;
  int64_t p0 = row_ptr[i], p1 = row_ptr[i + 1];
  int deg = (int)(p1 - p0);
  int64_t Kt = (int64_t)(k + 1) * di;
  float *Si = S + i * Kt;
  for (int64_t t = threadIdx.x; t < Kt; t += blockDim.x) Si[t] = 0.f;
  if (deg == 0) return;
  for (int q0 = 0; q0 < deg; q0 += kEdgeChunk) {
    int nq = min(kEdgeChunk, deg - q0);
    __syncthreads();
    for (int t = threadIdx.x; t < nq * di; t += blockDim.x) {
      int q = t / di, c = t - q * di;
      sv[t] = v[(int64_t)col[p0 + q0 + q] * di + c];
    }
    __syncthreads();
    for (int64_t t = threadIdx.x; t < Kt; t += blockDim.x) {
      int kap = (int)(t / di), c = (int)(t - (int64_t)kap * di);
      float s = Si[t];
      if (kap < k) {
        for (int q = 0; q < nq; ++q) s = fmaf(H[(p0 + q0 + q) * k + kap], sv[q * di + c], s);
      } else {
        for (int q = 0; q < nq; ++q) s += sv[q * di + c];
      }
      Si[t] = s;
    }
  }
  float inv = 1.0f / (float)deg;
  for (int64_t t = threadIdx.x; t < Kt; t += blockDim.x) Si[t] *= inv;
}

// node epilogue (a5): pre = agg (+ v_i if IDENTITY) + b; out = sigma(pre)
__global__ void node_epilogue_kernel(float *__restrict__ pre, const float *__restrict__ v_f32,
                                     const __nv_bfloat16 *__restrict__ v_bf16, const float *__restrict__ b,
                                     int64_t rb, int64_t re, int dout, int root, int act, float *__restrict__ out,
                                     __nv_bfloat16 *__restrict__ out_lowp) {
  int64_t total = (re - rb) * dout;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = rb + t / dout;
    int o = (int)(t % dout);
    int64_t idx = i * dout + o;
    float x = pre[idx];
    if (root == DSMPNN_ROOT_IDENTITY) x += v_f32 ? v_f32[idx] : __bfloat162float(v_bf16[idx]);
    x += b[o];
    pre[idx] = x;
    float y = (act == DSMPNN_ACT_RELU) ? fmaxf(x, 0.f) : x;
    out[idx] = y;
    if (out_lowp) out_lowp[idx] = __float2bfloat16_rn(y);
  }
}

// ghat = G * sigma'(pre) (ReLU'(0) = 0)
__global__ void ghat_kernel(const float *__restrict__ G, const float *__restrict__ pre, int64_t rb, int64_t re,
                            int dout, int act, float *__restrict__ gh) {
  int64_t total = (re - rb) * dout;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t idx = rb * dout + t;
    float g = G[idx];
    gh[idx] = (act == DSMPNN_ACT_RELU) ? (pre[idx] > 0.f ? g : 0.f) : g;
  }
}

__global__ void add_rows_kernel(const float *__restrict__ src, int64_t rb, int64_t re, int w, float *__restrict__ dst) {
  int64_t total = (re - rb) * w;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x)
    dst[rb * w + t] += src[rb * w + t];
}

// per edge of row i: dh_p[kap] = (1/deg) sum_c dS_i[kap,c] v_j[c]  -> dz2 = dh*[h>0]
//                    u_p[c]    = (1/deg) sum_{kap<=k} h~_p[kap] dS_i[kap,c]
__global__ void edge_bwd_f32_kernel(const float *__restrict__ dS, const float *__restrict__ H,
                                    const float *__restrict__ v, const int64_t *__restrict__ row_ptr,
                                    const int32_t *__restrict__ col, int64_t rb, int k, int di,
                                    float *__restrict__ dZ2, float *__restrict__ U) {
  extern __shared__ float sm[];
  int64_t i = rb + blockIdx.x;
  int64_t p0 = row_ptr[i], p1 = row_ptr[i + 1];
  int deg = (int)(p1 - p0);
  if (deg == 0) return;
  int64_t Kt = (int64_t)(k + 1) * di;
  float *sdS = sm;             // [Kt]
  float *sv = sm + Kt;         // [kEdgeChunk x di]
  float inv = 1.0f / (float)deg;
  for (int64_t t = threadIdx.x; t < Kt; t += blockDim.x) sdS[t] = dS[i * Kt + t] * inv;
  for (int q0 = 0; q0 < deg; q0 += kEdgeChunk) {
    int nq = min(kEdgeChunk, deg - q0);
    __syncthreads();
    for (int t = threadIdx.x; t < nq * di; t += blockDim.x) {
      int q = t / di, c = t - q * di;
      sv[t] = v[(int64_t)col[p0 + q0 + q] * di + c];
    }
    __syncthreads();
    for (int t = threadIdx.x; t < nq * k; t += blockDim.x) {
      int q = t / k, kap = t - q * k;
      float s = 0.f;
      for (int c = 0; c < di; ++c) s = fmaf(sdS[kap * di + c], sv[q * di + c], s);
      int64_t p = p0 + q0 + q;
      float h = H[p * k + kap];
      dZ2[p * k + kap] = h > 0.f ? s : 0.f;
    }
    for (int t = threadIdx.x; t < nq * di; t += blockDim.x) {
      int q = t / di, c = t - q * di;
      int64_t p = p0 + q0 + q;
      const float *hq = H + p * k;
      float s = 0.f;
      for (int kap = 0; kap < k; ++kap) s = fmaf(hq[kap], sdS[kap * di + c], s);
      s += sdS[(int64_t)k * di + c];
      U[p * di + c] = s;
    }
  }
}

__global__ void relu_mask_kernel(float *__restrict__ d, const float *__restrict__ a, int64_t n) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    if (!(a[t] > 0.f)) d[t] = 0.f;
}

// dv[j] += sum over edges p in csc(j) with eb <= p < ee of U[p]  (csc order: ascending edge id)
__global__ void scatter_csc_kernel(const float *__restrict__ U, const int32_t *__restrict__ perm,
                                   const int64_t *__restrict__ cptr, int64_t n_loc, int di, int64_t eb, int64_t ee,
                                   float *__restrict__ dv) {
  int64_t total = n_loc * di;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t j = t / di;
    int c = (int)(t - j * di);
    float s = 0.f;
    bool any = false;
    for (int64_t q = cptr[j]; q < cptr[j + 1]; ++q) {
      int64_t p = perm[q];
      if (p >= eb && p < ee) { s += U[p * di + c]; any = true; }
    }
    if (any) dv[t] += s;
  }
}

static int grid_of(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), 148 * 8)); }

static int splits_for(int64_t K) {
  int64_t s = K / 4096;
  return (int)std::max<int64_t>(1, std::min<int64_t>(s, 32));
}

// ---------------------------------------------------------- ws layouts ----
struct F32Fwd {
  float *A1, *H, *S, *pre;
};
static F32Fwd carve_f32_fwd(Carver &c, const dsmpnn_layer_desc &d, int64_t n_dst, int64_t E) {
  F32Fwd f;
  int64_t Kt = (int64_t)(d.k + 1) * d.d_in;
  f.A1 = c.take<float>(E * d.k);
  f.H = c.take<float>(E * d.k);
  f.S = c.take<float>(n_dst * Kt);
  f.pre = c.take<float>(n_dst * d.d_out);
  return f;
}

struct F32Bwd {
  float *gh, *dS, *dZ2, *dA1, *U, *dT, *partial;
};
static int64_t f32_partial_elems(const dsmpnn_layer_desc &d, int64_t n_dst, int64_t E) {
  int64_t Kt = (int64_t)(d.k + 1) * d.d_in;
  int64_t m = 0;
  m = std::max<int64_t>(m, splits_for(n_dst) * Kt * d.d_out);              // dTheta
  m = std::max<int64_t>(m, splits_for(n_dst) * (int64_t)d.d_out * d.d_in);  // dW_root
  m = std::max<int64_t>(m, splits_for(E) * (int64_t)d.k * d.k);            // dW2
  m = std::max<int64_t>(m, splits_for(E) * (int64_t)d.k * d.d_e);          // dW1
  return m;
}
static F32Bwd carve_f32_bwd(Carver &c, const dsmpnn_layer_desc &d, int64_t n_dst, int64_t n_loc, int64_t E) {
  F32Bwd b;
  int64_t Kt = (int64_t)(d.k + 1) * d.d_in;
  b.gh = c.take<float>(n_dst * d.d_out);
  b.dS = c.take<float>(n_dst * Kt);
  b.dZ2 = c.take<float>(E * d.k);
  b.dA1 = c.take<float>(E * d.k);
  b.U = c.take<float>(E * d.d_in);
  b.dT = c.take<float>(Kt * d.d_out);
  b.partial = c.take<float>(f32_partial_elems(d, n_dst, E));
  return b;
}

static dsmpnn_status check_desc(const dsmpnn_layer_desc *d) {
  DS_CHECK_ARG(d != nullptr, DSMPNN_ERR_INVALID_ARG, "layer: desc is NULL");
  DS_CHECK_ARG(d->d_e >= 1 && d->d_in >= 1 && d->d_out >= 1 && d->k >= 1, DSMPNN_ERR_INVALID_ARG,
               "layer: widths must be >= 1");
  DS_CHECK_ARG(d->root >= 0 && d->root <= 2 && d->act >= 0 && d->act <= 1, DSMPNN_ERR_INVALID_ARG,
               "layer: root/act out of range");
  DS_CHECK_ARG(d->root != DSMPNN_ROOT_IDENTITY || d->d_in == d->d_out, DSMPNN_ERR_SHAPE,
               "layer: ROOT_IDENTITY needs d_in == d_out");
  DS_CHECK_ARG(d->dtype == DSMPNN_F32 || d->dtype == DSMPNN_BF16, DSMPNN_ERR_INVALID_ARG, "layer: dtype");
  if (d->dtype == DSMPNN_F32) {
    DS_CHECK_ARG((int64_t)(d->k + 1) * d->d_in * 4 + 128 * d->d_in * 4 <= 200 * 1024, DSMPNN_ERR_UNSUPPORTED,
                 "layer F32: (k+1)*d_in too large for the per-row kernels");
  } else {
    DS_TRY(bf16_check_desc(*d));
  }
  return DSMPNN_OK;
}

static dsmpnn_status edge_range(const int64_t *row_ptr, const int64_t *row_ptr_host, int64_t rb, int64_t re,
                                int64_t *eb, int64_t *ee, cudaStream_t s) {
  if (row_ptr_host) {
    *eb = row_ptr_host[rb];
    *ee = row_ptr_host[re];
    return DSMPNN_OK;
  }
  int64_t h[2];
  DS_CUDA(cudaMemcpyAsync(&h[0], row_ptr + rb, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  DS_CUDA(cudaMemcpyAsync(&h[1], row_ptr + re, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  DS_CUDA(cudaStreamSynchronize(s));
  *eb = h[0];
  *ee = h[1];
  return DSMPNN_OK;
}

// ------------------------------------------------------- CSR validation ----
// BF16 edge tiles hold whole destination rows of at most kMaxRowEdgesBf16
// edges (edge_fwd2.cuh walk_tile); a longer row is UNSUPPORTED, checked here
// before any launch.  With DSMPNN_DEBUG set in the environment, every call
// also validates the CSR (row_ptr non-decreasing, 0 <= col < n_loc) and
// returns ERR_INDEX instead of reading out of bounds.
constexpr int kMaxRowEdgesBf16 = 128;

// flags[0] = max degree of rows [rb, re); flags[1] = number of bad entries
__global__ void csr_scan_kernel(const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col, int64_t rb,
                                int64_t re, int64_t n_loc, int check_cols, int *flags) {
  int mx = 0, bad = 0;
  for (int64_t i = rb + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < re; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = row_ptr[i], b = row_ptr[i + 1];
    if (b < a) { ++bad; continue; }
    const int64_t dg = b - a;
    mx = max(mx, dg > (1 << 30) ? (1 << 30) : (int)dg);
    if (check_cols)
      for (int64_t p = a; p < b; ++p) {
        const int32_t j = col[p];
        bad += (j < 0 || (n_loc >= 0 && j >= n_loc));
      }
  }
  if (mx) atomicMax(&flags[0], mx);
  if (bad) atomicAdd(&flags[1], bad);
}

static bool debug_checks() {
  static const bool on = getenv("DSMPNN_DEBUG") != nullptr;
  return on;
}

static dsmpnn_status check_rows(const dsmpnn_layer_desc &d, const int64_t *row_ptr, const int64_t *row_ptr_host,
                                const int32_t *col, int64_t rb, int64_t re, int64_t n_loc, cudaStream_t s) {
  const bool dbg = debug_checks();
  const bool need_deg = d.dtype == DSMPNN_BF16;
  if (!dbg && !need_deg) return DSMPNN_OK;
  int64_t maxdeg = 0;
  if (row_ptr_host && !dbg) {
    for (int64_t i = rb; i < re; ++i) maxdeg = std::max<int64_t>(maxdeg, row_ptr_host[i + 1] - row_ptr_host[i]);
  } else {
    int *flags = nullptr, h[2] = {0, 0};
    DS_CUDA(cudaMallocAsync((void **)&flags, 2 * sizeof(int), s));
    DS_CUDA(cudaMemsetAsync(flags, 0, 2 * sizeof(int), s));
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(re - rb, 256), kNumSMs * 4));
    csr_scan_kernel<<<blocks, 256, 0, s>>>(row_ptr, col, rb, re, n_loc, dbg ? 1 : 0, flags);
    DS_LAUNCH_CHECK();
    DS_CUDA(cudaMemcpyAsync(h, flags, sizeof(h), cudaMemcpyDeviceToHost, s));
    DS_CUDA(cudaFreeAsync(flags, s));
    DS_CUDA(cudaStreamSynchronize(s));
    DS_CHECK_ARG(h[1] == 0, DSMPNN_ERR_INDEX, "layer: CSR has %d invalid entries (row_ptr decreasing or col out of "
                 "range) in rows [%lld, %lld)", h[1], (long long)rb, (long long)re);
    maxdeg = h[0];
  }
  DS_CHECK_ARG(!need_deg || maxdeg <= kMaxRowEdgesBf16, DSMPNN_ERR_UNSUPPORTED,
               "layer BF16: a destination row has %lld edges; the fused edge kernels take rows of at most %d "
               "edges (cap the graph with n_e <= %d)", (long long)maxdeg, kMaxRowEdgesBf16, kMaxRowEdgesBf16);
  return DSMPNN_OK;
}

// ------------------------------------------------------------ F32 fwd ----
static dsmpnn_status fwd_f32(const dsmpnn_layer_desc &d, const dsmpnn_weights &w, const float *v, const float *e,
                             const int64_t *row_ptr, const int32_t *col, int64_t n_dst, int64_t E, int64_t rb,
                             int64_t re, int64_t eb, int64_t ee, float *out, __nv_bfloat16 *out_lowp, void *ws,
                             size_t ws_bytes, cudaStream_t s) {
  Carver c(ws, ws_bytes);
  F32Fwd f = carve_f32_fwd(c, d, n_dst, E);
  DS_CHECK_ARG(c.ok(), DSMPNN_ERR_CAPACITY, "layer_fwd: workspace too small");
  const float *T = static_cast<const float *>(w.packed);
  int64_t Kt = (int64_t)(d.k + 1) * d.d_in;
  int64_t nE = ee - eb, nR = re - rb;
  if (nE > 0) {
    // A1 = relu(e W1^T + b1);  H = relu(A1 W2^T + b2)
    SgemmArgs g1{nE, d.k, d.d_e, e + eb * d.d_e, d.d_e, 1, w.W1, 1, d.d_e, f.A1 + eb * d.k, d.k, w.b1, 1, 0, 1.f};
    DS_TRY(sgemm(g1, 1, nullptr, s));
    SgemmArgs g2{nE, d.k, d.k, f.A1 + eb * d.k, d.k, 1, w.W2, 1, d.k, f.H + eb * d.k, d.k, w.b2, 1, 0, 1.f};
    ProbeScope probe(DSMPNN_PROBE_F32_MLP2, s);
    DS_TRY(sgemm(g2, 1, nullptr, s));
  }
  if (nR > 0) {
    size_t smem = (size_t)kEdgeChunk * d.d_in * sizeof(float);
    s_form_f32_kernel<<<(unsigned)nR, 256, smem, s>>>(f.H, v, row_ptr, col, rb, d.k, d.d_in, f.S);
    DS_LAUNCH_CHECK();
    // agg = S~ Theta~  -> pre
    SgemmArgs g3{nR, d.d_out, Kt, f.S + rb * Kt, Kt, 1, T, d.d_out, 1, f.pre + rb * d.d_out, d.d_out, nullptr, 0, 0,
                 1.f};
    DS_TRY(sgemm(g3, 1, nullptr, s));
    if (d.root == DSMPNN_ROOT_DENSE) {
      SgemmArgs g4{nR, d.d_out, d.d_in, v + rb * d.d_in, d.d_in, 1, w.W_root, 1, d.d_in, f.pre + rb * d.d_out, d.d_out,
                   nullptr, 0, 1, 1.f};
      DS_TRY(sgemm(g4, 1, nullptr, s));
    }
    node_epilogue_kernel<<<grid_of(nR * d.d_out), 256, 0, s>>>(f.pre, v, nullptr, w.b, rb, re, d.d_out, d.root, d.act,
                                                               out, out_lowp);
    DS_LAUNCH_CHECK();
  }
  return DSMPNN_OK;
}

// ------------------------------------------------------------ F32 bwd ----
static dsmpnn_status bwd_f32(const dsmpnn_layer_desc &d, const dsmpnn_weights &w, const float *v, const float *e,
                             const int64_t *row_ptr, const int32_t *col, const int32_t *perm, const int64_t *cptr,
                             int64_t n_dst, int64_t n_loc, int64_t E, int64_t rb, int64_t re, int64_t eb, int64_t ee,
                             const float *G, float *dv, float *de, const dsmpnn_grads &gr, const void *ws,
                             size_t ws_bytes_unused, void *bws, size_t bws_bytes, cudaStream_t s) {
  Carver cf(const_cast<void *>(ws), SIZE_MAX);
  F32Fwd f = carve_f32_fwd(cf, d, n_dst, E);
  Carver cb(bws, bws_bytes);
  F32Bwd b = carve_f32_bwd(cb, d, n_dst, n_loc, E);
  DS_CHECK_ARG(cb.ok(), DSMPNN_ERR_CAPACITY, "layer_bwd: bwd workspace too small");
  const float *T = static_cast<const float *>(w.packed);
  int64_t Kt = (int64_t)(d.k + 1) * d.d_in;
  int64_t nE = ee - eb, nR = re - rb;
  if (nR <= 0) return DSMPNN_OK;
  ghat_kernel<<<grid_of(nR * d.d_out), 256, 0, s>>>(G, f.pre, rb, re, d.d_out, d.act, b.gh);
  DS_LAUNCH_CHECK();
  const float *gh = b.gh + rb * d.d_out;
  DS_TRY(colsum(gh, nR, d.d_out, d.d_out, gr.b, 1, s));
  if (d.root == DSMPNN_ROOT_DENSE) {
    if (gr.W_root) {  // dW_root += gh^T v_rows : [d_out x d_in], K = rows
      SgemmArgs g{d.d_out, d.d_in, nR, gh, 1, d.d_out, v + rb * d.d_in, d.d_in, 1, gr.W_root, d.d_in, nullptr, 0, 1,
                  1.f};
      DS_TRY(sgemm(g, splits_for(nR), b.partial, s));
    }
    if (dv) {  // dv[rows] += gh W_root
      SgemmArgs g{nR, d.d_in, d.d_out, gh, d.d_out, 1, w.W_root, d.d_in, 1, dv + rb * d.d_in, d.d_in, nullptr, 0, 1,
                  1.f};
      DS_TRY(sgemm(g, 1, nullptr, s));
    }
  } else if (d.root == DSMPNN_ROOT_IDENTITY && dv) {
    add_rows_kernel<<<grid_of(nR * d.d_out), 256, 0, s>>>(b.gh, rb, re, d.d_out, dv);
    DS_LAUNCH_CHECK();
  }
  // dTheta~ = S~^T gh  [Kt x d_out], K = rows
  if (gr.W3 || gr.b3) {
    SgemmArgs g{Kt, d.d_out, nR, f.S + rb * Kt, 1, Kt, gh, d.d_out, 1, b.dT, d.d_out, nullptr, 0, 0, 1.f};
    DS_TRY(sgemm(g, splits_for(nR), b.partial, s));
    unpack_dtheta_kernel<<<grid_of(Kt * d.d_out), 256, 0, s>>>(b.dT, d.k, d.d_in, d.d_out, gr.W3, gr.b3);
    DS_LAUNCH_CHECK();
  }
  // dS~ = gh Theta~^T  [rows x Kt]
  {
    SgemmArgs g{nR, Kt, d.d_out, gh, d.d_out, 1, T, 1, d.d_out, b.dS + rb * Kt, Kt, nullptr, 0, 0, 1.f};
    DS_TRY(sgemm(g, 1, nullptr, s));
  }
  if (nE <= 0) return DSMPNN_OK;
  {
    size_t smem = (size_t)(Kt + kEdgeChunk * d.d_in) * sizeof(float);
    DS_CUDA(cudaFuncSetAttribute(edge_bwd_f32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    ProbeScope probe(DSMPNN_PROBE_F32_EDGE_BWD, s);
    edge_bwd_f32_kernel<<<(unsigned)nR, 256, smem, s>>>(b.dS, f.H, v, row_ptr, col, rb, d.k, d.d_in, b.dZ2, b.U);
    DS_LAUNCH_CHECK();
  }
  float *dZ2 = b.dZ2 + eb * d.k;
  const float *A1 = f.A1 + eb * d.k;
  if (gr.W2) {  // dW2 += dZ2^T A1  [k x k], K = edges
    SgemmArgs g{d.k, d.k, nE, dZ2, 1, d.k, A1, d.k, 1, gr.W2, d.k, nullptr, 0, 1, 1.f};
    DS_TRY(sgemm(g, splits_for(nE), b.partial, s));
  }
  DS_TRY(colsum(dZ2, nE, d.k, d.k, gr.b2, 1, s));
  // dZ1 = (dZ2 W2) * [A1 > 0]
  float *dZ1 = b.dA1 + eb * d.k;
  {
    SgemmArgs g{nE, d.k, d.k, dZ2, d.k, 1, w.W2, d.k, 1, dZ1, d.k, nullptr, 0, 0, 1.f};
    DS_TRY(sgemm(g, 1, nullptr, s));
    relu_mask_kernel<<<grid_of(nE * d.k), 256, 0, s>>>(dZ1, A1, nE * d.k);
    DS_LAUNCH_CHECK();
  }
  if (gr.W1) {  // dW1 += dZ1^T e  [k x d_e]
    SgemmArgs g{d.k, d.d_e, nE, dZ1, 1, d.k, e + eb * d.d_e, d.d_e, 1, gr.W1, d.d_e, nullptr, 0, 1, 1.f};
    DS_TRY(sgemm(g, splits_for(nE), b.partial, s));
  }
  DS_TRY(colsum(dZ1, nE, d.k, d.k, gr.b1, 1, s));
  if (de) {  // de = dZ1 W1  [E x d_e]
    SgemmArgs g{nE, d.d_e, d.k, dZ1, d.k, 1, w.W1, d.d_e, 1, de + eb * d.d_e, d.d_e, nullptr, 0, 0, 1.f};
    DS_TRY(sgemm(g, 1, nullptr, s));
  }
  if (dv) {
    scatter_csc_kernel<<<grid_of(n_loc * d.d_in), 256, 0, s>>>(b.U, perm, cptr, n_loc, d.d_in, eb, ee, dv);
    DS_LAUNCH_CHECK();
  }
  return DSMPNN_OK;
}

}  // namespace dsmpnn

using namespace dsmpnn;

extern "C" {

dsmpnn_status dsmpnn_packed_weights_size(const dsmpnn_layer_desc *desc, size_t *bytes) {
  DS_TRY(check_desc(desc));
  if (desc->dtype == DSMPNN_F32) {
    *bytes = (size_t)(desc->k + 1) * desc->d_in * desc->d_out * sizeof(float);
    return DSMPNN_OK;
  }
  *bytes = bf16_packed_bytes(*desc);
  return DSMPNN_OK;
}

dsmpnn_status dsmpnn_pack_weights(const dsmpnn_layer_desc *desc, const dsmpnn_weights *w, void *packed, size_t bytes,
                                  void *stream) {
  DS_TRY(check_desc(desc));
  DS_CHECK_ARG(w && w->W1 && w->b1 && w->W2 && w->b2 && w->W3 && w->b3 && w->b, DSMPNN_ERR_INVALID_ARG,
               "pack_weights: NULL weight");
  size_t need;
  DS_TRY(dsmpnn_packed_weights_size(desc, &need));
  DS_CHECK_ARG(bytes >= need, DSMPNN_ERR_CAPACITY, "pack_weights: buffer %zu < %zu", bytes, need);
  cudaStream_t s = as_stream(stream);
  if (desc->dtype == DSMPNN_F32) {
    int64_t total = (int64_t)(desc->k + 1) * desc->d_in * desc->d_out;
    pack_theta_f32_kernel<<<grid_of(total), 256, 0, s>>>(w->W3, w->b3, desc->k, desc->d_in, desc->d_out,
                                                        (float *)packed);
    DS_LAUNCH_CHECK();
    return DSMPNN_OK;
  }
  return bf16_pack(*desc, *w, packed, s);
}

dsmpnn_status dsmpnn_layer_workspace_size(const dsmpnn_layer_desc *desc, int64_t n_dst, int64_t n_edges,
                                          size_t *bytes) {
  DS_TRY(check_desc(desc));
  DS_CHECK_ARG(n_dst >= 0 && n_edges >= 0, DSMPNN_ERR_INVALID_ARG, "layer_workspace_size: sizes");
  if (desc->dtype == DSMPNN_F32) {
    Carver c(nullptr, 0);
    carve_f32_fwd(c, *desc, n_dst, n_edges);
    *bytes = c.used();
    return DSMPNN_OK;
  }
  *bytes = bf16_fwd_ws_bytes(*desc, n_dst, n_edges);
  return DSMPNN_OK;
}

dsmpnn_status dsmpnn_layer_bwd_workspace_size(const dsmpnn_layer_desc *desc, int64_t n_dst, int64_t n_loc,
                                              int64_t n_edges, size_t *bytes) {
  DS_TRY(check_desc(desc));
  if (desc->dtype == DSMPNN_F32) {
    Carver c(nullptr, 0);
    carve_f32_bwd(c, *desc, n_dst, n_loc, n_edges);
    *bytes = c.used();
    return DSMPNN_OK;
  }
  *bytes = bf16_bwd_ws_bytes(*desc, n_dst, n_loc, n_edges);
  return DSMPNN_OK;
}

dsmpnn_status dsmpnn_layer_fwd(const dsmpnn_layer_desc *desc, const dsmpnn_weights *w, const void *v, const void *e,
                               const int64_t *row_ptr, const int64_t *row_ptr_host, const int32_t *col_idx,
                               int64_t n_dst, int64_t row_begin, int64_t row_end, float *out, void *out_lowp,
                               void *ws, size_t ws_bytes, void *stream) {
  DS_TRY(check_desc(desc));
  DS_CHECK_ARG(w && w->packed && w->W1 && w->b1 && w->W2 && w->b2 && w->b, DSMPNN_ERR_INVALID_ARG,
               "layer_fwd: NULL weight (packed weights are required)");
  DS_CHECK_ARG(desc->root != DSMPNN_ROOT_DENSE || w->W_root, DSMPNN_ERR_INVALID_ARG, "layer_fwd: W_root is NULL");
  DS_CHECK_ARG(0 <= row_begin && row_begin <= row_end && row_end <= n_dst, DSMPNN_ERR_INVALID_ARG,
               "layer_fwd: bad row range [%lld,%lld) of %lld", (long long)row_begin, (long long)row_end,
               (long long)n_dst);
  cudaStream_t s = as_stream(stream);
  if (row_end == row_begin) return DSMPNN_OK;
  int64_t eb, ee, E;
  DS_TRY(check_rows(*desc, row_ptr, row_ptr_host, col_idx, row_begin, row_end, -1, s));
  DS_TRY(edge_range(row_ptr, row_ptr_host, row_begin, row_end, &eb, &ee, s));
  if (row_ptr_host) E = row_ptr_host[n_dst];
  else {
    DS_CUDA(cudaMemcpyAsync(&E, row_ptr + n_dst, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    DS_CUDA(cudaStreamSynchronize(s));
  }
  size_t need;
  DS_TRY(dsmpnn_layer_workspace_size(desc, n_dst, E, &need));
  DS_CHECK_ARG(ws_bytes >= need, DSMPNN_ERR_CAPACITY, "layer_fwd: workspace %zu < %zu", ws_bytes, need);
  if (desc->dtype == DSMPNN_F32)
    return fwd_f32(*desc, *w, (const float *)v, (const float *)e, row_ptr, col_idx, n_dst, E, row_begin, row_end, eb,
                   ee, out, (__nv_bfloat16 *)out_lowp, ws, ws_bytes, s);
  return bf16_fwd(*desc, *w, (const __nv_bfloat16 *)v, (const __nv_bfloat16 *)e, row_ptr, col_idx, n_dst, E,
                  row_begin, row_end, eb, ee, out, (__nv_bfloat16 *)out_lowp, ws, ws_bytes, s);
}

dsmpnn_status dsmpnn_layer_bwd(const dsmpnn_layer_desc *desc, const dsmpnn_weights *w, const void *v, const void *e,
                               const int64_t *row_ptr, const int64_t *row_ptr_host, const int32_t *col_idx,
                               const int32_t *csc_perm, const int64_t *csc_ptr, int64_t n_dst, int64_t n_loc,
                               int64_t row_begin, int64_t row_end, const float *grad_out, float *grad_v,
                               float *grad_e, const dsmpnn_grads *grads, const void *ws, void *bwd_ws,
                               size_t bwd_ws_bytes, void *stream) {
  DS_TRY(check_desc(desc));
  DS_CHECK_ARG(w && w->packed && w->W2 && w->W1, DSMPNN_ERR_INVALID_ARG, "layer_bwd: NULL weight");
  DS_CHECK_ARG(grads != nullptr && grad_out != nullptr, DSMPNN_ERR_INVALID_ARG, "layer_bwd: NULL grads/grad_out");
  DS_CHECK_ARG(!grad_v || (csc_perm && csc_ptr), DSMPNN_ERR_INVALID_ARG, "layer_bwd: grad_v needs the CSC view");
  DS_CHECK_ARG(0 <= row_begin && row_begin <= row_end && row_end <= n_dst && n_dst <= n_loc, DSMPNN_ERR_INVALID_ARG,
               "layer_bwd: bad row range");
  cudaStream_t s = as_stream(stream);
  if (row_end == row_begin) return DSMPNN_OK;
  int64_t eb, ee, E;
  DS_TRY(check_rows(*desc, row_ptr, row_ptr_host, col_idx, row_begin, row_end, n_loc, s));
  DS_TRY(edge_range(row_ptr, row_ptr_host, row_begin, row_end, &eb, &ee, s));
  if (row_ptr_host) E = row_ptr_host[n_dst];
  else {
    DS_CUDA(cudaMemcpyAsync(&E, row_ptr + n_dst, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    DS_CUDA(cudaStreamSynchronize(s));
  }
  size_t need;
  DS_TRY(dsmpnn_layer_bwd_workspace_size(desc, n_dst, n_loc, E, &need));
  DS_CHECK_ARG(bwd_ws_bytes >= need, DSMPNN_ERR_CAPACITY, "layer_bwd: workspace %zu < %zu", bwd_ws_bytes, need);
  if (desc->dtype == DSMPNN_F32)
    return bwd_f32(*desc, *w, (const float *)v, (const float *)e, row_ptr, col_idx, csc_perm, csc_ptr, n_dst, n_loc, E,
                   row_begin, row_end, eb, ee, grad_out, grad_v, grad_e, *grads, ws, 0, bwd_ws, bwd_ws_bytes, s);
  return bf16_bwd(*desc, *w, (const __nv_bfloat16 *)v, (const __nv_bfloat16 *)e, row_ptr, col_idx, csc_perm, csc_ptr,
                  n_dst, n_loc, E, row_begin, row_end, eb, ee, grad_out, grad_v, grad_e, *grads, ws, bwd_ws,
                  bwd_ws_bytes, s);
}

}  // extern "C"

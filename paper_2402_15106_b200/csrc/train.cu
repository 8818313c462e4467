// train.cu - f1: the pieces of the DS-MPNN training step around the layer
// (PAPER.md eqs. (i), (iii), (iv), Alg. 1 :404-419; oracle/train.py O9), fp32:
//   3-layer node MLPs (encoder N_e, decoder N_d): forward / backward on the
//   library's deterministic SIMT GEMM (bias + ReLU epilogue, split-K dW);
//   backward of the edge refresh (iv) e_ij = (x_i - x_j, u_i - u_j);
//   MSE on owned rows (loss + gradient, fixed reduction order);
//   SGD (Alg. 1 :419) and Adam parameter updates.
#include <cmath>

#include "common.cuh"
#include "simt.cuh"

namespace dsmpnn {

__global__ void mlp_relu_mask_kernel(float *__restrict__ g, const float *__restrict__ h, int64_t total) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x)
    if (!(h[t] > 0.f)) g[t] = 0.f;
}

// du_j += (j < n_dst ? sum_{p in row j} de_p[off:off+w] : 0) - sum_{q in CSC(j)} de_{perm q}[off:off+w]
__global__ void edge_refresh_bwd_kernel(const float *__restrict__ de, int d_e, int off, int w,
                                        const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ perm,
                                        const int64_t *__restrict__ cptr, int64_t n_dst, int64_t n_loc,
                                        float *__restrict__ du) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n_loc * w; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = t / w;
    const int c = (int)(t - j * w);
    float a = 0.f;
    if (j < n_dst)
      for (int64_t p = row_ptr[j]; p < row_ptr[j + 1]; ++p) a += de[p * d_e + off + c];
    float b = 0.f;
    for (int64_t q = cptr[j]; q < cptr[j + 1]; ++q) b += de[(int64_t)perm[q] * d_e + off + c];
    du[t] += a - b;
  }
}

// one block: sse += sum (pred - y)^2 in a fixed order; grad = 2 (pred - y) * scale
__global__ void __launch_bounds__(1024) mse_kernel(const float *__restrict__ pred, const float *__restrict__ y,
                                                   int64_t total, float scale, float *__restrict__ grad,
                                                   float *__restrict__ sse) {
  __shared__ float red[1024];
  float s = 0.f;
  for (int64_t t = threadIdx.x; t < total; t += 1024) {
    const float d = pred[t] - y[t];
    s += d * d;
    if (grad) grad[t] = 2.f * d * scale;
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = 512; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *sse += red[0];
}

__global__ void sgd_kernel(float *__restrict__ w, const float *__restrict__ g, int64_t n, float lr) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    w[t] -= lr * g[t];
}

__global__ void adam_kernel(float *__restrict__ w, const float *__restrict__ g, float *__restrict__ m,
                            float *__restrict__ v, int64_t n, float lr, float b1, float b2, float eps, float c1,
                            float c2) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const float gt = g[t];
    const float mt = b1 * m[t] + (1.f - b1) * gt;
    const float vt = b2 * v[t] + (1.f - b2) * gt * gt;
    m[t] = mt;
    v[t] = vt;
    w[t] -= lr * (mt / c1) / (sqrtf(vt / c2) + eps);
  }
}

static int grid_n(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), 148 * 8)); }

struct MlpWs {
  float *d2, *d1, *partial, *cs;
};
static constexpr int kMlpSplits = 32;
static MlpWs carve_mlp(Carver &c, int in, int hid, int out, int64_t n) {
  MlpWs w;
  w.d2 = c.take<float>(n * hid);
  w.d1 = c.take<float>(n * hid);
  w.partial = c.take<float>((int64_t)kMlpSplits * std::max(hid * std::max(in, hid), out * hid));
  w.cs = c.take<float>((int64_t)kColsumChunks * std::max(hid, out));
  return w;
}

// dW (+)= dY^T X over n rows (M = rows of W, N = cols, K = n), split-K in a fixed order
static dsmpnn_status weight_grad(const float *dY, int m_out, const float *X, int n_in, int64_t n, float *dW,
                                 float *partial, cudaStream_t s) {
  if (!dW) return DSMPNN_OK;
  const int splits = (int)std::max<int64_t>(1, std::min<int64_t>(kMlpSplits, n / 256));
  SgemmArgs g{m_out, n_in, n, dY, 1, m_out, X, n_in, 1, dW, n_in, nullptr, 0, 1, 1.f};
  return sgemm(g, splits, partial, s);
}

}  // namespace dsmpnn

using namespace dsmpnn;

extern "C" {

dsmpnn_status dsmpnn_mlp3_fwd(int32_t in_dim, int32_t hid, int32_t out_dim, const float *const *Wb, const float *x,
                              int64_t n, float *h1, float *h2, float *y, void *stream) {
  DS_CHECK_ARG(in_dim > 0 && hid > 0 && out_dim > 0 && n >= 0, DSMPNN_ERR_INVALID_ARG, "mlp3_fwd: sizes");
  if (n == 0) return DSMPNN_OK;
  cudaStream_t s = as_stream(stream);
  // layer l: out = act(in W_l^T + b_l),  B(k, n) = W_l[n][k]
  SgemmArgs g0{n, hid, in_dim, x, in_dim, 1, Wb[0], 1, in_dim, h1, hid, Wb[1], 1, 0, 1.f};
  DS_TRY(sgemm(g0, 1, nullptr, s));
  SgemmArgs g1{n, hid, hid, h1, hid, 1, Wb[2], 1, hid, h2, hid, Wb[3], 1, 0, 1.f};
  DS_TRY(sgemm(g1, 1, nullptr, s));
  SgemmArgs g2{n, out_dim, hid, h2, hid, 1, Wb[4], 1, hid, y, out_dim, Wb[5], 0, 0, 1.f};
  return sgemm(g2, 1, nullptr, s);
}

dsmpnn_status dsmpnn_mlp3_bwd_workspace_size(int32_t in_dim, int32_t hid, int32_t out_dim, int64_t n, size_t *bytes) {
  DS_CHECK_ARG(in_dim > 0 && hid > 0 && out_dim > 0 && n >= 0, DSMPNN_ERR_INVALID_ARG, "mlp3_bwd: sizes");
  Carver c(nullptr, 0);
  carve_mlp(c, in_dim, hid, out_dim, n);
  *bytes = c.used();
  return DSMPNN_OK;
}

dsmpnn_status dsmpnn_mlp3_bwd(int32_t in_dim, int32_t hid, int32_t out_dim, const float *const *Wb, const float *x,
                              const float *h1, const float *h2, const float *dy, int64_t n, float *dx,
                              float *const *dWb, void *ws, size_t ws_bytes, void *stream) {
  DS_CHECK_ARG(in_dim > 0 && hid > 0 && out_dim > 0 && n >= 0, DSMPNN_ERR_INVALID_ARG, "mlp3_bwd: sizes");
  if (n == 0) return DSMPNN_OK;
  cudaStream_t s = as_stream(stream);
  Carver c(ws, ws_bytes);
  MlpWs w = carve_mlp(c, in_dim, hid, out_dim, n);
  DS_CHECK_ARG(c.ok(), DSMPNN_ERR_CAPACITY, "mlp3_bwd: workspace too small");
  // layer 2
  DS_TRY(weight_grad(dy, out_dim, h2, hid, n, dWb[4], w.partial, s));
  if (dWb[5]) DS_TRY(colsum_ws(dy, n, out_dim, out_dim, dWb[5], 1, w.cs, s));
  {
    SgemmArgs g{n, hid, out_dim, dy, out_dim, 1, Wb[4], hid, 1, w.d2, hid, nullptr, 0, 0, 1.f};
    DS_TRY(sgemm(g, 1, nullptr, s));
    mlp_relu_mask_kernel<<<grid_n(n * hid), 256, 0, s>>>(w.d2, h2, n * hid);
    DS_LAUNCH_CHECK();
  }
  // layer 1
  DS_TRY(weight_grad(w.d2, hid, h1, hid, n, dWb[2], w.partial, s));
  if (dWb[3]) DS_TRY(colsum_ws(w.d2, n, hid, hid, dWb[3], 1, w.cs, s));
  {
    SgemmArgs g{n, hid, hid, w.d2, hid, 1, Wb[2], hid, 1, w.d1, hid, nullptr, 0, 0, 1.f};
    DS_TRY(sgemm(g, 1, nullptr, s));
    mlp_relu_mask_kernel<<<grid_n(n * hid), 256, 0, s>>>(w.d1, h1, n * hid);
    DS_LAUNCH_CHECK();
  }
  // layer 0
  DS_TRY(weight_grad(w.d1, hid, x, in_dim, n, dWb[0], w.partial, s));
  if (dWb[1]) DS_TRY(colsum_ws(w.d1, n, hid, hid, dWb[1], 1, w.cs, s));
  if (dx) {
    SgemmArgs g{n, in_dim, hid, w.d1, hid, 1, Wb[0], in_dim, 1, dx, in_dim, nullptr, 0, 1, 1.f};  // dx +=
    DS_TRY(sgemm(g, 1, nullptr, s));
  }
  return DSMPNN_OK;
}

dsmpnn_status dsmpnn_edge_refresh_bwd(const float *grad_e, int32_t d_e, int32_t off, int32_t width,
                                      const int64_t *row_ptr, const int32_t *csc_perm, const int64_t *csc_ptr,
                                      int64_t n_dst, int64_t n_loc, float *grad_u, void *stream) {
  DS_CHECK_ARG(d_e > 0 && off >= 0 && width > 0 && off + width <= d_e && n_dst >= 0 && n_loc >= n_dst,
               DSMPNN_ERR_INVALID_ARG, "edge_refresh_bwd: sizes");
  if (n_loc == 0) return DSMPNN_OK;
  edge_refresh_bwd_kernel<<<grid_n(n_loc * width), 256, 0, as_stream(stream)>>>(
      grad_e, d_e, off, width, row_ptr, csc_perm, csc_ptr, n_dst, n_loc, grad_u);
  DS_LAUNCH_CHECK();
  return DSMPNN_OK;
}

dsmpnn_status dsmpnn_mse(const float *pred, const float *target, int64_t n_elems, float scale, float *grad,
                         float *sse, void *stream) {
  DS_CHECK_ARG(n_elems >= 0 && sse, DSMPNN_ERR_INVALID_ARG, "mse: arguments");
  if (n_elems == 0) return DSMPNN_OK;
  mse_kernel<<<1, 1024, 0, as_stream(stream)>>>(pred, target, n_elems, scale, grad, sse);
  DS_LAUNCH_CHECK();
  return DSMPNN_OK;
}

__global__ void mse_mean_kernel(const float *__restrict__ sse, double count, float *__restrict__ loss) {
  loss[0] = (float)((double)sse[0] / count);
}

dsmpnn_status dsmpnn_mse_mean(const float *sse, int64_t count, float *loss, void *stream) {
  DS_CHECK_ARG(sse && loss && count > 0, DSMPNN_ERR_INVALID_ARG, "mse_mean: arguments");
  mse_mean_kernel<<<1, 1, 0, as_stream(stream)>>>(sse, (double)count, loss);
  DS_LAUNCH_CHECK();
  return DSMPNN_OK;
}

dsmpnn_status dsmpnn_sgd(float *w, const float *g, int64_t n, float lr, void *stream) {
  DS_CHECK_ARG(n >= 0, DSMPNN_ERR_INVALID_ARG, "sgd: n");
  if (n == 0) return DSMPNN_OK;
  sgd_kernel<<<grid_n(n), 256, 0, as_stream(stream)>>>(w, g, n, lr);
  DS_LAUNCH_CHECK();
  return DSMPNN_OK;
}

dsmpnn_status dsmpnn_adam(float *w, const float *g, float *m, float *v, int64_t n, float lr, float beta1, float beta2,
                          float eps, int32_t step, void *stream) {
  DS_CHECK_ARG(n >= 0 && step >= 1, DSMPNN_ERR_INVALID_ARG, "adam: n / step");
  if (n == 0) return DSMPNN_OK;
  const float c1 = (float)(1.0 - std::pow((double)beta1, step)), c2 = (float)(1.0 - std::pow((double)beta2, step));
  adam_kernel<<<grid_n(n), 256, 0, as_stream(stream)>>>(w, g, m, v, n, lr, beta1, beta2, eps, c1, c2);
  DS_LAUNCH_CHECK();
  return DSMPNN_OK;
}

}  // extern "C"

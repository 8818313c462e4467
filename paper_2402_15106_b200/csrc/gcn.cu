// gcn.cu - f3: the paper's node-based comparison model ("GCN here
// uses 6 hidden layers with a size of 378"), one layer
//   agg_i = (v_i + sum_{p in row i} v_{col p}) / (deg_i + 1)    (mean over N(i) u {i})
//   out_i = act(W agg_i + c)
// on the radius graph built as for the MPNN (R24), fp32 (F32 mode of
// reading R18: SIMT FFMA).  The aggregation is HBM-bound (one warp per row,
// lanes over channels, four neighbour rows in flight, fixed summation order);
// the dense parts use the library's deterministic SIMT GEMM.
#include "common.cuh"
#include "simt.cuh"

namespace dsmpnn {

// agg_i = (v_i + sum_p v_{col p}) / (deg_i + 1); self first, then the row in CSR order
__global__ void gcn_mean_kernel(const float *__restrict__ v, const int64_t *__restrict__ row_ptr,
                                const int32_t *__restrict__ col, int64_t n_dst, int d, float *__restrict__ agg) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n_dst; i += nw) {
    const int64_t p0 = row_ptr[i], p1 = row_ptr[i + 1];
    const float inv = 1.0f / (float)(p1 - p0 + 1);
    for (int c0 = 0; c0 < d; c0 += 32) {
      const int c = c0 + lane;
      if (c >= d) break;
      float acc = v[i * d + c];
      int64_t p = p0;
      for (; p + 4 <= p1; p += 4) {
        int32_t j[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) j[u] = __ldg(col + p + u);
        float x[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) x[u] = __ldg(v + (int64_t)j[u] * d + c);
#pragma unroll
        for (int u = 0; u < 4; ++u) acc += x[u];
      }
      for (; p < p1; ++p) acc += __ldg(v + (int64_t)__ldg(col + p) * d + c);
      agg[i * d + c] = acc * inv;
    }
  }
}

// ghat = G * act'(pre), with act'(pre) = [out > 0] for ReLU (ReLU'(0) = 0)
__global__ void gcn_ghat_kernel(const float *__restrict__ G, const float *__restrict__ out, int64_t total, int act,
                                float *__restrict__ gh) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x)
    gh[t] = (act == DSMPNN_ACT_RELU && !(out[t] > 0.f)) ? 0.f : G[t];
}

// dv_j += dagg_j / (deg_j + 1)  (self, j < n_dst)  +  sum over the CSC list of j
// of dagg_i / (deg_i + 1), i = destination of the edge (binary search)
__global__ void gcn_scatter_kernel(const float *__restrict__ dagg, const int64_t *__restrict__ row_ptr,
                                   const int32_t *__restrict__ perm, const int64_t *__restrict__ cptr, int64_t n_dst,
                                   int64_t n_loc, int d, float *__restrict__ dv) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; j < n_loc; j += nw) {
    const int64_t q0 = cptr[j], q1 = cptr[j + 1];
    for (int c0 = 0; c0 < d; c0 += 32) {
      const int c = c0 + lane;
      float acc = 0.f;
      if (j < n_dst && c < d) acc = dagg[j * d + c] / (float)(row_ptr[j + 1] - row_ptr[j] + 1);
      for (int64_t q = q0; q < q1; ++q) {
        const int64_t p = perm[q];
        int64_t lo = 0, hi = n_dst;  // largest i with row_ptr[i] <= p
        while (hi - lo > 1) {
          const int64_t mid = (lo + hi) >> 1;
          if (row_ptr[mid] <= p) lo = mid; else hi = mid;
        }
        if (c < d) acc += dagg[lo * d + c] / (float)(row_ptr[lo + 1] - row_ptr[lo] + 1);
      }
      if (c < d && (q1 > q0 || j < n_dst)) dv[j * d + c] += acc;
    }
  }
}

static int warps_grid(int64_t rows) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(rows, 8), 148 * 16));
}

struct GcnWs {
  float *gh, *dagg, *partial, *cs;
};
static constexpr int kGcnSplits = 32;
static GcnWs carve_gcn(Carver &c, int d_in, int d_out, int64_t n_dst) {
  GcnWs w;
  w.gh = c.take<float>(n_dst * d_out);
  w.dagg = c.take<float>(n_dst * d_in);
  w.partial = c.take<float>((int64_t)kGcnSplits * d_in * d_out);
  w.cs = c.take<float>((int64_t)kColsumChunks * d_out);
  return w;
}

}  // namespace dsmpnn

using namespace dsmpnn;

extern "C" {

dsmpnn_status dsmpnn_gcn_fwd(int32_t d_in, int32_t d_out, int32_t act, const float *W, const float *c,
                             const float *v, const int64_t *row_ptr, const int32_t *col_idx, int64_t n_dst,
                             float *agg, float *out, void *stream) {
  DS_CHECK_ARG(d_in > 0 && d_out > 0 && n_dst >= 0, DSMPNN_ERR_INVALID_ARG, "gcn_fwd: sizes");
  DS_CHECK_ARG(act == DSMPNN_ACT_IDENTITY || act == DSMPNN_ACT_RELU, DSMPNN_ERR_INVALID_ARG, "gcn_fwd: act");
  if (n_dst == 0) return DSMPNN_OK;
  cudaStream_t s = as_stream(stream);
  gcn_mean_kernel<<<warps_grid(n_dst), 256, 0, s>>>(v, row_ptr, col_idx, n_dst, d_in, agg);
  DS_LAUNCH_CHECK();
  // out = act(agg W^T + c):  B(k, n) = W[n][k]
  SgemmArgs g{n_dst, d_out, d_in, agg, d_in, 1, W, 1, d_in, out, d_out, c, act == DSMPNN_ACT_RELU, 0, 1.f};
  return sgemm(g, 1, nullptr, s);
}

dsmpnn_status dsmpnn_gcn_bwd_workspace_size(int32_t d_in, int32_t d_out, int64_t n_dst, size_t *bytes) {
  DS_CHECK_ARG(d_in > 0 && d_out > 0 && n_dst >= 0, DSMPNN_ERR_INVALID_ARG, "gcn_bwd_workspace_size: sizes");
  Carver c(nullptr, 0);
  carve_gcn(c, d_in, d_out, n_dst);
  *bytes = c.used();
  return DSMPNN_OK;
}

dsmpnn_status dsmpnn_gcn_bwd(int32_t d_in, int32_t d_out, int32_t act, const float *W, const int64_t *row_ptr,
                             const int32_t *col_idx, const int32_t *csc_perm, const int64_t *csc_ptr, int64_t n_dst,
                             int64_t n_loc, const float *agg, const float *out, const float *grad_out, float *grad_v,
                             float *grad_W, float *grad_c, void *ws, size_t ws_bytes, void *stream) {
  DS_CHECK_ARG(d_in > 0 && d_out > 0 && n_dst >= 0 && n_loc >= n_dst, DSMPNN_ERR_INVALID_ARG, "gcn_bwd: sizes");
  DS_CHECK_ARG(act == DSMPNN_ACT_IDENTITY || act == DSMPNN_ACT_RELU, DSMPNN_ERR_INVALID_ARG, "gcn_bwd: act");
  if (n_dst == 0) return DSMPNN_OK;
  cudaStream_t s = as_stream(stream);
  Carver cv(ws, ws_bytes);
  GcnWs w = carve_gcn(cv, d_in, d_out, n_dst);
  DS_CHECK_ARG(cv.ok(), DSMPNN_ERR_CAPACITY, "gcn_bwd: workspace too small");
  const int64_t total = n_dst * d_out;
  gcn_ghat_kernel<<<(int)std::min<int64_t>(ceil_div(total, 256), 148 * 8), 256, 0, s>>>(grad_out, out, total, act,
                                                                                        w.gh);
  DS_LAUNCH_CHECK();
  if (grad_c) DS_TRY(colsum_ws(w.gh, n_dst, d_out, d_out, grad_c, 1, w.cs, s));
  if (grad_W) {  // dW += ghat^T agg   (M = d_out, N = d_in, K = rows), split-K in a fixed order
    const int splits = (int)std::max<int64_t>(1, std::min<int64_t>(kGcnSplits, n_dst / 256));
    SgemmArgs g{d_out, d_in, n_dst, w.gh, 1, d_out, agg, d_in, 1, grad_W, d_in, nullptr, 0, 1, 1.f};
    DS_TRY(sgemm(g, splits, w.partial, s));
  }
  if (grad_v) {  // dagg = ghat W, then the transposed mean
    SgemmArgs g{n_dst, d_in, d_out, w.gh, d_out, 1, W, d_in, 1, w.dagg, d_in, nullptr, 0, 0, 1.f};
    DS_TRY(sgemm(g, 1, nullptr, s));
    gcn_scatter_kernel<<<warps_grid(n_loc), 256, 0, s>>>(w.dagg, row_ptr, csc_perm, csc_ptr, n_dst, n_loc, d_in,
                                                         grad_v);
    DS_LAUNCH_CHECK();
  }
  return DSMPNN_OK;
}

}  // extern "C"

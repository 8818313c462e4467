// misc.cu - error text, version, row gathers, edge attributes, halo gather /
// scatter-add, loopback exchange, CSC view.
#include <cub/cub.cuh>
#include <stdarg.h>

#include <vector>

#include "common.cuh"
#include "halo.cuh"

namespace dsmpnn {

static thread_local std::string g_last_error;

bool pdl_enabled() {
  static const bool on = [] {
    const char *e = getenv("DSMPNN_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

void set_error(const char *fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
}

// ---------------------------------------------------------------- gathers --
template <typename T>
__global__ void gather_rows_kernel(const T *__restrict__ in, const int64_t *__restrict__ rows, int64_t n_rows,
                                   int64_t row_elems, T *__restrict__ out) {
  int64_t total = n_rows * row_elems;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = t / row_elems, c = t - r * row_elems;
    out[t] = in[rows[r] * row_elems + c];
  }
}

// fp32 rows -> bf16 rows (round to nearest even): the BF16 mode's layer-0 operand
__global__ void gather_rows_bf16_kernel(const float *__restrict__ in, const int64_t *__restrict__ rows,
                                        int64_t n_rows, int64_t row_elems, __nv_bfloat16 *__restrict__ out) {
  int64_t total = n_rows * row_elems;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = t / row_elems, c = t - r * row_elems;
    out[t] = __float2bfloat16_rn(in[(rows ? rows[r] : r) * row_elems + c]);
  }
}

// ------------------------------------------------------- edge attributes --
// PAPER.md:27 / Alg. 1 :397, reading R21.  One thread per (edge, column).
__global__ void edge_features_kernel(int32_t mode, const float *__restrict__ x, int dim, const float *__restrict__ a,
                                     int n_attr, const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                                     int64_t n_dst, int64_t n_edges, float *__restrict__ e32,
                                     __nv_bfloat16 *__restrict__ e16) {
  int de = (mode == DSMPNN_EDGE_DIFF) ? (dim + n_attr) : 2 * (dim + n_attr);
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n_edges; p += (int64_t)gridDim.x * blockDim.x) {
    // destination row of edge p: binary search in row_ptr
    int64_t lo = 0, hi = n_dst;  // find largest i with row_ptr[i] <= p
    while (hi - lo > 1) {
      int64_t mid = (lo + hi) >> 1;
      if (row_ptr[mid] <= p) lo = mid; else hi = mid;
    }
    int64_t i = lo, j = col[p];
    if (de <= 16) {
      // value k of the edge attribute, k unrolled so everything stays in registers
      float vals[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        float v = 0.f;
        if (mode == DSMPNN_EDGE_DIFF) {
          if (k < dim) v = __fsub_rn(x[i * dim + k], x[j * dim + k]);
          else if (k < dim + n_attr) v = __fsub_rn(a[i * n_attr + (k - dim)], a[j * n_attr + (k - dim)]);
        } else {
          if (k < dim) v = x[i * dim + k];
          else if (k < 2 * dim) v = x[j * dim + (k - dim)];
          else if (k < 2 * dim + n_attr) v = a[i * n_attr + (k - 2 * dim)];
          else if (k < de) v = a[j * n_attr + (k - 2 * dim - n_attr)];
        }
        vals[k] = v;
      }
      if (e32)
#pragma unroll
        for (int k = 0; k < 16; ++k)
          if (k < de) e32[p * de + k] = vals[k];
      if (e16) {
        uint32_t w[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          __nv_bfloat162 h = __floats2bfloat162_rn(vals[2 * k], vals[2 * k + 1]);
          w[k] = *reinterpret_cast<uint32_t *>(&h);
        }
        uint4 *o = reinterpret_cast<uint4 *>(e16 + p * 16);
        o[0] = make_uint4(w[0], w[1], w[2], w[3]);
        o[1] = make_uint4(w[4], w[5], w[6], w[7]);
      }
      continue;
    }
    float vals[32];
    int c = 0;
    if (mode == DSMPNN_EDGE_DIFF) {
      for (int d = 0; d < dim; ++d) vals[c++] = __fsub_rn(x[i * dim + d], x[j * dim + d]);
      for (int d = 0; d < n_attr; ++d) vals[c++] = __fsub_rn(a[i * n_attr + d], a[j * n_attr + d]);
    } else {
      for (int d = 0; d < dim; ++d) vals[c++] = x[i * dim + d];
      for (int d = 0; d < dim; ++d) vals[c++] = x[j * dim + d];
      for (int d = 0; d < n_attr; ++d) vals[c++] = a[i * n_attr + d];
      for (int d = 0; d < n_attr; ++d) vals[c++] = a[j * n_attr + d];
    }
    if (e32)
      for (int d = 0; d < de; ++d) e32[p * de + d] = vals[d];
  }
}

// ------------------------------------------------------------------ halo --
template <typename T>
__global__ void halo_gather_kernel(const T *__restrict__ v, const int32_t *__restrict__ rows, int64_t n_rows,
                                   int width, T *__restrict__ out) {
  pdl_wait();
  pdl_trigger();
  int64_t total = n_rows * width;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = t / width, c = t - r * width;
    out[t] = v[(int64_t)rows[r] * width + c];
  }
}

__global__ void halo_scatter_add_kernel(const float *__restrict__ in, const int32_t *__restrict__ rows,
                                        int64_t n_rows, int width, float *__restrict__ v) {
  // rows within one call are distinct (a send list), so plain read-modify-write is race free
  int64_t total = n_rows * width;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = t / width, c = t - r * width;
    float *dst = v + (int64_t)rows[r] * width + c;
    *dst = __fadd_rn(*dst, in[t]);
  }
}

// ------------------------------------------------------------ f4 reassembly --
__global__ void reassemble_acc_kernel(const float *__restrict__ pred, const int64_t *__restrict__ gid, int64_t n,
                                      int width, float *__restrict__ sum, int32_t *__restrict__ count) {
  // gids within one call are distinct: plain read-modify-write is race free
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n * width; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = t / width, c = t - k * width, g = gid[k];
    sum[g * width + c] = __fadd_rn(sum[g * width + c], pred[t]);
    if (c == 0) count[g] += 1;
  }
}
__global__ void reassemble_fin_kernel(const float *__restrict__ sum, const int32_t *__restrict__ count,
                                      int64_t n_points, int width, float *__restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n_points * width;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int32_t c = count[t / width];
    out[t] = c > 0 ? __fdiv_rn(sum[t], (float)c) : 0.f;
  }
}

// ------------------------------------------------------------------- CSC --
__global__ void iota_i32(int32_t *o, int64_t n) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    o[t] = (int32_t)t;
}
// csc_ptr[j] = first position in sorted keys with key >= j (lower bound)
__global__ void csc_ptr_kernel(const int32_t *__restrict__ sorted_col, int64_t n_edges, int64_t n_loc,
                               int64_t *__restrict__ ptr) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j <= n_loc; j += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = n_edges;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (sorted_col[mid] < j) lo = mid + 1; else hi = mid;
    }
    ptr[j] = lo;
  }
}

// ---------------------------------------------------------------- probe --
struct Probe {
  int id = 0;
  int cap = 0;
  int n = 0;
  std::vector<cudaEvent_t> ev;  // 2 per launch
};
static Probe g_probe;

bool probe_armed(int id) { return g_probe.id == id && id != 0 && g_probe.n < g_probe.cap; }
void probe_before(int id, cudaStream_t s) { cudaEventRecord(g_probe.ev[2 * g_probe.n], s); }
void probe_after(int id, cudaStream_t s) {
  cudaEventRecord(g_probe.ev[2 * g_probe.n + 1], s);
  g_probe.n++;
}

static int grid_for(int64_t n, int block = 256) {
  int64_t g = ceil_div(n, block);
  if (g < 1) g = 1;
  if (g > 148 * 16) g = 148 * 16;
  return (int)g;
}

}  // namespace dsmpnn

using namespace dsmpnn;

extern "C" {

const char *dsmpnn_last_error(void) { return g_last_error.c_str(); }
int32_t dsmpnn_version(void) { return 1; }

dsmpnn_status dsmpnn_probe_begin(int32_t kernel_id, int32_t max_launches) {
  DS_CHECK_ARG(max_launches >= 0 && max_launches <= 1 << 20, DSMPNN_ERR_INVALID_ARG, "probe: max_launches");
  while ((int)g_probe.ev.size() < 2 * max_launches) {
    cudaEvent_t e;
    DS_CUDA(cudaEventCreate(&e));
    g_probe.ev.push_back(e);
  }
  g_probe.id = kernel_id;
  g_probe.cap = max_launches;
  g_probe.n = 0;
  return DSMPNN_OK;
}

dsmpnn_status dsmpnn_probe_end(float *total_ms, int64_t *launches) {
  double tot = 0.0;
  for (int i = 0; i < g_probe.n; ++i) {
    DS_CUDA(cudaEventSynchronize(g_probe.ev[2 * i + 1]));
    float ms = 0.f;
    DS_CUDA(cudaEventElapsedTime(&ms, g_probe.ev[2 * i], g_probe.ev[2 * i + 1]));
    tot += ms;
  }
  if (total_ms) *total_ms = (float)tot;
  if (launches) *launches = g_probe.n;
  g_probe.id = 0;
  g_probe.n = 0;
  return DSMPNN_OK;
}

dsmpnn_status dsmpnn_gather_rows(const void *in, const int64_t *rows, int64_t n_rows, int64_t row_elems,
                                 int32_t elem_bytes, void *out, void *stream) {
  DS_CHECK_ARG(n_rows >= 0 && row_elems >= 0, DSMPNN_ERR_INVALID_ARG, "gather_rows: negative size");
  if (n_rows == 0 || row_elems == 0) return DSMPNN_OK;
  cudaStream_t s = as_stream(stream);
  int g = grid_for(n_rows * row_elems);
  if (elem_bytes == 4)
    gather_rows_kernel<uint32_t><<<g, 256, 0, s>>>((const uint32_t *)in, rows, n_rows, row_elems, (uint32_t *)out);
  else if (elem_bytes == 8)
    gather_rows_kernel<uint64_t><<<g, 256, 0, s>>>((const uint64_t *)in, rows, n_rows, row_elems, (uint64_t *)out);
  else if (elem_bytes == 2)
    gather_rows_kernel<uint16_t><<<g, 256, 0, s>>>((const uint16_t *)in, rows, n_rows, row_elems, (uint16_t *)out);
  else
    DS_CHECK_ARG(false, DSMPNN_ERR_INVALID_ARG, "gather_rows: elem_bytes must be 2, 4 or 8");
  DS_LAUNCH_CHECK();
  return DSMPNN_OK;
}

dsmpnn_status dsmpnn_gather_rows_bf16(const float *in, const int64_t *rows, int64_t n_rows, int64_t row_elems,
                                      void *out, void *stream) {
  DS_CHECK_ARG(n_rows >= 0 && row_elems >= 0, DSMPNN_ERR_INVALID_ARG, "gather_rows_bf16: negative size");
  if (n_rows == 0 || row_elems == 0) return DSMPNN_OK;
  gather_rows_bf16_kernel<<<grid_for(n_rows * row_elems), 256, 0, as_stream(stream)>>>(in, rows, n_rows, row_elems,
                                                                                     (__nv_bfloat16 *)out);
  DS_LAUNCH_CHECK();
  return DSMPNN_OK;
}

dsmpnn_status dsmpnn_edge_features(int32_t mode, const float *coords, int dim, const float *attr, int n_attr,
                                   const int64_t *row_ptr, const int32_t *col_idx, int64_t n_dst,
                                   int64_t n_edges, float *e32, void *e16, void *stream) {
  DS_CHECK_ARG(mode == DSMPNN_EDGE_DIFF || mode == DSMPNN_EDGE_CONCAT, DSMPNN_ERR_INVALID_ARG, "edge_features: mode");
  DS_CHECK_ARG(dim == 2 || dim == 3, DSMPNN_ERR_INVALID_ARG, "edge_features: dim must be 2 or 3");
  DS_CHECK_ARG(n_attr >= 0 && n_attr <= 6, DSMPNN_ERR_INVALID_ARG, "edge_features: n_attr in [0,6]");
  int de = (mode == DSMPNN_EDGE_DIFF) ? (dim + n_attr) : 2 * (dim + n_attr);
  DS_CHECK_ARG(!e16 || de <= 16, DSMPNN_ERR_SHAPE, "edge_features: d_e=%d > 16 for bf16 output", de);
  if (n_edges <= 0) return DSMPNN_OK;
  edge_features_kernel<<<grid_for(n_edges), 256, 0, as_stream(stream)>>>(
      mode, coords, dim, attr, n_attr, row_ptr, col_idx, n_dst, n_edges, e32, (__nv_bfloat16 *)e16);
  DS_LAUNCH_CHECK();
  return DSMPNN_OK;
}

dsmpnn_status dsmpnn_halo_gather(const void *values, const int32_t *rows, int64_t n_rows, int32_t width,
                                 int32_t dtype, void *out, void *stream) {
  DS_CHECK_ARG(width > 0 && n_rows >= 0, DSMPNN_ERR_INVALID_ARG, "halo_gather: bad size");
  if (n_rows == 0) return DSMPNN_OK;
  cudaStream_t s = as_stream(stream);
  int g = grid_for(n_rows * width);
  if (dtype == DSMPNN_F32)
    DS_CUDA(launch_pdl(halo_gather_kernel<float>, g, 256, 0, s, (const float *)values, rows, n_rows, width, (float *)out));
  else if (dtype == DSMPNN_BF16)
    DS_CUDA(launch_pdl(halo_gather_kernel<uint16_t>, g, 256, 0, s, (const uint16_t *)values, rows, n_rows, width, (uint16_t *)out));
  else
    DS_CHECK_ARG(false, DSMPNN_ERR_INVALID_ARG, "halo_gather: dtype");
  DS_LAUNCH_CHECK();
  return DSMPNN_OK;
}

__global__ void accumulate_f32_kernel(float *__restrict__ dst, const float *__restrict__ src, int64_t n) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    dst[t] += src[t];
}

dsmpnn_status dsmpnn_accumulate_f32(float *dst, const float *src, int64_t n, void *stream) {
  DS_CHECK_ARG(n >= 0, DSMPNN_ERR_INVALID_ARG, "accumulate_f32: n < 0");
  if (n == 0) return DSMPNN_OK;
  accumulate_f32_kernel<<<grid_for(n), 256, 0, as_stream(stream)>>>(dst, src, n);
  DS_LAUNCH_CHECK();
  return DSMPNN_OK;
}

dsmpnn_status dsmpnn_halo_scatter_add(const float *in, const int32_t *rows, int64_t n_rows, int32_t width,
                                      float *values, void *stream) {
  DS_CHECK_ARG(width > 0 && n_rows >= 0, DSMPNN_ERR_INVALID_ARG, "halo_scatter_add: bad size");
  if (n_rows == 0) return DSMPNN_OK;
  halo_scatter_add_kernel<<<grid_for(n_rows * width), 256, 0, as_stream(stream)>>>(in, rows, n_rows, width, values);
  DS_LAUNCH_CHECK();
  return DSMPNN_OK;
}

dsmpnn_status dsmpnn_halo_exchange_loopback(int32_t nparts, void *const *values, const int64_t *const *halo_ptr,
                                            const int64_t *const *send_ptr, const int32_t *const *send_idx,
                                            int32_t width, int32_t dtype, void *stream) {
  DS_CHECK_ARG(nparts >= 1, DSMPNN_ERR_INVALID_ARG, "halo_exchange_loopback: nparts");
  size_t esz = dtype == DSMPNN_BF16 ? 2 : 4;
  // rows of whole 16-byte chunks: every copy of the refresh in one launch
  if ((width * esz) % 16 == 0) {
    HaloJobs jobs;
    int nj = 0;
    int64_t most = 0;
    bool fits = true;
    for (int q = 0; q < nparts && fits; ++q)
      for (int p = 0; p < nparts; ++p) {
        if (p == q) continue;
        int64_t a = halo_ptr[q][p], b = halo_ptr[q][p + 1];
        int64_t s0 = send_ptr[p][q], s1 = send_ptr[p][q + 1];
        DS_CHECK_ARG(b - a == s1 - s0, DSMPNN_ERR_SHAPE, "halo_exchange_loopback: %d->%d sizes differ", p, q);
        if (b == a) continue;
        if (nj == HaloJobs::kMax) { fits = false; break; }
        const char *srcp = (const char *)values[p];
        char *dstp = (char *)values[q] + (size_t)a * width * esz;
        if (((uintptr_t)srcp & 15) || ((uintptr_t)dstp & 15)) { fits = false; break; }
        jobs.src[nj] = reinterpret_cast<const uint4 *>(srcp);
        jobs.rows[nj] = send_idx[p] + s0;
        jobs.dst[nj] = reinterpret_cast<uint4 *>(dstp);
        jobs.n_rows[nj] = b - a;
        most = std::max(most, b - a);
        ++nj;
      }
    if (fits) {
      if (nj == 0) return DSMPNN_OK;
      const int row16 = (int)(width * esz / 16);
      const int gx = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(most * row16, 256), 64));
      halo_gather_jobs_kernel<<<dim3(gx, nj), 256, 0, as_stream(stream)>>>(jobs, row16);
      DS_LAUNCH_CHECK();
      return DSMPNN_OK;
    }
  }
  for (int q = 0; q < nparts; ++q)
    for (int p = 0; p < nparts; ++p) {
      if (p == q) continue;
      int64_t a = halo_ptr[q][p], b = halo_ptr[q][p + 1];
      int64_t s0 = send_ptr[p][q], s1 = send_ptr[p][q + 1];
      DS_CHECK_ARG(b - a == s1 - s0, DSMPNN_ERR_SHAPE, "halo_exchange_loopback: %d->%d sizes differ", p, q);
      if (b == a) continue;
      char *dst = (char *)values[q] + (size_t)a * width * esz;
      DS_TRY(dsmpnn_halo_gather(values[p], send_idx[p] + s0, b - a, width, dtype, dst, stream));
    }
  return DSMPNN_OK;
}

dsmpnn_status dsmpnn_halo_reverse_add_loopback(int32_t nparts, float *const *values, const int64_t *const *halo_ptr,
                                               const int64_t *const *send_ptr, const int32_t *const *send_idx,
                                               int32_t width, void *stream) {
  DS_CHECK_ARG(nparts >= 1 && width > 0, DSMPNN_ERR_INVALID_ARG, "halo_reverse_add_loopback: nparts / width");
  for (int p = 0; p < nparts; ++p)
    for (int q = 0; q < nparts; ++q) {
      if (q == p) continue;
      int64_t s0 = send_ptr[p][q], s1 = send_ptr[p][q + 1];
      int64_t a = halo_ptr[q][p], b = halo_ptr[q][p + 1];
      DS_CHECK_ARG(b - a == s1 - s0, DSMPNN_ERR_SHAPE, "halo_reverse_add_loopback: %d<-%d sizes differ", p, q);
      if (b == a) continue;
      DS_TRY(dsmpnn_halo_scatter_add(values[q] + a * width, send_idx[p] + s0, b - a, width, values[p], stream));
    }
  return DSMPNN_OK;
}

dsmpnn_status dsmpnn_reassemble_accumulate(const float *pred, const int64_t *gid, int64_t n, int32_t width,
                                           float *sum, int32_t *count, void *stream) {
  DS_CHECK_ARG(n >= 0 && width > 0, DSMPNN_ERR_INVALID_ARG, "reassemble_accumulate: sizes");
  if (n == 0) return DSMPNN_OK;
  reassemble_acc_kernel<<<grid_for(n * width), 256, 0, as_stream(stream)>>>(pred, gid, n, width, sum, count);
  DS_LAUNCH_CHECK();
  return DSMPNN_OK;
}

dsmpnn_status dsmpnn_reassemble_finalize(const float *sum, const int32_t *count, int64_t n_points, int32_t width,
                                         float *out, void *stream) {
  DS_CHECK_ARG(n_points >= 0 && width > 0, DSMPNN_ERR_INVALID_ARG, "reassemble_finalize: sizes");
  if (n_points == 0) return DSMPNN_OK;
  reassemble_fin_kernel<<<grid_for(n_points * width), 256, 0, as_stream(stream)>>>(sum, count, n_points, width, out);
  DS_LAUNCH_CHECK();
  return DSMPNN_OK;
}

dsmpnn_status dsmpnn_csc_workspace_size(int64_t n_edges, int64_t n_loc, size_t *bytes) {
  size_t tmp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp, (const int32_t *)nullptr, (int32_t *)nullptr,
                                  (const int32_t *)nullptr, (int32_t *)nullptr, (int)n_edges);
  Carver c(nullptr, 0);
  c.take<int32_t>(n_edges);  // iota
  c.take<int32_t>(n_edges);  // sorted keys
  c.take<char>(tmp);
  *bytes = c.used();
  return DSMPNN_OK;
}

dsmpnn_status dsmpnn_csc(const int32_t *col_idx, int64_t n_edges, int64_t n_loc, int32_t *csc_perm,
                         int64_t *csc_ptr, void *ws, size_t ws_bytes, void *stream) {
  DS_CHECK_ARG(n_edges >= 0 && n_loc >= 0 && n_edges < (1ll << 31), DSMPNN_ERR_INVALID_ARG, "csc: sizes");
  cudaStream_t s = as_stream(stream);
  size_t tmp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp, (const int32_t *)nullptr, (int32_t *)nullptr,
                                  (const int32_t *)nullptr, (int32_t *)nullptr, (int)n_edges);
  Carver c(ws, ws_bytes);
  int32_t *iota = c.take<int32_t>(n_edges);
  int32_t *keys = c.take<int32_t>(n_edges);
  void *t = c.take<char>(tmp);
  DS_CHECK_ARG(c.ok(), DSMPNN_ERR_CAPACITY, "csc: workspace too small");
  if (n_edges > 0) {
    iota_i32<<<grid_for(n_edges), 256, 0, s>>>(iota, n_edges);
    int end_bit = 1;
    while ((1ll << end_bit) <= n_loc) ++end_bit;
    DS_CUDA(cub::DeviceRadixSort::SortPairs(t, tmp, col_idx, keys, iota, csc_perm, (int)n_edges, 0, end_bit, s));
  }
  csc_ptr_kernel<<<grid_for(n_loc + 1), 256, 0, s>>>(keys, n_edges, n_loc, csc_ptr);
  DS_LAUNCH_CHECK();
  return DSMPNN_OK;
}

}  // extern "C"

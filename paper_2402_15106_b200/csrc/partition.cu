// partition.cu - a3 domain decomposition with overlap l (
// Alg. 1 :392, :403; readings R12, R13, R23).
//
// Median RCB level by level: per-part bounding boxes (exact min/max via
// ordered-int atomics), longest axis per part, one radix sort of
// (part, orderable x[a*]) keys to read the lower median c* of every part,
// then every point moves to child 2*part + (x > c*).  After log2(P) levels the
// part index is the owner (the first split is the most significant bit, which
// matches RCB(lower, p0, P/2), RCB(upper, p0 + P/2, P/2)).
// The plan of one rank is then a classification (deep / near / halo / other)
// followed by a radix sort on (class, owner, gid), and the send lists a sort on
// (destination rank, gid) over owned points that fall in other ranks'
// extended boxes.
#include <cub/cub.cuh>

#include "common.cuh"

namespace dsmpnn {

constexpr int kMaxParts = 64;

__device__ __forceinline__ uint32_t f2ord(float v) {
  uint32_t u = __float_as_uint(__fadd_rn(v, 0.0f));  // -0 -> +0
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ord2f(uint32_t o) {
  uint32_t u = (o & 0x80000000u) ? (o & 0x7fffffffu) : ~o;
  return __uint_as_float(u);
}

struct PartState {
  unsigned int lo_ord[kMaxParts][3];  // per-part bbox (ordered ints), current level
  unsigned int hi_ord[kMaxParts][3];
  int count[kMaxParts];
  int upper[kMaxParts];
  int axis[kMaxParts];
  float cut[kMaxParts];
  float box_lo[kMaxParts][3], box_hi[kMaxParts][3];
  unsigned char in_lo[kMaxParts][3], in_hi[kMaxParts][3];
  int degenerate;
  // plan counters for one rank
  int cls_count[4];
  int halo_count[kMaxParts];
  int send_count[kMaxParts];
};

__global__ void part_init_kernel(PartState *st, int nparts_cur) {
  int t = threadIdx.x;
  if (t < kMaxParts) {
    for (int d = 0; d < 3; ++d) { st->lo_ord[t][d] = 0xffffffffu; st->hi_ord[t][d] = 0u; }
    st->count[t] = 0;
    st->upper[t] = 0;
  }
}

__global__ void part_bbox_kernel(const float *__restrict__ x, int64_t n, int dim, const int32_t *__restrict__ part,
                                 int nparts_cur, PartState *st) {
  __shared__ unsigned int slo[kMaxParts][3], shi[kMaxParts][3];
  __shared__ int scnt[kMaxParts];
  for (int t = threadIdx.x; t < nparts_cur; t += blockDim.x) {
    for (int d = 0; d < 3; ++d) { slo[t][d] = 0xffffffffu; shi[t][d] = 0u; }
    scnt[t] = 0;
  }
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int p = part[i];
    atomicAdd(&scnt[p], 1);
    for (int d = 0; d < dim; ++d) {
      uint32_t o = f2ord(x[i * dim + d]);
      atomicMin(&slo[p][d], o);
      atomicMax(&shi[p][d], o);
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < nparts_cur; t += blockDim.x) {
    if (scnt[t] == 0) continue;
    atomicAdd(&st->count[t], scnt[t]);
    for (int d = 0; d < dim; ++d) {
      atomicMin(&st->lo_ord[t][d], slo[t][d]);
      atomicMax(&st->hi_ord[t][d], shi[t][d]);
    }
  }
}

// level 0 only: the root box is the fp32 bounding box of all points
__global__ void root_box_kernel(PartState *st, int dim) {
  for (int d = 0; d < 3; ++d) {
    st->box_lo[0][d] = d < dim ? ord2f(st->lo_ord[0][d]) : 0.f;
    st->box_hi[0][d] = d < dim ? ord2f(st->hi_ord[0][d]) : 0.f;
    st->in_lo[0][d] = 0;
    st->in_hi[0][d] = 0;
  }
  st->degenerate = 0;
}

__global__ void part_axis_kernel(PartState *st, int nparts_cur, int dim) {
  int p = threadIdx.x;
  if (p >= nparts_cur) return;
  int best = 0;
  float bext = -INFINITY;
  for (int d = 0; d < dim; ++d) {
    float ext = __fsub_rn(ord2f(st->hi_ord[p][d]), ord2f(st->lo_ord[p][d]));
    if (ext > bext) { bext = ext; best = d; }  // first maximum
  }
  st->axis[p] = best;
}

__global__ void part_key_kernel(const float *__restrict__ x, int64_t n, int dim, const int32_t *__restrict__ part,
                                const PartState *st, uint64_t *__restrict__ keys) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int p = part[i];
    keys[i] = ((uint64_t)p << 32) | f2ord(x[i * dim + st->axis[p]]);
  }
}

// c*(p) = x[a*] of the ceil(|S_p|/2)-th element of part p in sorted order
__global__ void part_cut_kernel(const uint64_t *__restrict__ sorted, PartState *st, int nparts_cur) {
  if (threadIdx.x != 0) return;
  int64_t off = 0;
  for (int p = 0; p < nparts_cur; ++p) {
    int c = st->count[p];
    int m = (c + 1) / 2;
    st->cut[p] = c > 0 ? ord2f((uint32_t)(sorted[off + m - 1] & 0xffffffffu)) : 0.f;
    if (c == 0) st->degenerate = 1;
    off += c;
  }
}

__global__ void part_split_kernel(const float *__restrict__ x, int64_t n, int dim, int32_t *__restrict__ part,
                                  PartState *st) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int p = part[i];
    float v = __fadd_rn(x[i * dim + st->axis[p]], 0.0f);
    int up = v > st->cut[p] ? 1 : 0;
    if (up) atomicAdd(&st->upper[p], 1);
    part[i] = 2 * p + up;
  }
}

// children boxes: lower child (2p) gets hi[a*] = c*, upper child (2p+1) lo[a*] = c*
__global__ void part_boxes_kernel(PartState *st, int nparts_cur) {
  if (threadIdx.x != 0) return;
  float lo[kMaxParts][3], hi[kMaxParts][3];
  unsigned char il[kMaxParts][3], ih[kMaxParts][3];
  for (int p = 0; p < nparts_cur; ++p)
    for (int d = 0; d < 3; ++d) {
      lo[p][d] = st->box_lo[p][d]; hi[p][d] = st->box_hi[p][d];
      il[p][d] = st->in_lo[p][d]; ih[p][d] = st->in_hi[p][d];
    }
  for (int p = 0; p < nparts_cur; ++p) {
    if (st->upper[p] == 0) st->degenerate = 1;
    int a = st->axis[p];
    float c = st->cut[p];
    for (int d = 0; d < 3; ++d) {
      st->box_lo[2 * p][d] = lo[p][d]; st->box_hi[2 * p][d] = hi[p][d];
      st->box_lo[2 * p + 1][d] = lo[p][d]; st->box_hi[2 * p + 1][d] = hi[p][d];
      st->in_lo[2 * p][d] = il[p][d]; st->in_hi[2 * p][d] = ih[p][d];
      st->in_lo[2 * p + 1][d] = il[p][d]; st->in_hi[2 * p + 1][d] = ih[p][d];
    }
    st->box_hi[2 * p][a] = c;
    st->in_hi[2 * p][a] = 1;
    st->box_lo[2 * p + 1][a] = c;
    st->in_lo[2 * p + 1][a] = 1;
  }
}

__global__ void part_out_boxes_kernel(const PartState *st, int nparts, int dim, float *boxes, uint8_t *internal) {
  int p = threadIdx.x;
  if (p >= nparts) return;
  for (int d = 0; d < dim; ++d) {
    boxes[(p * 2 + 0) * dim + d] = st->box_lo[p][d];
    boxes[(p * 2 + 1) * dim + d] = st->box_hi[p][d];
    internal[(p * 2 + 0) * dim + d] = st->in_lo[p][d];
    internal[(p * 2 + 1) * dim + d] = st->in_hi[p][d];
  }
}

__global__ void plan_reset_kernel(PartState *st) {
  int t = threadIdx.x;
  if (t < 4) st->cls_count[t] = 0;
  if (t < kMaxParts) { st->halo_count[t] = 0; st->send_count[t] = 0; }
}

__device__ __forceinline__ bool in_ext_box(const float *xj, int dim, const PartState *st, int q, float l) {
  for (int d = 0; d < dim; ++d) {
    float lo = __fsub_rn(st->box_lo[q][d], l), hi = __fadd_rn(st->box_hi[q][d], l);
    if (!(xj[d] >= lo && xj[d] <= hi)) return false;
  }
  return true;
}

// key = class<<(gb+7) | owner<<gb (halo only) | gid ; class 0 deep, 1 near, 2
// halo, 3 other.  gb = 52 without a gid bound (gid < 2^52), else the bound.
__global__ void plan_classify_kernel(const float *__restrict__ x, const int64_t *__restrict__ gid, int64_t n, int dim,
                                     const int32_t *__restrict__ owner, PartState *st, int q, float l, float t,
                                     int gb, uint64_t *__restrict__ keys, int32_t *__restrict__ vals) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    float xj[3] = {0.f, 0.f, 0.f};
    for (int d = 0; d < dim; ++d) xj[d] = x[j * dim + d];
    int o = owner[j];
    uint64_t cls;
    if (o == q) {
      bool near = false;
      for (int d = 0; d < dim; ++d) {
        if (st->in_lo[q][d] && xj[d] <= __fadd_rn(st->box_lo[q][d], t)) near = true;
        if (st->in_hi[q][d] && xj[d] >= __fsub_rn(st->box_hi[q][d], t)) near = true;
      }
      cls = near ? 1 : 0;
    } else if (in_ext_box(xj, dim, st, q, l)) {
      cls = 2;
      atomicAdd(&st->halo_count[o], 1);
    } else {
      cls = 3;
    }
    atomicAdd(&st->cls_count[cls], 1);
    keys[j] = (cls << (gb + 7)) | (cls == 2 ? ((uint64_t)o << gb) : 0) | (uint64_t)gid[j];
    vals[j] = (int32_t)j;
  }
}

__global__ void plan_local_kernel(const int32_t *__restrict__ sorted_vals, int64_t n, const PartState *st,
                                  int64_t *__restrict__ local_rows, int32_t *__restrict__ pos) {
  int64_t n_loc = st->cls_count[0] + st->cls_count[1] + st->cls_count[2];
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    int32_t j = sorted_vals[k];
    if (k < n_loc) { local_rows[k] = j; pos[j] = (int32_t)k; }
    else pos[j] = -1;
  }
}

// candidate (q', gid) keys for owned points in other ranks' extended boxes
__global__ void plan_send_kernel(const float *__restrict__ x, const int64_t *__restrict__ gid, int64_t n, int dim,
                                 const int32_t *__restrict__ owner, const int32_t *__restrict__ pos, PartState *st,
                                 int q, int nparts, float l, int gb, uint64_t *__restrict__ keys,
                                 int32_t *__restrict__ vals) {
  int64_t total = n * nparts;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t j = t / nparts;
    int qq = (int)(t - j * nparts);
    uint64_t key = ~0ull;
    int32_t v = -1;
    if (owner[j] == q && qq != q) {
      float xj[3] = {0.f, 0.f, 0.f};
      for (int d = 0; d < dim; ++d) xj[d] = x[j * dim + d];
      if (in_ext_box(xj, dim, st, qq, l)) {
        key = ((uint64_t)qq << gb) | (uint64_t)gid[j];
        v = pos[j];
        atomicAdd(&st->send_count[qq], 1);
      }
    }
    keys[t] = key;
    vals[t] = v;
  }
}

__global__ void plan_counts_kernel(const PartState *st, int nparts, int q, int64_t *counts) {
  if (threadIdx.x != 0) return;
  int64_t nd = st->cls_count[0], nn = st->cls_count[1], nh = st->cls_count[2];
  int64_t ns = 0;
  for (int p = 0; p < nparts; ++p) ns += st->send_count[p];
  counts[0] = nd; counts[1] = nn; counts[2] = nh; counts[3] = ns;
  int64_t *halo_ptr = counts + 4, *send_ptr = counts + 4 + nparts + 1;
  halo_ptr[0] = nd + nn;
  send_ptr[0] = 0;
  for (int p = 0; p < nparts; ++p) {
    halo_ptr[p + 1] = halo_ptr[p] + (p == q ? 0 : st->halo_count[p]);
    send_ptr[p + 1] = send_ptr[p] + st->send_count[p];
  }
  counts[4 + 2 * (nparts + 1)] = st->degenerate;  // extra slot (workspace copy only)
}

__global__ void copy_send_kernel(const int32_t *__restrict__ sorted_vals, const int64_t *__restrict__ counts,
                                 int32_t *__restrict__ send_idx) {
  int64_t ns = counts[3];
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < ns; k += (int64_t)gridDim.x * blockDim.x)
    send_idx[k] = sorted_vals[k];
}

static size_t partition_ws(int64_t n, int nparts, size_t *sort1, size_t *sort2) {
  cub::DeviceRadixSort::SortKeys(nullptr, *sort1, (const uint64_t *)nullptr, (uint64_t *)nullptr, (int)n);
  cub::DeviceRadixSort::SortPairs(nullptr, *sort2, (const uint64_t *)nullptr, (uint64_t *)nullptr,
                                  (const int32_t *)nullptr, (int32_t *)nullptr, (int)(n * nparts));
  Carver c(nullptr, 0);
  c.take<PartState>(1);
  c.take<int32_t>(n);                 // part
  c.take<uint64_t>(n * nparts);       // keys
  c.take<uint64_t>(n * nparts);       // keys sorted
  c.take<int32_t>(n * nparts);        // vals
  c.take<int32_t>(n * nparts);        // vals sorted
  c.take<int32_t>(n);                 // pos
  c.take<int64_t>(8 + 2 * (kMaxParts + 1));
  c.take<char>(std::max(*sort1, *sort2));
  return c.used();
}

}  // namespace dsmpnn

using namespace dsmpnn;

extern "C" {

dsmpnn_status dsmpnn_partition_workspace_size(int64_t n, int dim, int nparts, size_t *bytes) {
  DS_CHECK_ARG(n >= 1 && nparts >= 1 && nparts <= kMaxParts && n * nparts < (1ll << 31), DSMPNN_ERR_INVALID_ARG,
               "partition: sizes");
  size_t a, b;
  *bytes = partition_ws(n, nparts, &a, &b);
  return DSMPNN_OK;
}

}  // extern "C"

namespace dsmpnn {

struct PartWs {
  PartState *st;
  int32_t *part, *vals, *vals2, *pos;
  uint64_t *keys, *keys2;
  int64_t *cnt_ws;
  void *tmp;
  size_t tmp_bytes;
};

static dsmpnn_status carve_part(int64_t n, int nparts, void *ws, size_t ws_bytes, PartWs &w) {
  size_t sort1, sort2;
  size_t need = partition_ws(n, nparts, &sort1, &sort2);
  DS_CHECK_ARG(ws_bytes >= need, DSMPNN_ERR_CAPACITY, "partition: workspace %zu < %zu", ws_bytes, need);
  Carver c(ws, ws_bytes);
  w.st = c.take<PartState>(1);
  w.part = c.take<int32_t>(n);
  w.keys = c.take<uint64_t>(n * nparts);
  w.keys2 = c.take<uint64_t>(n * nparts);
  w.vals = c.take<int32_t>(n * nparts);
  w.vals2 = c.take<int32_t>(n * nparts);
  w.pos = c.take<int32_t>(n);
  w.cnt_ws = c.take<int64_t>(8 + 2 * (kMaxParts + 1));
  w.tmp_bytes = std::max(sort1, sort2);
  w.tmp = c.take<char>(w.tmp_bytes);
  return DSMPNN_OK;
}

static dsmpnn_status check_part_args(int64_t n, int dim, int nparts, float overlap_l, float radius) {
  DS_CHECK_ARG(dim == 2 || dim == 3, DSMPNN_ERR_INVALID_ARG, "partition: dim must be 2 or 3");
  DS_CHECK_ARG(nparts >= 1 && (nparts & (nparts - 1)) == 0 && nparts <= kMaxParts && nparts <= n,
               DSMPNN_ERR_INVALID_ARG, "partition: nparts must be a power of two <= min(n, %d)", kMaxParts);
  DS_CHECK_ARG(overlap_l >= 0.f && radius > 0.f, DSMPNN_ERR_INVALID_ARG, "partition: need l >= 0 and r > 0");
  DS_CHECK_ARG(n * nparts < (1ll << 31), DSMPNN_ERR_INVALID_ARG, "partition: n*P too large");
  return DSMPNN_OK;
}

// recursive coordinate bisection (R12): owner, boxes, internal faces
static dsmpnn_status run_rcb(const float *coords, int64_t n, int dim, int nparts, const PartWs &w, int32_t *owner,
                             float *boxes, uint8_t *internal, cudaStream_t s) {
  const int g = (int)std::min<int64_t>(ceil_div(n, 256), 148 * 4);
  DS_CUDA(cudaMemsetAsync(w.part, 0, n * sizeof(int32_t), s));
  int levels = 0;
  while ((1 << levels) < nparts) ++levels;
  for (int L = 0; L <= levels; ++L) {
    int cur = 1 << L;
    part_init_kernel<<<1, kMaxParts, 0, s>>>(w.st, cur);
    part_bbox_kernel<<<g, 256, 0, s>>>(coords, n, dim, w.part, cur, w.st);
    if (L == 0) root_box_kernel<<<1, 1, 0, s>>>(w.st, dim);
    if (L == levels) break;
    part_axis_kernel<<<1, kMaxParts, 0, s>>>(w.st, cur, dim);
    part_key_kernel<<<g, 256, 0, s>>>(coords, n, dim, w.part, w.st, w.keys);
    size_t tb = w.tmp_bytes;
    DS_CUDA(cub::DeviceRadixSort::SortKeys(w.tmp, tb, w.keys, w.keys2, (int)n, 0, 32 + levels + 1, s));
    part_cut_kernel<<<1, 32, 0, s>>>(w.keys2, w.st, cur);
    part_split_kernel<<<g, 256, 0, s>>>(coords, n, dim, w.part, w.st);
    part_boxes_kernel<<<1, 32, 0, s>>>(w.st, cur);
  }
  DS_CUDA(cudaMemcpyAsync(owner, w.part, n * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
  part_out_boxes_kernel<<<1, kMaxParts, 0, s>>>(w.st, nparts, dim, boxes, internal);
  DS_LAUNCH_CHECK();
  return DSMPNN_OK;
}

// plan of one rank from the RCB state in w (R13, R23); counts gets
// 4 + 2(P+1) entries plus the degenerate flag when with_flag
static dsmpnn_status run_plan(const float *coords, const int64_t *gid, int64_t n, int dim, int nparts,
                              float overlap_l, float radius, int rank, int gid_bits, const PartWs &w,
                              int64_t *local_rows, int64_t *counts, bool with_flag, int32_t *send_idx,
                              cudaStream_t s) {
  const int g = (int)std::min<int64_t>(ceil_div(n, 256), 148 * 4);
  const int gb = (gid_bits >= 1 && gid_bits <= 52) ? gid_bits : 52;  // key fields: gid | owner (7) | class (2)
  float m = overlap_l > radius ? overlap_l : radius;
  float t = m * 1.0009765625f;  // fl(max(l, r) * (1 + 2^-10)), single RNE product
  plan_reset_kernel<<<1, kMaxParts, 0, s>>>(w.st);
  plan_classify_kernel<<<g, 256, 0, s>>>(coords, gid, n, dim, w.part, w.st, rank, overlap_l, t, gb, w.keys, w.vals);
  size_t tb = w.tmp_bytes;
  DS_CUDA(cub::DeviceRadixSort::SortPairs(w.tmp, tb, w.keys, w.keys2, w.vals, w.vals2, (int)n, 0, gb + 9, s));
  plan_local_kernel<<<g, 256, 0, s>>>(w.vals2, n, w.st, local_rows, w.pos);
  int g2 = (int)std::min<int64_t>(ceil_div(n * nparts, 256), 148 * 8);
  plan_send_kernel<<<g2, 256, 0, s>>>(coords, gid, n, dim, w.part, w.pos, w.st, rank, nparts, overlap_l, gb, w.keys,
                                      w.vals);
  tb = w.tmp_bytes;
  DS_CUDA(cub::DeviceRadixSort::SortPairs(w.tmp, tb, w.keys, w.keys2, w.vals, w.vals2, (int)(n * nparts), 0, gb + 7,
                                          s));
  plan_counts_kernel<<<1, 32, 0, s>>>(w.st, nparts, rank, w.cnt_ws);
  const int nc = 4 + 2 * (nparts + 1) + (with_flag ? 1 : 0);
  DS_CUDA(cudaMemcpyAsync(counts, w.cnt_ws, nc * sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
  copy_send_kernel<<<g, 256, 0, s>>>(w.vals2, w.cnt_ws, send_idx);
  DS_LAUNCH_CHECK();
  return DSMPNN_OK;
}

}  // namespace dsmpnn

extern "C" {

dsmpnn_status dsmpnn_partition(const float *coords, const int64_t *gid, int64_t n, int dim, int nparts,
                               float overlap_l, float radius, int rank, int32_t *owner, float *boxes,
                               uint8_t *internal, int64_t *local_rows, int64_t *counts, int32_t *send_idx,
                               int64_t *counts_host, void *ws, size_t ws_bytes, void *stream) {
  DS_TRY(check_part_args(n, dim, nparts, overlap_l, radius));
  DS_CHECK_ARG(rank >= 0 && rank < nparts, DSMPNN_ERR_INVALID_ARG, "partition: rank out of range");
  cudaStream_t s = as_stream(stream);
  PartWs w;
  DS_TRY(carve_part(n, nparts, ws, ws_bytes, w));
  DS_TRY(run_rcb(coords, n, dim, nparts, w, owner, boxes, internal, s));
  DS_TRY(run_plan(coords, gid, n, dim, nparts, overlap_l, radius, rank, 0, w, local_rows, counts, false, send_idx,
                  s));
  if (counts_host) {
    int64_t tmp_host[4 + 2 * (kMaxParts + 1) + 1];
    int nc = 4 + 2 * (nparts + 1) + 1;
    DS_CUDA(cudaMemcpyAsync(tmp_host, w.cnt_ws, nc * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    DS_CUDA(cudaStreamSynchronize(s));
    for (int k = 0; k < nc - 1; ++k) counts_host[k] = tmp_host[k];
    if (tmp_host[nc - 1]) {
      set_error("partition: a split left an empty side (all split coordinates tied)");
      return DSMPNN_ERR_DEGENERATE;
    }
  }
  return DSMPNN_OK;
}

dsmpnn_status dsmpnn_partition_all(const float *coords, const int64_t *gid, int64_t n, int dim, int nparts,
                                   float overlap_l, float radius, int32_t gid_bits, int32_t *owner, float *boxes,
                                   uint8_t *internal, int64_t *local_rows, int64_t *counts, int32_t *send_idx,
                                   void *ws, size_t ws_bytes, void *stream) {
  DS_TRY(check_part_args(n, dim, nparts, overlap_l, radius));
  DS_CHECK_ARG(gid_bits >= 0 && gid_bits <= 63, DSMPNN_ERR_INVALID_ARG, "partition_all: gid_bits in 0..63");
  cudaStream_t s = as_stream(stream);
  PartWs w;
  DS_TRY(carve_part(n, nparts, ws, ws_bytes, w));
  DS_TRY(run_rcb(coords, n, dim, nparts, w, owner, boxes, internal, s));
  const int64_t nc = 5 + 2 * (nparts + 1), cap = n * std::max(1, nparts - 1);
  for (int q = 0; q < nparts; ++q)
    DS_TRY(run_plan(coords, gid, n, dim, nparts, overlap_l, radius, q, gid_bits, w, local_rows + q * n,
                    counts + q * nc, true, send_idx + q * cap, s));
  return DSMPNN_OK;
}

}  // extern "C"

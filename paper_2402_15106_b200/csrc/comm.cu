// comm.cu - a6: the per-layer halo exchange between processes, over NCCL
// point-to-point ("the overlap area of a given domain is updated
// from the neighboring domains' interiors"; Alg. 1 :411 Comm(i_b, Omega,
// v_L)), and the gradient sum (Alg. 1 :418 "sum gradients").
//
// A process holds one or more sub-domains; the plan of each (halo_ptr,
// send_ptr, send_idx from dsmpnn_partition) makes every receive slice a
// contiguous run of halo rows, so a FORWARD exchange is: gather the send rows
// into a staging buffer, ncclSend / ncclRecv straight into the halo rows.
// REVERSE_ADD (reading R16) sends the contiguous halo slices
// back and adds them into the owner's send rows in ascending holder order.
//
// Message matching: NCCL pairs the sends and receives between two ranks in
// issue order.  Every rank walks the same global (source, destination)
// sub-domain order, so the k-th send of rank A to rank B is the k-th receive
// of B from A (dsmpnn_halo_schedule builds this list; it is host-only code,
// testable without a GPU).
//
// Streams: the exchange runs on the context's own comm stream, ordered after
// the caller's stream; the caller's stream waits for it unless
// DSMPNN_HALO_ASYNC is given (then dsmpnn_halo_wait joins it later, which is
// how the deep rows of the next layer overlap the transfer).
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <chrono>
#include <thread>
#include <vector>

#include "common.cuh"
#include "halo.cuh"

#define DS_NCCL(expr)                                                                                  \
  do {                                                                                                 \
    ncclResult_t _r = (expr);                                                                          \
    if (_r != ncclSuccess) {                                                                           \
      ::dsmpnn::set_error("NCCL error %d at %s:%d: %s", (int)_r, __FILE__, __LINE__, ncclGetErrorString(_r)); \
      return DSMPNN_ERR_NCCL;                                                                          \
    }                                                                                                  \
  } while (0)

struct dsmpnn_ctx_s {
  int device = -1, rank = 0, nranks = 1;
  ncclComm_t comm = nullptr;
  cudaStream_t cs = nullptr;      // comm stream
  cudaEvent_t ev_in = nullptr;    // caller's stream -> comm stream
  cudaEvent_t ev_done = nullptr;  // last exchange / all-reduce done
  void *stage = nullptr;
  size_t stage_bytes = 0;
  bool aborted = false;
  std::vector<dsmpnn_halo_op> ops;  // scratch
};

namespace dsmpnn {

static int find_local(int32_t n_local, const int32_t *local_parts, int32_t part) {
  for (int i = 0; i < n_local; ++i)
    if (local_parts[i] == part) return i;
  return -1;
}

// the op list of one exchange (see dsmpnn_halo_schedule in include/dsmpnn.h)
static dsmpnn_status build_schedule(int32_t nparts, const int32_t *part_rank, int32_t my_rank, int32_t n_local,
                                    const int32_t *local_parts, const int64_t *const *halo_ptr,
                                    const int64_t *const *send_ptr, int32_t direction, int32_t flags,
                                    std::vector<dsmpnn_halo_op> &ops, int64_t *stage_rows) {
  DS_CHECK_ARG(nparts >= 1 && n_local >= 0 && n_local <= nparts, DSMPNN_ERR_INVALID_ARG, "halo: nparts / n_local");
  DS_CHECK_ARG(direction == DSMPNN_HALO_FORWARD || direction == DSMPNN_HALO_REVERSE_ADD, DSMPNN_ERR_INVALID_ARG,
               "halo: direction");
  std::vector<int> loc(nparts, -1);
  for (int i = 0; i < n_local; ++i) {
    const int p = local_parts[i];
    DS_CHECK_ARG(p >= 0 && p < nparts && loc[p] < 0, DSMPNN_ERR_INVALID_ARG, "halo: local part %d invalid or repeated",
                 p);
    DS_CHECK_ARG(part_rank[p] == my_rank, DSMPNN_ERR_INVALID_ARG, "halo: local part %d belongs to rank %d, not %d", p,
                 part_rank[p], my_rank);
    loc[p] = i;
  }
  for (int p = 0; p < nparts; ++p)
    DS_CHECK_ARG(part_rank[p] != my_rank || loc[p] >= 0, DSMPNN_ERR_INVALID_ARG,
                 "halo: part %d of this rank is missing from local_parts", p);
  const bool via = (flags & DSMPNN_HALO_VIA_NCCL) != 0;
  ops.clear();
  int64_t stage = 0;
  auto push = [&](int32_t kind, int32_t peer, int32_t src, int32_t dst, int64_t rows, int64_t off) {
    dsmpnn_halo_op o;
    o.kind = kind;
    o.peer_rank = peer;
    o.src_part = src;
    o.dst_part = dst;
    o.rows = rows;
    o.offset = off;
    ops.push_back(o);
  };
  if (direction == DSMPNN_HALO_FORWARD) {
    // values[t][halo_ptr_t[s] ..] <- values[s][send_idx_s[send_ptr_s[t] ..]]
    for (int s = 0; s < nparts; ++s)
      for (int t = 0; t < nparts; ++t) {
        if (s == t) continue;
        const int sl = loc[s], tl = loc[t];
        if (sl < 0 && tl < 0) continue;
        const int64_t ns = sl >= 0 ? send_ptr[sl][t + 1] - send_ptr[sl][t] : -1;
        const int64_t nh = tl >= 0 ? halo_ptr[tl][s + 1] - halo_ptr[tl][s] : -1;
        DS_CHECK_ARG(ns >= -1 && nh >= -1 && (ns < 0 || nh < 0 || ns == nh), DSMPNN_ERR_SHAPE,
                     "halo: %d -> %d sends %lld rows but receives %lld", s, t, (long long)ns, (long long)nh);
        if (sl >= 0 && tl >= 0 && !via) {
          if (nh > 0) push(DSMPNN_HALO_OP_LOCAL, my_rank, s, t, nh, halo_ptr[tl][s]);
          continue;
        }
        if (sl >= 0 && ns > 0) {
          push(DSMPNN_HALO_OP_SEND, part_rank[t], s, t, ns, stage);
          stage += ns;
        }
        if (tl >= 0 && nh > 0) push(DSMPNN_HALO_OP_RECV, part_rank[s], s, t, nh, halo_ptr[tl][s]);
      }
  } else {
    // values[p][send_idx_p[send_ptr_p[q] + r]] += values[q][halo_ptr_q[p] + r], q ascending per p
    for (int p = 0; p < nparts; ++p)
      for (int q = 0; q < nparts; ++q) {
        if (p == q) continue;
        const int pl = loc[p], ql = loc[q];
        if (pl < 0 && ql < 0) continue;
        const int64_t ns = pl >= 0 ? send_ptr[pl][q + 1] - send_ptr[pl][q] : -1;
        const int64_t nh = ql >= 0 ? halo_ptr[ql][p + 1] - halo_ptr[ql][p] : -1;
        DS_CHECK_ARG(ns >= -1 && nh >= -1 && (ns < 0 || nh < 0 || ns == nh), DSMPNN_ERR_SHAPE,
                     "halo: reverse %d <- %d: %lld send rows, %lld halo rows", p, q, (long long)ns, (long long)nh);
        if (pl >= 0 && ql >= 0 && !via) {
          if (nh > 0) push(DSMPNN_HALO_OP_LOCAL, my_rank, q, p, nh, halo_ptr[ql][p]);
          continue;
        }
        if (ql >= 0 && nh > 0) push(DSMPNN_HALO_OP_SEND, part_rank[p], q, p, nh, halo_ptr[ql][p]);
        if (pl >= 0 && ns > 0) {
          push(DSMPNN_HALO_OP_RECV, part_rank[q], q, p, ns, stage);
          stage += ns;
        }
      }
  }
  *stage_rows = stage;
  return DSMPNN_OK;
}

template <typename T>
__global__ void gather_rows_any_kernel(const T *__restrict__ v, const int32_t *__restrict__ rows, int64_t n_rows,
                                       int width, T *__restrict__ out) {
  const int64_t total = n_rows * width;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / width, c = t - r * width;
    out[t] = v[(int64_t)rows[r] * width + c];
  }
}

// spins for `ns` nanoseconds of the global timer (test hook, see below)
__global__ void stall_kernel(unsigned long long ns) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    __nanosleep(100000);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while (t - t0 < ns);
}

struct Gather {
  const char *src;
  const int32_t *rows;
  char *dst;
  int64_t n;
};

// all gathers of one exchange: 16-byte rows in batched launches (HaloJobs),
// other widths one launch each
static dsmpnn_status run_gathers(const std::vector<Gather> &g, int width, size_t esz, cudaStream_t s) {
  const size_t rowb = (size_t)width * esz;
  bool vec = rowb % 16 == 0;
  for (const Gather &x : g) vec = vec && !((uintptr_t)x.src & 15) && !((uintptr_t)x.dst & 15);
  if (vec) {
    const int row16 = (int)(rowb / 16);
    for (size_t b = 0; b < g.size(); b += HaloJobs::kMax) {
      HaloJobs jobs;
      const int nj = (int)std::min<size_t>(HaloJobs::kMax, g.size() - b);
      int64_t most = 0;
      for (int j = 0; j < nj; ++j) {
        jobs.src[j] = reinterpret_cast<const uint4 *>(g[b + j].src);
        jobs.rows[j] = g[b + j].rows;
        jobs.dst[j] = reinterpret_cast<uint4 *>(g[b + j].dst);
        jobs.n_rows[j] = g[b + j].n;
        most = std::max(most, g[b + j].n);
      }
      const int gx = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(most * row16, 256), 64));
      halo_gather_jobs_kernel<<<dim3(gx, nj), 256, 0, s>>>(jobs, row16);
      DS_LAUNCH_CHECK();
    }
    return DSMPNN_OK;
  }
  for (const Gather &x : g) {
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(x.n * width, 256), 148 * 8));
    if (esz == 2)
      gather_rows_any_kernel<uint16_t><<<blocks, 256, 0, s>>>((const uint16_t *)x.src, x.rows, x.n, width,
                                                              (uint16_t *)x.dst);
    else
      gather_rows_any_kernel<uint32_t><<<blocks, 256, 0, s>>>((const uint32_t *)x.src, x.rows, x.n, width,
                                                              (uint32_t *)x.dst);
    DS_LAUNCH_CHECK();
  }
  return DSMPNN_OK;
}

static dsmpnn_status ensure_stage(dsmpnn_ctx_s *c, size_t bytes) {
  if (bytes <= c->stage_bytes) return DSMPNN_OK;
  // rare: wait for every exchange that may still use the old buffer
  DS_CUDA(cudaStreamSynchronize(c->cs));
  if (c->stage) DS_CUDA(cudaFree(c->stage));
  c->stage = nullptr;
  c->stage_bytes = 0;
  const size_t nb = std::max<size_t>(bytes + bytes / 4, 1 << 16);
  DS_CUDA(cudaMalloc(&c->stage, nb));
  c->stage_bytes = nb;
  return DSMPNN_OK;
}

}  // namespace dsmpnn

using namespace dsmpnn;

extern "C" {

dsmpnn_status dsmpnn_comm_unique_id(void *id) {
  DS_CHECK_ARG(id != nullptr, DSMPNN_ERR_INVALID_ARG, "comm_unique_id: NULL");
  static_assert(sizeof(ncclUniqueId) == DSMPNN_UNIQUE_ID_BYTES, "ncclUniqueId size");
  ncclUniqueId u;
  DS_NCCL(ncclGetUniqueId(&u));
  memcpy(id, &u, sizeof(u));
  return DSMPNN_OK;
}

dsmpnn_status dsmpnn_ctx_create(int32_t device, const void *unique_id, int32_t rank, int32_t nranks,
                                dsmpnn_ctx *ctx) {
  DS_CHECK_ARG(ctx && unique_id, DSMPNN_ERR_INVALID_ARG, "ctx_create: NULL argument");
  DS_CHECK_ARG(nranks >= 1 && rank >= 0 && rank < nranks, DSMPNN_ERR_INVALID_ARG, "ctx_create: rank %d of %d", rank,
               nranks);
  *ctx = nullptr;
  DS_CUDA(cudaSetDevice(device));
  dsmpnn_ctx_s *c = new dsmpnn_ctx_s();
  c->device = device;
  c->rank = rank;
  c->nranks = nranks;
  ncclUniqueId u;
  memcpy(&u, unique_id, sizeof(u));
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  cudaError_t e = cudaStreamCreateWithPriority(&c->cs, cudaStreamNonBlocking, hi);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_in, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_done, cudaEventDisableTiming);
  if (e != cudaSuccess) {
    set_error("ctx_create: %s", cudaGetErrorString(e));
    dsmpnn_ctx_destroy(c);
    return DSMPNN_ERR_CUDA;
  }
  ncclResult_t r = ncclCommInitRank(&c->comm, nranks, u, rank);
  if (r != ncclSuccess) {
    set_error("ctx_create: ncclCommInitRank: %s", ncclGetErrorString(r));
    c->comm = nullptr;
    dsmpnn_ctx_destroy(c);
    return DSMPNN_ERR_NCCL;
  }
  *ctx = c;
  return DSMPNN_OK;
}

dsmpnn_status dsmpnn_ctx_destroy(dsmpnn_ctx c) {
  if (!c) return DSMPNN_OK;
  if (c->device >= 0) cudaSetDevice(c->device);
  if (c->cs) cudaStreamSynchronize(c->cs);
  if (c->comm) {
    if (c->aborted) ncclCommAbort(c->comm);
    else ncclCommDestroy(c->comm);
  }
  if (c->stage) cudaFree(c->stage);
  if (c->ev_in) cudaEventDestroy(c->ev_in);
  if (c->ev_done) cudaEventDestroy(c->ev_done);
  if (c->cs) cudaStreamDestroy(c->cs);
  delete c;
  return DSMPNN_OK;
}

dsmpnn_status dsmpnn_ctx_info(dsmpnn_ctx c, int32_t *rank, int32_t *nranks, void **comm_stream) {
  DS_CHECK_ARG(c, DSMPNN_ERR_INVALID_ARG, "ctx_info: NULL ctx");
  if (rank) *rank = c->rank;
  if (nranks) *nranks = c->nranks;
  if (comm_stream) *comm_stream = (void *)c->cs;
  return DSMPNN_OK;
}

dsmpnn_status dsmpnn_halo_schedule(int32_t nparts, const int32_t *part_rank, int32_t my_rank, int32_t n_local,
                                   const int32_t *local_parts, const int64_t *const *halo_ptr,
                                   const int64_t *const *send_ptr, int32_t direction, int32_t flags,
                                   dsmpnn_halo_op *ops, int32_t capacity, int32_t *n_ops, int64_t *stage_rows) {
  DS_CHECK_ARG(part_rank && n_ops && stage_rows && (n_local == 0 || (local_parts && halo_ptr && send_ptr)),
               DSMPNN_ERR_INVALID_ARG, "halo_schedule: NULL argument");
  std::vector<dsmpnn_halo_op> v;
  DS_TRY(build_schedule(nparts, part_rank, my_rank, n_local, local_parts, halo_ptr, send_ptr, direction, flags, v,
                        stage_rows));
  *n_ops = (int32_t)v.size();
  DS_CHECK_ARG((int64_t)v.size() <= capacity, DSMPNN_ERR_CAPACITY, "halo_schedule: %zu ops > capacity %d", v.size(),
               capacity);
  if (!v.empty()) memcpy(ops, v.data(), v.size() * sizeof(dsmpnn_halo_op));
  return DSMPNN_OK;
}

dsmpnn_status dsmpnn_halo_exchange(dsmpnn_ctx c, int32_t nparts, const int32_t *part_rank, int32_t n_local,
                                   const int32_t *local_parts, void *const *values, const int64_t *const *halo_ptr,
                                   const int64_t *const *send_ptr, const int32_t *const *send_idx, int32_t width,
                                   int32_t dtype, int32_t direction, int32_t flags, void *stream) {
  DS_CHECK_ARG(c, DSMPNN_ERR_INVALID_ARG, "halo_exchange: no context");
  DS_CHECK_ARG(!c->aborted && c->comm, DSMPNN_ERR_NCCL, "halo_exchange: the communicator was aborted");
  DS_CHECK_ARG(part_rank && (n_local == 0 || (local_parts && values && halo_ptr && send_ptr && send_idx)),
               DSMPNN_ERR_INVALID_ARG, "halo_exchange: NULL argument");
  DS_CHECK_ARG(width > 0, DSMPNN_ERR_INVALID_ARG, "halo_exchange: width");
  DS_CHECK_ARG(dtype == DSMPNN_F32 || dtype == DSMPNN_BF16, DSMPNN_ERR_INVALID_ARG, "halo_exchange: dtype");
  DS_CHECK_ARG(direction != DSMPNN_HALO_REVERSE_ADD || dtype == DSMPNN_F32, DSMPNN_ERR_UNSUPPORTED,
               "halo_exchange: REVERSE_ADD takes fp32 gradients");
  for (int p = 0; p < nparts; ++p)
    DS_CHECK_ARG(part_rank[p] >= 0 && part_rank[p] < c->nranks, DSMPNN_ERR_INVALID_ARG,
                 "halo_exchange: part %d on rank %d of %d", p, part_rank[p], c->nranks);
  int64_t stage_rows = 0;
  DS_TRY(build_schedule(nparts, part_rank, c->rank, n_local, local_parts, halo_ptr, send_ptr, direction, flags, c->ops,
                        &stage_rows));
  const size_t esz = dtype == DSMPNN_BF16 ? 2 : 4;
  const size_t rowb = (size_t)width * esz;
  DS_TRY(ensure_stage(c, (size_t)stage_rows * rowb));
  cudaStream_t s = as_stream(stream), cs = c->cs;
  DS_CUDA(cudaEventRecord(c->ev_in, s));
  DS_CUDA(cudaStreamWaitEvent(cs, c->ev_in, 0));
  char *stage = (char *)c->stage;
  auto L = [&](int part) { return find_local(n_local, local_parts, part); };
  bool any_nccl = false;
  for (const dsmpnn_halo_op &o : c->ops) any_nccl = any_nccl || o.kind != DSMPNN_HALO_OP_LOCAL;
  // test hook: stall the comm stream for DSMPNN_TEST_HALO_STALL_MS ms before
  // the exchange (a bounded stand-in for a peer that never answers; exercises
  // the dsmpnn_ctx_sync watchdog; never set in production)
  static const int stall_ms = getenv("DSMPNN_TEST_HALO_STALL_MS") ? atoi(getenv("DSMPNN_TEST_HALO_STALL_MS")) : 0;
  if (stall_ms > 0) {
    stall_kernel<<<1, 1, 0, cs>>>((unsigned long long)stall_ms * 1000000ull);
    DS_LAUNCH_CHECK();
  }
  if (direction == DSMPNN_HALO_FORWARD) {
    std::vector<Gather> g;
    for (const dsmpnn_halo_op &o : c->ops) {
      if (o.kind == DSMPNN_HALO_OP_RECV) continue;
      const int sl = L(o.src_part);
      const int32_t *rows = send_idx[sl] + send_ptr[sl][o.dst_part];
      char *dst = o.kind == DSMPNN_HALO_OP_LOCAL ? (char *)values[L(o.dst_part)] + (size_t)o.offset * rowb
                                                 : stage + (size_t)o.offset * rowb;
      g.push_back(Gather{(const char *)values[sl], rows, dst, o.rows});
    }
    DS_TRY(run_gathers(g, width, esz, cs));
    if (any_nccl) {
      DS_NCCL(ncclGroupStart());
      for (const dsmpnn_halo_op &o : c->ops) {
        if (o.kind == DSMPNN_HALO_OP_SEND)
          DS_NCCL(ncclSend(stage + (size_t)o.offset * rowb, (size_t)o.rows * rowb, ncclUint8, o.peer_rank, c->comm, cs));
        if (o.kind == DSMPNN_HALO_OP_RECV)
          DS_NCCL(ncclRecv((char *)values[L(o.dst_part)] + (size_t)o.offset * rowb, (size_t)o.rows * rowb, ncclUint8,
                           o.peer_rank, c->comm, cs));
      }
      DS_NCCL(ncclGroupEnd());
    }
  } else {
    if (any_nccl) {
      DS_NCCL(ncclGroupStart());
      for (const dsmpnn_halo_op &o : c->ops) {
        if (o.kind == DSMPNN_HALO_OP_SEND)
          DS_NCCL(ncclSend((char *)values[L(o.src_part)] + (size_t)o.offset * rowb, (size_t)o.rows * rowb, ncclUint8,
                           o.peer_rank, c->comm, cs));
        else if (o.kind == DSMPNN_HALO_OP_RECV)
          DS_NCCL(ncclRecv(stage + (size_t)o.offset * rowb, (size_t)o.rows * rowb, ncclUint8, o.peer_rank, c->comm,
                           cs));
      }
      DS_NCCL(ncclGroupEnd());
    }
    // additions in (owner, holder ascending) order: the schedule's order
    for (const dsmpnn_halo_op &o : c->ops) {
      if (o.kind == DSMPNN_HALO_OP_SEND) continue;
      const int pl = L(o.dst_part);
      const float *src = o.kind == DSMPNN_HALO_OP_LOCAL
                             ? (const float *)values[L(o.src_part)] + (size_t)o.offset * width
                             : (const float *)(stage + (size_t)o.offset * rowb);
      DS_TRY(dsmpnn_halo_scatter_add(src, send_idx[pl] + send_ptr[pl][o.src_part], o.rows, width,
                                     (float *)values[pl], (void *)cs));
    }
  }
  DS_CUDA(cudaEventRecord(c->ev_done, cs));
  if (!(flags & DSMPNN_HALO_ASYNC)) DS_CUDA(cudaStreamWaitEvent(s, c->ev_done, 0));
  return DSMPNN_OK;
}

dsmpnn_status dsmpnn_halo_wait(dsmpnn_ctx c, void *stream) {
  DS_CHECK_ARG(c, DSMPNN_ERR_INVALID_ARG, "halo_wait: no context");
  DS_CUDA(cudaStreamWaitEvent(as_stream(stream), c->ev_done, 0));
  return DSMPNN_OK;
}

dsmpnn_status dsmpnn_allreduce_sum_f32(dsmpnn_ctx c, float *buf, int64_t n, void *stream) {
  DS_CHECK_ARG(c, DSMPNN_ERR_INVALID_ARG, "allreduce: no context");
  DS_CHECK_ARG(!c->aborted && c->comm, DSMPNN_ERR_NCCL, "allreduce: the communicator was aborted");
  DS_CHECK_ARG(n >= 0, DSMPNN_ERR_INVALID_ARG, "allreduce: n < 0");
  cudaStream_t s = as_stream(stream);
  if (n > 0) DS_NCCL(ncclAllReduce(buf, buf, (size_t)n, ncclFloat32, ncclSum, c->comm, s));
  DS_CUDA(cudaEventRecord(c->ev_done, s));
  return DSMPNN_OK;
}

dsmpnn_status dsmpnn_ctx_sync(dsmpnn_ctx c, int32_t timeout_ms) {
  DS_CHECK_ARG(c, DSMPNN_ERR_INVALID_ARG, "ctx_sync: no context");
  DS_CHECK_ARG(!c->aborted && c->comm, DSMPNN_ERR_NCCL, "ctx_sync: the communicator was aborted");
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    cudaError_t q = cudaEventQuery(c->ev_done);
    if (q == cudaSuccess) break;
    if (q != cudaErrorNotReady) DS_CUDA(q);
    ncclResult_t ar = ncclSuccess;
    DS_NCCL(ncclCommGetAsyncError(c->comm, &ar));
    if (ar != ncclSuccess && ar != ncclInProgress) {
      c->aborted = true;
      ncclCommAbort(c->comm);
      c->comm = nullptr;
      set_error("ctx_sync: NCCL asynchronous error: %s", ncclGetErrorString(ar));
      return DSMPNN_ERR_NCCL;
    }
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (timeout_ms >= 0 && ms > timeout_ms) {
      c->aborted = true;
      ncclCommAbort(c->comm);
      c->comm = nullptr;
      set_error("ctx_sync: the last exchange did not finish within %d ms; communicator aborted", timeout_ms);
      return DSMPNN_ERR_TIMEOUT;
    }
    std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
  return DSMPNN_OK;
}

}  // extern "C"

// batch.cu - the sub-domains held by one process as ONE disjoint-union graph
// (dsmpnn_batch_subdomains, include/dsmpnn.h "a8").
//
// PAPER.md:58 gives each GPU one sub-domain; with more sub-domains than
// processes (one GPU running the 4-sub-domain Darcy case) the P local graphs
// are independent between halo refreshes (Alg. 1 :404-411), so the layer can
// run over their disjoint union in one launch per kernel instead of P: the
// per-launch fill / drain of the persistent edge kernels and the small node
// kernels are paid once per layer, not once per sub-domain.
//
// Union node order: the owned rows of part 0, 1, ..., P-1, then the halo rows
// of part 0, 1, ..., P-1 (so rows [0, N_own) are the ones a layer computes and
// a halo refresh is one gather into [N_own, N_loc)).  Union edge order: the
// parts' edge arrays concatenated (a part's rows keep their CSR order).  The
// union CSC lists keep every part's list order, so the backward scatter adds
// in the same order as per part.
#include <algorithm>

#include "common.cuh"

namespace dsmpnn {

namespace {

constexpr int kMaxBatch = 16;

int grid_for(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 8)); }

struct BatchGeom {
  int P;
  int64_t n_own[kMaxBatch], n_loc[kMaxBatch], E[kMaxBatch];
  int64_t own_off[kMaxBatch + 1], halo_off[kMaxBatch + 1], edge_off[kMaxBatch + 1];
  const int64_t *row_ptr[kMaxBatch];
  const int32_t *col[kMaxBatch];
  const int32_t *perm[kMaxBatch];
  const int64_t *cptr[kMaxBatch];
  const int64_t *rows[kMaxBatch];
  int64_t N_own, N_loc, E_tot;
};

// part holding union index u of an offset table off[0..P] (off[P] = end)
__device__ __forceinline__ int part_of(const int64_t *off, int P, int64_t u) {
  int q = 0;
  while (q + 1 < P && off[q + 1] <= u) ++q;
  return q;
}

__device__ __forceinline__ int64_t map_col(const BatchGeom &g, int q, int64_t j) {
  return j < g.n_own[q] ? g.own_off[q] + j : g.halo_off[q] + (j - g.n_own[q]);
}

// CSC segment bases: own[q] = sum_{q' < q} |own-column lists of q'|,
// halo[q] = (all own lists) + sum_{q' < q} |halo-column lists of q'|
__global__ void batch_bases_kernel(BatchGeom g, int64_t *bases) {
  if (threadIdx.x != 0) return;
  int64_t acc = 0;
  for (int q = 0; q < g.P; ++q) {
    bases[q] = acc;
    acc += g.cptr[q][g.n_own[q]];
  }
  bases[g.P] = acc;
  for (int q = 0; q < g.P; ++q) {
    bases[kMaxBatch + 1 + q] = acc;
    acc += g.E[q] - g.cptr[q][g.n_own[q]];
  }
  bases[kMaxBatch + 1 + g.P] = acc;
}

__global__ void batch_nodes_kernel(BatchGeom g, const int64_t *__restrict__ bases, int64_t *__restrict__ row_ptr,
                                   int64_t *__restrict__ cptr, int64_t *__restrict__ rows) {
  __shared__ int64_t sb[2 * (kMaxBatch + 1)];
  for (int i = threadIdx.x; i < 2 * (kMaxBatch + 1); i += blockDim.x) sb[i] = bases[i];
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u <= g.N_loc; u += stride) {
    if (u <= g.N_own && row_ptr) {
      if (u == g.N_own) {
        row_ptr[u] = g.E_tot;
      } else {
        const int q = part_of(g.own_off, g.P, u);
        row_ptr[u] = g.row_ptr[q][u - g.own_off[q]] + g.edge_off[q];
      }
    }
    if (u == g.N_loc) {
      if (cptr) cptr[u] = g.E_tot;
      continue;
    }
    int q;
    int64_t j, c;
    if (u < g.N_own) {
      q = part_of(g.own_off, g.P, u);
      j = u - g.own_off[q];
      if (cptr) c = g.cptr[q][j] + sb[q];
    } else {
      q = part_of(g.halo_off, g.P, u);
      j = g.n_own[q] + (u - g.halo_off[q]);
      if (cptr) c = g.cptr[q][j] - g.cptr[q][g.n_own[q]] + sb[kMaxBatch + 1 + q];
    }
    if (cptr) cptr[u] = c;
    if (rows) rows[u] = g.rows[q][j];
  }
}

__global__ void batch_edges_kernel(BatchGeom g, const int64_t *__restrict__ bases, int32_t *__restrict__ col,
                                   int32_t *__restrict__ perm) {
  __shared__ int64_t sb[2 * (kMaxBatch + 1)];
  for (int i = threadIdx.x; i < 2 * (kMaxBatch + 1); i += blockDim.x) sb[i] = bases[i];
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < g.E_tot; p += stride) {
    if (col) {
      const int q = part_of(g.edge_off, g.P, p);
      col[p] = (int32_t)map_col(g, q, g.col[q][p - g.edge_off[q]]);
    }
    if (perm) {
      // CSC position p: the own-column segment of part q, or its halo-column segment
      int q;
      int64_t src;
      if (p < sb[g.P]) {
        q = part_of(sb, g.P, p);
        src = p - sb[q];
      } else {
        q = part_of(sb + kMaxBatch + 1, g.P, p);
        src = g.cptr[q][g.n_own[q]] + (p - sb[kMaxBatch + 1 + q]);
      }
      perm[p] = (int32_t)(g.perm[q][src] + g.edge_off[q]);
    }
  }
}

struct HaloJobsU {
  int n;
  int64_t dst0[kMaxBatch * kMaxBatch + 1];  // start of the job's rows in the halo region
  int64_t src_off[kMaxBatch * kMaxBatch];   // union row of the source part's row 0
  const int32_t *send[kMaxBatch * kMaxBatch];
};

// the job table is a kernel parameter (< 7 KB; CUDA 12.1+ takes up to 32 KB)
__global__ void batch_halo_kernel(const __grid_constant__ HaloJobsU J, int64_t n_halo, int32_t *__restrict__ src) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t h = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; h < n_halo; h += stride) {
    int lo = 0, hi = J.n;  // largest job with dst0 <= h
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (J.dst0[mid] <= h) lo = mid; else hi = mid;
    }
    src[h] = (int32_t)(J.src_off[lo] + J.send[lo][h - J.dst0[lo]]);
  }
}

}  // namespace

}  // namespace dsmpnn

using namespace dsmpnn;

extern "C" dsmpnn_status dsmpnn_batch_workspace_size(int32_t nparts, size_t *bytes) {
  DS_CHECK_ARG(bytes != nullptr, DSMPNN_ERR_INVALID_ARG, "batch_workspace_size: bytes is NULL");
  DS_CHECK_ARG(nparts >= 1 && nparts <= kMaxBatch, DSMPNN_ERR_UNSUPPORTED,
               "batch_workspace_size: 1 <= nparts <= %d (got %d)", kMaxBatch, nparts);
  *bytes = 2 * (kMaxBatch + 1) * sizeof(int64_t);
  return DSMPNN_OK;
}

extern "C" dsmpnn_status dsmpnn_batch_subdomains(int32_t nparts, const dsmpnn_batch_part *parts, int32_t e_row_bytes,
                                                 int64_t *row_ptr, int32_t *col_idx, void *e, int32_t *csc_perm,
                                                 int64_t *csc_ptr, int64_t *rows, int32_t *halo_src, void *ws,
                                                 size_t ws_bytes, void *stream) {
  DS_CHECK_ARG(nparts >= 1 && nparts <= kMaxBatch, DSMPNN_ERR_UNSUPPORTED,
               "batch_subdomains: 1 <= nparts <= %d (got %d)", kMaxBatch, nparts);
  DS_CHECK_ARG(parts != nullptr, DSMPNN_ERR_INVALID_ARG, "batch_subdomains: parts is NULL");
  size_t need = 0;
  DS_TRY(dsmpnn_batch_workspace_size(nparts, &need));
  DS_CHECK_ARG(ws != nullptr && ws_bytes >= need, DSMPNN_ERR_CAPACITY, "batch_subdomains: workspace too small");
  cudaStream_t s = as_stream(stream);
  BatchGeom g{};
  g.P = nparts;
  int64_t no = 0, nl = 0, ne = 0;
  for (int q = 0; q < nparts; ++q) {
    const dsmpnn_batch_part &b = parts[q];
    DS_CHECK_ARG(b.n_own >= 0 && b.n_loc >= b.n_own && b.n_edges >= 0, DSMPNN_ERR_INVALID_ARG,
                 "batch_subdomains: part %d sizes (n_own %lld, n_loc %lld, E %lld)", q, (long long)b.n_own,
                 (long long)b.n_loc, (long long)b.n_edges);
    DS_CHECK_ARG(b.row_ptr && (b.n_edges == 0 || b.col_idx), DSMPNN_ERR_INVALID_ARG,
                 "batch_subdomains: part %d row_ptr / col_idx NULL", q);
    DS_CHECK_ARG(!csc_perm == !csc_ptr && (!csc_ptr || (b.csc_perm && b.csc_ptr)), DSMPNN_ERR_INVALID_ARG,
                 "batch_subdomains: part %d CSC inputs / outputs incomplete", q);
    DS_CHECK_ARG(!rows || b.rows, DSMPNN_ERR_INVALID_ARG, "batch_subdomains: part %d rows NULL", q);
    DS_CHECK_ARG(!e || (e_row_bytes > 0 && (b.n_edges == 0 || b.e)), DSMPNN_ERR_INVALID_ARG,
                 "batch_subdomains: part %d edge attributes NULL / e_row_bytes", q);
    g.n_own[q] = b.n_own;
    g.n_loc[q] = b.n_loc;
    g.E[q] = b.n_edges;
    g.row_ptr[q] = b.row_ptr;
    g.col[q] = b.col_idx;
    g.perm[q] = b.csc_perm;
    g.cptr[q] = b.csc_ptr;
    g.rows[q] = b.rows;
    g.own_off[q] = no;
    g.edge_off[q] = ne;
    no += b.n_own;
    ne += b.n_edges;
  }
  for (int q = 0; q < nparts; ++q) {
    g.halo_off[q] = no + nl;
    nl += parts[q].n_loc - parts[q].n_own;
  }
  g.own_off[nparts] = no;
  g.halo_off[nparts] = no + nl;
  g.edge_off[nparts] = ne;
  g.N_own = no;
  g.N_loc = no + nl;
  g.E_tot = ne;
  DS_CHECK_ARG(g.N_loc < INT32_MAX && g.E_tot < INT32_MAX, DSMPNN_ERR_UNSUPPORTED,
               "batch_subdomains: union sizes exceed int32 indices");

  // halo jobs: rows [halo_ptr_q[p], halo_ptr_q[p+1]) of part q <- rows send_idx_p[send_ptr_p[q] ..] of part p
  HaloJobsU J{};
  const int64_t n_halo = g.N_loc - g.N_own;
  if (halo_src) {
    for (int q = 0; q < nparts; ++q) {
      const dsmpnn_batch_part &b = parts[q];
      DS_CHECK_ARG(b.halo_ptr && b.send_ptr, DSMPNN_ERR_INVALID_ARG, "batch_subdomains: part %d halo_ptr / send_ptr NULL", q);
      DS_CHECK_ARG(b.halo_ptr[0] == b.n_own && b.halo_ptr[nparts] == b.n_loc, DSMPNN_ERR_SHAPE,
                   "batch_subdomains: part %d halo_ptr does not span its halo rows", q);
      for (int p = 0; p < nparts; ++p) {
        const int64_t a = b.halo_ptr[p], z = b.halo_ptr[p + 1];
        DS_CHECK_ARG(z >= a, DSMPNN_ERR_SHAPE, "batch_subdomains: part %d halo_ptr not ascending", q);
        if (z == a) continue;
        DS_CHECK_ARG(p != q, DSMPNN_ERR_SHAPE, "batch_subdomains: part %d lists halo rows from itself", q);
        const int64_t s0 = parts[p].send_ptr[q], s1 = parts[p].send_ptr[q + 1];
        DS_CHECK_ARG(s1 - s0 == z - a, DSMPNN_ERR_SHAPE, "batch_subdomains: %d<-%d sizes differ (%lld vs %lld)", q, p,
                     (long long)(z - a), (long long)(s1 - s0));
        DS_CHECK_ARG(parts[p].send_idx != nullptr, DSMPNN_ERR_INVALID_ARG, "batch_subdomains: part %d send_idx NULL", p);
        J.dst0[J.n] = g.halo_off[q] - g.N_own + (a - b.n_own);
        J.src_off[J.n] = g.own_off[p];
        J.send[J.n] = parts[p].send_idx + s0;
        ++J.n;
      }
    }
  }

  int64_t *bases = static_cast<int64_t *>(ws);
  if (csc_ptr) {
    batch_bases_kernel<<<1, 32, 0, s>>>(g, bases);
    DS_LAUNCH_CHECK();
  }
  if (row_ptr || csc_ptr || rows) {
    batch_nodes_kernel<<<grid_for(g.N_loc + 1), 256, 0, s>>>(g, bases, row_ptr, csc_ptr, rows);
    DS_LAUNCH_CHECK();
  }
  if (g.E_tot > 0 && (col_idx || csc_perm)) {
    batch_edges_kernel<<<grid_for(g.E_tot), 256, 0, s>>>(g, bases, col_idx, csc_perm);
    DS_LAUNCH_CHECK();
  }
  if (e) {
    for (int q = 0; q < nparts; ++q)
      if (parts[q].n_edges > 0)
        DS_CUDA(cudaMemcpyAsync(static_cast<char *>(e) + g.edge_off[q] * e_row_bytes, parts[q].e,
                                (size_t)parts[q].n_edges * e_row_bytes, cudaMemcpyDeviceToDevice, s));
  }
  if (halo_src && n_halo > 0 && J.n > 0) {
    batch_halo_kernel<<<grid_for(n_halo), 256, 0, s>>>(J, n_halo, halo_src);
    DS_LAUNCH_CHECK();
  }
  return DSMPNN_OK;
}

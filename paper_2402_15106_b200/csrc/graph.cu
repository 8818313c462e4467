// graph.cu - a2 radius graph kernel with random edge cap (PAPER.md:27,
// Alg. 1 :395-396; readings R7, R8, R10, R11).
//
// Cell list: points are binned into cells of edge h >= r(1+2^-8) over the
// local bounding box and sorted by cell (stable radix sort); coordinates, the
// local index and gid are then stored in cell order (xs, gs) so a candidate
// scan is one coalesced 16-byte load per point.  One warp owns one
// destination row and scans the 3^dim neighbouring cells (32 candidates per
// step, ballot-compacted).
//  pass 1 (count2): candidate count and a 2^10-bin histogram of the top key
//          bits; for a capped row the bin holding the n_e-th smallest key and
//          how many to take from it;
//  CSR offsets = exclusive scan of min(count, n_e);
//  pass 2 (select2): keeps the candidates below the boundary bin, selects the
//          remaining ones from the boundary bin by full (key_edge, gid) rank,
//          orders the kept row by gid (rank sort) and writes it.
// A row whose boundary bin overflows the per-warp buffer (not expected for
// hash keys) is finished by the general most-significant-digit radix select
// (select_kernel, 8-bit digits over the full 128-bit (key, gid) composite).
// Large sub-domains use the one-pass kernel graph1 instead (see below); the
// candidate coordinates and gids are loaded together (scan_sorted_g).
#include <cub/cub.cuh>
#include <cstdlib>

#include "common.cuh"
#include "hash.cuh"

namespace dsmpnn {

constexpr int kReach = 3;

struct GridParams {
  float lo[3];
  float inv_h;
  int n[3];
  int n_cells;
  int reach;  // neighbour cells scanned on each side: cell edge >= r / reach
};

// fp32 predicate in the fixed order of R7 (no FMA contraction)
__device__ __forceinline__ bool within(const float *xi, const float *xj, int dim, float r2) {
  float dx = __fsub_rn(xi[0], xj[0]);
  float d2 = __fmul_rn(dx, dx);
  dx = __fsub_rn(xi[1], xj[1]);
  d2 = __fadd_rn(d2, __fmul_rn(dx, dx));
  if (dim == 3) {
    dx = __fsub_rn(xi[2], xj[2]);
    d2 = __fadd_rn(d2, __fmul_rn(dx, dx));
  }
  return d2 <= r2;
}

__global__ void bbox_kernel(const float *__restrict__ x, int64_t n, int dim, float *__restrict__ out /*lo[3],hi[3]*/) {
  __shared__ float slo[3][32], shi[3][32];
  float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x)
    for (int d = 0; d < dim; ++d) {
      float v = x[i * dim + d];
      lo[d] = fminf(lo[d], v);
      hi[d] = fmaxf(hi[d], v);
    }
  for (int d = 0; d < 3; ++d)
    for (int o = 16; o; o >>= 1) {
      lo[d] = fminf(lo[d], __shfl_xor_sync(0xffffffffu, lo[d], o));
      hi[d] = fmaxf(hi[d], __shfl_xor_sync(0xffffffffu, hi[d], o));
    }
  int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0)
    for (int d = 0; d < 3; ++d) { slo[d][w] = lo[d]; shi[d][w] = hi[d]; }
  __syncthreads();
  if (threadIdx.x < 3) {
    int d = threadIdx.x;
    float a = INFINITY, b = -INFINITY;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) { a = fminf(a, slo[d][k]); b = fmaxf(b, shi[d][k]); }
    out[d] = a;
    out[3 + d] = b;
  }
}

__global__ void grid_params_kernel(const float *__restrict__ bb, int dim, float h0, int64_t max_cells,
                                   GridParams *__restrict__ gp) {
  float h = h0;
  int n[3] = {1, 1, 1};
  for (int it = 0; it < 200; ++it) {
    int64_t tot = 1;
    for (int d = 0; d < dim; ++d) {
      float ext = bb[3 + d] - bb[d];
      n[d] = (int)floorf(ext / h) + 1;
      tot *= n[d];
    }
    if (tot <= max_cells) break;
    h *= 1.25f;
  }
  GridParams p;
  for (int d = 0; d < 3; ++d) { p.lo[d] = d < dim ? bb[d] : 0.f; p.n[d] = d < dim ? n[d] : 1; }
  p.inv_h = 1.0f / h;
  p.n_cells = p.n[0] * p.n[1] * p.n[2];
  p.reach = kReach;
  *gp = p;
}

__device__ __forceinline__ int cell_coord(float v, float lo, float inv_h, int n) {
  int c = (int)floorf((v - lo) * inv_h);
  return c < 0 ? 0 : (c >= n ? n - 1 : c);
}

__global__ void cell_id_kernel(const float *__restrict__ x, int64_t n, int dim, const GridParams *__restrict__ gp,
                               int32_t *__restrict__ cell, int32_t *__restrict__ idx) {
  GridParams p = *gp;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int c[3] = {0, 0, 0};
    for (int d = 0; d < dim; ++d) c[d] = cell_coord(x[i * dim + d], p.lo[d], p.inv_h, p.n[d]);
    cell[i] = (c[2] * p.n[1] + c[1]) * p.n[0] + c[0];
    idx[i] = (int32_t)i;
  }
}

__global__ void cell_start_kernel(const int32_t *__restrict__ sorted_cell, int64_t n, const GridParams *__restrict__ gp,
                                  int32_t *__restrict__ start, int64_t max_cells) {
  int64_t nc = gp->n_cells;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c <= nc; c += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (sorted_cell[mid] < c) lo = mid + 1; else hi = mid;
    }
    start[c] = (int32_t)lo;
  }
}

// Visit every candidate j != i of row i; F(j, ok) is called warp-uniformly per
// 32-wide step with `ok` this lane's predicate result.
template <typename F>
__device__ __forceinline__ void scan_candidates(int64_t i, const float *__restrict__ x, int dim, float r2,
                                                const GridParams &p, const int32_t *__restrict__ start,
                                                const int32_t *__restrict__ sorted_idx, F &&f) {
  int lane = threadIdx.x & 31;
  float xi[3] = {0.f, 0.f, 0.f};
  for (int d = 0; d < dim; ++d) xi[d] = x[i * dim + d];
  int c[3] = {0, 0, 0};
  for (int d = 0; d < dim; ++d) c[d] = cell_coord(xi[d], p.lo[d], p.inv_h, p.n[d]);
  const int R = p.reach;
  int z0 = dim == 3 ? max(c[2] - R, 0) : 0, z1 = dim == 3 ? min(c[2] + R, p.n[2] - 1) : 0;
  int y0 = max(c[1] - R, 0), y1 = min(c[1] + R, p.n[1] - 1);
  int x0 = max(c[0] - R, 0), x1 = min(c[0] + R, p.n[0] - 1);
  for (int cz = z0; cz <= z1; ++cz)
    for (int cy = y0; cy <= y1; ++cy) {
      // cells (x0..x1, cy, cz) are contiguous in the sorted order
      int base = (cz * p.n[1] + cy) * p.n[0];
      int a = start[base + x0], b = start[base + x1 + 1];
      for (int t0 = a; t0 < b; t0 += 32) {
        int t = t0 + lane;
        int j = -1;
        bool ok = false;
        if (t < b) {
          j = sorted_idx[t];
          float xj[3] = {0.f, 0.f, 0.f};
          for (int d = 0; d < dim; ++d) xj[d] = x[(int64_t)j * dim + d];
          ok = (j != i) && within(xi, xj, dim, r2);
        }
        f(j, ok);
      }
    }
}

constexpr int kMaxNe = 128;
constexpr int kSelWarps = 4;

// digit d (0..15) of the 128-bit composite (key, gid), most significant first
__device__ __forceinline__ uint32_t comp_digit(uint64_t key, uint64_t gid, int d) {
  return d < 8 ? (uint32_t)(key >> (56 - 8 * d)) & 0xffu : (uint32_t)(gid >> (56 - 8 * (d - 8))) & 0xffu;
}
// does the composite's top D digits equal (pk, pg)'s top D digits?
__device__ __forceinline__ bool comp_prefix_eq(uint64_t key, uint64_t gid, uint64_t pk, uint64_t pg, int D) {
  if (D == 0) return true;
  if (D <= 8) {
    int sh = 64 - 8 * D;
    return (key >> sh) == (pk >> sh);
  }
  if (key != pk) return false;
  int sh = 64 - 8 * (D - 8);
  return D == 16 ? gid == pg : (gid >> sh) == (pg >> sh);
}
__device__ __forceinline__ bool comp_prefix_le(uint64_t key, uint64_t gid, uint64_t pk, uint64_t pg, int D) {
  if (D <= 8) {
    int sh = 64 - 8 * D;
    return D == 0 ? true : (key >> sh) <= (pk >> sh);
  }
  if (key != pk) return key < pk;
  int sh = 64 - 8 * (D - 8);
  return D == 16 ? gid <= pg : (gid >> sh) <= (pg >> sh);
}

__global__ void __launch_bounds__(kSelWarps * 32) select_kernel(
    const float *__restrict__ x, const int64_t *__restrict__ gid, int64_t n_dst, int dim, float r, int32_t n_e,
    uint64_t s0, const GridParams *__restrict__ gp, const int32_t *__restrict__ start,
    const int32_t *__restrict__ sorted_idx, const int32_t *__restrict__ counts, const int64_t *__restrict__ row_ptr,
    int32_t *__restrict__ col, const int32_t *__restrict__ rows, const int32_t *__restrict__ nrows) {
  __shared__ uint32_t hist[kSelWarps][256];
  __shared__ int32_t lidx[kSelWarps][kMaxNe];
  __shared__ int64_t lgid[kSelWarps][kMaxNe];
  GridParams p = *gp;
  float r2 = __fmul_rn(r, r);
  int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nr = rows ? (int64_t)*nrows : n_dst;
  for (int64_t ii = warp; ii < nr; ii += nwarps) {
    const int64_t i = rows ? (int64_t)rows[ii] : ii;
    int cnt = counts[i];
    uint64_t gi = (uint64_t)gid[i];
    uint64_t si = smx(s0 ^ gi);
    uint64_t pk = 0, pg = 0;
    int D = 0;
    if (cnt > n_e) {
      int need = n_e;
      for (int d = 0; d < 16; ++d) {
        for (int b = lane; b < 256; b += 32) hist[w][b] = 0;
        __syncwarp();
        scan_candidates(i, x, dim, r2, p, start, sorted_idx, [&](int j, bool ok) {
          if (ok) {
            uint64_t gj = (uint64_t)gid[j];
            uint64_t k = key_edge(si, gj);
            if (comp_prefix_eq(k, gj, pk, pg, d)) atomicAdd(&hist[w][comp_digit(k, gj, d)], 1u);
          }
        });
        __syncwarp();
        // find bucket b with cum_before < need <= cum_before + hist[b]; lane owns bins 8*lane..8*lane+7
        uint32_t loc[8];
        uint32_t s = 0;
        for (int q = 0; q < 8; ++q) { loc[q] = hist[w][lane * 8 + q]; s += loc[q]; }
        uint32_t incl = s;
        for (int o = 1; o < 32; o <<= 1) {
          uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += v;
        }
        uint32_t excl = incl - s;
        int found = -1, taken_before = 0, bcnt = 0;
        if ((int)excl < need && need <= (int)incl) {
          uint32_t c0 = excl;
          for (int q = 0; q < 8; ++q) {
            if ((int)(c0 + loc[q]) >= need) { found = lane * 8 + q; taken_before = c0; bcnt = loc[q]; break; }
            c0 += loc[q];
          }
        }
        unsigned m = __ballot_sync(0xffffffffu, found >= 0);
        int src = __ffs(m) - 1;
        found = __shfl_sync(0xffffffffu, found, src);
        taken_before = __shfl_sync(0xffffffffu, taken_before, src);
        bcnt = __shfl_sync(0xffffffffu, bcnt, src);
        if (d < 8) pk |= (uint64_t)found << (56 - 8 * d);
        else pg |= (uint64_t)found << (56 - 8 * (d - 8));
        need -= taken_before;
        D = d + 1;
        __syncwarp();
        if (bcnt == need) break;
      }
    }
    // collect the kept candidates (all, or those with top-D digits <= prefix)
    int nk = 0;
    scan_candidates(i, x, dim, r2, p, start, sorted_idx, [&](int j, bool ok) {
      bool keep = false;
      uint64_t gj = 0;
      if (ok) {
        gj = (uint64_t)gid[j];
        keep = (cnt <= n_e) || comp_prefix_le(key_edge(si, gj), gj, pk, pg, D);
      }
      unsigned m = __ballot_sync(0xffffffffu, keep);
      if (keep) {
        int slot = nk + __popc(m & ((1u << lane) - 1));
        lidx[w][slot] = j;
        lgid[w][slot] = (int64_t)gj;
      }
      nk += __popc(m);
    });
    __syncwarp();
    int64_t off = row_ptr[i];
    for (int a = lane; a < nk; a += 32) {
      int64_t g = lgid[w][a];
      int rank = 0;
      for (int b = 0; b < nk; ++b) rank += lgid[w][b] < g;
      col[off + rank] = lidx[w][a];
    }
    __syncwarp();
  }
}


// ----------------------------------------------------------- fast path --
#ifndef DSMPNN_KHB
#define DSMPNN_KHB 9  // 512 bins: smaller per-warp histograms, more resident warps in graph1 (airfoil build -4 %)
#endif
constexpr int kHB = DSMPNN_KHB, kHBins = 1 << kHB;  // top key bits of the pass-1 histogram
constexpr int kCapB = 384;                  // boundary-bin buffer per warp
constexpr int kGWarps = 8;

__global__ void permute_points_kernel(const float *__restrict__ x, const int64_t *__restrict__ gid, int64_t n,
                                      int dim, const int32_t *__restrict__ sorted_idx, float4 *__restrict__ xs,
                                      int64_t *__restrict__ gs) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int32_t j = sorted_idx[t];
    float4 p;
    p.x = x[(int64_t)j * dim];
    p.y = x[(int64_t)j * dim + 1];
    p.z = dim == 3 ? x[(int64_t)j * dim + 2] : 0.f;
    p.w = __int_as_float(j);
    xs[t] = p;
    if (gs) gs[t] = gid[j];
  }
}

// Visit the candidates of row i in cell order; F(t, j, ok) per 32-wide step
// (warp-uniform call), t = cell-order position, j = local index.
template <typename F>
__device__ __forceinline__ void scan_sorted(int64_t i, const float *__restrict__ x, int dim, float r2,
                                            const GridParams &p, const int32_t *__restrict__ start,
                                            const float4 *__restrict__ xs, F &&f) {
  const int lane = threadIdx.x & 31;
  float xi[3] = {0.f, 0.f, 0.f};
  for (int d = 0; d < dim; ++d) xi[d] = x[i * dim + d];
  int c[3] = {0, 0, 0};
  for (int d = 0; d < dim; ++d) c[d] = cell_coord(xi[d], p.lo[d], p.inv_h, p.n[d]);
  const int R = p.reach;
  const int z0 = dim == 3 ? max(c[2] - R, 0) : 0, z1 = dim == 3 ? min(c[2] + R, p.n[2] - 1) : 0;
  const int y0 = max(c[1] - R, 0), y1 = min(c[1] + R, p.n[1] - 1);
  const int x0 = max(c[0] - R, 0), x1 = min(c[0] + R, p.n[0] - 1);
  for (int cz = z0; cz <= z1; ++cz)
    for (int cy = y0; cy <= y1; ++cy) {
      const int base = (cz * p.n[1] + cy) * p.n[0];
      const int a = start[base + x0], b = start[base + x1 + 1];
      for (int t0 = a; t0 < b; t0 += 64) {  // two loads in flight per lane
        const int ta = t0 + lane, tb = t0 + 32 + lane;
        const float4 pa = ta < b ? xs[ta] : make_float4(0.f, 0.f, 0.f, __int_as_float(-1));
        const float4 pb = tb < b ? xs[tb] : make_float4(0.f, 0.f, 0.f, __int_as_float(-1));
        {
          const int j = __float_as_int(pa.w);
          const float xj[3] = {pa.x, pa.y, pa.z};
          f(ta, j, ta < b && j != i && within(xi, xj, dim, r2));
        }
        if (t0 + 32 < b) {
          const int j = __float_as_int(pb.w);
          const float xj[3] = {pb.x, pb.y, pb.z};
          f(tb, j, tb < b && j != i && within(xi, xj, dim, r2));
        }
      }
    }
}

// As scan_sorted, with the candidate's gid loaded together with its
// coordinates (both loads in flight before the predicate): F(t, j, ok, g).
template <typename F>
__device__ __forceinline__ void scan_sorted_g(int64_t i, const float *__restrict__ x, int dim, float r2,
                                              const GridParams &p, const int32_t *__restrict__ start,
                                              const float4 *__restrict__ xs, const int64_t *__restrict__ gs, F &&f) {
  const int lane = threadIdx.x & 31;
  float xi[3] = {0.f, 0.f, 0.f};
  for (int d = 0; d < dim; ++d) xi[d] = x[i * dim + d];
  int c[3] = {0, 0, 0};
  for (int d = 0; d < dim; ++d) c[d] = cell_coord(xi[d], p.lo[d], p.inv_h, p.n[d]);
  const int R = p.reach;
  const int z0 = dim == 3 ? max(c[2] - R, 0) : 0, z1 = dim == 3 ? min(c[2] + R, p.n[2] - 1) : 0;
  const int y0 = max(c[1] - R, 0), y1 = min(c[1] + R, p.n[1] - 1);
  const int x0 = max(c[0] - R, 0), x1 = min(c[0] + R, p.n[0] - 1);
  for (int cz = z0; cz <= z1; ++cz)
    for (int cy = y0; cy <= y1; ++cy) {
      const int base = (cz * p.n[1] + cy) * p.n[0];
      const int a = start[base + x0], b = start[base + x1 + 1];
      for (int t0 = a; t0 < b; t0 += 64) {
        const int ta = t0 + lane, tb = t0 + 32 + lane;
        const float4 pa = ta < b ? xs[ta] : make_float4(0.f, 0.f, 0.f, __int_as_float(-1));
        const float4 pb = tb < b ? xs[tb] : make_float4(0.f, 0.f, 0.f, __int_as_float(-1));
        const int64_t ga = ta < b ? __ldg(gs + ta) : 0, gb = tb < b ? __ldg(gs + tb) : 0;
        {
          const int j = __float_as_int(pa.w);
          const float xj[3] = {pa.x, pa.y, pa.z};
          f(ta, j, ta < b && j != i && within(xi, xj, dim, r2), ga);
        }
        if (t0 + 32 < b) {
          const int j = __float_as_int(pb.w);
          const float xj[3] = {pb.x, pb.y, pb.z};
          f(tb, j, tb < b && j != i && within(xi, xj, dim, r2), gb);
        }
      }
    }
}

__device__ unsigned long long g_graph_tests;  // candidate tests (fp32 predicate evaluations), dsmpnn_graph_stats

// pass 1: counts, deg = min(count, n_e), and for capped rows the boundary
// bin b* of the top-kHB key bits and the number `take` kept from it
template <bool HIST>
__global__ void __launch_bounds__(kGWarps * 32) count2_kernel(
    const float *__restrict__ x, const int64_t *__restrict__ gs, const int64_t *__restrict__ gid, int64_t n_dst,
    int dim, float r, int32_t n_e, uint64_t s0, const GridParams *__restrict__ gp, const int32_t *__restrict__ start,
    const float4 *__restrict__ xs, int32_t *__restrict__ counts, int64_t *__restrict__ deg, int2 *__restrict__ bnd,
    int64_t n_loc = 0, int cell_order = 0) {
  __shared__ uint32_t hist_all[HIST ? kGWarps : 1][HIST ? kHBins : 1];
  const GridParams p = *gp;
  const float r2 = __fmul_rn(r, r);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t *hist = hist_all[HIST ? w : 0];
  if (HIST)
    for (int q = lane; q < kHBins; q += 32) hist[q] = 0;
  __syncwarp();
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long nscan = 0;
  const int64_t n_iter = cell_order ? n_loc : n_dst;
  for (int64_t tt = warp; tt < n_iter; tt += nwarps) {
    const int64_t i = cell_order ? (int64_t)__float_as_int(xs[tt].w) : tt;  // rows in cell order: L1 reuse
    if (i >= n_dst) continue;
    const uint64_t si = HIST ? smx(s0 ^ (uint64_t)gid[i]) : 0;
    int cnt = 0;
    scan_sorted_g(i, x, dim, r2, p, start, xs, gs, [&](int, int jj, bool ok, int64_t gt) {
      if (HIST && ok) atomicAdd(&hist[key_edge(si, (uint64_t)gt) >> (64 - kHB)], 1u);
      cnt += __popc(__ballot_sync(0xffffffffu, ok));
      nscan += jj >= 0;
    });
    if (lane == 0) {
      if (counts) counts[i] = cnt;
      if (deg) deg[i] = cnt < n_e ? cnt : n_e;
    }
    if (HIST) {
      __syncwarp();
      constexpr int PER = kHBins / 32;
      if (cnt > n_e) {
        uint32_t sum = 0;
        for (int q = 0; q < PER; ++q) sum += hist[lane * PER + q];
        uint32_t incl = sum;
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += v;
        }
        const uint32_t excl = incl - sum;
        if ((int)excl < n_e && n_e <= (int)incl) {
          uint32_t c0 = excl;
          for (int q = 0; q < PER; ++q) {
            const uint32_t hq = hist[lane * PER + q];
            if ((int)(c0 + hq) >= n_e) {
              bnd[i] = make_int2(lane * PER + q, n_e - (int)c0);
              break;
            }
            c0 += hq;
          }
        }
      }
      __syncwarp();
      for (int q = lane; q < kHBins; q += 32) hist[q] = 0;
      __syncwarp();
    }
  }
  if (HIST) {  // one atomic per warp
    const unsigned int wsum = __reduce_add_sync(0xffffffffu, (unsigned int)nscan);
    if ((threadIdx.x & 31) == 0 && wsum) atomicAdd(&g_graph_tests, (unsigned long long)wsum);
  }
}

// pass 2 (capped rows select from the boundary bin; uncapped rows keep all)
__global__ void __launch_bounds__(kGWarps * 32) select2_kernel(
    const float *__restrict__ x, const int64_t *__restrict__ gs, const int64_t *__restrict__ gid, int64_t n_dst,
    int dim, float r, int32_t n_e, uint64_t s0, const GridParams *__restrict__ gp, const int32_t *__restrict__ start,
    const float4 *__restrict__ xs, const int32_t *__restrict__ counts, const int2 *__restrict__ bnd,
    const int64_t *__restrict__ row_ptr, int32_t *__restrict__ col, int32_t *__restrict__ fl_rows,
    int32_t *__restrict__ fl_n, int force_fallback, int64_t n_loc = 0, int cell_order = 0) {
  __shared__ int32_t Lt[kGWarps][kMaxNe];
  __shared__ int64_t Lg[kGWarps][kMaxNe];
  __shared__ uint64_t Bk[kGWarps][kCapB];
  __shared__ int32_t Bt[kGWarps][kCapB];
  const GridParams p = *gp;
  const float r2 = __fmul_rn(r, r);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t lt = (1u << lane) - 1u;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t n_iter = cell_order ? n_loc : n_dst;
  for (int64_t tt = warp; tt < n_iter; tt += nwarps) {
    const int64_t i = cell_order ? (int64_t)__float_as_int(xs[tt].w) : tt;
    if (i >= n_dst) continue;
    const int cnt = counts[i];
    const bool capped = cnt > n_e;
    const int2 bt = capped ? bnd[i] : make_int2(kHBins, 0);
    const uint64_t si = smx(s0 ^ (uint64_t)gid[i]);
    int nl = 0, nb = 0;
    scan_sorted_g(i, x, dim, r2, p, start, xs, gs, [&](int t, int, bool ok, int64_t gt) {
      uint32_t top = 0;
      uint64_t key = 0;
      if (ok && capped) {
        key = key_edge(si, (uint64_t)gt);
        top = (uint32_t)(key >> (64 - kHB));
      }
      const bool inL = ok && (!capped || (int)top < bt.x);
      const bool inB = ok && capped && (int)top == bt.x;
      const uint32_t mL = __ballot_sync(0xffffffffu, inL), mB = __ballot_sync(0xffffffffu, inB);
      if (inL) Lt[w][nl + __popc(mL & lt)] = t;
      if (inB) {
        const int q = nb + __popc(mB & lt);
        if (q < kCapB) {
          Bk[w][q] = key;
          Bt[w][q] = t;
        }
      }
      nl += __popc(mL);
      nb += __popc(mB);
    });
    if (nb > kCapB || (force_fallback && capped)) {  // finish this row with the general select
      if (lane == 0) fl_rows[atomicAdd(fl_n, 1)] = (int32_t)i;
      __syncwarp();
      continue;
    }
    __syncwarp();
    // the `take` smallest (key, gid) of the boundary bin
    for (int a0 = 0; a0 < nb; a0 += 32) {
      const int a = a0 + lane;
      bool keep = false;
      if (a < nb) {
        const uint64_t ka = Bk[w][a];
        int rank = 0;
        for (int b = 0; b < nb; ++b) {
          const uint64_t kb = Bk[w][b];
          rank += kb < ka || (kb == ka && gs[Bt[w][b]] < gs[Bt[w][a]]);
        }
        keep = rank < bt.y;
      }
      const uint32_t m = __ballot_sync(0xffffffffu, keep);
      if (keep) Lt[w][nl + __popc(m & lt)] = Bt[w][a];
      nl += __popc(m);
    }
    __syncwarp();
    for (int q = lane; q < nl; q += 32) Lg[w][q] = gs[Lt[w][q]];
    __syncwarp();
    const int64_t off = row_ptr[i];
    for (int a = lane; a < nl; a += 32) {
      const int64_t g = Lg[w][a];
      int rank = 0;
      for (int b = 0; b < nl; ++b) rank += Lg[w][b] < g;
      col[off + rank] = __float_as_int(xs[Lt[w][a]].w);
    }
    __syncwarp();
  }
}

// ------------------------------------------------------ one-pass path --
// graph1_kernel: the candidate scan of each row runs ONCE.  Besides the
// count and the histogram of the top kHB key bits, the warp keeps the
// candidates whose bin is <= T in a shared list, where T is the boundary bin
// of the histogram so far: the final boundary bin b* can only be lower (bins
// only gain counts), so no candidate the selection needs is ever dropped.
// When the list fills up, T is recomputed and the list compacted.  At the end
// of the row the kept set (all candidates of an uncapped row; bins < b* plus
// the `take` smallest (key, gid) of bin b* of a capped row) is ordered by gid
// (rank sort) and written to the row's n_e-wide slot of `tmp`; after the
// exclusive scan of the degrees a copy kernel packs the slots into col.  A
// list overflow (many equal top bits, not expected for hash keys) flags the
// row for the general radix select (select_kernel), as before.
constexpr int kG1Warps = 4;

__device__ __forceinline__ int warp_boundary_bin(const uint32_t *hist, int lane, int n_e, int *below) {
  // bin b with (count in bins < b) < n_e <= (count in bins <= b); lane owns 32 consecutive bins
  constexpr int PER = kHBins / 32;
  uint32_t sum = 0;
  for (int q = 0; q < PER; ++q) sum += hist[lane * PER + q];
  uint32_t incl = sum;
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  const uint32_t excl = incl - sum;
  int found = -1, bl = 0;
  if ((int)excl < n_e && n_e <= (int)incl) {
    uint32_t c0 = excl;
    for (int q = 0; q < PER; ++q) {
      const uint32_t hq = hist[lane * PER + q];
      if ((int)(c0 + hq) >= n_e) {
        found = lane * PER + q;
        bl = (int)c0;
        break;
      }
      c0 += hq;
    }
  }
  const uint32_t m = __ballot_sync(0xffffffffu, found >= 0);
  const int src = m ? __ffs(m) - 1 : 0;
  found = __shfl_sync(0xffffffffu, found, src);
  bl = __shfl_sync(0xffffffffu, bl, src);
  *below = bl;
  return found;
}

template <int kCap1>  // shared candidate list per warp
__global__ void __launch_bounds__(kG1Warps * 32, 6) graph1_kernel(
    const float *__restrict__ x, const int64_t *__restrict__ gs, const int64_t *__restrict__ gid, int64_t n_loc,
    int64_t n_dst,
    int dim, float r, int32_t n_e, uint64_t s0, const GridParams *__restrict__ gp, const int32_t *__restrict__ start,
    const float4 *__restrict__ xs, int32_t *__restrict__ counts, int64_t *__restrict__ deg, int32_t *__restrict__ tmp,
    int32_t *__restrict__ fl_rows, int32_t *__restrict__ fl_n, int force_fallback, unsigned long long *scanned,
    int cell_order) {
  __shared__ uint32_t hist_all[kG1Warps][kHBins];
  __shared__ int32_t lt_all[kG1Warps][kCap1];
  __shared__ uint64_t lk_all[kG1Warps][kCap1];
  __shared__ int32_t kj_all[kG1Warps][kMaxNe];
  __shared__ int64_t kg_all[kG1Warps][kMaxNe];
  const GridParams p = *gp;
  const float r2 = __fmul_rn(r, r);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t lt_mask = (1u << lane) - 1u;
  uint32_t *hist = hist_all[w];
  int32_t *lt = lt_all[w];
  uint64_t *lk = lk_all[w];
  int32_t *kj = kj_all[w];
  int64_t *kg = kg_all[w];
  unsigned long long nscan = 0;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // rows in cell order: the warps of a block (and neighbouring blocks) scan
  // overlapping cells, so candidate loads hit in L1; halo points are skipped
  const int64_t n_iter = cell_order ? n_loc : n_dst;
  for (int64_t tt = warp; tt < n_iter; tt += nwarps) {
    const int64_t i = cell_order ? (int64_t)__float_as_int(xs[tt].w) : tt;
    if (i >= n_dst) continue;
    for (int q = lane; q < kHBins; q += 32) hist[q] = 0;
    __syncwarp();
    const uint64_t si = smx(s0 ^ (uint64_t)gid[i]);
    int cnt = 0, ns = 0, T = kHBins - 1;
    bool overflow = false;
    scan_sorted_g(i, x, dim, r2, p, start, xs, gs, [&](int t, int jj, bool ok, int64_t gt) {
      uint64_t key = 0;
      int bin = kHBins;
      if (ok) {
        key = key_edge(si, (uint64_t)gt);
        bin = (int)(key >> (64 - kHB));
        // bins above T can no longer hold b*: their counts are never needed
        if (bin <= T) atomicAdd(&hist[bin], 1u);
      }
      nscan += jj >= 0;
      cnt += __popc(__ballot_sync(0xffffffffu, ok));
      const bool keep = ok && bin <= T;
      const uint32_t m = __ballot_sync(0xffffffffu, keep);
      if (keep) {
        const int q = ns + __popc(m & lt_mask);
        if (q < kCap1) {
          lt[q] = t;
          lk[q] = key;
        }
      }
      ns += __popc(m);
      if (ns > kCap1 - 64 && !overflow) {  // lower T to the boundary bin so far and compact the list
        __syncwarp();
        if (cnt > n_e) {
          int below;
          T = warp_boundary_bin(hist, lane, n_e, &below);
          int nk = 0;
          const int n0 = min(ns, kCap1);
          for (int a0 = 0; a0 < n0; a0 += 32) {
            const int a = a0 + lane;
            int ta = 0;
            uint64_t ka = 0;
            bool k2 = false;
            if (a < n0) {
              ta = lt[a];
              ka = lk[a];
              k2 = (int)(ka >> (64 - kHB)) <= T;
            }
            __syncwarp();
            const uint32_t m2 = __ballot_sync(0xffffffffu, k2);
            if (k2) {
              const int q = nk + __popc(m2 & lt_mask);
              lt[q] = ta;
              lk[q] = ka;
            }
            nk += __popc(m2);
            __syncwarp();
          }
          ns = nk;
        }
        if (ns > kCap1 - 64) overflow = true;  // keep counting; the general select finishes the row
      }
    });
    __syncwarp();
    if (lane == 0) {
      counts[i] = cnt;
      deg[i] = cnt < n_e ? cnt : n_e;
    }
    if (overflow || ns > kCap1 || (force_fallback && cnt > n_e)) {
      if (lane == 0) fl_rows[atomicAdd(fl_n, 1)] = (int32_t)i;
      __syncwarp();
      continue;
    }
    // the kept set: everything (uncapped), or bins < b* plus the `take` smallest (key, gid) of bin b*
    int bstar = kHBins, take = 0;
    if (cnt > n_e) {
      int below;
      bstar = warp_boundary_bin(hist, lane, n_e, &below);
      take = n_e - below;
    }
    int nk = 0;
    for (int a0 = 0; a0 < ns; a0 += 32) {
      const int a = a0 + lane;
      bool keep = false;
      int ta = 0;
      if (a < ns) {
        ta = lt[a];
        const uint64_t ka = lk[a];
        const int ba = (int)(ka >> (64 - kHB));
        if (ba < bstar) {
          keep = true;
        } else if (ba == bstar) {
          const uint64_t ga = (uint64_t)gs[ta];
          int rank = 0;
          for (int b = 0; b < ns; ++b) {
            const uint64_t kb = lk[b];
            if ((int)(kb >> (64 - kHB)) != bstar) continue;
            rank += kb < ka || (kb == ka && (uint64_t)gs[lt[b]] < ga);
          }
          keep = rank < take;
        }
      }
      const uint32_t m = __ballot_sync(0xffffffffu, keep);
      if (keep) {
        const int q = nk + __popc(m & lt_mask);
        kj[q] = __float_as_int(xs[ta].w);
        kg[q] = gs[ta];
      }
      nk += __popc(m);
    }
    __syncwarp();
    // order the row by gid (R11): rank sort, write the row's slot of tmp
    for (int a = lane; a < nk; a += 32) {
      const int64_t g = kg[a];
      int rank = 0;
      for (int b = 0; b < nk; ++b) rank += kg[b] < g;
      tmp[i * (int64_t)n_e + rank] = kj[a];
    }
    __syncwarp();
  }
  {  // candidate tests (predicate evaluations), one atomic per warp
    const unsigned int wsum = __reduce_add_sync(0xffffffffu, (unsigned int)nscan);
    if (lane == 0 && wsum) atomicAdd(scanned ? scanned : &g_graph_tests, (unsigned long long)wsum);
  }
}

// col[row_ptr[i] + k] = tmp[i * n_e + k], k < deg_i (rows finished by the general select are skipped)
__global__ void pack_rows_kernel(const int32_t *__restrict__ tmp, const int64_t *__restrict__ row_ptr,
                                 const int32_t *__restrict__ counts, int64_t n_dst, int32_t n_e,
                                 int32_t *__restrict__ col) {
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (int64_t i = warp; i < n_dst; i += nwarps) {
    const int64_t a = row_ptr[i], d = row_ptr[i + 1] - a;
    for (int k = lane; k < d; k += 32) col[a + k] = tmp[i * (int64_t)n_e + k];
  }
}

static int64_t max_cells_for(int64_t n_loc) { return std::max<int64_t>(4 * n_loc, 4096); }

static size_t graph_ws(int64_t n_loc, int64_t n_dst, size_t *sort_tmp, size_t *scan_tmp) {
  cub::DeviceRadixSort::SortPairs(nullptr, *sort_tmp, (const int32_t *)nullptr, (int32_t *)nullptr,
                                  (const int32_t *)nullptr, (int32_t *)nullptr, (int)n_loc);
  cub::DeviceScan::ExclusiveSum(nullptr, *scan_tmp, (const int64_t *)nullptr, (int64_t *)nullptr, (int)(n_dst + 1));
  Carver c(nullptr, 0);
  c.take<float>(8);
  c.take<GridParams>(1);
  c.take<int32_t>(n_loc); c.take<int32_t>(n_loc); c.take<int32_t>(n_loc); c.take<int32_t>(n_loc);
  c.take<int32_t>(max_cells_for(n_loc) + 1);
  c.take<int32_t>(n_dst);
  c.take<int64_t>(n_dst + 1);
  c.take<float4>(n_loc);
  c.take<int64_t>(n_loc);
  c.take<int2>(n_dst);
  c.take<int32_t>(n_dst + 1);
  c.take<char>(*sort_tmp);
  c.take<char>(*scan_tmp);
  c.take<int32_t>(n_dst * (int64_t)kMaxNe);  // one-pass row slots
  c.take<unsigned long long>(2);
  return c.used();
}

struct GraphState {
  GridParams *gp;
  int32_t *sorted_idx, *start, *counts;
  int64_t *deg;
  float4 *xs;
  int64_t *gs;
  int2 *bnd;
  int32_t *fl;  // [0] = count, [1..] = rows
  void *scan_tmp;
  size_t scan_bytes;
  int32_t *tmp;                  // [n_dst x n_e] row slots of the one-pass kernel
  unsigned long long *scanned;   // candidate tests of the last build (diagnostics)
};

static dsmpnn_status build_cells(const float *coords, const int64_t *gid, int64_t n_loc, int64_t n_dst, int dim,
                                 float r, void *ws, size_t ws_bytes, cudaStream_t s, GraphState &st) {
  size_t sort_tmp, scan_tmp;
  size_t need = graph_ws(n_loc, n_dst, &sort_tmp, &scan_tmp);
  DS_CHECK_ARG(ws_bytes >= need, DSMPNN_ERR_CAPACITY, "radius_graph: workspace %zu < %zu", ws_bytes, need);
  Carver c(ws, ws_bytes);
  float *bb = c.take<float>(8);
  st.gp = c.take<GridParams>(1);
  int32_t *cell = c.take<int32_t>(n_loc), *cell_sorted = c.take<int32_t>(n_loc);
  int32_t *idx = c.take<int32_t>(n_loc);
  st.sorted_idx = c.take<int32_t>(n_loc);
  int64_t maxc = max_cells_for(n_loc);
  st.start = c.take<int32_t>(maxc + 1);
  st.counts = c.take<int32_t>(n_dst);
  st.deg = c.take<int64_t>(n_dst + 1);
  st.xs = c.take<float4>(n_loc);
  st.gs = c.take<int64_t>(n_loc);
  st.bnd = c.take<int2>(n_dst);
  st.fl = c.take<int32_t>(n_dst + 1);
  void *t1 = c.take<char>(sort_tmp);
  st.scan_tmp = c.take<char>(scan_tmp);
  st.scan_bytes = scan_tmp;
  st.tmp = c.take<int32_t>(n_dst * (int64_t)kMaxNe);
  st.scanned = c.take<unsigned long long>(2);
  bbox_kernel<<<1, 1024, 0, s>>>(coords, n_loc, dim, bb);
  // cell edge r(1+2^-8)/kReach: kReach cells on each side cover r with a margin
  // for the rounding of the cell index; smaller cells scan less area per row
  // ((2 kReach + 1)^dim cells of edge r/kReach: 6.25 r^2 instead of 9 r^2 in 2-D)
  float h0 = r * 1.00390625f / (float)kReach;
  grid_params_kernel<<<1, 1, 0, s>>>(bb, dim, h0, maxc, st.gp);
  int g = (int)std::min<int64_t>(ceil_div(n_loc, 256), 148 * 8);
  cell_id_kernel<<<g, 256, 0, s>>>(coords, n_loc, dim, st.gp, cell, idx);
  DS_LAUNCH_CHECK();
  int end_bit = 1;
  while ((1ll << end_bit) <= maxc) ++end_bit;
  DS_CUDA(cub::DeviceRadixSort::SortPairs(t1, sort_tmp, cell, cell_sorted, idx, st.sorted_idx, (int)n_loc, 0,
                                          end_bit, s));
  cell_start_kernel<<<(int)std::min<int64_t>(ceil_div(maxc + 1, 256), 148 * 8), 256, 0, s>>>(cell_sorted, n_loc,
                                                                                            st.gp, st.start, maxc);
  DS_LAUNCH_CHECK();
  permute_points_kernel<<<g, 256, 0, s>>>(coords, gid, n_loc, dim, st.sorted_idx, st.xs, gid ? st.gs : nullptr);
  DS_LAUNCH_CHECK();
  return DSMPNN_OK;
}

}  // namespace dsmpnn

using namespace dsmpnn;

extern "C" {

dsmpnn_status dsmpnn_graph_stats(uint64_t *candidate_tests, int32_t reset) {
  unsigned long long v = 0;
  DS_CUDA(cudaMemcpyFromSymbol(&v, g_graph_tests, sizeof(v)));
  if (candidate_tests) *candidate_tests = v;
  if (reset) {
    const unsigned long long z = 0;
    DS_CUDA(cudaMemcpyToSymbol(g_graph_tests, &z, sizeof(z)));
  }
  return DSMPNN_OK;
}

dsmpnn_status dsmpnn_radius_graph_workspace_size(int64_t n_loc, int64_t n_dst, int dim, size_t *bytes) {
  DS_CHECK_ARG(n_loc >= 0 && n_dst >= 0 && n_dst <= n_loc && n_loc < (1ll << 31), DSMPNN_ERR_INVALID_ARG,
               "radius_graph: sizes");
  size_t a, b;
  *bytes = graph_ws(n_loc, n_dst, &a, &b);
  return DSMPNN_OK;
}

dsmpnn_status dsmpnn_radius_counts(const float *coords, int64_t n_loc, int64_t n_dst, int dim, float r,
                                   int32_t *counts, void *ws, size_t ws_bytes, void *stream) {
  DS_CHECK_ARG(r > 0.f && (dim == 2 || dim == 3) && n_dst <= n_loc && n_loc < (1ll << 31), DSMPNN_ERR_INVALID_ARG,
               "radius_counts: bad arguments");
  if (n_dst == 0) return DSMPNN_OK;
  cudaStream_t s = as_stream(stream);
  GraphState st;
  DS_TRY(build_cells(coords, nullptr, n_loc, n_dst, dim, r, ws, ws_bytes, s, st));
  int blocks = (int)std::min<int64_t>(ceil_div(n_dst, kGWarps), 148 * 16);
  count2_kernel<false><<<blocks, kGWarps * 32, 0, s>>>(coords, nullptr, nullptr, n_dst, dim, r, 1, 0, st.gp, st.start,
                                                       st.xs, counts, nullptr, nullptr);
  DS_LAUNCH_CHECK();
  return DSMPNN_OK;
}

dsmpnn_status dsmpnn_radius_graph(const float *coords, const int64_t *gid, int64_t n_loc, int64_t n_dst, int dim,
                                  float r, int32_t n_e, uint64_t seed, int64_t *row_ptr, int32_t *col_idx,
                                  int64_t col_capacity, int64_t *n_edges, void *ws, size_t ws_bytes, void *stream) {
  DS_CHECK_ARG(r > 0.f, DSMPNN_ERR_INVALID_ARG, "radius_graph: r must be > 0");
  DS_CHECK_ARG(n_e >= 1, DSMPNN_ERR_INVALID_ARG, "radius_graph: n_e must be >= 1");
  DS_CHECK_ARG(n_e <= kMaxNe, DSMPNN_ERR_UNSUPPORTED, "radius_graph: n_e <= %d supported", kMaxNe);
  DS_CHECK_ARG(dim == 2 || dim == 3, DSMPNN_ERR_INVALID_ARG, "radius_graph: dim must be 2 or 3");
  DS_CHECK_ARG(n_loc >= 0 && n_dst >= 0 && n_dst <= n_loc && n_loc < (1ll << 31), DSMPNN_ERR_INVALID_ARG,
               "radius_graph: need 0 <= n_dst <= n_loc < 2^31");
  cudaStream_t s = as_stream(stream);
  if (n_dst == 0) {
    DS_CUDA(cudaMemsetAsync(row_ptr, 0, sizeof(int64_t), s));
    if (n_edges) *n_edges = 0;
    return DSMPNN_OK;
  }
  if (!n_edges)
    DS_CHECK_ARG(col_capacity >= n_dst * (int64_t)n_e, DSMPNN_ERR_CAPACITY,
                 "radius_graph: without n_edges, col_capacity must be >= n_dst*n_e");
  GraphState st;
  DS_TRY(build_cells(coords, gid, n_loc, n_dst, dim, r, ws, ws_bytes, s, st));
  const uint64_t s0 = smx(seed);
  const bool force_fb = getenv("DSMPNN_TEST_GRAPH_FALLBACK") != nullptr;
  // One pass (graph1, rows in cell order) or two passes (count2 + select2,
  // rows in index order).  Measured per Darcy sub-domain (4.1k rows, index
  // order already spatially coherent): two passes 441 us, one pass 618 us;
  // airfoil (25k rows per sub-domain, unordered cloud, up to 12k candidates
  // per row): one pass 14.4 ms, two passes 22 ms per build of 8; step: 2.95 vs
  // 3.3 ms.  Both give the same graph bit for bit; the choice is by size.
  // DSMPNN_GRAPH_TWO_PASS=0|1 forces one (A/B timing).
  static const int force_tp = getenv("DSMPNN_GRAPH_TWO_PASS") ? atoi(getenv("DSMPNN_GRAPH_TWO_PASS")) : -1;
  const bool two_pass = force_tp >= 0 ? force_tp != 0 : n_dst < 16384;
  int blocks = (int)std::min<int64_t>(ceil_div(n_dst, kGWarps), 148 * 16);
  // rows of the two-pass kernels in index order (cell order with DSMPNN_GRAPH_ROWORDER=1)
  static const int roworder2 = getenv("DSMPNN_GRAPH_ROWORDER") ? atoi(getenv("DSMPNN_GRAPH_ROWORDER")) : 0;
  const int roworder = 1;
  const int blocks2 = (int)std::min<int64_t>(ceil_div(roworder2 ? n_loc : n_dst, kGWarps), 148 * 16);
  DS_CUDA(cudaMemsetAsync(st.fl, 0, sizeof(int32_t), s));
  DS_CUDA(cudaMemsetAsync(st.deg + n_dst, 0, sizeof(int64_t), s));
  if (!two_pass) {
    const int blocks1 = (int)std::min<int64_t>(ceil_div(n_loc, kG1Warps), 148 * 32);
    static const int cap = getenv("DSMPNN_GRAPH_CAP") ? atoi(getenv("DSMPNN_GRAPH_CAP")) : 320;
    auto k1 = cap >= 512 ? graph1_kernel<512> : graph1_kernel<320>;
    k1<<<blocks1, kG1Warps * 32, 0, s>>>(coords, st.gs, gid, n_loc, n_dst, dim, r, n_e, s0, st.gp, st.start,
                                                   st.xs,
                                                   st.counts, st.deg, st.tmp, st.fl + 1, st.fl, force_fb ? 1 : 0,
                                                   nullptr, roworder);
  } else {
    count2_kernel<true><<<blocks2, kGWarps * 32, 0, s>>>(coords, st.gs, gid, n_dst, dim, r, n_e, s0, st.gp, st.start,
                                                         st.xs, st.counts, st.deg, st.bnd, n_loc, roworder2);
  }
  DS_LAUNCH_CHECK();
  size_t sb = st.scan_bytes;
  DS_CUDA(cub::DeviceScan::ExclusiveSum(st.scan_tmp, sb, st.deg, row_ptr, (int)(n_dst + 1), s));
  if (n_edges) {
    DS_CUDA(cudaMemcpyAsync(n_edges, row_ptr + n_dst, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    DS_CUDA(cudaStreamSynchronize(s));
    if (*n_edges > col_capacity) {
      set_error("radius_graph: col_capacity %lld < E %lld", (long long)col_capacity, (long long)*n_edges);
      return DSMPNN_ERR_CAPACITY;
    }
  }
  if (!two_pass) {
    pack_rows_kernel<<<(int)std::min<int64_t>(ceil_div(n_dst, 8), 148 * 16), 256, 0, s>>>(st.tmp, row_ptr, st.counts,
                                                                                         n_dst, n_e, col_idx);
  } else {
    select2_kernel<<<blocks2, kGWarps * 32, 0, s>>>(coords, st.gs, gid, n_dst, dim, r, n_e, s0, st.gp, st.start, st.xs,
                                                   st.counts, st.bnd, row_ptr, col_idx, st.fl + 1, st.fl, force_fb, n_loc,
                                                   roworder2);
  }
  DS_LAUNCH_CHECK();
  // rows whose boundary bin overflowed (row list on the device; usually empty)
  select_kernel<<<148, kSelWarps * 32, 0, s>>>(coords, gid, n_dst, dim, r, n_e, s0, st.gp, st.start, st.sorted_idx,
                                               st.counts, row_ptr, col_idx, st.fl + 1, st.fl);
  DS_LAUNCH_CHECK();
  return DSMPNN_OK;
}

}  // extern "C"

/*
 * dsmpnn.h - C ABI of libdsmpnn.so, the B200 (sm_100a) hot path of DS-MPNN
 * (arXiv 2402.15106): the edge-conditioned message-passing layer on
 * ball-radius graphs over Nystrom-sampled nodes of overlapping sub-domains.
 *
 * Citations are PAPER.md:<line> of the paper's LaTeX source; "R<n>" are the
 * readings listed in DESIGN.md §2.
 *
 * Conventions (all calls):
 *  - Every call returns dsmpnn_status; DSMPNN_OK == 0.  On error, a text is
 *    available from dsmpnn_last_error() (thread-local).  No call aborts.
 *  - Pointers are DEVICE pointers unless the argument says "host".  The caller
 *    owns every buffer (it allocates them, e.g. with PyTorch); the library never
 *    frees or retains them past the enqueued work.
 *  - `stream` is a cudaStream_t passed as void*; NULL is the legacy default
 *    stream.  Calls are stream-ordered and asynchronous, except where a
 *    "host" output is requested (then the call synchronises `stream`).
 *  - Layouts are row-major and contiguous.  Index types: int64 row_ptr and
 *    global ids, int32 local column indices.
 *  - Workspace: calls that need scratch take (ws, ws_bytes) sized by the
 *    matching *_workspace_size query; DSMPNN_ERR_CAPACITY is returned if it
 *    is too small.
 *  - Determinism: equal inputs give bit-equal outputs on every run (no
 *    floating-point atomics on any result).
 */
#ifndef DSMPNN_H
#define DSMPNN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  DSMPNN_OK = 0,
  DSMPNN_ERR_INVALID_ARG = -1, /* r<=0, s<1, n_e<1, P not 2^m or P>n, dim not 2/3, ... */
  DSMPNN_ERR_SHAPE = -2,       /* width mismatch, ROOT_IDENTITY with d_in!=d_out, misalignment */
  DSMPNN_ERR_INDEX = -3,       /* index out of range */
  DSMPNN_ERR_CAPACITY = -4,    /* output or workspace buffer too small */
  DSMPNN_ERR_CUDA = -5,        /* a CUDA runtime error (text in dsmpnn_last_error) */
  DSMPNN_ERR_NCCL = -6,        /* an NCCL error, or a communicator aborted by the watchdog */
  DSMPNN_ERR_TIMEOUT = -7,     /* dsmpnn_ctx_sync: the exchange did not finish in time (communicator aborted) */
  DSMPNN_ERR_UNSUPPORTED = -8, /* shape/dtype combination not implemented */
  DSMPNN_ERR_DEGENERATE = -9   /* RCB split leaves an empty side (R12) */
} dsmpnn_status;

typedef enum { DSMPNN_F32 = 0, DSMPNN_BF16 = 1 } dsmpnn_dtype;
typedef enum { DSMPNN_ROOT_NONE = 0, DSMPNN_ROOT_IDENTITY = 1, DSMPNN_ROOT_DENSE = 2 } dsmpnn_root;
typedef enum { DSMPNN_ACT_IDENTITY = 0, DSMPNN_ACT_RELU = 1 } dsmpnn_act;
typedef enum { DSMPNN_EDGE_DIFF = 0, DSMPNN_EDGE_CONCAT = 1 } dsmpnn_edge_mode;

/* Layer description.  kappa_phi (R5) = Linear(d_e,k) -> ReLU -> Linear(k,k)
 * -> ReLU -> Linear(k, d_in*d_out); K[c][o] = kappa_out[c*d_out+o] (R4). */
typedef struct {
  int32_t d_e, d_in, d_out, k;
  int32_t dtype; /* dsmpnn_dtype: F32 = fp32 SIMT arithmetic; BF16 = tcgen05 bf16 MMA, fp32 accumulate */
  int32_t root;  /* dsmpnn_root (R2) */
  int32_t act;   /* dsmpnn_act (R1) */
  int32_t reserved;
} dsmpnn_layer_desc;

/* fp32 master weights in PyTorch Linear layout [out, in] (device). */
typedef struct {
  const float *W1, *b1;         /* [k x d_e], [k] */
  const float *W2, *b2;         /* [k x k], [k] */
  const float *W3, *b3;         /* [d_in*d_out x k], [d_in*d_out] */
  const float *W_root, *b;      /* [d_out x d_in] (ROOT_DENSE only, else may be NULL), [d_out] */
  const void *packed;           /* BF16 mode: buffer filled by dsmpnn_pack_weights (required) */
} dsmpnn_weights;

/* fp32 weight gradients, ACCUMULATED (+=) by dsmpnn_layer_bwd. Any may be NULL. */
typedef struct {
  float *W1, *b1, *W2, *b2, *W3, *b3, *W_root, *b;
} dsmpnn_grads;

const char *dsmpnn_last_error(void);
int32_t dsmpnn_version(void);

/* ------------------------------------------------------------------ a1 --- */
/* Nystrom node sampling ("randomly sampling nodes, |V_s| = s";
 * Alg. 1 :391).  R9: the min(s,N) ids g in [0,N) with the smallest
 * (key_node(seed,g), g), key_node = smx(smx(seed) ^ g), written ascending.
 * ids: int32[min(s,N)].  Errors: s < 1 or N < 0 -> INVALID_ARG. */
dsmpnn_status dsmpnn_sample_workspace_size(int64_t n_points, size_t *bytes /*host*/);
dsmpnn_status dsmpnn_sample(int64_t n_points, int64_t s, uint64_t seed, int32_t *ids,
                            void *ws, size_t ws_bytes, void *stream);

/* ------------------------------------------------------------------ a2 --- */
/* Radius graph kernel + random edge cap (Alg. 1 :395-396).
 * For each destination row i < n_dst: candidates C_i = {j < n_loc, j != i :
 * pred_fp32(x_i, x_j, r)} (R7, inclusive, no FMA); if |C_i| > n_e keep the n_e
 * smallest (key_edge(seed, gid_i, gid_j), gid_j) (R10); the row is ordered by
 * gid_j ascending (R11).  Cell-list search over cells of edge r(1+2^-8).
 *   coords   float32[n_loc x dim] (dim 2 or 3), local order
 *   gid      int64[n_loc] global ids (unique)
 *   row_ptr  int64[n_dst+1] (out), col_idx int32[col_capacity] (out, local ids)
 *   n_edges  host int64 out (may be NULL: then the call stays asynchronous and
 *            row_ptr[n_dst] holds the count); if col_capacity < E the call
 *            returns CAPACITY and *n_edges holds E (requires n_edges != NULL).
 * Errors: r <= 0, n_e < 1, dim not in {2,3}, n_dst > n_loc -> INVALID_ARG. */
dsmpnn_status dsmpnn_radius_graph_workspace_size(int64_t n_loc, int64_t n_dst, int dim, size_t *bytes);
dsmpnn_status dsmpnn_radius_graph(const float *coords, const int64_t *gid, int64_t n_loc, int64_t n_dst,
                                  int dim, float r, int32_t n_e, uint64_t seed, int64_t *row_ptr,
                                  int32_t *col_idx, int64_t col_capacity, int64_t *n_edges /*host*/,
                                  void *ws, size_t ws_bytes, void *stream);

/* Diagnostics of the radius-graph search: the number of candidate tests (fp32
 * predicate evaluations) of dsmpnn_radius_graph calls since the last reset,
 * summed over calls and devices' default context (synchronising read).
 * candidate_tests: host uint64 out (may be NULL); reset != 0 zeroes the counter. */
dsmpnn_status dsmpnn_graph_stats(uint64_t *candidate_tests /*host*/, int32_t reset);

/* Candidate counts |C_i| (pre-cap) per destination row; same search as above.
 * counts int32[n_dst].  Used for diagnostics and tests. */
dsmpnn_status dsmpnn_radius_counts(const float *coords, int64_t n_loc, int64_t n_dst, int dim, float r,
                                   int32_t *counts, void *ws, size_t ws_bytes, void *stream);

/* CSC view of a CSR graph for deterministic scatters (backward a7):
 * csc_perm int32[E] = edge ids sorted by (col_idx, edge id); csc_ptr int64[n_loc+1]. */
dsmpnn_status dsmpnn_csc_workspace_size(int64_t n_edges, int64_t n_loc, size_t *bytes);
dsmpnn_status dsmpnn_csc(const int32_t *col_idx, int64_t n_edges, int64_t n_loc, int32_t *csc_perm,
                         int64_t *csc_ptr, void *ws, size_t ws_bytes, void *stream);

/* ------------------------------------------------------------------ a3 --- */
/* Domain decomposition with overlap l ("extended overlap of
 * length l", :70 "equally partitioned based on their coordinates"; Alg. 1
 * :392, :403).  R12 median RCB on the longest axis, ties to the lower rank;
 * R13 closed L-inf box extension by l; R23 near/deep split at
 * t = fl(max(l,r)(1+2^-10)) from internal faces.  Computes the plan of `rank`:
 *   owner      int32[n]            owner rank of every sampled point
 *   boxes      float32[P x 2 x dim] lo/hi per rank
 *   internal   uint8[P x 2 x dim]   1 if that face was created by a split
 *   local_rows int64[n] (capacity)  indices into the n points, local order
 *                                   deep (gid asc) | near (gid asc) | halo (owner asc, gid asc)
 *   counts     int64[4 + 2(P+1)]    n_deep, n_near, n_halo, n_send_total,
 *                                   halo_ptr[P+1] (absolute local rows, halo_ptr[0] = n_own),
 *                                   send_ptr[P+1] (offsets into send_idx)
 *   send_idx   int32[n*(P-1)] (capacity; n if P == 1): local rows sent to each q,
 *                                   q ascending, gid ascending within q
 *   counts_host host int64[4 + 2(P+1)] copy of counts (may be NULL: asynchronous)
 * Errors: P not a power of two or P > n, l < 0, r <= 0 -> INVALID_ARG;
 * DEGENERATE if a split leaves an empty side (only detected when
 * counts_host != NULL, which synchronises). */
dsmpnn_status dsmpnn_partition_workspace_size(int64_t n, int dim, int nparts, size_t *bytes);
dsmpnn_status dsmpnn_partition(const float *coords, const int64_t *gid, int64_t n, int dim, int nparts,
                               float overlap_l, float radius, int rank, int32_t *owner, float *boxes,
                               uint8_t *internal, int64_t *local_rows, int64_t *counts, int32_t *send_idx,
                               int64_t *counts_host, void *ws, size_t ws_bytes, void *stream);

/* The plans of ALL P ranks from one RCB, with no host synchronisation (the
 * same arithmetic and outputs as P calls of dsmpnn_partition):
 *   owner, boxes, internal   as above
 *   local_rows int64[P x n]               rank q's local order at q*n
 *   counts     int64[P x (5 + 2(P+1))]    rank q's counts at q*(5+2(P+1)), as above,
 *                                         followed by the DEGENERATE flag (nonzero: a
 *                                         split left an empty side; the caller checks
 *                                         it after synchronising)
 *   send_idx   int32[P x n*max(1,P-1)]    rank q's send lists at q*n*max(1,P-1)
 *   gid_bits   0, or b in 1..52 with every gid < 2^b: the plan's radix sorts
 *              then use b+9 / b+7 key bits instead of 61 / 59.
 * Workspace: dsmpnn_partition_workspace_size.  Errors as dsmpnn_partition
 * (DEGENERATE is reported through the flag). */
dsmpnn_status dsmpnn_partition_all(const float *coords, const int64_t *gid, int64_t n, int dim, int nparts,
                                   float overlap_l, float radius, int32_t gid_bits, int32_t *owner, float *boxes,
                                   uint8_t *internal, int64_t *local_rows, int64_t *counts, int32_t *send_idx,
                                   void *ws, size_t ws_bytes, void *stream);

/* Gather rows (local order) of a float32 array: out[k] = in[rows[k]].  Used to
 * form local coordinates / attributes / global ids from a plan. elem_bytes 4 or 8. */
dsmpnn_status dsmpnn_gather_rows(const void *in, const int64_t *rows, int64_t n_rows, int64_t row_elems,
                                 int32_t elem_bytes, void *out, void *stream);

/* The same gather from float32 rows into bfloat16 rows, rounded to nearest
 * even (the BF16 mode's layer-0 operand); rows may be NULL
 * (then row k is row k). */
dsmpnn_status dsmpnn_gather_rows_bf16(const float *in, const int64_t *rows, int64_t n_rows, int64_t row_elems,
                                      void *out, void *stream);

/* Edge attributes ("relative difference between node coordinates
 * and attributes"; Alg. 1 :397; R21).  For edge p of row i with source j:
 *   DIFF:   e_p = (x_i - x_j, a_i - a_j)            d_e = dim + n_attr
 *   CONCAT: e_p = (x_i, x_j, a_i, a_j)              d_e = 2(dim + n_attr)
 * Each value is one fp32 operation or a copy.  Writes e32 float32[E x d_e]
 * and/or e16 bf16[E x 16] (zero-padded to 16 columns; d_e <= 16), either may be NULL. */
dsmpnn_status dsmpnn_edge_features(int32_t mode, const float *coords, int dim, const float *attr, int n_attr,
                                   const int64_t *row_ptr, const int32_t *col_idx, int64_t n_dst,
                                   int64_t n_edges, float *e32, void *e16, void *stream);

/* -------------------------------------------------------------- a4 + a5 --- */
/* Bytes of the bf16 packed-weight buffer, and packing (BF16 mode). */
dsmpnn_status dsmpnn_packed_weights_size(const dsmpnn_layer_desc *desc, size_t *bytes);
dsmpnn_status dsmpnn_pack_weights(const dsmpnn_layer_desc *desc, const dsmpnn_weights *w, void *packed,
                                  size_t bytes, void *stream);

/* Layer forward, Eq. (1) / eq. (ii) (:40) with Alg. 1's residual
 * (:407-409) and the north_star root/sigma (R1-R5):
 *   out_i = sigma( [deg_i>0] (1/deg_i) sum_{p in row i} K_p^T v_{j(p)} + root(v_i) + b )
 * for destination rows [row_begin, row_end).  K_p is never materialised: the
 * row sum is contracted as vec(sum_p h~_p (x) v_j) . Theta~.
 *   v        [n_loc x d_in]  fp32 (F32) or bf16 (BF16); rows 0..n_dst-1 are the destinations
 *   e        [E x d_e] fp32 (F32) or [E x 16] bf16 zero-padded (BF16)
 *   row_ptr  int64[n_dst+1] device; row_ptr_host: host copy (may be NULL: then the
 *            call reads row_ptr[row_begin], row_ptr[row_end] synchronously)
 *   col_idx  int32[E]
 *   out      float32[n_dst x d_out] (rows row_begin.. written)
 *   out_lowp bf16[n_dst x d_out] copy of out, or NULL
 *   ws       saved activations for dsmpnn_layer_bwd, sized by
 *            dsmpnn_layer_workspace_size(desc, n_dst, E); pass the same ws to bwd.
 * Errors: SHAPE for ROOT_IDENTITY with d_in != d_out or BF16 with d_e > 13 (the
 * padded edge columns 13..15 carry the first kappa layer bias, layer_bf16.cu);
 * UNSUPPORTED for BF16 widths other than d_in = d_out in {32, 64} and k <= 256
 * (the BF16 kernels run k = 256; a smaller k is zero-padded to 256 by
 * dsmpnn_pack_weights: the padded units are exact zeros, the results and
 * gradients are those of width k, the cost that of width 256), and for a BF16 call whose rows [row_begin, row_end) include a row of more
 * than 128 edges (the fused edge kernels tile whole rows; checked on the host
 * from row_ptr_host, else from row_ptr with a synchronising scan).
 * With DSMPNN_DEBUG set in the environment, layer_fwd / layer_bwd also
 * validate the CSR (row_ptr non-decreasing, 0 <= col_idx < n_loc) and return
 * INDEX on a violation (synchronising). */
dsmpnn_status dsmpnn_layer_workspace_size(const dsmpnn_layer_desc *desc, int64_t n_dst, int64_t n_edges,
                                          size_t *bytes);
dsmpnn_status dsmpnn_layer_fwd(const dsmpnn_layer_desc *desc, const dsmpnn_weights *w, const void *v,
                               const void *e, const int64_t *row_ptr, const int64_t *row_ptr_host,
                               const int32_t *col_idx, int64_t n_dst, int64_t row_begin, int64_t row_end,
                               float *out, void *out_lowp, void *ws, size_t ws_bytes, void *stream);

/* ------------------------------------------------------------------ a7 --- */
/* Layer backward (Alg. 1 :417 "Backprop", local gradients; R16 detach).
 * Given grad_out = dL/dout (fp32 [n_dst x d_out], rows [row_begin,row_end)
 * used), accumulates:
 *   grad_v [n_loc x d_in] fp32  +=  dL/dv (root term on destination rows and
 *                                   messages on source rows, incl. halo rows)
 *   grad_e [E x d_e] fp32       =   dL/de for edges of the rows (NULL: skipped)
 *   grads                       +=  weight gradients (fp32)
 * csc_perm/csc_ptr from dsmpnn_csc (deterministic scatter to source rows).
 * ws: the workspace passed to the matching dsmpnn_layer_fwd (unmodified);
 * bwd_ws: scratch sized by dsmpnn_layer_bwd_workspace_size. */
dsmpnn_status dsmpnn_layer_bwd_workspace_size(const dsmpnn_layer_desc *desc, int64_t n_dst, int64_t n_loc,
                                              int64_t n_edges, size_t *bytes);
dsmpnn_status dsmpnn_layer_bwd(const dsmpnn_layer_desc *desc, const dsmpnn_weights *w, const void *v,
                               const void *e, const int64_t *row_ptr, const int64_t *row_ptr_host,
                               const int32_t *col_idx, const int32_t *csc_perm, const int64_t *csc_ptr,
                               int64_t n_dst, int64_t n_loc, int64_t row_begin, int64_t row_end,
                               const float *grad_out, float *grad_v, float *grad_e, const dsmpnn_grads *grads,
                               const void *ws, void *bwd_ws, size_t bwd_ws_bytes, void *stream);

/* ------------------------------------------------------------------ a6 --- */
/* Halo exchange building blocks ("the overlap area of a given
 * domain is updated from the neighboring domains' interiors"; Alg. 1 :411).
 * The plan makes every receive slice contiguous, so a FORWARD exchange is:
 * gather the send rows into a contiguous buffer, transfer (NCCL send/recv via
 * torch.distributed, or a device copy between virtual ranks), done.  The
 * REVERSE_ADD direction gathers the contiguous halo slice, transfers it, and
 * scatter-adds it into the owner's send rows in ascending peer order.
 * width elements of dtype (F32 or BF16) per row. */
dsmpnn_status dsmpnn_halo_gather(const void *values, const int32_t *rows, int64_t n_rows, int32_t width,
                                 int32_t dtype, void *out, void *stream);
dsmpnn_status dsmpnn_halo_scatter_add(const float *in, const int32_t *rows, int64_t n_rows, int32_t width,
                                      float *values, void *stream);

/* Loopback exchange among P virtual ranks resident on ONE device (no NCCL):
 * for every ordered pair (p -> q), values[q][halo_ptr_q[p] .. halo_ptr_q[p+1])
 * <- values[p][send_idx_p[send_ptr_p[q] .. send_ptr_p[q+1])].
 * values, send_idx: host arrays of P device pointers; halo_ptr, send_ptr:
 * host arrays of P host pointers to int64[P+1]. */
dsmpnn_status dsmpnn_halo_exchange_loopback(int32_t nparts, void *const *values, const int64_t *const *halo_ptr,
                                            const int64_t *const *send_ptr, const int32_t *const *send_idx,
                                            int32_t width, int32_t dtype, void *stream);

/* Loopback REVERSE_ADD among P virtual ranks on ONE device (SURVEY §8(f) f2,
 * reading R16): the transpose of dsmpnn_halo_exchange_loopback for fp32
 * gradients.  For p = 0..P-1 and q ascending (q != p):
 *   values[p][send_idx_p[send_ptr_p[q] + t]] += values[q][halo_ptr_q[p] + t]
 * so a halo row's gradient reaches the row it was copied from.  Halo rows are
 * only read; the order of the additions is fixed (deterministic).  Same
 * argument layout as dsmpnn_halo_exchange_loopback; values are float32. */
dsmpnn_status dsmpnn_halo_reverse_add_loopback(int32_t nparts, float *const *values, const int64_t *const *halo_ptr,
                                               const int64_t *const *send_ptr, const int32_t *const *send_idx,
                                               int32_t width, void *stream);

/* ------------------------------------------------------------------ a8 --- */
/* Sub-domain batch: the P sub-domains one process holds as ONE disjoint-union
 * graph, so a layer (a4 + a5 + a7) runs once over all of them.
 * places one sub-domain on each GPU; with more sub-domains than processes the
 * local graphs are independent between two halo refreshes (Alg. 1 :404-411),
 * and the union gives the same per-row results as P separate calls (reading
 * R31).  Union node order: owned rows of part 0..P-1, then halo rows of part
 * 0..P-1 (N_own = sum n_own, N_loc = sum n_loc); own row i of part q is union
 * row own_off_q + i, halo row n_own_q + h of part q is union row halo_off_q + h.
 * Union edges: the parts' edges concatenated (edge_off_q = sum of earlier E).
 * Every part whose halo rows source another part must have that part in the
 * batch (a process-local batch: all P parts).  1 <= P <= 16.
 *
 * parts: host array of P descriptors (device pointers inside, except the host
 * halo_ptr / send_ptr: int64[P+1] each, the plan of dsmpnn_partition_all).
 * Outputs (device, caller-allocated; any may be NULL to skip it):
 *   row_ptr  int64[N_own+1]   union CSR (row_ptr[N_own] = E_tot)
 *   col_idx  int32[E_tot]     union column ids
 *   e        E_tot x e_row_bytes bytes: the parts' edge attribute rows
 *   csc_perm int32[E_tot], csc_ptr int64[N_loc+1]: the union CSC view; each
 *            union column's list is its part's list (order kept) + edge_off_q
 *   rows     int64[N_loc]     the parts' `rows` entries in union order
 *   halo_src int32[N_loc-N_own] union row each union halo row is copied from:
 *            a FORWARD halo refresh is dsmpnn_halo_gather(values, halo_src,
 *            N_loc - N_own, width, dtype, values + N_own * width)
 * ws: sized by dsmpnn_batch_workspace_size.  Errors: P out of range ->
 * UNSUPPORTED; inconsistent halo / send plans -> SHAPE; union sizes >= 2^31 ->
 * UNSUPPORTED; missing inputs for a requested output -> INVALID_ARG. */
typedef struct {
  int64_t n_own, n_loc, n_edges;
  const int64_t *row_ptr;   /* int64[n_own+1] */
  const int32_t *col_idx;   /* int32[n_edges], local ids < n_loc */
  const void *e;            /* n_edges x e_row_bytes (or NULL when e is not requested) */
  const int32_t *csc_perm;  /* int32[n_edges] (dsmpnn_csc) */
  const int64_t *csc_ptr;   /* int64[n_loc+1] */
  const int64_t *rows;      /* int64[n_loc] per-row payload (e.g. sampled-set rows), or NULL */
  const int64_t *halo_ptr;  /* host int64[P+1]: halo rows from part p are [halo_ptr[p], halo_ptr[p+1]) */
  const int64_t *send_ptr;  /* host int64[P+1]: rows sent to part q are send_idx[send_ptr[q] ..] */
  const int32_t *send_idx;  /* int32[n_send] local own rows */
} dsmpnn_batch_part;
dsmpnn_status dsmpnn_batch_workspace_size(int32_t nparts, size_t *bytes);
dsmpnn_status dsmpnn_batch_subdomains(int32_t nparts, const dsmpnn_batch_part *parts, int32_t e_row_bytes,
                                      int64_t *row_ptr, int32_t *col_idx, void *e, int32_t *csc_perm,
                                      int64_t *csc_ptr, int64_t *rows, int32_t *halo_src, void *ws, size_t ws_bytes,
                                      void *stream);

/* ------------------------------------------------------- a6 over NCCL --- */
/* The halo exchange between processes ("the overlap area of a
 * given domain is updated from the neighboring domains' interiors"; Alg. 1
 * :411 Comm(i_b, Omega, v_L)) and the gradient sum (Alg. 1 :418), over an NCCL
 * communicator owned by a context.  One process per GPU; a process may hold
 * several sub-domains ("parts").
 *
 * dsmpnn_comm_unique_id: rank 0 creates the communicator id (host buffer of
 *   DSMPNN_UNIQUE_ID_BYTES); the caller distributes it to every rank (e.g. a
 *   torch.distributed broadcast) before dsmpnn_ctx_create.
 * dsmpnn_ctx_create: collective over the nranks processes (blocks until all
 *   have joined); sets `device` current; creates the communicator, a
 *   high-priority comm stream and the events of the exchange.
 *   dsmpnn_ctx_destroy frees them (NULL is a no-op).
 * dsmpnn_halo_exchange: for the parts this rank holds (local_parts[i], with
 *   values[i] / halo_ptr[i] / send_ptr[i] / send_idx[i] from that part's
 *   plan, dsmpnn_partition; part_rank[p] = rank holding part p, host int32
 *   [nparts]; every part with part_rank == this rank must be listed):
 *     FORWARD:     values_t[halo_ptr_t[s] + r] = values_s[send_idx_s[send_ptr_s[t] + r]]
 *                  for every ordered pair s != t with s or t local;
 *     REVERSE_ADD: values_p[send_idx_p[send_ptr_p[q] + r]] += values_q[halo_ptr_q[p] + r]
 *                  (fp32 only; for each local p the holders q are added in
 *                  ascending order, the loopback call's order: deterministic).
 *   Same-rank pairs are device copies/adds; other pairs are ncclSend/ncclRecv
 *   (send rows gathered into a context-owned staging buffer; FORWARD receives
 *   land directly in the contiguous halo rows).  The work runs on the comm
 *   stream after everything enqueued on `stream`; unless flags has
 *   DSMPNN_HALO_ASYNC, `stream` then waits for it.  With ASYNC the caller joins
 *   later with dsmpnn_halo_wait(ctx, stream) (e.g. after the deep rows of the
 *   next layer, which read no halo row, reading R23).  DSMPNN_HALO_VIA_NCCL
 *   routes same-rank pairs through NCCL too (send/recv to self: exercises the
 *   NCCL path on one GPU).  Both ranks of a pair derive the same message
 *   sizes from their own plans; a mismatch is SHAPE.  Errors: INVALID_ARG
 *   (bad parts, width, dtype), UNSUPPORTED (REVERSE_ADD of bf16), NCCL.
 * dsmpnn_halo_schedule: the host-only op list that dsmpnn_halo_exchange
 *   issues (no GPU needed; used by the multi-process CPU tests): kind LOCAL /
 *   SEND / RECV, the peer rank, source and destination part, rows, and offset
 *   (FORWARD: LOCAL/RECV = first halo row in the destination part, SEND = first
 *   staging row; REVERSE_ADD: LOCAL/SEND = first halo row in the holder part
 *   (src_part), RECV = first staging row).  Sends and receives between two
 *   ranks are issued in this (global source, destination) order on both
 *   sides, which is how NCCL matches them.  stage_rows = staging rows needed.
 * dsmpnn_allreduce_sum_f32: in-place sum over the ranks (ncclAllReduce on `stream`).
 * dsmpnn_ctx_sync: host watchdog: waits for the context's last exchange or
 *   all-reduce; polls ncclCommGetAsyncError; after timeout_ms (< 0: no limit)
 *   aborts the communicator and returns TIMEOUT (NCCL on an asynchronous
 *   error).  An aborted context fails every later call with NCCL. */
#define DSMPNN_UNIQUE_ID_BYTES 128
typedef struct dsmpnn_ctx_s *dsmpnn_ctx;
typedef enum { DSMPNN_HALO_FORWARD = 0, DSMPNN_HALO_REVERSE_ADD = 1 } dsmpnn_halo_dir;
typedef enum { DSMPNN_HALO_ASYNC = 1, DSMPNN_HALO_VIA_NCCL = 2 } dsmpnn_halo_flags;
typedef enum { DSMPNN_HALO_OP_LOCAL = 0, DSMPNN_HALO_OP_SEND = 1, DSMPNN_HALO_OP_RECV = 2 } dsmpnn_halo_op_kind;
typedef struct {
  int32_t kind, peer_rank, src_part, dst_part;
  int64_t rows, offset;
} dsmpnn_halo_op;

dsmpnn_status dsmpnn_comm_unique_id(void *id /*host, DSMPNN_UNIQUE_ID_BYTES*/);
dsmpnn_status dsmpnn_ctx_create(int32_t device, const void *unique_id /*host*/, int32_t rank, int32_t nranks,
                                dsmpnn_ctx *ctx /*host out*/);
dsmpnn_status dsmpnn_ctx_destroy(dsmpnn_ctx ctx);
dsmpnn_status dsmpnn_ctx_info(dsmpnn_ctx ctx, int32_t *rank, int32_t *nranks, void **comm_stream);
dsmpnn_status dsmpnn_halo_schedule(int32_t nparts, const int32_t *part_rank, int32_t my_rank, int32_t n_local,
                                   const int32_t *local_parts, const int64_t *const *halo_ptr,
                                   const int64_t *const *send_ptr, int32_t direction, int32_t flags,
                                   dsmpnn_halo_op *ops /*host*/, int32_t capacity, int32_t *n_ops /*host*/,
                                   int64_t *stage_rows /*host*/);
dsmpnn_status dsmpnn_halo_exchange(dsmpnn_ctx ctx, int32_t nparts, const int32_t *part_rank, int32_t n_local,
                                   const int32_t *local_parts, void *const *values, const int64_t *const *halo_ptr,
                                   const int64_t *const *send_ptr, const int32_t *const *send_idx, int32_t width,
                                   int32_t dtype, int32_t direction, int32_t flags, void *stream);
dsmpnn_status dsmpnn_halo_wait(dsmpnn_ctx ctx, void *stream);
dsmpnn_status dsmpnn_allreduce_sum_f32(dsmpnn_ctx ctx, float *buf, int64_t n, void *stream);
dsmpnn_status dsmpnn_ctx_sync(dsmpnn_ctx ctx, int32_t timeout_ms);

/* ----------------------------------------------------------- f4 --------- */
/* Inference by sub-domain reassembly ("randomly selected
 * sub-domains ... sequentially fed into the trained model ... reassembled in
 * post-processing").  Each pass (sample, partition, L-layer
 * forward) contributes its owned rows' predictions; the assembled field is
 * their per-node average.
 *   accumulate: sum[gid[k]] += pred[k] (width floats), count[gid[k]] += 1, for
 *               k < n.  gid values within one call must be distinct (one
 *               sub-domain's owned rows); calls are applied in stream order,
 *               so the result is deterministic.
 *   finalize:   out[g] = count[g] ? sum[g] / count[g] : 0, g < n_points. */
dsmpnn_status dsmpnn_reassemble_accumulate(const float *pred, const int64_t *gid, int64_t n, int32_t width,
                                           float *sum, int32_t *count, void *stream);
dsmpnn_status dsmpnn_reassemble_finalize(const float *sum, const int32_t *count, int64_t n_points, int32_t width,
                                         float *out, void *stream);

/* ----------------------------------------------------------- f3 --------- */
/* GCN layer, the paper's node-based comparison model ("GCN here
 * uses 6 hidden layers with a size of 378"; SURVEY §8(f) f3;
 * reading R24: same radius graph as the MPNN, mean over N(i) u {i}), fp32:
 *   agg_i = (v_i + sum_{p in row i} v_{col p}) / (deg_i + 1)
 *   out_i = act(W agg_i + c),  W float32 [d_out x d_in] (PyTorch layout), c [d_out]
 * v [n_loc x d_in] (rows 0..n_dst-1 are the destinations), CSR by destination.
 * gcn_fwd writes agg [n_dst x d_in] (kept for the backward) and out
 * [n_dst x d_out].  gcn_bwd, for grad_out [n_dst x d_out], ACCUMULATES
 * grad_v [n_loc x d_in] (+=, any may be NULL), grad_W, grad_c; csc_perm /
 * csc_ptr from dsmpnn_csc.  Deterministic (fixed summation orders). */
dsmpnn_status dsmpnn_gcn_fwd(int32_t d_in, int32_t d_out, int32_t act, const float *W, const float *c,
                             const float *v, const int64_t *row_ptr, const int32_t *col_idx, int64_t n_dst,
                             float *agg, float *out, void *stream);
dsmpnn_status dsmpnn_gcn_bwd_workspace_size(int32_t d_in, int32_t d_out, int64_t n_dst, size_t *bytes);
dsmpnn_status dsmpnn_gcn_bwd(int32_t d_in, int32_t d_out, int32_t act, const float *W, const int64_t *row_ptr,
                             const int32_t *col_idx, const int32_t *csc_perm, const int64_t *csc_ptr, int64_t n_dst,
                             int64_t n_loc, const float *agg, const float *out, const float *grad_out, float *grad_v,
                             float *grad_W, float *grad_c, void *ws, size_t ws_bytes, void *stream);

/* ----------------------------------------------------------- f1 --------- */
/* The training step around the layer (PAPER.md eqs. (i), (iii), (iv) :39-42,
 * Alg. 1 :404-419), fp32:
 * mlp3: 3 Linear layers, ReLU after the first two (encoder N_e, decoder N_d).
 *   Wb = {W0, b0, W1, b1, W2, b2}, W_l PyTorch [out, in]; x [n x in_dim],
 *   h1, h2 [n x hid] (kept for the backward), y [n x out_dim].
 *   mlp3_bwd ACCUMULATES dWb (+=, entries may be NULL) and dx (+=, may be
 *   NULL) for dy [n x out_dim].
 * edge_refresh_bwd: backward of (iv) e_ij = (.., u_i - u_j, ..) where the u
 *   difference occupies columns [off, off + width) of the d_e-wide edge
 *   attribute: grad_u[j] += sum_{p in row j} grad_e[p] - sum_{p: col p = j}
 *   grad_e[p] (rows j < n_dst are destinations; CSC view from dsmpnn_csc).
 * mse: *sse += sum (pred - target)^2 (one block, fixed order) and, if grad is
 *   not NULL, grad = 2 (pred - target) * scale.  mse_mean: *loss = *sse / count
 *   (device scalars; count = number of terms over all ranks).
 * sgd: w -= lr g (Alg. 1 :419).  adam: Adam with bias
 *   correction for step >= 1, m / v updated in place. */
dsmpnn_status dsmpnn_mlp3_fwd(int32_t in_dim, int32_t hid, int32_t out_dim, const float *const *Wb, const float *x,
                              int64_t n, float *h1, float *h2, float *y, void *stream);
dsmpnn_status dsmpnn_mlp3_bwd_workspace_size(int32_t in_dim, int32_t hid, int32_t out_dim, int64_t n, size_t *bytes);
dsmpnn_status dsmpnn_mlp3_bwd(int32_t in_dim, int32_t hid, int32_t out_dim, const float *const *Wb, const float *x,
                              const float *h1, const float *h2, const float *dy, int64_t n, float *dx,
                              float *const *dWb, void *ws, size_t ws_bytes, void *stream);
dsmpnn_status dsmpnn_edge_refresh_bwd(const float *grad_e, int32_t d_e, int32_t off, int32_t width,
                                      const int64_t *row_ptr, const int32_t *csc_perm, const int64_t *csc_ptr,
                                      int64_t n_dst, int64_t n_loc, float *grad_u, void *stream);
dsmpnn_status dsmpnn_mse(const float *pred, const float *target, int64_t n_elems, float scale, float *grad,
                         float *sse, void *stream);
dsmpnn_status dsmpnn_mse_mean(const float *sse, int64_t count, float *loss, void *stream);
dsmpnn_status dsmpnn_sgd(float *w, const float *g, int64_t n, float lr, void *stream);
dsmpnn_status dsmpnn_adam(float *w, const float *g, float *m, float *v, int64_t n, float lr, float beta1, float beta2,
                          float eps, int32_t step, void *stream);

/* --------------------------------------------------------------- GEMM --- */
/* Dense bf16 GEMM on the tcgen05 tensor cores, fp32 accumulate:
 *   C[M x N] (+)= A[M x K] . B[K x N]
 * A stored [M][K] (a_mn_major = 0) or [K][M] (1) with row stride lda elements;
 * B stored [N][K] (b_mn_major = 0) or [K][N] (1) with row stride ldb.  Base
 * pointers and row strides must be 16-byte aligned.  splits > 1 splits K
 * across CTAs into `partial` (fp32 [splits x M x N], caller-owned) and sums
 * the slices in a fixed order (deterministic).  The building block of the
 * BF16 layer's dense contractions, exported for testing. */
dsmpnn_status dsmpnn_gemm_bf16(int64_t M, int64_t N, int64_t K, const void *A, int64_t lda, int32_t a_mn_major,
                               const void *B, int64_t ldb, int32_t b_mn_major, float *C, int64_t ldc, int32_t splits,
                               float *partial, int32_t accumulate, void *stream);

/* Gradient sum of sub-domains processed on separate CUDA streams (Alg. 1
 * :418 "sum gradients"): dst[i] += src[i] for i < n (fp32, device pointers,
 * element-wise, deterministic).  The caller orders the streams. */
dsmpnn_status dsmpnn_accumulate_f32(float *dst, const float *src, int64_t n, void *stream);

/* ------------------------------------------------------------ probes --- */
/* Live kernel timing for the benchmark's roofline figure: while a probe is
 * armed, the library records a CUDA event pair on the launching stream around
 * every launch of the selected kernel; dsmpnn_probe_end synchronises those
 * events and returns the summed duration and the number of launches.
 * kernel_id: one of dsmpnn_probe_kernel.  Not thread safe (bench use). */
typedef enum {
  DSMPNN_PROBE_NONE = 0,
  DSMPNN_PROBE_F32_MLP2 = 1,      /* F32: h = relu(a1 W2^T + b2) GEMM */
  DSMPNN_PROBE_F32_EDGE_BWD = 2,  /* F32: per-row dh / u kernel */
  DSMPNN_PROBE_BF16_EDGE_FWD = 3, /* BF16: fused kappa MLP + S formation (tcgen05) */
  DSMPNN_PROBE_BF16_NODE_GEMM = 4,/* BF16: [S~ | v] . [Theta~ ; W_root^T] GEMM + epilogue (tcgen05) */
  DSMPNN_PROBE_BF16_EDGE_BWD = 5, /* BF16: fused edge backward (tcgen05) */
  DSMPNN_PROBE_BF16_DZ1W1 = 6,    /* BF16: fused dz1 = (dz2 W2)[a1>0] -> dW1, db1 (tcgen05) */
  DSMPNN_PROBE_BF16_DW2 = 7       /* BF16: dW2 = dz2^T a1 with a1 recomputed (tcgen05) */
} dsmpnn_probe_kernel;
dsmpnn_status dsmpnn_probe_begin(int32_t kernel_id, int32_t max_launches);
dsmpnn_status dsmpnn_probe_end(float *total_ms /*host*/, int64_t *launches /*host*/);

#ifdef __cplusplus
}
#endif
#endif /* DSMPNN_H */

"""Orchestration of the hot path over the C ABI (no arithmetic here).

Graph build per Alg. 1: sample -> decompose
-> local arrays -> radius graph -> edge attributes (+ CSC view for the
backward scatter); then the layer loop of lines 404-417 with the halo refresh
of line 411.  Every step is one call into libdsmpnn.so; torch
only allocates device memory and provides streams / process groups.
"""
from dataclasses import dataclass, field

import torch

from . import _lib as L


@dataclass
class Subdomain:
    rank: int
    nparts: int
    n_deep: int
    n_near: int
    n_halo: int
    halo_ptr: list
    send_ptr: list
    local_rows: torch.Tensor        # int64 [n_loc] indices into the sampled set
    send_idx: torch.Tensor          # int32 [n_send]
    coords: torch.Tensor            # float32 [n_loc x dim]
    gid: torch.Tensor               # int64 [n_loc]
    attr: torch.Tensor              # float32 [n_loc x n_attr]
    row_ptr: torch.Tensor = None    # int64 [n_own+1]
    row_ptr_host: torch.Tensor = None
    col_idx: torch.Tensor = None    # int32 [E]
    n_edges: int = 0
    e32: torch.Tensor = None
    e16: torch.Tensor = None
    csc_perm: torch.Tensor = None
    csc_ptr: torch.Tensor = None
    extra: dict = field(default_factory=dict)

    @property
    def n_own(self):
        return self.n_deep + self.n_near

    @property
    def n_loc(self):
        return self.n_own + self.n_halo


class Pool:
    """Persistent device buffers of one graph slot: `empty(key, shape, dtype)`
    returns a view of a cached byte buffer (grown on demand with 25 %
    headroom), so steady-state graph builds allocate nothing.  HotPath keeps
    two slots and alternates them build by build: a build overwrites the
    arrays of the build before last, which no queued work reads any more
    (the pipelined build waits for the previous step's layers)."""

    def __init__(self, device):
        self.dev = device
        self.bufs = {}

    def empty(self, key, shape, dtype):
        shape = tuple(int(x) for x in (shape if isinstance(shape, (tuple, list)) else (shape,)))
        count = 1
        for x in shape:
            count *= x
        esz = torch.empty((), dtype=dtype).element_size()
        nbytes = max(1, count) * esz
        b = self.bufs.get(key)
        if b is None or b.numel() < nbytes:
            b = torch.empty(int(nbytes * 1.25) + 256, dtype=torch.uint8, device=self.dev)
            self.bufs[key] = b
        return b[:nbytes].view(dtype)[:count].view(shape)


def _empty(pool, key, shape, dtype, device):
    if pool is None:
        return torch.empty(shape, dtype=dtype, device=device)
    return pool.empty(key, shape, dtype)


def sample_nodes(n_points, s, seed, device, pool=None):
    ids = _empty(pool, "ids", min(s, n_points), torch.int32, device)
    L.sample(n_points, s, seed, ids)
    return ids


def decompose(coords_s, gid_s, attr_s, nparts, overlap_l, radius, ranks, gid_bits=0, pool=None):
    """Partition the sampled set (all ranks' plans from one RCB, one host
    synchronisation) and build the local arrays of the given ranks.
    gid_bits: every gid < 2^gid_bits (0 = unknown), shortens the plan sorts.
    pool: optional Pool the arrays are taken from."""
    dev = coords_s.device
    n, dim = coords_s.shape
    owner = _empty(pool, "owner", n, torch.int32, dev)
    boxes = _empty(pool, "boxes", nparts * 2 * dim, torch.float32, dev)
    internal = _empty(pool, "internal", nparts * 2 * dim, torch.uint8, dev)
    nc = 5 + 2 * (nparts + 1)
    cap = n * max(1, nparts - 1)
    local_rows = _empty(pool, "local_rows", (nparts, n), torch.int64, dev)
    counts = _empty(pool, "counts", (nparts, nc), torch.int64, dev)
    send_idx = _empty(pool, "send_idx", (nparts, cap), torch.int32, dev)
    L.partition_all(coords_s, gid_s, nparts, overlap_l, radius, owner, boxes, internal, local_rows, counts,
                    send_idx, gid_bits=gid_bits)
    hcounts = counts.cpu().tolist()  # the one synchronisation
    if any(h[-1] for h in hcounts):
        raise L.DsmpnnError(-9, "partition_all", "partition: a split left an empty side (all split coordinates tied)")
    out = []
    for q in ranks:
        h = hcounts[q]
        nd, nn, nh, ns = h[0], h[1], h[2], h[3]
        halo_ptr = h[4:4 + nparts + 1]
        send_ptr = h[4 + nparts + 1:4 + 2 * (nparts + 1)]
        n_loc = nd + nn + nh
        lr = local_rows[q, :n_loc]
        c = _empty(pool, ("coords", q), (n_loc, dim), torch.float32, dev)
        L.gather_rows(coords_s, lr, c)
        g = _empty(pool, ("gid", q), n_loc, torch.int64, dev)
        L.gather_rows(gid_s, lr, g)
        a = _empty(pool, ("attr", q), (n_loc, attr_s.shape[1]), torch.float32, dev)
        L.gather_rows(attr_s, lr, a)
        out.append(Subdomain(q, nparts, nd, nn, nh, halo_ptr, send_ptr, lr, send_idx[q, :max(ns, 0)], c, g, a))
    return out, dict(owner=owner, boxes=boxes.view(nparts, 2, dim), internal=internal.view(nparts, 2, dim))


def build_graphs(subs, r, n_e, seed, edge_mode, want_f32=True, want_bf16=True, streams=None, ws_cache=None,
                 pool=None):
    """build_graph for several sub-domains with one host synchronisation: all
    radius graphs are enqueued (capacity n_own * n_e), then the edge counts and
    the host copies of row_ptr are read back together, then edge attributes
    and CSC views are enqueued.  streams: optional CUDA streams; sub-domain q's
    kernels go to streams[q % len(streams)] (arrays are allocated on the
    current stream, which waits for every stream before returning).
    ws_cache: optional dict keeping the radius-graph / CSC workspaces of each
    sub-domain slot across calls (grown on demand).  pool: optional Pool the
    graph arrays are taken from.  The edge attributes of all sub-domains are
    views of one array (sub-domain q at its edge offset), so the union graph
    (batch_subdomains) needs no copy of them."""
    if not subs:
        return subs
    dev = subs[0].coords.device
    main = torch.cuda.current_stream(dev)

    def fan_out(work):
        if not streams:
            for q, sd in enumerate(subs):
                work(q, sd)
            return
        fork = torch.cuda.Event()
        fork.record(main)
        for st in streams:
            st.wait_event(fork)
        for q, sd in enumerate(subs):
            with torch.cuda.stream(streams[q % len(streams)]):
                work(q, sd)
        for st in streams:
            done = torch.cuda.Event()
            done.record(st)
            main.wait_event(done)

    def ws(key, nbytes):
        if ws_cache is None:
            return None
        t = ws_cache.get(key)
        if t is None or t.numel() < nbytes:
            t = torch.empty(max(1, int(nbytes * 1.25)), dtype=torch.uint8, device=dev)  # headroom for the next step
            ws_cache[key] = t
        return t

    cols, rws = [], []
    for q, sd in enumerate(subs):
        sd.row_ptr = _empty(pool, ("row_ptr", q), sd.n_own + 1, torch.int64, dev)
        cols.append(_empty(pool, ("col", q), max(1, sd.n_own * n_e), torch.int32, dev))
        rws.append(ws(("radius", q), L.radius_graph_workspace_size(sd.n_loc, sd.n_own, sd.coords.shape[1])))
    fan_out(lambda q, sd: L.radius_graph(sd.coords, sd.gid, sd.n_own, r, n_e, seed, sd.row_ptr, cols[q],
                                         want_count=False, ws=rws[q]))
    host = torch.cat([sd.row_ptr for sd in subs]).cpu()  # the one synchronisation
    off = 0
    for sd, col in zip(subs, cols):
        sd.row_ptr_host = host[off:off + sd.n_own + 1]
        off += sd.n_own + 1
        E = int(sd.row_ptr_host[-1])
        sd.col_idx = col[:E]
        sd.n_edges = E
    E_tot = sum(sd.n_edges for sd in subs)
    de = (subs[0].coords.shape[1] + subs[0].attr.shape[1]) * (1 if edge_mode == L.EDGE_DIFF else 2)
    e32_all = _empty(pool, "e32", (E_tot + 1, de), torch.float32, dev) if want_f32 else None
    e16_all = _empty(pool, "e16", (E_tot + 1, 16), torch.bfloat16, dev) if want_bf16 else None  # all 16 written
    eoff = 0
    for q, sd in enumerate(subs):
        E = sd.n_edges
        # (an empty sub-domain's one-row view is never written)
        sd.e32 = e32_all[eoff:eoff + max(E, 1)] if want_f32 else None
        sd.e16 = e16_all[eoff:eoff + max(E, 1)] if want_bf16 else None
        sd.csc_perm = _empty(pool, ("csc_perm", q), max(E, 1), torch.int32, dev)
        sd.csc_ptr = _empty(pool, ("csc_ptr", q), sd.n_loc + 1, torch.int64, dev)
        eoff += E
    cws = [ws(("csc", q), L.csc_workspace_size(sd.n_edges, sd.n_loc)) for q, sd in enumerate(subs)]
    fan_out(lambda q, sd: _edge_arrays(sd, edge_mode, cws[q]))
    return subs


def _edge_arrays(sd, edge_mode, csc_ws=None):
    L.edge_features(edge_mode, sd.coords, sd.attr, sd.row_ptr, sd.col_idx, sd.n_own, sd.e32, sd.e16)
    L.csc(sd.col_idx, sd.n_loc, sd.csc_perm, sd.csc_ptr, ws=csc_ws)


def build_graph(sd: Subdomain, r, n_e, seed, edge_mode, want_f32=True, want_bf16=True):
    return build_graphs([sd], r, n_e, seed, edge_mode, want_f32, want_bf16)[0]


def halo_exchange_loopback(subs, values, dtype, stream=None):
    """FORWARD halo refresh among virtual ranks resident on this device."""
    L.halo_exchange_loopback(values, [s.halo_ptr for s in subs], [s.send_ptr for s in subs],
                             [s.send_idx for s in subs], dtype, stream=stream)


def halo_reverse_loopback(subs, grads):
    """REVERSE_ADD among virtual ranks on this device:
    fp32 gradients of halo rows are added to the rows they were copied from."""
    L.halo_reverse_add_loopback(grads, [s.halo_ptr for s in subs], [s.send_ptr for s in subs],
                                [s.send_idx for s in subs])


def halo_exchange_comm(comm, subs, values, dtype, proc_of, direction, flags=0, stream=None):
    """Halo refresh (FORWARD) or gradient return (REVERSE_ADD, fp32) of this
    process's sub-domains through the library's NCCL context
    (dsmpnn_halo_exchange): same-process pairs are device copies, the others
    ncclSend/ncclRecv; proc_of[p] is the process holding sub-domain p."""
    comm.halo_exchange(subs[0].nparts, proc_of, [sd.rank for sd in subs], values, [sd.halo_ptr for sd in subs],
                       [sd.send_ptr for sd in subs], [sd.send_idx for sd in subs], dtype, direction, flags,
                       stream=stream)


@dataclass
class Batch:
    """The local sub-domains as one disjoint-union graph (dsmpnn_batch_subdomains,
    reading R31): owned rows of every part first, then every part's halo rows."""
    subs: list
    n_own: int
    n_loc: int
    n_edges: int
    own_off: list                   # union row of part q's row 0
    halo_off: list                  # union row of part q's first halo row
    row_ptr: torch.Tensor
    row_ptr_host: torch.Tensor
    col_idx: torch.Tensor
    e32: torch.Tensor
    e16: torch.Tensor
    csc_perm: torch.Tensor
    csc_ptr: torch.Tensor
    local_rows: torch.Tensor        # int64 [n_loc] sampled-set rows in union order
    halo_src: torch.Tensor          # int32 [n_loc - n_own]


def batch_subdomains(subs, ws=None, pool=None):
    """Union graph of `subs` (every sub-domain of the plan, all on this device).
    When the sub-domains' edge attributes are consecutive views of one array
    (build_graphs), the union uses that array as is."""
    dev = subs[0].coords.device
    n_own = sum(sd.n_own for sd in subs)
    n_loc = sum(sd.n_loc for sd in subs)
    E = sum(sd.n_edges for sd in subs)
    own_off, halo_off, a, h = [], [], 0, n_own
    for sd in subs:
        own_off.append(a)
        halo_off.append(h)
        a += sd.n_own
        h += sd.n_halo
    # host copy of the union row_ptr (the layer calls read edge ranges from it)
    parts_h, eoff = [], 0
    for sd in subs:
        parts_h.append(sd.row_ptr_host[:-1] + eoff)
        eoff += sd.n_edges
    parts_h.append(torch.tensor([E], dtype=torch.int64))
    rph = torch.cat(parts_h)
    e_arr = subs[0].e16 if subs[0].e16 is not None else subs[0].e32
    e_row_bytes = e_arr.shape[1] * e_arr.element_size()
    b = Batch(subs, n_own, n_loc, E, own_off, halo_off,
              row_ptr=_empty(pool, "u_row_ptr", n_own + 1, torch.int64, dev), row_ptr_host=rph,
              col_idx=_empty(pool, "u_col", max(E, 1), torch.int32, dev), e32=None, e16=None,
              csc_perm=_empty(pool, "u_csc_perm", max(E, 1), torch.int32, dev),
              csc_ptr=_empty(pool, "u_csc_ptr", n_loc + 1, torch.int64, dev),
              local_rows=_empty(pool, "u_rows", n_loc, torch.int64, dev),
              halo_src=_empty(pool, "u_halo_src", max(n_loc - n_own, 1), torch.int32, dev))
    # the parts' attributes already form the union array when they are consecutive views of one buffer
    base, eoff, contiguous = e_arr.data_ptr(), 0, True
    for sd in subs:
        t = sd.e16 if subs[0].e16 is not None else sd.e32
        contiguous &= t.data_ptr() == base + eoff * e_row_bytes
        eoff += sd.n_edges
    if contiguous:
        e_out, e_copy = torch.as_strided(e_arr, (max(E, 1), e_arr.shape[1]), e_arr.stride()), None
    else:
        e_out = _empty(pool, "u_e", (max(E, 1), e_arr.shape[1]), e_arr.dtype, dev)
        e_copy = e_out
    if subs[0].e16 is not None:
        b.e16 = e_out
    else:
        b.e32 = e_out
    parts = [dict(n_own=sd.n_own, n_loc=sd.n_loc, n_edges=sd.n_edges, row_ptr=sd.row_ptr, col_idx=sd.col_idx,
                  e=sd.e16 if sd.e16 is not None else sd.e32, csc_perm=sd.csc_perm, csc_ptr=sd.csc_ptr,
                  rows=sd.local_rows, halo_ptr=sd.halo_ptr, send_ptr=sd.send_ptr, send_idx=sd.send_idx)
             for sd in subs]
    L.batch_subdomains(parts, e_row_bytes, b.row_ptr, b.col_idx, e_copy, b.csc_perm, b.csc_ptr, b.local_rows,
                       b.halo_src, ws=ws)
    return b


def batch_halo(b, values, dtype, stream=None):
    """FORWARD halo refresh of a union value array [n_loc x width]: one gather."""
    if b.n_loc > b.n_own:
        L.halo_gather(values, b.halo_src[: b.n_loc - b.n_own], values[b.n_own:], dtype, stream=stream)


def batch_halo_reverse(b, grads):
    """REVERSE_ADD of a union fp32 gradient array, pair by pair in the order of
    dsmpnn_halo_reverse_add_loopback (bitwise the same sums)."""
    subs = b.subs
    for p, sp in enumerate(subs):
        for q, sq in enumerate(subs):
            if q == p:
                continue
            s0, s1 = sp.send_ptr[q], sp.send_ptr[q + 1]
            a, z = sq.halo_ptr[p], sq.halo_ptr[p + 1]
            if z == a:
                continue
            h0 = b.halo_off[q] + (a - sq.n_own)
            L.halo_scatter_add(grads[h0:h0 + (z - a)], sp.send_idx[s0:s1], grads[b.own_off[p]:])

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


def sample_nodes(n_points, s, seed, device):
    ids = torch.empty(min(s, n_points), dtype=torch.int32, device=device)
    L.sample(n_points, s, seed, ids)
    return ids


def decompose(coords_s, gid_s, attr_s, nparts, overlap_l, radius, ranks, gid_bits=0):
    """Partition the sampled set (all ranks' plans from one RCB, one host
    synchronisation) and build the local arrays of the given ranks.
    gid_bits: every gid < 2^gid_bits (0 = unknown), shortens the plan sorts."""
    dev = coords_s.device
    n, dim = coords_s.shape
    owner = torch.empty(n, dtype=torch.int32, device=dev)
    boxes = torch.empty(nparts * 2 * dim, dtype=torch.float32, device=dev)
    internal = torch.empty(nparts * 2 * dim, dtype=torch.uint8, device=dev)
    nc = 5 + 2 * (nparts + 1)
    cap = n * max(1, nparts - 1)
    local_rows = torch.empty((nparts, n), dtype=torch.int64, device=dev)
    counts = torch.empty((nparts, nc), dtype=torch.int64, device=dev)
    send_idx = torch.empty((nparts, cap), dtype=torch.int32, device=dev)
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
        c = torch.empty((n_loc, dim), dtype=torch.float32, device=dev)
        L.gather_rows(coords_s, lr, c)
        g = torch.empty(n_loc, dtype=torch.int64, device=dev)
        L.gather_rows(gid_s, lr, g)
        a = torch.empty((n_loc, attr_s.shape[1]), dtype=torch.float32, device=dev)
        L.gather_rows(attr_s, lr, a)
        out.append(Subdomain(q, nparts, nd, nn, nh, halo_ptr, send_ptr, lr, send_idx[q, :max(ns, 0)], c, g, a))
    return out, dict(owner=owner, boxes=boxes.view(nparts, 2, dim), internal=internal.view(nparts, 2, dim))


def build_graphs(subs, r, n_e, seed, edge_mode, want_f32=True, want_bf16=True, streams=None, ws_cache=None):
    """build_graph for several sub-domains with one host synchronisation: all
    radius graphs are enqueued (capacity n_own * n_e), then the edge counts and
    the host copies of row_ptr are read back together, then edge attributes
    and CSC views are enqueued.  streams: optional CUDA streams; sub-domain q's
    kernels go to streams[q % len(streams)] (arrays are allocated on the
    current stream, which waits for every stream before returning).
    ws_cache: optional dict keeping the radius-graph / CSC workspaces of each
    sub-domain slot across calls (grown on demand)."""
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
        sd.row_ptr = torch.empty(sd.n_own + 1, dtype=torch.int64, device=dev)
        cols.append(torch.empty(max(1, sd.n_own * n_e), dtype=torch.int32, device=dev))
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
        _alloc_edge_arrays(sd, edge_mode, want_f32, want_bf16)
    cws = [ws(("csc", q), L.csc_workspace_size(sd.n_edges, sd.n_loc)) for q, sd in enumerate(subs)]
    fan_out(lambda q, sd: _edge_arrays(sd, edge_mode, cws[q]))
    return subs


def _alloc_edge_arrays(sd, edge_mode, want_f32, want_bf16):
    dev = sd.coords.device
    E = sd.n_edges
    de = (sd.coords.shape[1] + sd.attr.shape[1]) * (1 if edge_mode == L.EDGE_DIFF else 2)
    sd.e32 = torch.empty((max(E, 1), de), dtype=torch.float32, device=dev) if want_f32 else None
    sd.e16 = torch.empty((max(E, 1), 16), dtype=torch.bfloat16, device=dev) if want_bf16 else None  # all 16 written
    sd.csc_perm = torch.empty(max(E, 1), dtype=torch.int32, device=dev)
    sd.csc_ptr = torch.empty(sd.n_loc + 1, dtype=torch.int64, device=dev)


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


def halo_reverse_mixed(subs, grads, proc_of, my_proc, group=None, scatter_add=None):
    """REVERSE_ADD when sub-domains are spread over processes: the halo slice
    of q received from p is sent back to p's process (NCCL send/recv, issued in
    (destination, source) order on both sides), then every owner adds the
    slices into its send rows with q ascending (the oracle's order).  fp32.
    `scatter_add(inp, rows, values)` defaults to the library kernel."""
    import torch.distributed as dist
    if scatter_add is None:
        scatter_add = L.halo_scatter_add
    local = {sd.rank: (sd, g) for sd, g in zip(subs, grads)}
    nparts = subs[0].nparts
    ops, recv = [], {}
    for p_id in range(nparts):          # owner of the rows
        for q_id in range(nparts):      # holder of the halo copy
            if p_id == q_id:
                continue
            own_local, halo_local = p_id in local, q_id in local
            if own_local and not halo_local:
                psd, _ = local[p_id]
                s0, s1 = psd.send_ptr[q_id], psd.send_ptr[q_id + 1]
                if s1 > s0:
                    buf = torch.empty((s1 - s0, grads[0].shape[1]), dtype=torch.float32, device=grads[0].device)
                    recv[(p_id, q_id)] = buf
                    ops.append(dist.P2POp(dist.irecv, buf, proc_of[q_id], group))
            elif halo_local and not own_local:
                qsd, qg = local[q_id]
                a, b = qsd.halo_ptr[p_id], qsd.halo_ptr[p_id + 1]
                if b > a:
                    ops.append(dist.P2POp(dist.isend, qg[a:b].contiguous(), proc_of[p_id], group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    for p_id in range(nparts):
        if p_id not in local:
            continue
        psd, pg = local[p_id]
        for q_id in range(nparts):
            if q_id == p_id:
                continue
            s0, s1 = psd.send_ptr[q_id], psd.send_ptr[q_id + 1]
            if s1 <= s0:
                continue
            if q_id in local:
                qsd, qg = local[q_id]
                a, b = qsd.halo_ptr[p_id], qsd.halo_ptr[p_id + 1]
                src = qg[a:b]
            else:
                src = recv[(p_id, q_id)]
            scatter_add(src, psd.send_idx[s0:s1], pg)


def halo_exchange_mixed(subs, values, dtype, proc_of, my_proc, group=None, gather=None, stream=None):
    """FORWARD halo refresh when sub-domains are spread over processes.

    subs/values: this process's sub-domains and their [n_loc x width] arrays.
    proc_of[p]: process holding sub-domain p.  A peer on the same process is a
    device gather straight into the halo slice; a peer on another process is
    a contiguous send buffer + NCCL send/recv (torch.distributed
    batch_isend_irecv).  Receive slices are contiguous halo rows, so they land
    in place.  Messages between two processes are issued in (source
    sub-domain, destination sub-domain) order on both sides, which is how
    NCCL matches them.  `gather(values, rows, out)` defaults to the library's
    halo gather kernel."""
    import torch.distributed as dist
    if gather is None:
        def gather(vals, rows, out):
            L.halo_gather(vals, rows, out, dtype, stream=stream)
    local = {sd.rank: (sd, v) for sd, v in zip(subs, values)}
    nparts = subs[0].nparts
    ops = []
    keep = []
    for s_id in range(nparts):
        for t_id in range(nparts):
            if s_id == t_id:
                continue
            src_local, dst_local = s_id in local, t_id in local
            if src_local and dst_local:
                ssd, sv = local[s_id]
                tsd, tv = local[t_id]
                s0, s1 = ssd.send_ptr[t_id], ssd.send_ptr[t_id + 1]
                a, b = tsd.halo_ptr[s_id], tsd.halo_ptr[s_id + 1]
                if b > a:
                    gather(sv, ssd.send_idx[s0:s1], tv[a:b])
            elif src_local:
                ssd, sv = local[s_id]
                s0, s1 = ssd.send_ptr[t_id], ssd.send_ptr[t_id + 1]
                if s1 > s0:
                    buf = torch.empty((s1 - s0, sv.shape[1]), dtype=sv.dtype, device=sv.device)
                    gather(sv, ssd.send_idx[s0:s1], buf)
                    keep.append(buf)
                    ops.append(dist.P2POp(dist.isend, buf, proc_of[t_id], group))
            elif dst_local:
                tsd, tv = local[t_id]
                a, b = tsd.halo_ptr[s_id], tsd.halo_ptr[s_id + 1]
                if b > a:
                    ops.append(dist.P2POp(dist.irecv, tv[a:b], proc_of[s_id], group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()

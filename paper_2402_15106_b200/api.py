"""Public API: one DS-MPNN hot-path step (graph build + L layers forward with a
halo refresh after each + L layers backward + gradient sum) over the C ABI.

PAPER.md Alg. 1 (:385-422): lines 391-397 (sample, decompose, edge index,
edge sampling, edge attributes), 404-411 (per-hop convolution with residual
and overlap communication), 417-418 (local backprop, gradient sum).  The
encoder/decoder and the optimiser are outside the hot path.

A process owns one or more sub-domains ("virtual ranks"); halos between
sub-domains on the same device are device copies, halos between processes go
through the library's NCCL context (dsmpnn_halo_exchange, dsmpnn_allreduce_sum_f32);
torch.distributed only distributes the communicator id.  Gradients through halo
rows (reading R16): DETACH (default, the paper's local backprop) drops them;
REVERSE_ADD adds them to the owning rows after every
layer's backward, which makes the decomposed gradient equal the
undecomposed one.
"""
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from . import pipeline

GNAMES = ("W1", "b1", "W2", "b2", "W3", "b3", "W_root", "b")
DETACH, REVERSE_ADD = 0, 1


@dataclass
class StepConfig:
    n_points: int
    s: int
    dim: int
    n_attr: int
    nparts: int
    r: float
    overlap_l: float
    n_e: int
    d: int
    k: int
    L: int
    edge_mode: int
    dtype: int = L.BF16
    root: int = L.ROOT_DENSE
    act: int = L.ACT_RELU
    seed_sampling: int = 0
    seed_capping: int = 0
    grad_mode: int = DETACH
    overlap_halo: int = -1  # 1: deep rows of a layer run while the previous halo refresh is in flight; -1: when world > 1
    streams: int = 2  # CUDA streams the local sub-domains' layer work is spread over (1: one stream)
    halo: int = 1  # 0: skip the per-layer halo refresh (bench --no-comm: measures the exposed exchange time)
    halo_flags: int = 0  # extra dsmpnn_halo_exchange flags (L.HALO_VIA_NCCL: same-process pairs through NCCL too)
    batch: int = -1  # 1/-1: without a communicator, run the local sub-domains as one union graph (a8, R31); 0: per part


def parts_of_process(nparts, world, rank):
    """Block mapping of sub-domains to processes (nparts is a multiple of world)."""
    per = nparts // world
    return list(range(rank * per, (rank + 1) * per))


def make_comm(device, rank, world, group=None):
    """The library's NCCL context for this process: rank 0 creates the
    communicator id, torch.distributed broadcasts it (the only thing torch
    carries), every rank joins (collective)."""
    import torch.distributed as dist
    uid = [L.comm_unique_id() if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(uid, src=0, group=group)
    return L.Comm(device, uid[0], rank, world)


class HotPath:
    def __init__(self, cfg: StepConfig, weights: dict, device, rank=0, world=1, group=None, comm=None):
        """comm: the library NCCL context (make_comm); created here when
        world > 1 and none is given.  With world == 1 and no comm, halos are
        device copies (dsmpnn_halo_exchange_loopback)."""
        assert cfg.nparts % world == 0, "sub-domain count must be a multiple of the process count"
        self.cfg, self.dev, self.rank, self.world, self.group = cfg, device, rank, world, group
        if comm is None and world > 1:
            comm = make_comm(device, rank, world, group)
        self.comm = comm
        self.my_parts = parts_of_process(cfg.nparts, world, rank)
        self.proc_of = [p // (cfg.nparts // world) for p in range(cfg.nparts)]
        d_e = (cfg.dim + cfg.n_attr) * (1 if cfg.edge_mode == L.EDGE_DIFF else 2)
        self.d_e = d_e
        self.desc = L.make_desc(d_e, cfg.d, cfg.d, cfg.k, cfg.dtype, cfg.root, cfg.act)
        self.W = {n: torch.as_tensor(np.ascontiguousarray(weights[n]), dtype=torch.float32).to(device)
                  for n in GNAMES}
        self.packed = torch.empty(L.packed_weights_size(self.desc), dtype=torch.uint8, device=device)
        L.pack_weights(self.desc, self.W, self.packed)
        self.grads = {n: torch.zeros_like(t) for n, t in self.W.items()}
        self.flat_grads = None
        self.subs = []
        self.ws = {}

    # ------------------------------------------------------------- graph --
    def build(self, coords, attr):
        """Alg. 1 lines 391-397 on device-resident points (float32 [N x dim], [N x n_attr])."""
        c = self.cfg
        # graph arrays come from two alternating slots of persistent buffers
        # (pipeline.Pool): a build overwrites the arrays of the build before
        # last, whose step has finished (step_pipelined waits for it)
        if not hasattr(self, "_pools"):
            self._pools, self._slot = [pipeline.Pool(self.dev), pipeline.Pool(self.dev)], 1
        self._slot ^= 1
        pool = self._pools[self._slot]
        ids = pipeline.sample_nodes(c.n_points, c.s, c.seed_sampling, self.dev, pool=pool)
        self.ids = ids
        ids64 = pool.empty("ids64", ids.numel(), torch.int64)
        ids64.copy_(ids)
        cs = pool.empty("cs", (ids.numel(), c.dim), torch.float32)
        L.gather_rows(coords, ids64, cs)
        a = pool.empty("as", (ids.numel(), c.n_attr), torch.float32)
        L.gather_rows(attr, ids64, a)
        gid_bits = max(1, int(c.n_points - 1).bit_length())  # sampled ids are < n_points
        self.subs, self.plan = pipeline.decompose(cs, ids64, a, c.nparts, c.overlap_l, c.r, self.my_parts,
                                                  gid_bits=gid_bits, pool=pool)
        pipeline.build_graphs(self.subs, c.r, c.n_e, c.seed_capping, c.edge_mode, want_f32=(c.dtype == L.F32),
                              want_bf16=(c.dtype == L.BF16), streams=self._side_streams(),
                              ws_cache=self.ws.setdefault("graph", {}), pool=pool)
        self.bat = pipeline.batch_subdomains(self.subs, pool=pool) if self._batched() else None
        return self

    def _batched(self):
        """Union-graph mode (a8): every sub-domain is on this device (no
        communicator), more than one of them, and no deep-row overlap asked for."""
        c = self.cfg
        return (c.batch != 0 and self.comm is None and 1 < len(self.subs) <= 16 and c.overlap_halo != 1)

    @property
    def n_edges(self):
        return sum(sd.n_edges for sd in self.subs)

    # ------------------------------------------------------------ layers --
    def _ws(self, key, nbytes):
        t = self.ws.get(key)
        if t is None or t.numel() < nbytes:
            t = torch.empty(max(1, int(nbytes)), dtype=torch.uint8, device=self.dev)
            self.ws[key] = t
        return t

    def _side_streams(self):
        """Streams for concurrent sub-domains (StepConfig.streams > 1 and more
        than one local sub-domain); the sub-domains of a layer are independent
        once their inputs (including halo rows) are in place."""
        S = min(self.cfg.streams, len(self.subs))
        if S <= 1:
            return []
        if getattr(self, "_side", None) is None or len(self._side) != S:
            # stream 0 at high priority, the others fill its gaps and kernel tails
            lo, hi = torch.cuda.Stream.priority_range()
            self._side = [torch.cuda.Stream(self.dev, priority=hi if k == 0 else lo) for k in range(S)]
        return self._side

    def _comm_stream(self):
        if getattr(self, "_comm", None) is None:
            self._comm = torch.cuda.Stream(self.dev)
        return self._comm

    def halo(self, vals, dtype, stream=None, flags=0):
        """Overlap update (Alg. 1) for every local sub-domain: the
        library's NCCL exchange when a communicator exists, else device
        copies among the sub-domains of this device."""
        if not self.cfg.halo:
            return
        if self.comm is None:
            pipeline.halo_exchange_loopback(self.subs, vals, dtype, stream=stream)
        else:
            pipeline.halo_exchange_comm(self.comm, self.subs, vals, dtype, self.proc_of, L.HALO_FORWARD,
                                        flags | self.cfg.halo_flags, stream=stream)

    def halo_reverse(self, grads):
        """REVERSE_ADD of fp32 gradients (f2) for every local sub-domain."""
        if self.comm is None:
            pipeline.halo_reverse_loopback(self.subs, grads)
        else:
            pipeline.halo_exchange_comm(self.comm, self.subs, grads, L.F32, self.proc_of, L.HALO_REVERSE_ADD,
                                        self.cfg.halo_flags)

    def _halo_async(self, vals, dtype, main, side):
        """Start the refresh of `vals` behind the work enqueued on `main`;
        returns a callable that makes `main` wait for it.  With the library
        communicator the exchange runs on its own comm stream
        (DSMPNN_HALO_ASYNC + dsmpnn_halo_wait); the loopback path uses `side`."""
        if self.comm is not None:
            self.halo(vals, dtype, flags=L.HALO_ASYNC)
            return lambda: self.comm.halo_wait(main)
        ready = torch.cuda.Event()
        ready.record(main)
        side.wait_event(ready)
        for t in vals:
            t.record_stream(side)
        with torch.cuda.stream(side):
            self.halo(vals, dtype, stream=side)
        done = torch.cuda.Event()
        done.record(side)
        return lambda: main.wait_event(done)

    def forward(self, v0):
        """L layers forward (Alg. 1 :404-411) with a halo refresh after each.
        v0: [s x d] initial latent of the sampled nodes (sampled order).
        Returns (acts, outs): every layer's input per sub-domain (local order)
        and the last layer's fp32 outputs of each sub-domain's owned rows."""
        if getattr(self, "bat", None) is not None:
            return self._forward_batch(v0)
        c, desc = self.cfg, self.desc
        lowp = c.dtype == L.BF16
        vdt = torch.bfloat16 if lowp else torch.float32
        # layer-0 inputs of every sub-domain (local order)
        vals = []
        for sd in self.subs:
            v = torch.empty((sd.n_loc, c.d), dtype=vdt, device=self.dev)
            if lowp:  # bf16 operand rounding inside the library
                L.gather_rows_bf16(v0, sd.local_rows, v)
            else:
                L.gather_rows(v0, sd.local_rows, v)
            vals.append(v)
        acts = [vals]
        overlap = c.overlap_halo == 1 or (c.overlap_halo < 0 and self.world > 1)
        main = torch.cuda.current_stream(self.dev)
        comm = self._comm_stream() if overlap and self.comm is None else None
        ex_done = None

        def run(layer, q, sd, out, nv, a, b):
            if b <= a:
                return
            ws = self._ws(("fwd", layer, q), L.layer_workspace_size(desc, sd.n_own, sd.n_edges))
            e = sd.e16 if lowp else sd.e32
            L.layer_fwd(desc, self.W, self.packed, acts[-1][q], e, sd.row_ptr, sd.col_idx, sd.n_own, a, b,
                        out, nv[: sd.n_own] if lowp else None, ws, row_ptr_host=sd.row_ptr_host)
            if not lowp:
                nv[a:b].copy_(out[a:b])

        for layer in range(c.L):
            nxt, outs_l = [], []
            for q, sd in enumerate(self.subs):
                outs_l.append(self._ws(("out", q), sd.n_own * c.d * 4).view(torch.float32)[: sd.n_own * c.d]
                              .view(sd.n_own, c.d))
                nxt.append(torch.empty((sd.n_loc, c.d), dtype=vdt, device=self.dev))
            if not overlap:
                side = self._side_streams()
                if side:  # sub-domain q on stream q % S, joined before the halo refresh
                    for q, sd in enumerate(self.subs):  # workspaces exist before the fork
                        self._ws(("fwd", layer, q), L.layer_workspace_size(desc, sd.n_own, sd.n_edges))
                    fork = torch.cuda.Event()
                    fork.record(main)
                    for st in side:
                        st.wait_event(fork)
                    for q, sd in enumerate(self.subs):
                        with torch.cuda.stream(side[q % len(side)]):
                            run(layer, q, sd, outs_l[q], nxt[q], 0, sd.n_own)
                    for st in side:
                        done = torch.cuda.Event()
                        done.record(st)
                        main.wait_event(done)
                else:
                    for q, sd in enumerate(self.subs):
                        run(layer, q, sd, outs_l[q], nxt[q], 0, sd.n_own)
                self.halo(nxt, L.BF16 if lowp else L.F32)
            else:
                # deep rows have no halo neighbour (R23): they run while the
                # previous layer's halo refresh is still in flight
                for q, sd in enumerate(self.subs):
                    run(layer, q, sd, outs_l[q], nxt[q], 0, sd.n_deep)
                if ex_done is not None:
                    ex_done()
                for q, sd in enumerate(self.subs):
                    run(layer, q, sd, outs_l[q], nxt[q], sd.n_deep, sd.n_own)
                # only near rows are sent (R23): the refresh can start now
                ex_done = self._halo_async(nxt, L.BF16 if lowp else L.F32, main, comm)
            acts.append(nxt)
        if ex_done is not None:
            ex_done()
        outs = [self.ws[("out", q)].view(torch.float32)[: sd.n_own * c.d].view(sd.n_own, c.d)
                for q, sd in enumerate(self.subs)]
        return acts, outs

    def forward_backward(self, v0, G):
        """v0: [s x d] initial latent of the sampled nodes (sampled order);
        G: [s x d] dL/d(last layer output) (rows of owned nodes are used).
        Returns the accumulated weight gradients (dict of device tensors)."""
        c, desc = self.cfg, self.desc
        lowp = c.dtype == L.BF16
        for g in self.grads.values():
            g.zero_()
        if getattr(self, "bat", None) is not None:
            return self._forward_backward_batch(v0, G)
        acts, _ = self.forward(v0)
        # backward: DETACH or REVERSE_ADD halo rows (R16, f2)
        gouts = []
        for sd in self.subs:
            g = torch.empty((sd.n_own, c.d), dtype=torch.float32, device=self.dev)
            L.gather_rows(G, sd.local_rows[: sd.n_own], g)
            gouts.append(g)
        side = self._side_streams() if c.grad_mode == DETACH else []
        if side:
            # DETACH: a sub-domain's backward needs nothing from the others, so
            # sub-domain q runs all its layers on stream q % S with its own
            # gradient accumulator; the accumulators are summed in stream order
            main = torch.cuda.current_stream(self.dev)
            accs = [self.grads] + [self._ws_grads(k) for k in range(1, len(side))]
            for q, sd in enumerate(self.subs):
                self._ws(("bwd", q), L.layer_bwd_workspace_size(desc, sd.n_own, sd.n_loc, sd.n_edges))
            gvs = {(layer, q): torch.zeros((sd.n_loc, c.d), dtype=torch.float32, device=self.dev)
                   for layer in range(1, c.L) for q, sd in enumerate(self.subs)}
            fork = torch.cuda.Event()
            fork.record(main)
            for st in side:
                st.wait_event(fork)
            for q, sd in enumerate(self.subs):
                k = q % len(side)
                g = gouts[q]
                with torch.cuda.stream(side[k]):
                    for layer in reversed(range(c.L)):
                        gv = gvs.get((layer, q))
                        e = sd.e16 if lowp else sd.e32
                        L.layer_bwd(desc, self.W, self.packed, acts[layer][q], e, sd.row_ptr, sd.col_idx,
                                    sd.csc_perm, sd.csc_ptr, sd.n_own, sd.n_loc, 0, sd.n_own, g, gv, None, accs[k],
                                    self.ws[("fwd", layer, q)], self.ws[("bwd", q)], row_ptr_host=sd.row_ptr_host)
                        if gv is not None:
                            g = gv[: sd.n_own]
            for st in side:
                done = torch.cuda.Event()
                done.record(st)
                main.wait_event(done)
            for k in range(1, len(side)):
                for n in GNAMES:
                    L.accumulate_f32(self.grads[n], accs[k][n])
        else:
            for layer in reversed(range(c.L)):
                new_g = []
                for q, sd in enumerate(self.subs):
                    ws = self.ws[("fwd", layer, q)]
                    bws = self._ws(("bwd", q), L.layer_bwd_workspace_size(desc, sd.n_own, sd.n_loc, sd.n_edges))
                    gv = torch.zeros((sd.n_loc, c.d), dtype=torch.float32, device=self.dev)
                    e = sd.e16 if lowp else sd.e32
                    # the input gradient of the first layer is not needed (no scatter / root term)
                    L.layer_bwd(desc, self.W, self.packed, acts[layer][q], e, sd.row_ptr, sd.col_idx, sd.csc_perm,
                                sd.csc_ptr, sd.n_own, sd.n_loc, 0, sd.n_own, gouts[q], gv if layer > 0 else None,
                                None, self.grads, ws, bws, row_ptr_host=sd.row_ptr_host)
                    new_g.append(gv)
                if c.grad_mode == REVERSE_ADD:
                    self.halo_reverse(new_g)
                gouts = [gv[: sd.n_own] for gv, sd in zip(new_g, self.subs)]
        if self.world > 1:
            self._allreduce_grads()
        return self.grads

    # ------------------------------------------------ union-graph mode (a8) --
    def _forward_batch(self, v0):
        """forward() over the union graph: one layer call per layer for all
        local sub-domains, then one gather refreshes every halo row.  Returns
        (acts, outs) with acts[l] the union layer inputs and outs the per-part
        views of the last layer's fp32 outputs."""
        c, desc, b = self.cfg, self.desc, self.bat
        lowp = c.dtype == L.BF16
        vdt = torch.bfloat16 if lowp else torch.float32
        v = torch.empty((b.n_loc, c.d), dtype=vdt, device=self.dev)
        if lowp:
            L.gather_rows_bf16(v0, b.local_rows, v)
        else:
            L.gather_rows(v0, b.local_rows, v)
        acts = [v]
        out = self._ws(("out", "B"), b.n_own * c.d * 4).view(torch.float32)[: b.n_own * c.d].view(b.n_own, c.d)
        e = b.e16 if lowp else b.e32
        for layer in range(c.L):
            nv = torch.empty((b.n_loc, c.d), dtype=vdt, device=self.dev)
            ws = self._ws(("fwd", layer, "B"), L.layer_workspace_size(desc, b.n_own, b.n_edges))
            L.layer_fwd(desc, self.W, self.packed, acts[-1], e, b.row_ptr, b.col_idx, b.n_own, 0, b.n_own, out,
                        nv[: b.n_own] if lowp else None, ws, row_ptr_host=b.row_ptr_host)
            if not lowp:
                nv[: b.n_own].copy_(out)
            if c.halo:
                pipeline.batch_halo(b, nv, L.BF16 if lowp else L.F32)
            acts.append(nv)
        outs = [out[o:o + sd.n_own] for o, sd in zip(b.own_off, self.subs)]
        return acts, outs

    def _forward_backward_batch(self, v0, G):
        c, desc, b = self.cfg, self.desc, self.bat
        lowp = c.dtype == L.BF16
        acts, _ = self._forward_batch(v0)
        g = torch.empty((b.n_own, c.d), dtype=torch.float32, device=self.dev)
        L.gather_rows(G, b.local_rows[: b.n_own], g)
        bws = self._ws(("bwd", "B"), L.layer_bwd_workspace_size(desc, b.n_own, b.n_loc, b.n_edges))
        e = b.e16 if lowp else b.e32
        for layer in reversed(range(c.L)):
            # the input gradient of the first layer is not needed (no scatter / root term)
            gv = torch.zeros((b.n_loc, c.d), dtype=torch.float32, device=self.dev) if layer > 0 else None
            L.layer_bwd(desc, self.W, self.packed, acts[layer], e, b.row_ptr, b.col_idx, b.csc_perm, b.csc_ptr,
                        b.n_own, b.n_loc, 0, b.n_own, g, gv, None, self.grads, self.ws[("fwd", layer, "B")], bws,
                        row_ptr_host=b.row_ptr_host)
            if gv is not None:
                if c.grad_mode == REVERSE_ADD:
                    pipeline.batch_halo_reverse(b, gv)
                g = gv[: b.n_own]
        return self.grads

    def _ws_grads(self, k):
        """Zeroed gradient accumulator of side stream k (k >= 1)."""
        if not hasattr(self, "_acc"):
            self._acc = {}
        if k not in self._acc:
            self._acc[k] = {n: torch.zeros_like(t) for n, t in self.W.items()}
        for t in self._acc[k].values():
            t.zero_()
        return self._acc[k]

    def _allreduce_grads(self):
        """Gradient sum over processes (Alg. 1): one all-reduce of
        the flattened gradients through the library communicator."""
        flat = torch.cat([self.grads[n].reshape(-1) for n in GNAMES])
        self.comm.allreduce_sum_f32(flat)
        off = 0
        for n in GNAMES:
            m = self.grads[n].numel()
            self.grads[n].copy_(flat[off:off + m].view_as(self.grads[n]))
            off += m

    def infer(self, coords, attr, v0_global, seeds):
        """Inference by sub-domain reassembly:
        for every sampling seed, sample / decompose / build graphs and run the
        L-layer forward; each owned row's output is added to its global node,
        and the field is the per-node average over the passes that visited it
        (0 where none did).  v0_global: [n_points x d] initial latent of every
        point.  Returns (field [n_points x d] fp32, count [n_points] int32)."""
        import dataclasses
        c0 = self.cfg
        N, d = c0.n_points, c0.d
        acc = torch.zeros((N, d), dtype=torch.float32, device=self.dev)
        cnt = torch.zeros(N, dtype=torch.int32, device=self.dev)
        try:
            for seed in seeds:
                self.cfg = dataclasses.replace(c0, seed_sampling=int(seed))
                self.build(coords, attr)
                ids64 = self.ids.to(torch.int64)
                v0 = torch.empty((ids64.numel(), d), dtype=torch.float32, device=self.dev)
                L.gather_rows(v0_global, ids64, v0)
                _, outs = self.forward(v0)
                for sd, o in zip(self.subs, outs):
                    L.reassemble_accumulate(o, sd.gid[: sd.n_own], acc, cnt)
        finally:
            self.cfg = c0
        if self.world > 1:  # each process holds some sub-domains of every pass
            self.comm.allreduce_sum_f32(acc)
            cntf = cnt.to(torch.float32)  # counts <= len(seeds): exact in fp32
            self.comm.allreduce_sum_f32(cntf)
            cnt.copy_(cntf.round().to(torch.int32))
        field = torch.empty_like(acc)
        L.reassemble_finalize(acc, cnt, field)
        return field, cnt

    def step(self, coords, attr, v0, G):
        """One full hot-path step on device inputs."""
        self.build(coords, attr)
        return self.forward_backward(v0, G)

    # ------------------------------------------------------ pipelined steps --
    # Alg. 1 builds every sample's graph (lines 391-397) in a loop of its own,
    # ahead of the training loop (the trainloader).  step_pipelined keeps that
    # order within a run of steps: while the layers of step t run on the
    # current stream, the host builds the graph of step t+1 on a separate
    # high-priority stream, so the build's host synchronisations (plan sizes,
    # edge counts) wait for the build's own kernels only and its kernels fill
    # the SMs the layer kernels leave idle.  Every step still does its full
    # build and its full layer work.
    def _build_stream(self):
        if getattr(self, "_bstream", None) is None:
            import os
            lo, hi = torch.cuda.Stream.priority_range()
            self._bstream = torch.cuda.Stream(self.dev, priority=lo if os.environ.get("DSMPNN_BUILD_PRIO") == "lo"
                                              else hi)
        return self._bstream

    def _graph_state(self):
        return (self.subs, getattr(self, "bat", None), getattr(self, "ids", None), getattr(self, "plan", None))

    def _set_graph_state(self, st):
        self.subs, self.bat, self.ids, self.plan = st

    @staticmethod
    def _state_tensors(st):
        subs, bat, ids, plan = st
        objs = list(subs) + ([bat] if bat is not None else [])
        out = [ids] + (list(plan.values()) if plan else [])
        for o in objs:
            out += [v for v in vars(o).values() if isinstance(v, torch.Tensor) and v.is_cuda]
        return [t for t in out if isinstance(t, torch.Tensor) and t.is_cuda]

    def prefetch(self, coords, attr, after=()):
        """Enqueue the graph build of the next step on the build stream (it
        first waits for the events in `after`, e.g. the inputs' copy); the
        host returns when the build's host-side work is done.  The next
        step_pipelined call adopts the result."""
        bs = self._build_stream()
        for ev in after:
            if ev is not None:
                bs.wait_event(ev)
        coords.record_stream(bs)
        attr.record_stream(bs)
        cur = self._graph_state()
        try:
            with torch.cuda.stream(bs):
                self.build(coords, attr)
                done = torch.cuda.Event()
                done.record(bs)
            self._next = (self._graph_state(), done)
        finally:
            self._set_graph_state(cur)

    def step_pipelined(self, coords, attr, v0, G, next_inputs=None, next_ready=None):
        """One step (build + forward_backward) whose graph was prefetched by
        the previous call, or is built now; then, if next_inputs = (coords,
        attr) is given, the next step's graph is built on the build stream
        (after next_ready, an event, if given) while this step's layers run.
        Returns the gradients as forward_backward does."""
        main = torch.cuda.current_stream(self.dev)
        nxt = getattr(self, "_next", None)
        if nxt is not None:
            st, done = nxt
            self._next = None
            main.wait_event(done)
            for t in self._state_tensors(st):  # used on this stream from now on
                t.record_stream(main)
            self._set_graph_state(st)
        else:
            self.build(coords, attr)
        fence = torch.cuda.Event()
        fence.record(main)  # the next build may reuse the graph workspaces once this step's build is done
        grads = self.forward_backward(v0, G)
        if next_inputs is not None:
            self.prefetch(next_inputs[0], next_inputs[1], after=(fence, next_ready))
        return grads


class TrainStep:
    """one DS-MPNN training step (PAPER.md eqs. (i)-(iv),
    Alg. 1 :404-419) over the C ABI, fp32.  Per sub-domain: the encoder N_e on
    every local row, then `hops` times {residual convolution (the layer in
    paper form: identity root = the residual, identity sigma) on owned rows,
    halo refresh of the latent values, decoder N_d on every local row, edge
    refresh (iv) e_ij = (x_i - x_j, u_i - u_j)}; MSE of the last decoded values
    on owned rows; backward with received values detached (R16); gradient sum
    over processes; SGD (Alg. 1 :419) or Adam.  The oracle is
    oracle/train.py (O9).  F32 or BF16 mode (cfg.dtype): in BF16 the latent
    values, the decoder and the optimiser stay fp32, and each hop's
    convolution reads a bf16 copy of its input and the bf16 edge attributes
    (the tensor-core kernels; reading R27), as oracle.train's bf16 mode.

    params: dict enc=[(W, b)] * 3, dec=[(W, b)] * 3 (PyTorch [out, in]),
    conv=layer weights (W1, b1, W2, b2, W3, b3, b)."""

    CONV = ("W1", "b1", "W2", "b2", "W3", "b3", "W_root", "b")

    def __init__(self, cfg: StepConfig, params: dict, hops: int, device, rank=0, world=1, group=None,
                 optimizer="sgd", lr=1e-3, comm=None, decoded_exchange=True):
        """decoded_exchange: after every hop's decoder, also refresh the halo
        rows of the decoded values from their owners (Alg. 1 :412, the second
        per-hop Comm); the values equal the local decode of the refreshed
        latent rows bit for bit (reading R26), so this models the paper's
        communication, not a different result."""
        import dataclasses
        cfg = dataclasses.replace(cfg, root=L.ROOT_IDENTITY, act=L.ACT_IDENTITY, grad_mode=DETACH, L=hops, batch=0)
        conv = dict(params["conv"])
        conv.setdefault("W_root", np.zeros((cfg.d, cfg.d), np.float32))  # identity root: unused
        self.hp = HotPath(cfg, conv, device, rank, world, group, comm=comm)
        self.dev, self.hops, self.opt, self.lr = device, hops, optimizer, lr
        self.decoded_exchange = decoded_exchange
        T = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float32).to(device)
        self.enc = [T(x) for Wl, bl in params["enc"] for x in (Wl, bl)]
        self.dec = [T(x) for Wl, bl in params["dec"] for x in (Wl, bl)]
        self.g_enc = [torch.zeros_like(t) for t in self.enc]
        self.g_dec = [torch.zeros_like(t) for t in self.dec]
        self.m = self.v = None
        self.t = 0

    def build(self, coords, attr):
        self.hp.build(coords, attr)
        self.coords = coords
        return self

    def _mlp(self, Wb, x):
        n = x.shape[0]
        hid, out_dim = Wb[0].shape[0], Wb[4].shape[0]
        h1 = torch.empty((n, hid), device=self.dev)
        h2 = torch.empty((n, hid), device=self.dev)
        y = torch.empty((n, out_dim), device=self.dev)
        L.mlp3_fwd(Wb, x, h1, h2, y)
        return y, (x, h1, h2)

    def _conv_input(self, v):
        """The convolution's operand: v itself (F32) or its bf16 copy (BF16)."""
        if self.hp.cfg.dtype == L.F32:
            return v
        vb = torch.empty(v.shape, dtype=torch.bfloat16, device=self.dev)
        L.gather_rows_bf16(v, None, vb)
        return vb

    def loss_and_grads(self, v0_global, Y_global):
        """v0_global [N x (dim + n_attr)] initial node values, Y_global
        [N x n_attr] targets (rows = point ids).  Returns (loss, grads) with
        grads = dict(enc=[...], dec=[...], conv=HotPath.grads)."""
        hp, c = self.hp, self.hp.cfg
        desc, subs = hp.desc, hp.subs
        n_attr, dim = c.n_attr, c.dim
        for g in self.g_enc + self.g_dec + list(hp.grads.values()):
            g.zero_()
        gidx = [sd.gid.to(torch.int64) for sd in subs]  # local rows -> point ids
        enc_cache, vL, e = [], [], []
        for sd, gi in zip(subs, gidx):
            v0 = torch.empty((sd.n_loc, v0_global.shape[1]), device=self.dev)
            L.gather_rows(v0_global, gi, v0)
            y, cache = self._mlp(self.enc, v0)
            enc_cache.append(cache)
            vL.append(y)
            e.append(sd.e32 if c.dtype == L.F32 else sd.e16)
        hist = []
        for hop in range(self.hops):
            new, vin = [], []
            for q, sd in enumerate(subs):
                ws = hp._ws(("fwd", hop, q), L.layer_workspace_size(desc, sd.n_own, sd.n_edges))
                out = torch.empty((sd.n_own, c.d), device=self.dev)
                vin.append(self._conv_input(vL[q]))
                L.layer_fwd(desc, hp.W, hp.packed, vin[q], e[q], sd.row_ptr, sd.col_idx, sd.n_own, 0, sd.n_own, out,
                            None, ws, row_ptr_host=sd.row_ptr_host)
                nv = vL[q].clone()
                nv[: sd.n_own].copy_(out)
                new.append(nv)
            hp.halo(new, L.F32)
            dec_cache, u, e_next = [], [], []
            for q, sd in enumerate(subs):
                uq, cache = self._mlp(self.dec, new[q])
                dec_cache.append(cache)
                u.append(uq)
            if self.decoded_exchange:  # Alg. 1 :412 v^l <- Comm(i_b, Omega, v^l)
                hp.halo(u, L.F32)
            for q, sd in enumerate(subs):
                uq = u[q]
                if c.dtype == L.F32:
                    en = torch.empty((max(sd.n_edges, 1), dim + n_attr), device=self.dev)
                    L.edge_features(L.EDGE_DIFF, sd.coords, uq, sd.row_ptr, sd.col_idx, sd.n_own, e32=en)
                else:
                    en = torch.empty((max(sd.n_edges, 1), 16), dtype=torch.bfloat16, device=self.dev)
                    L.edge_features(L.EDGE_DIFF, sd.coords, uq, sd.row_ptr, sd.col_idx, sd.n_own, e16=en)
                e_next.append(en)
            hist.append(dict(vin=vin, e=e, vout=new, dec_cache=dec_cache, u=u))
            vL, e = new, e_next
        # loss: MSE of the last decoded values on owned rows, over all ranks
        count = sum(sd.n_own for sd in subs) * n_attr
        if hp.world > 1:
            ct = torch.tensor([float(count)], dtype=torch.float32, device=self.dev)  # < 2^24 rows: exact
            hp.comm.allreduce_sum_f32(ct)
            count = int(ct.item())
        sse = torch.zeros(1, device=self.dev)
        du = []
        for q, sd in enumerate(subs):
            d = torch.zeros((sd.n_loc, n_attr), device=self.dev)
            yq = torch.empty((sd.n_own, n_attr), device=self.dev)
            L.gather_rows(Y_global, gidx[q][: sd.n_own], yq)
            L.mse(hist[-1]["u"][q][: sd.n_own].contiguous(), yq, 1.0 / count, d, sse)
            du.append(d)
        # backward
        dvL_in = None
        for hop in reversed(range(self.hops)):
            H = hist[hop]
            dvout = []
            for q, sd in enumerate(subs):
                dd = du[q]
                dd[sd.n_own:].zero_()  # decoded halo values are received (detached)
                # gradient of the hop's output: from the next hop's input (if any)
                # plus the decoder's (mlp3_bwd accumulates dx)
                dx = dvL_in[q] if dvL_in is not None else torch.zeros((sd.n_loc, c.d), device=self.dev)
                x_, h1, h2 = H["dec_cache"][q]
                L.mlp3_bwd(self.dec, x_, h1, h2, dd, dx, self.g_dec)
                dvout.append(dx)
            dvL_in, du = [], []
            for q, sd in enumerate(subs):
                ws = hp.ws[("fwd", hop, q)]
                bws = hp._ws(("bwd", q), L.layer_bwd_workspace_size(desc, sd.n_own, sd.n_loc, sd.n_edges))
                dv = torch.zeros((sd.n_loc, c.d), device=self.dev)
                de = torch.zeros((max(sd.n_edges, 1), dim + n_attr), device=self.dev) if hop > 0 else None
                G = dvout[q][: sd.n_own].contiguous()
                L.layer_bwd(desc, hp.W, hp.packed, H["vin"][q], H["e"][q], sd.row_ptr, sd.col_idx, sd.csc_perm,
                            sd.csc_ptr, sd.n_own, sd.n_loc, 0, sd.n_own, G, dv, de, hp.grads, ws, bws,
                            row_ptr_host=sd.row_ptr_host)
                dp = torch.zeros((sd.n_loc, n_attr), device=self.dev)
                if hop > 0:
                    dv[sd.n_own:].zero_()  # halo latent values of hops > 1 are received (detached)
                    L.edge_refresh_bwd(de, dim, n_attr, sd.row_ptr, sd.csc_perm, sd.csc_ptr, sd.n_own, sd.n_loc,
                                       dp)
                dvL_in.append(dv)
                du.append(dp)
        for q, sd in enumerate(subs):
            x_, h1, h2 = enc_cache[q]
            L.mlp3_bwd(self.enc, x_, h1, h2, dvL_in[q], None, self.g_enc)
        if hp.world > 1:
            flat = torch.cat([t.reshape(-1) for t in self.g_enc + self.g_dec + [hp.grads[n] for n in self.CONV]]
                             + [sse])
            hp.comm.allreduce_sum_f32(flat)
            off = 0
            for t in self.g_enc + self.g_dec + [hp.grads[n] for n in self.CONV] + [sse]:
                t.copy_(flat[off:off + t.numel()].view_as(t))
                off += t.numel()
        loss_t = torch.empty(1, dtype=torch.float32, device=self.dev)
        L.mse_mean(sse, count, loss_t)
        loss = float(loss_t.item())
        return loss, dict(enc=self.g_enc, dec=self.g_dec, conv=hp.grads)

    def _params(self):
        conv = [self.hp.W[n] for n in self.CONV if n != "W_root"]
        convg = [self.hp.grads[n] for n in self.CONV if n != "W_root"]
        return self.enc + self.dec + conv, self.g_enc + self.g_dec + convg

    def step(self, v0_global, Y_global):
        """loss_and_grads, then the parameter update; returns the loss."""
        loss, _ = self.loss_and_grads(v0_global, Y_global)
        ws, gs = self._params()
        self.t += 1
        if self.opt == "adam":
            if self.m is None:
                self.m = [torch.zeros_like(w) for w in ws]
                self.v = [torch.zeros_like(w) for w in ws]
            for w, g, m, v in zip(ws, gs, self.m, self.v):
                L.adam(w, g, m, v, self.lr, self.t)
        else:
            for w, g in zip(ws, gs):
                L.sgd(w, g, self.lr)
        L.pack_weights(self.hp.desc, self.hp.W, self.hp.packed)  # the layer reads the packed copy
        return loss

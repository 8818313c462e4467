"""N>1 host-side logic on CPU (gloo, world_size 2).

The cross-process halo exchange of Alg. 1 line 411 is dsmpnn_halo_exchange:
host code that builds an op list (dsmpnn_halo_schedule) and device code that
gathers rows and calls ncclSend / ncclRecv in that order.  Here each process
asks the LIBRARY for its op list (no GPU needed) and carries it out over gloo
with the same pairing rule NCCL uses (the k-th send of rank A to rank B meets
the k-th receive of B from A); the result must equal oracle.halo.  This pins
the part of the exchange a single-GPU box cannot: that two processes'
schedules match message for message.  The device half (gathers, NCCL calls,
scatter-adds) is checked on the GPU through NCCL send/recv to self
(tests/test_gpu_comm.py).  The gradient sum of line 418
(HotPath._allreduce_grads) is checked with the all-reduce carried by gloo.
Sub-domains are mapped to processes in blocks (api.parts_of_process), as
bench.py does for --gpus N."""
import os
import socket
import types

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import halo as ohalo
from oracle import partition as opart

WORLD = 2
NPARTS = 4


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _plan(nparts=NPARTS):
    g = np.random.default_rng(5)
    x = g.random((600, 2)).astype(np.float32)
    gid = np.arange(600, dtype=np.int64) * 7 + 3
    _, _, _, ranks = opart.plan(x, gid, nparts, 0.05, 0.04)
    vals = []
    for q, rk in enumerate(ranks):
        n_loc = len(rk["local_rows"])
        n_own = rk["n_deep"] + rk["n_near"]
        v = g.normal(size=(n_loc, 5)).astype(np.float32)
        v[n_own:] = np.nan  # halo rows: stale until the refresh
        vals.append(v)
    return ranks, vals


def run_schedule(L, ranks, mine, values, proc_of, rank, direction, flags=0):
    """Carry out the library's op list for this rank: gathers / adds with
    numpy, transfers with gloo P2P in the list's order."""
    ops, stage_rows = L.halo_schedule(len(ranks), proc_of, rank, mine, [ranks[p]["halo_ptr"] for p in mine],
                                      [ranks[p]["send_ptr"] for p in mine], direction, flags)
    loc = {p: i for i, p in enumerate(mine)}
    width = values[0].shape[1]
    stage = np.zeros((stage_rows, width), values[0].dtype)
    send_rows = lambda p, q: ranks[p]["send_idx"][int(ranks[p]["send_ptr"][q]):int(ranks[p]["send_ptr"][q + 1])]
    reqs, recvd = [], []
    if direction == L.HALO_FORWARD:
        for o in ops:  # gathers first (into the halo rows or the staging rows)
            if o["kind"] == L.HALO_OP_RECV:
                continue
            rows = values[loc[o["src_part"]]][send_rows(o["src_part"], o["dst_part"])]
            assert len(rows) == o["rows"]
            if o["kind"] == L.HALO_OP_LOCAL:
                values[loc[o["dst_part"]]][o["offset"]:o["offset"] + o["rows"]] = rows
            else:
                stage[o["offset"]:o["offset"] + o["rows"]] = rows
    to_self = []  # gloo has no send-to-self: the k-th self send meets the k-th self receive here
    for o in ops:  # transfers, in schedule order (as in ncclGroupStart .. ncclGroupEnd)
        a, n = o["offset"], o["rows"]
        if o["kind"] == L.HALO_OP_SEND:
            src = stage if direction == L.HALO_FORWARD else values[loc[o["src_part"]]]
            msg = torch.from_numpy(np.ascontiguousarray(src[a:a + n]))
            if o["peer_rank"] == rank:
                to_self.append(msg)
            else:
                reqs.append(dist.isend(msg, o["peer_rank"]))
        elif o["kind"] == L.HALO_OP_RECV:
            buf = torch.empty((n, width), dtype=torch.float32)
            if o["peer_rank"] != rank:
                reqs.append(dist.irecv(buf, o["peer_rank"]))
            recvd.append((o, buf))
    for r in reqs:
        r.wait()
    for o, buf in recvd:
        if o["peer_rank"] == rank:
            buf.copy_(to_self.pop(0))
    assert not to_self
    for o, buf in recvd:
        dst = values[loc[o["dst_part"]]] if direction == L.HALO_FORWARD else stage
        dst[o["offset"]:o["offset"] + o["rows"]] = buf.numpy()
    if direction == L.HALO_REVERSE_ADD:
        for o in ops:  # additions in schedule order (owner, holder ascending)
            if o["kind"] == L.HALO_OP_SEND:
                continue
            a, n = o["offset"], o["rows"]
            src = values[loc[o["src_part"]]][a:a + n] if o["kind"] == L.HALO_OP_LOCAL else stage[a:a + n]
            values[loc[o["dst_part"]]][send_rows(o["dst_part"], o["src_part"])] += src
    return ops


def _worker(rank, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    dist.barrier()  # connect the gloo pairs before the first point-to-point message
    try:
        from paper_2402_15106_b200 import _lib as L
        from paper_2402_15106_b200 import api
        ranks, vals = _plan()
        mine = api.parts_of_process(NPARTS, WORLD, rank)
        proc_of = [p // (NPARTS // WORLD) for p in range(NPARTS)]
        tv = [vals[p].copy() for p in mine]
        ops = run_schedule(L, ranks, mine, tv, proc_of, rank, L.HALO_FORWARD)
        want = ohalo.halo_forward(ranks, vals)
        ok_halo = all(np.array_equal(t, want[p], equal_nan=True) for t, p in zip(tv, mine))
        n_remote = sum(o["kind"] != L.HALO_OP_LOCAL for o in ops)

        # REVERSE_ADD (f2): halo slices go back to their owners, added in q order
        gv = [np.nan_to_num(vals[p]).astype(np.float32) for p in mine]
        run_schedule(L, ranks, mine, gv, proc_of, rank, L.HALO_REVERSE_ADD)
        want_r = ohalo.halo_reverse_add(ranks, [np.nan_to_num(v).astype(np.float64) for v in vals])
        ok_rev = all(np.allclose(t, want_r[p], rtol=1e-6, atol=1e-6) for t, p in zip(gv, mine))

        # VIA_NCCL routes same-process pairs through send/recv to self: same result
        tv2 = [vals[p].copy() for p in mine]
        run_schedule(L, ranks, mine, tv2, proc_of, rank, L.HALO_FORWARD, L.HALO_VIA_NCCL)
        ok_via = all(np.array_equal(t, want[p], equal_nan=True) for t, p in zip(tv2, mine))

        # gradient sum over processes through the communicator's all-reduce
        names = api.GNAMES
        grads = {n: torch.full((3, 2), float(rank + 1) * (i + 1)) for i, n in enumerate(names)}
        comm = types.SimpleNamespace(allreduce_sum_f32=lambda t: dist.all_reduce(t))
        stub = types.SimpleNamespace(grads=grads, comm=comm)
        api.HotPath._allreduce_grads(stub)
        ok_red = all(torch.equal(grads[n], torch.full((3, 2), 3.0 * (i + 1))) for i, n in enumerate(names))
        q.put((rank, ok_halo, ok_rev, ok_via, ok_red, n_remote))
    except Exception as ex:  # report instead of leaving the parent waiting
        q.put((rank, repr(ex)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_halo_schedule_and_allreduce_world2():
    from paper_2402_15106_b200 import build
    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(WORLD)]
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    for r in res:
        assert len(r) == 6, f"worker failed: {r}"
    for rank, ok_halo, ok_rev, ok_via, ok_red, n_remote in sorted(res):
        assert n_remote > 0, f"rank {rank}: no cross-process message in the fixture"
        assert ok_halo, f"rank {rank}: halo refresh differs from oracle.halo"
        assert ok_rev, f"rank {rank}: reverse add differs from oracle.halo"
        assert ok_via, f"rank {rank}: VIA_NCCL schedule differs from oracle.halo"
        assert ok_red, f"rank {rank}: gradient all-reduce wrong"


def test_schedules_pair_up_for_every_rank_count():
    """For P = 8 parts over 1, 2, 4, 8 processes: every rank's k-th send to a
    peer has the size of the peer's k-th receive from it (NCCL's pairing
    rule), in both directions; single-process schedules are all LOCAL."""
    from paper_2402_15106_b200 import _lib as L
    ranks, _ = _plan(8)
    for world in (1, 2, 4, 8):
        proc_of = [p // (8 // world) for p in range(8)]
        for direction in (L.HALO_FORWARD, L.HALO_REVERSE_ADD):
            sched = {}
            for r in range(world):
                mine = [p for p in range(8) if proc_of[p] == r]
                sched[r], _ = L.halo_schedule(8, proc_of, r, mine, [ranks[p]["halo_ptr"] for p in mine],
                                              [ranks[p]["send_ptr"] for p in mine], direction)
            for a in range(world):
                for b in range(world):
                    sends = [o["rows"] for o in sched[a] if o["kind"] == L.HALO_OP_SEND and o["peer_rank"] == b]
                    recvs = [o["rows"] for o in sched[b] if o["kind"] == L.HALO_OP_RECV and o["peer_rank"] == a]
                    assert sends == recvs, (world, direction, a, b)
            if world == 1:
                assert all(o["kind"] == L.HALO_OP_LOCAL for o in sched[0])
            # every cross-part slice of the plan appears exactly once
            tot = sum(o["rows"] for r in sched for o in sched[r] if o["kind"] != L.HALO_OP_SEND)
            assert tot == sum(int(ranks[p]["halo_ptr"][-1] - ranks[p]["halo_ptr"][0]) for p in range(8))


def test_schedule_rejects_inconsistent_parts():
    from paper_2402_15106_b200 import _lib as L
    ranks, _ = _plan()
    proc_of = [0, 0, 1, 1]
    with pytest.raises(L.DsmpnnError):  # part 1 of rank 0 missing from local_parts
        L.halo_schedule(4, proc_of, 0, [0], [ranks[0]["halo_ptr"]], [ranks[0]["send_ptr"]], L.HALO_FORWARD)
    with pytest.raises(L.DsmpnnError):  # part 2 belongs to rank 1
        L.halo_schedule(4, proc_of, 0, [0, 1, 2], [ranks[p]["halo_ptr"] for p in (0, 1, 2)],
                        [ranks[p]["send_ptr"] for p in (0, 1, 2)], L.HALO_FORWARD)

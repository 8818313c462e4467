"""a8 on the GPU: the local sub-domains as one disjoint-union graph
(dsmpnn_batch_subdomains, include/dsmpnn.h; reading R31).

The union arrays are pinned to their definition (concatenation with the
header's offsets) and to the library's own CSC of the union column ids; the
union halo refresh / REVERSE_ADD to oracle.halo (bit-exact: copies and the
same fp32 addition order); the union layer chain to the per-part chain (the
same per-row arithmetic except the node GEMM's split-K order) and, through
test_gpu_grad_modes.py's batch=1 cases, to the fp64 oracle."""
import dataclasses

import numpy as np
import pytest
import torch

from oracle import halo, partition
from paper_2402_15106_b200 import synth
from gpu_util import T, N, cuda, nerr

pytestmark = pytest.mark.gpu

NAMES = ("W1", "b1", "W2", "b2", "W3", "b3", "W_root", "b")


@pytest.fixture(scope="module")
def L():
    from paper_2402_15106_b200 import build
    build.build()
    from paper_2402_15106_b200 import _lib
    return _lib


def _subs(L, n=3000, P=4, r=0.05, n_e=24, seed=3, dim=2):
    from paper_2402_15106_b200 import pipeline
    g = np.random.default_rng(seed)
    x = g.random((n, dim)).astype(np.float32)
    gid = np.arange(n, dtype=np.int64)
    a = g.normal(size=(n, 1)).astype(np.float32)
    subs, _ = pipeline.decompose(T(x), T(gid), T(a), P, r, r, range(P))
    pipeline.build_graphs(subs, r, n_e, 7, L.EDGE_DIFF, want_f32=False, want_bf16=True)
    return x, gid, a, subs


@pytest.mark.parametrize("P", [2, 4, 8])
def test_union_graph_is_the_concatenation(L, P):
    from paper_2402_15106_b200 import pipeline
    x, gid, a, subs = _subs(L, P=P)
    b = pipeline.batch_subdomains(subs)
    torch.cuda.synchronize()
    own_off = np.cumsum([0] + [sd.n_own for sd in subs])
    halo_off = own_off[-1] + np.cumsum([0] + [sd.n_halo for sd in subs])
    edge_off = np.cumsum([0] + [sd.n_edges for sd in subs])
    assert (b.n_own, b.n_loc, b.n_edges) == (own_off[-1], halo_off[-1], edge_off[-1])
    rp, col, e16, rows = [], [], [], np.zeros(b.n_loc, np.int64)
    for q, sd in enumerate(subs):
        r = N(sd.row_ptr)
        rp.append(r[:-1] + edge_off[q])
        c = N(sd.col_idx).astype(np.int64)
        col.append(np.where(c < sd.n_own, own_off[q] + c, halo_off[q] + c - sd.n_own))
        e16.append(N(sd.e16[: sd.n_edges]))
        lr = N(sd.local_rows)
        rows[own_off[q]:own_off[q + 1]] = lr[: sd.n_own]
        rows[halo_off[q]:halo_off[q + 1]] = lr[sd.n_own:]
    rp.append(np.array([edge_off[-1]]))
    assert np.array_equal(N(b.row_ptr), np.concatenate(rp))
    assert np.array_equal(N(b.row_ptr_host), np.concatenate(rp))
    ucol = np.concatenate(col)
    assert np.array_equal(N(b.col_idx[: b.n_edges]).astype(np.int64), ucol)
    assert np.array_equal(N(b.e16[: b.n_edges]), np.concatenate(e16))
    assert np.array_equal(N(b.local_rows), rows)
    # the union CSC keeps each part's (column, edge id) order, so it is the
    # CSC of the union column ids (dsmpnn_csc's definition, pinned in test_gpu_graph)
    perm = np.argsort(ucol, kind="stable")
    assert np.array_equal(N(b.csc_perm[: b.n_edges]), perm)
    assert np.array_equal(N(b.csc_ptr), np.searchsorted(ucol[perm], np.arange(b.n_loc + 1), side="left"))


def _to_union(b, vals):
    parts_own = [v[: sd.n_own] for v, sd in zip(vals, b.subs)]
    parts_halo = [v[sd.n_own:] for v, sd in zip(vals, b.subs)]
    return np.concatenate(parts_own + parts_halo)


def _from_union(b, u):
    out = []
    for q, sd in enumerate(b.subs):
        out.append(np.concatenate([u[b.own_off[q]:b.own_off[q] + sd.n_own],
                                   u[b.halo_off[q]:b.halo_off[q] + sd.n_halo]]))
    return out


@pytest.mark.parametrize("dt", [0, 1], ids=["f32", "bf16"])
def test_union_halo_refresh_matches_oracle(L, dt):
    from paper_2402_15106_b200 import pipeline
    x, gid, a, subs = _subs(L, seed=4)
    _, _, _, ranks = partition.plan(x, gid, 4, 0.05, 0.05)
    b = pipeline.batch_subdomains(subs)
    g = np.random.default_rng(5)
    vals = [g.normal(size=(len(q["local_rows"]), 64)).astype(np.float32) for q in ranks]
    if dt == 1:
        vals = [synth.round_bf16(v) for v in vals]
    u = T(_to_union(b, vals)).to(torch.bfloat16 if dt else torch.float32)
    pipeline.batch_halo(b, u, dt)
    want = halo.halo_forward(ranks, vals)
    for got, w in zip(_from_union(b, N(u).astype(np.float32)), want):
        assert np.array_equal(got, w.astype(np.float32))


def test_union_reverse_add_matches_oracle(L):
    from paper_2402_15106_b200 import pipeline
    x, gid, a, subs = _subs(L, seed=6)
    _, _, _, ranks = partition.plan(x, gid, 4, 0.05, 0.05)
    b = pipeline.batch_subdomains(subs)
    g = np.random.default_rng(7)
    vals = [g.normal(size=(len(q["local_rows"]), 64)).astype(np.float32) for q in ranks]
    u = T(_to_union(b, vals))
    pipeline.batch_halo_reverse(b, u)
    want = halo.halo_reverse_add(ranks, vals)
    for got, w in zip(_from_union(b, N(u)), want):
        assert np.array_equal(got, w)


def test_batch_rejects_inconsistent_plans(L):
    from paper_2402_15106_b200 import pipeline
    _, _, _, subs = _subs(L, seed=8)
    bad = dataclasses.replace(subs[1], halo_ptr=list(subs[1].halo_ptr))
    bad.halo_ptr[-1] += 1  # does not end at n_loc
    with pytest.raises(L.DsmpnnError) as ei:
        pipeline.batch_subdomains([subs[0], bad, subs[2], subs[3]])
    assert ei.value.status == -2  # SHAPE


def _step(c, dtype, batch, mode=0, L_=None):
    from paper_2402_15106_b200 import _lib as Lib
    from paper_2402_15106_b200.api import HotPath, StepConfig
    l = c["r"] * (1 + 2 ** -12)
    sc = StepConfig(n_points=c["n"], s=c["n"], dim=c["dim"], n_attr=1, nparts=c["P"], r=c["r"], overlap_l=l,
                    n_e=c["n_e"], d=c["d"], k=c["k"], L=L_ or c["L"], edge_mode=Lib.EDGE_DIFF, dtype=dtype,
                    seed_sampling=3, seed_capping=5, grad_mode=mode, batch=batch, streams=1)
    hp = HotPath(sc, c["W"], cuda())
    hp.build(T(c["x"]), T(c["a"]))
    assert (hp.bat is not None) == bool(batch)
    _, outs = hp.forward(T(c["v0"]))
    o = np.concatenate([N(t) for t in outs])
    g = hp.forward_backward(T(c["v0"]), T(c["G"]))
    torch.cuda.synchronize()
    return o, {n: N(g[n]).copy() for n in NAMES}


@pytest.mark.parametrize("dtype,mode", [(0, 0), (0, 1), (1, 0)], ids=["f32-detach", "f32-reverse", "bf16-detach"])
def test_union_step_matches_per_part(L, dtype, mode):
    """The union chain against the per-part chain: the per-row arithmetic is
    the same except the node GEMM's split-K order (it depends on the row
    count), so outputs and weight gradients agree to fp32 rounding.  BF16 is
    compared on one layer (deeper, a rounding difference can move a bf16
    operand across a ReLU kink; the deep BF16 chains are compared with the
    oracle in test_gpu_grad_modes.py)."""
    from test_gpu_grad_modes import _case
    c = _case(seed=81) if dtype == 0 else _case(seed=81, d=64, k=256)
    Ln = None if dtype == 0 else 1
    o0, g0 = _step(c, dtype, 0, mode, Ln)
    o1, g1 = _step(c, dtype, 1, mode, Ln)
    assert nerr(o1, o0) <= 1e-5
    for n in NAMES:
        assert nerr(g1[n], g0[n]) <= 1e-5, n


@pytest.mark.parametrize("batch", [0, 1], ids=["per-part", "union"])
def test_pipelined_steps_match_serial_steps(L, batch):
    """HotPath.step_pipelined (the next step's graph built on the build
    stream while this step's layers run) gives, step by step, bitwise the
    gradients of HotPath.step on the same inputs -- also when consecutive
    steps have different point clouds (the prefetched graph is the next
    step's, not the current one's)."""
    from paper_2402_15106_b200 import _lib as Lib
    from paper_2402_15106_b200.api import HotPath, StepConfig
    from test_gpu_grad_modes import _case
    cs = [_case(seed=91 + i, d=64, k=256) for i in range(3)]
    c = cs[0]
    l = c["r"] * (1 + 2 ** -12)
    sc = StepConfig(n_points=c["n"], s=c["n"] - 50, dim=c["dim"], n_attr=1, nparts=c["P"], r=c["r"], overlap_l=l,
                    n_e=c["n_e"], d=c["d"], k=c["k"], L=2, edge_mode=Lib.EDGE_DIFF, dtype=Lib.BF16,
                    seed_sampling=3, seed_capping=5, batch=batch)
    inp = [[T(x[n]) for n in ("x", "a", "v0", "G")] for x in (cs[0], cs[1], cs[2], cs[1])]
    hs = HotPath(sc, c["W"], cuda())
    want = []
    for x in inp:
        g = hs.step(*x)
        want.append({n: N(g[n]).copy() for n in NAMES})
    hp = HotPath(sc, c["W"], cuda())
    for i, x in enumerate(inp):
        nxt = inp[i + 1][:2] if i + 1 < len(inp) else None
        g = hp.step_pipelined(*x, next_inputs=nxt)
        got = {n: N(g[n]).copy() for n in NAMES}
        for n in NAMES:
            assert np.array_equal(got[n], want[i][n]), (i, n)
    assert getattr(hp, "_next", None) is None

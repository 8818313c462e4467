"""GPU halo exchange (a6) and decomposition self-check (§8(e)): P virtual ranks
on one device through the C ABI, against the oracle plan/halo and against the
undecomposed GPU run."""
import numpy as np
import pytest
import torch

from oracle import halo, partition, sample
from paper_2402_15106_b200 import synth
from gpu_util import T, N, cuda, nerr

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    from paper_2402_15106_b200 import build
    build.build()
    from paper_2402_15106_b200 import _lib
    return _lib


def _build(L, x, a, gid, P, l, r, n_e, seed, mode):
    from paper_2402_15106_b200 import pipeline
    subs, glob = pipeline.decompose(T(x), T(gid), T(a), P, l, r, range(P))
    for sd in subs:
        pipeline.build_graph(sd, r, n_e, seed, mode)
    return subs


@pytest.mark.parametrize("width", [8, 5, 6], ids=["w8", "w5", "w6"])
def test_halo_loopback_matches_oracle(L, width):
    # rows of whole 16-byte chunks (w8) take the one-launch job-table path,
    # the others the per-peer gathers
    g = np.random.default_rng(3)
    x = g.random((3000, 2)).astype(np.float32)
    gid = np.arange(3000, dtype=np.int64)
    a = g.normal(size=(3000, 1)).astype(np.float32)
    P, r = 4, 0.05
    from paper_2402_15106_b200 import pipeline
    subs, _ = pipeline.decompose(T(x), T(gid), T(a), P, r, r, range(P))
    _, _, _, ranks = partition.plan(x, gid, P, r, r)
    for dt, tdt in ((0, torch.float32), (1, torch.bfloat16)):
        vals_np = [g.normal(size=(len(q["local_rows"]), width)).astype(np.float32) for q in ranks]
        if dt == 1:
            vals_np = [synth.round_bf16(v) for v in vals_np]
        vals = [T(v).to(tdt) for v in vals_np]
        pipeline.halo_exchange_loopback(subs, vals, dt)
        want = halo.halo_forward(ranks, vals_np)
        for got, w in zip(vals, want):
            assert np.array_equal(N(got).astype(np.float32), w.astype(np.float32))


def test_accumulate_f32(L):
    g = np.random.default_rng(4)
    for n in (1, 257, 1 << 20):
        a, b = g.normal(size=n).astype(np.float32), g.normal(size=n).astype(np.float32)
        ta, tb = T(a), T(b)
        L.accumulate_f32(ta, tb)
        assert np.array_equal(N(ta), a + b)


def test_scatter_add_reverse(L):
    v = torch.zeros((10, 3), device=cuda())
    src = torch.arange(12, dtype=torch.float32, device=cuda()).view(4, 3)
    rows = torch.tensor([7, 1, 3, 9], dtype=torch.int32, device=cuda())
    L.halo_scatter_add(src, rows, v)
    want = np.zeros((10, 3), np.float32)
    want[[7, 1, 3, 9]] = np.arange(12).reshape(4, 3)
    assert np.array_equal(N(v), want)


@pytest.mark.parametrize("dtype", [0])
def test_decomposed_equals_undecomposed_gpu(L, dtype):
    # north_star: decomposed graph with full-width halo reproduces the
    # undecomposed output on owned nodes (2 layers, halo refresh in between)
    cfg = synth.CONFIGS["darcy"]
    coords, attr = synth.points(cfg)
    ids = sample.sample(len(coords), 4096, 5)
    x, a, gid = coords[ids], attr[ids], ids.astype(np.int64)
    r, n_e, d, k = 0.1, 32, 16, 32
    l = r * (1 + 2 ** -12)
    from paper_2402_15106_b200 import pipeline
    W = synth.weights(3, d, d, k)
    Wd = {n: T(W[n]) for n in W}
    desc = L.make_desc(3, d, d, k, dtype, L.ROOT_DENSE, L.ACT_RELU)
    packed = torch.empty(L.packed_weights_size(desc), dtype=torch.uint8, device=cuda())
    L.pack_weights(desc, Wd, packed)
    vg = synth.node_features(len(x), d)

    def run(P):
        subs = _build(L, x, a, gid, P, l, r, n_e, 9, L.EDGE_DIFF)
        vals = [T(vg[N(sd.local_rows)]) for sd in subs]
        outs = None
        for layer_i in range(2):
            outs = []
            for sd, v in zip(subs, vals):
                out = torch.empty((sd.n_own, d), device=cuda())
                ws = torch.empty(L.layer_workspace_size(desc, sd.n_own, sd.n_edges), dtype=torch.uint8,
                                 device=cuda())
                L.layer_fwd(desc, Wd, packed, v, sd.e32, sd.row_ptr, sd.col_idx, sd.n_own, 0, sd.n_own, out, None, ws,
                            row_ptr_host=sd.row_ptr_host)
                outs.append(out)
            vals = [torch.cat([o, v[sd.n_own:]], 0).contiguous() for o, v, sd in zip(outs, vals, subs)]
            pipeline.halo_exchange_loopback(subs, vals, 0)
        return subs, outs

    s1, o1 = run(1)
    pos = {int(rw): i for i, rw in enumerate(N(s1[0].local_rows))}
    ref = N(o1[0])
    s4, o4 = run(4)
    for sd, o in zip(s4, o4):
        idx = [pos[int(rw)] for rw in N(sd.local_rows)[:sd.n_own]]
        assert np.array_equal(N(o), ref[idx])

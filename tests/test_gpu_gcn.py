"""GPU parity for f3 (GCN layer) against the
fp64 oracle/gcn.py on the same seeded inputs: forward (out, agg) and backward
(dv, dW, dc), normwise-inf <= 1e-5 (fp32), at the paper's width 378 on a
radius graph with isolated rows, n_dst < n_loc, and a 6-layer chain."""
import numpy as np
import pytest
import torch

from oracle import gcn, graph
from gpu_util import T, N, cuda, nerr

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    from paper_2402_15106_b200 import build
    build.build()
    from paper_2402_15106_b200 import _lib
    return _lib


def _problem(seed, n=900, n_dst=800, d_in=378, d_out=378, r=0.07, n_e=24, isolated=4):
    g = np.random.default_rng(seed)
    x = g.random((n, 2)).astype(np.float32)
    x[n_dst - isolated:n_dst] += 10.0 + np.arange(isolated, dtype=np.float32)[:, None] * 3  # isolated rows
    rp, col = graph.radius_graph(x, np.arange(n), n_dst, r, n_e, seed)
    W = (g.uniform(-1, 1, (d_out, d_in)) / np.sqrt(d_in)).astype(np.float32)
    c = g.uniform(-0.1, 0.1, d_out).astype(np.float32)
    v = g.normal(size=(n, d_in)).astype(np.float32)
    G = g.normal(size=(n_dst, d_out)).astype(np.float32)
    return rp, col, W, c, v, G, n, n_dst


def _run(L, rp, col, W, c, v, G, n, n_dst, act):
    d_out, d_in = W.shape
    E = len(col)
    rpt, colt = T(rp), T(col) if E else torch.zeros(1, dtype=torch.int32, device=cuda())
    agg = torch.empty((n_dst, d_in), device=cuda())
    out = torch.empty((n_dst, d_out), device=cuda())
    Wt, ct, vt = T(W), T(c), T(v)
    L.gcn_fwd(Wt, ct, act, vt, rpt, colt, n_dst, agg, out)
    perm = torch.empty(max(E, 1), dtype=torch.int32, device=cuda())
    cptr = torch.empty(n + 1, dtype=torch.int64, device=cuda())
    L.csc(colt[:E], n, perm, cptr)
    gv = torch.zeros((n, d_in), device=cuda())
    gW = torch.zeros_like(Wt)
    gc = torch.zeros_like(ct)
    L.gcn_bwd(Wt, act, rpt, colt, perm, cptr, n_dst, n, agg, out, T(G), gv, gW, gc)
    torch.cuda.synchronize()
    return N(out), N(agg), N(gv), N(gW), N(gc)


@pytest.mark.parametrize("act", [gcn.ACT_RELU, gcn.ACT_IDENTITY], ids=["relu", "identity"])
def test_gcn_layer_matches_oracle(L, act):
    rp, col, W, c, v, G, n, n_dst = _problem(5 + act)
    out, agg, gv, gW, gc = _run(L, rp, col, W, c, v, G, n, n_dst, act)
    o_out, o_agg = gcn.gcn_fwd(W, c, act, v, rp, col)
    # kink-masked upstream gradient for ReLU: entries whose pre-activation is
    # within 1e-6 of 0 are decisions the two precisions may take differently
    if act == gcn.ACT_RELU:
        pre = o_agg @ W.astype(np.float64).T + c
        G = np.where(np.abs(pre) < 1e-6, 0.0, G).astype(np.float32)
        out, agg, gv, gW, gc = _run(L, rp, col, W, c, v, G, n, n_dst, act)
    dv, dW, dc = gcn.gcn_bwd(W, c, act, v, rp, col, G)
    assert nerr(agg, o_agg) <= 1e-5
    assert nerr(out, o_out) <= 1e-5
    assert nerr(gv, dv) <= 1e-5
    assert nerr(gW, dW) <= 1e-5
    assert nerr(gc, dc) <= 1e-5


def test_gcn_six_layer_chain(L):
    # 6 hidden layers of width 378 (forward chain; each layer's
    # input is the previous output, n_dst = n)
    rp, col, W, c, v, G, n, n_dst = _problem(9, n=600, n_dst=600, isolated=2)
    Wt, ct = T(W), T(c)
    rpt, colt = T(rp), T(col)
    x = T(v)
    ref = v.astype(np.float64)
    for _ in range(6):
        agg = torch.empty((n, W.shape[1]), device=cuda())
        out = torch.empty((n, W.shape[0]), device=cuda())
        L.gcn_fwd(Wt, ct, gcn.ACT_RELU, x, rpt, colt, n, agg, out)
        x = out
        ref, _ = gcn.gcn_fwd(W, c, gcn.ACT_RELU, ref, rp, col)
    torch.cuda.synchronize()
    assert nerr(N(x), ref) <= 1e-5


def test_gcn_bad_args(L):
    W = torch.zeros((4, 3), device=cuda())
    with pytest.raises(L.DsmpnnError):
        L.gcn_fwd(W, torch.zeros(4, device=cuda()), 7, torch.zeros((2, 3), device=cuda()),
                  torch.zeros(3, dtype=torch.int64, device=cuda()), torch.zeros(1, dtype=torch.int32, device=cuda()),
                  2, torch.empty((2, 3), device=cuda()), torch.empty((2, 4), device=cuda()))

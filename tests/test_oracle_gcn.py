"""Pins for oracle/gcn.py (O8) against what the definition
fixes independently of the oracle's own code."""
import numpy as np
import scipy.sparse as sp

from oracle import gcn, graph


def _case(seed, n=60, d_in=5, d_out=4, r=0.3, n_e=6):
    g = np.random.default_rng(seed)
    x = g.random((n, 2)).astype(np.float32)
    rp, col = graph.radius_graph(x, np.arange(n), n, r, n_e, seed)
    W = g.normal(size=(d_out, d_in))
    c = g.normal(size=d_out)
    v = g.normal(size=(n, d_in))
    return rp, col, W, c, v


def test_isolated_node_is_its_own_mlp():
    # SPEC.md:255 "single isolated node -> MLP applied to its own features"
    W = np.array([[1.0, -2.0], [0.5, 3.0]])
    c = np.array([0.25, -1.0])
    v = np.array([[2.0, 1.0]])
    out, agg = gcn.gcn_fwd(W, c, gcn.ACT_RELU, v, [0, 0], [])
    assert np.array_equal(agg, v)
    assert np.allclose(out, np.maximum(v @ W.T + c, 0.0), rtol=0, atol=0)


def test_two_node_symmetry():
    # two-node complete graph with equal features -> equal outputs
    W = np.random.default_rng(1).normal(size=(3, 3))
    v = np.array([[1.0, 2.0, 3.0], [1.0, 2.0, 3.0]])
    out, _ = gcn.gcn_fwd(W, np.zeros(3), gcn.ACT_IDENTITY, v, [0, 1, 2], [1, 0])
    assert np.array_equal(out[0], out[1])


def test_mean_with_self_equals_normalised_adjacency_spmm():
    # agg = D^-1 (A + I) v with A the capped adjacency: scipy sparse product
    rp, col, W, c, v = _case(3)
    n = len(rp) - 1
    A = sp.csr_matrix((np.ones(len(col)), col, rp), shape=(n, n)) + sp.identity(n)
    deg = np.asarray(A.sum(axis=1)).ravel()
    want = sp.diags(1.0 / deg) @ A @ v
    _, agg = gcn.gcn_fwd(W, c, gcn.ACT_IDENTITY, v, rp, col)
    assert np.allclose(agg, want, rtol=1e-13, atol=1e-13)


def test_permutation_invariance_of_neighbour_order():
    rp, col, W, c, v = _case(4)
    g = np.random.default_rng(0)
    col2 = col.copy()
    for i in range(len(rp) - 1):
        seg = col2[rp[i]:rp[i + 1]]
        col2[rp[i]:rp[i + 1]] = seg[g.permutation(len(seg))]
    a, _ = gcn.gcn_fwd(W, c, gcn.ACT_RELU, v, rp, col)
    b, _ = gcn.gcn_fwd(W, c, gcn.ACT_RELU, v, rp, col2)
    assert np.allclose(a, b, rtol=1e-14, atol=1e-14)


def test_backward_central_differences():
    rp, col, W, c, v = _case(5, n=25, d_in=3, d_out=2, r=0.4)
    G = np.random.default_rng(9).normal(size=(25, 2))
    dv, dW, dc = gcn.gcn_bwd(W, c, gcn.ACT_RELU, v, rp, col, G)
    loss = lambda W_, c_, v_: float((gcn.gcn_fwd(W_, c_, gcn.ACT_RELU, v_, rp, col)[0] * G).sum())
    h = 1e-6
    for arr, grad, name in ((v, dv, "v"), (W, dW, "W"), (c, dc, "c")):
        num = np.zeros_like(arr)
        it = np.nditer(arr, flags=["multi_index"])
        for _ in it:
            idx = it.multi_index
            args = {"v": v.copy(), "W": W.copy(), "c": c.copy()}
            args[name][idx] += h
            up = loss(args["W"], args["c"], args["v"])
            args[name][idx] -= 2 * h
            dn = loss(args["W"], args["c"], args["v"])
            num[idx] = (up - dn) / (2 * h)
        assert np.allclose(grad, num, rtol=1e-5, atol=1e-6), name

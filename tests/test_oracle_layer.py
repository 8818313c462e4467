"""Pins for oracle O5/O6 (Eq. 1 forward/backward), R1-R5, R18."""
import json
import os

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import decomp, graph, layer, sample
from oracle.layer import ACT_IDENTITY, ACT_RELU, ROOT_DENSE, ROOT_IDENTITY, ROOT_NONE, LayerDesc

ROOTS = {"none": ROOT_NONE, "identity": ROOT_IDENTITY, "dense": ROOT_DENSE}
ACTS = {"identity": ACT_IDENTITY, "relu": ACT_RELU}


def _load(golden_dir, name):
    with open(os.path.join(golden_dir, name)) as f:
        fx = json.load(f)
    desc = LayerDesc(fx["d_e"], fx["d_in"], fx["d_out"], fx["k"], ROOTS[fx["root"]], ACTS[fx["act"]])
    W = {k: np.array(fx[k], float) for k in ("W1", "b1", "W2", "b2", "W3", "b3", "W_root", "b")}
    return fx, desc, W


def _rand_problem(seed, n=40, d_e=3, d_in=4, d_out=5, k=6, root=ROOT_DENSE, act=ACT_RELU,
                  r=0.3, n_e=7):
    g = np.random.default_rng(seed)
    x = g.random((n, 2)).astype(np.float32)
    rp, ci = graph.radius_graph(x, np.arange(n), n, r, n_e, seed)
    E = int(rp[-1])
    desc = LayerDesc(d_e, d_in, d_out, k, root, act)
    W = dict(W1=g.normal(size=(k, d_e)), b1=g.normal(size=k), W2=g.normal(size=(k, k)) / np.sqrt(k),
             b2=g.normal(size=k), W3=g.normal(size=(d_in * d_out, k)) / np.sqrt(k),
             b3=g.normal(size=d_in * d_out), W_root=g.normal(size=(d_out, d_in)),
             b=g.normal(size=d_out))
    v = g.normal(size=(n, d_in))
    e = g.normal(size=(E, d_e))
    return desc, W, v, e, rp, ci


def test_orientation_hand_fixture(golden_dir):
    fx, desc, W = _load(golden_dir, "layer_orientation.json")
    out, _ = layer.layer_fwd(desc, W, np.array(fx["v"]), np.array(fx["e"]), fx["row_ptr"], fx["col_idx"])
    assert np.allclose(out[0], fx["expected_out_row0"], atol=0, rtol=0)


def test_scalar_mlp_hand_fixture(golden_dir):
    fx, desc, W = _load(golden_dir, "layer_scalar_mlp.json")
    out, pre = layer.layer_fwd(desc, W, np.array(fx["v"]), np.array(fx["e"]), fx["row_ptr"], fx["col_idx"])
    assert np.allclose(out, fx["expected_out"], atol=1e-12)
    assert np.allclose(pre, fx["expected_pre"], atol=1e-12)


@pytest.mark.parametrize("root,act", [(ROOT_NONE, ACT_IDENTITY), (ROOT_DENSE, ACT_RELU),
                                      (ROOT_IDENTITY, ACT_RELU)])
def test_identity_kernel_is_csr_spmm(root, act):
    # K == I (W3 = 0, b3 = vec(I)) -> sigma(D^-1 A V + root + b): a textbook
    # CSR SpMM, computed here with scipy.sparse
    d = 4
    desc, W, v, e, rp, ci = _rand_problem(0, d_in=d, d_out=d, root=root, act=act)
    W["W3"] = np.zeros_like(W["W3"])
    W["b3"] = np.eye(d).reshape(-1)
    n = len(rp) - 1
    deg = np.diff(rp)
    A = sp.csr_matrix((np.ones(len(ci)), ci, rp), shape=(n, v.shape[0]))
    Dinv = sp.diags(np.where(deg > 0, 1.0 / np.maximum(deg, 1), 0.0))
    want = Dinv @ (A @ v)
    if root == ROOT_DENSE:
        want = want + v[:n] @ W["W_root"].T
    elif root == ROOT_IDENTITY:
        want = want + v[:n]
    want = want + W["b"]
    if act == ACT_RELU:
        want = np.maximum(want, 0)
    out, _ = layer.layer_fwd(desc, W, v, e, rp, ci)
    assert np.allclose(out, want, rtol=1e-12, atol=1e-12)


def test_empty_rows_get_root_plus_bias():
    desc, W, v, e, rp, ci = _rand_problem(1)
    rp0 = np.zeros_like(rp)
    out, pre = layer.layer_fwd(desc, W, v, e[:0], rp0, ci[:0])
    assert np.allclose(pre, v[: len(rp) - 1] @ W["W_root"].T + W["b"], atol=1e-12)


def test_constant_field_invariance():
    # v == c and W1 == 0: every edge has the same K, so every row with deg >= 1
    # has the same output whatever its degree (pins the 1/|E_i| reading R3)
    desc, W, v, e, rp, ci = _rand_problem(2, n=60, n_e=9)
    W["W1"] = np.zeros_like(W["W1"])
    c = np.random.default_rng(0).normal(size=desc.d_in)
    v = np.tile(c, (v.shape[0], 1))
    out, _ = layer.layer_fwd(desc, W, v, e, rp, ci)
    deg = np.diff(rp)
    assert len(set(deg[deg > 0])) > 2
    ref = out[np.nonzero(deg > 0)[0][0]]
    assert np.allclose(out[deg > 0], ref, rtol=1e-13, atol=1e-13)


def test_linearity_in_v():
    desc, W, v, e, rp, ci = _rand_problem(3, act=ACT_IDENTITY)
    W["b"] = np.zeros_like(W["b"])
    g = np.random.default_rng(1)
    v2 = g.normal(size=v.shape)
    f = lambda vv: layer.layer_fwd(desc, W, vv, e, rp, ci)[1]
    assert np.allclose(f(2.5 * v - 1.5 * v2), 2.5 * f(v) - 1.5 * f(v2), atol=1e-12)


def test_duplicate_edges_leave_mean_unchanged():
    desc, W, v, e, rp, ci = _rand_problem(4)
    deg = np.diff(rp)
    rp2 = np.concatenate([[0], np.cumsum(2 * deg)])
    ci2 = np.concatenate([np.concatenate([ci[a:b], ci[a:b]]) for a, b in zip(rp[:-1], rp[1:])])
    e2 = np.concatenate([np.concatenate([e[a:b], e[a:b]]) for a, b in zip(rp[:-1], rp[1:])])
    o1, _ = layer.layer_fwd(desc, W, v, e, rp, ci)
    o2, _ = layer.layer_fwd(desc, W, v, e2, rp2, ci2)
    assert np.allclose(o1, o2, rtol=1e-12, atol=1e-12)


def test_contraction_formulation_matches_materialised_K():
    # (h~ (x) v_j) . Theta~ == K_p^T v_j to 1e-12: pins the index algebra the GPU uses
    desc, W, v, e, rp, ci = _rand_problem(5, d_in=3, d_out=5, k=7)
    E = len(ci)
    m1 = layer.messages(desc, W, v, e, ci, 0, E)
    m2 = layer.messages_contraction(desc, W, v, e, ci, 0, E)
    assert np.allclose(m1, m2, rtol=1e-12, atol=1e-12)


def test_node_permutation_invariance():
    # relabelling the nodes (rows re-sorted by gid) permutes outputs bitwise
    g = np.random.default_rng(6)
    n = 50
    x = g.random((n, 2)).astype(np.float32)
    gid = np.arange(n) + 1000
    attr = g.normal(size=(n, 1)).astype(np.float32)
    desc, W, _, _, _, _ = _rand_problem(6, d_e=3)
    v = g.normal(size=(n, desc.d_in))
    from oracle import features

    def run(perm):
        xs, gs, vs, at = x[perm], gid[perm], v[perm], attr[perm]
        rp, ci = graph.radius_graph(xs, gs, n, 0.3, 7, 3)
        e = features.edge_features("diff", xs, at, features.dst_of_edges(rp), ci)
        return layer.layer_fwd(desc, W, vs, e, rp, ci)[0]

    base = run(np.arange(n))
    perm = g.permutation(n)
    o = run(perm)
    assert np.array_equal(o, base[perm])


def _fd_check(desc, W, v, e, rp, ci, G, eps=1e-6):
    dv, de, grads = layer.layer_bwd(desc, W, v, e, rp, ci, G)
    f = lambda W_, v_, e_: float(np.sum(G * layer.layer_fwd(desc, W_, v_, e_, rp, ci)[0]))
    g = np.random.default_rng(11)
    worst = 0.0
    for name in list(grads) + ["v", "e"]:
        base = v if name == "v" else e if name == "e" else W[name]
        for _ in range(3):
            dlt = g.normal(size=base.shape)
            if name == "v":
                fp, fm = f(W, v + eps * dlt, e), f(W, v - eps * dlt, e)
                an = np.sum(dv * dlt)
            elif name == "e":
                fp, fm = f(W, v, e + eps * dlt), f(W, v, e - eps * dlt)
                an = np.sum(de * dlt)
            else:
                Wp = dict(W); Wp[name] = W[name] + eps * dlt
                Wm = dict(W); Wm[name] = W[name] - eps * dlt
                fp, fm = f(Wp, v, e), f(Wm, v, e)
                an = np.sum(grads[name] * dlt)
            num = (fp - fm) / (2 * eps)
            worst = max(worst, abs(num - an) / max(1e-8, abs(num), abs(an)))
    return worst


def _kink_margin(desc, W, v, e, rp, ci):
    a1, h, _ = layer.kappa(W, e)
    z1 = e @ W["W1"].T + W["b1"]
    z2 = a1 @ W["W2"].T + W["b2"]
    _, pre = layer.layer_fwd(desc, W, v, e, rp, ci)
    return min(np.abs(z1).min(), np.abs(z2).min(), np.abs(pre).min())


@pytest.mark.parametrize("root,act", [(ROOT_DENSE, ACT_RELU), (ROOT_IDENTITY, ACT_IDENTITY),
                                      (ROOT_NONE, ACT_RELU)])
def test_backward_finite_differences(root, act):
    # central differences in fp64, directional, every input and parameter
    # (SPEC.md:73,77); draws too close to a ReLU kink are re-drawn
    for seed in range(20, 60):
        desc, W, v, e, rp, ci = _rand_problem(seed, n=25, d_in=3, d_out=3, k=5, root=root, act=act)
        if _kink_margin(desc, W, v, e, rp, ci) > 1e-3:
            break
    G = np.random.default_rng(seed).normal(size=(len(rp) - 1, desc.d_out))
    assert _fd_check(desc, W, v, e, rp, ci, G) < 1e-6


def test_backward_mutation_is_caught():
    # a corrupted backward (x2) must fail the same check
    for seed in range(20, 60):
        desc, W, v, e, rp, ci = _rand_problem(seed, n=25, d_in=3, d_out=3, k=5)
        if _kink_margin(desc, W, v, e, rp, ci) > 1e-3:
            break
    G = np.random.default_rng(seed).normal(size=(len(rp) - 1, desc.d_out))
    orig = layer.layer_bwd
    try:
        def bad(*a, **kw):
            dv, de, g = orig(*a, **kw)
            g["W2"] = 2 * g["W2"]
            return dv, de, g
        layer.layer_bwd = bad
        assert _fd_check(desc, W, v, e, rp, ci, G) > 1e-3
    finally:
        layer.layer_bwd = orig


def test_backward_mass_conservation():
    # K == I, root NONE, sigma identity: sum_j dv_j = sum_{i: deg>=1} g_i
    desc, W, v, e, rp, ci = _rand_problem(7, d_in=4, d_out=4, root=ROOT_NONE, act=ACT_IDENTITY)
    W["W3"] = np.zeros_like(W["W3"])
    W["b3"] = np.eye(4).reshape(-1)
    G = np.random.default_rng(2).normal(size=(len(rp) - 1, 4))
    dv, _, _ = layer.layer_bwd(desc, W, v, e, rp, ci, G)
    deg = np.diff(rp)
    assert np.allclose(dv.sum(0), G[deg > 0].sum(0), atol=1e-12)


def test_backward_masked_upstream_equals_subset():
    # gradient with G restricted to a row subset == backward over those rows only
    desc, W, v, e, rp, ci = _rand_problem(8)
    n = len(rp) - 1
    rows = np.array([1, 5, 9, 17])
    G = np.random.default_rng(3).normal(size=(n, desc.d_out))
    Gm = np.zeros_like(G); Gm[rows] = G[rows]
    full = layer.layer_bwd(desc, W, v, e, rp, ci, Gm)
    sub = layer.layer_bwd(desc, W, v, e, rp, ci, G[rows], rows=rows)
    assert np.allclose(full[0], sub[0], atol=1e-12)
    for k in full[2]:
        assert np.allclose(full[2][k], sub[2][k], atol=1e-12)


def test_backward_adjoint_linearity():
    # the backward is linear in G
    desc, W, v, e, rp, ci = _rand_problem(9, act=ACT_IDENTITY)
    g = np.random.default_rng(4)
    n = len(rp) - 1
    G1, G2 = g.normal(size=(n, desc.d_out)), g.normal(size=(n, desc.d_out))
    a = layer.layer_bwd(desc, W, v, e, rp, ci, G1)
    b = layer.layer_bwd(desc, W, v, e, rp, ci, G2)
    c = layer.layer_bwd(desc, W, v, e, rp, ci, 2 * G1 - G2)
    assert np.allclose(c[0], 2 * a[0] - b[0], atol=1e-10)
    assert np.allclose(c[2]["W1"], 2 * a[2]["W1"] - b[2]["W1"], atol=1e-10)


def _decomp_case(seed, P, l_factor, dim=2):
    g = np.random.default_rng(seed)
    n = 400
    x = g.random((n, dim)).astype(np.float32)
    gid = g.permutation(10 * n)[:n]
    attr = g.normal(size=(n, 1)).astype(np.float32)
    r = 0.12
    desc = LayerDesc(dim + 1, 4, 4, 6, ROOT_DENSE, ACT_RELU)
    W = _rand_problem(seed, d_e=dim + 1, d_in=4, d_out=4, k=6)[1]
    vg = g.normal(size=(n, 4))
    return x, gid, attr, r, desc, W, vg


@pytest.mark.parametrize("P,dim", [(2, 2), (4, 2), (4, 3)])
def test_decomposed_equals_undecomposed(P, dim):
    # north_star: a decomposed graph with full-width halo reproduces the
    # undecomposed layer output on owned nodes - bitwise, over 2 layers (R10, R11)
    x, gid, attr, r, desc, W, vg = _decomp_case(30 + P + dim, P, 1, dim)
    l = r * (1 + 2 ** -12)
    _, _, _, ranks = decomp.build_local(x, gid, attr, P, l, r, 8, 5, "diff")
    outs = decomp.ds_forward(desc, W, ranks, lambda rows: vg[rows], 2)
    _, _, _, single = decomp.build_local(x, gid, attr, 1, l, r, 8, 5, "diff")
    ref = decomp.ds_forward(desc, W, single, lambda rows: vg[rows], 2)[0]
    pos = {int(rw): k for k, rw in enumerate(single[0]["local_rows"])}
    for q, o in zip(ranks, outs):
        n_own = q["n_deep"] + q["n_near"]
        idx = [pos[int(rw)] for rw in q["local_rows"][:n_own]]
        assert np.array_equal(o, ref[idx])


def test_zero_overlap_differs():
    # with l = 0 the decomposed output generically differs
    x, gid, attr, r, desc, W, vg = _decomp_case(41, 4, 0)
    _, _, _, ranks = decomp.build_local(x, gid, attr, 4, 0.0, r, 8, 5, "diff")
    outs = decomp.ds_forward(desc, W, ranks, lambda rows: vg[rows], 1)
    _, _, _, single = decomp.build_local(x, gid, attr, 1, 0.0, r, 8, 5, "diff")
    ref = decomp.ds_forward(desc, W, single, lambda rows: vg[rows], 1)[0]
    pos = {int(rw): k for k, rw in enumerate(single[0]["local_rows"])}
    diff = 0
    for q, o in zip(ranks, outs):
        n_own = q["n_deep"] + q["n_near"]
        idx = [pos[int(rw)] for rw in q["local_rows"][:n_own]]
        diff += int(np.sum(np.any(o != ref[idx], axis=1)))
    assert diff > 0


def test_round_bf16_matches_torch():
    # the oracle's own bf16 rounding == torch's CPU float32 -> bfloat16 conversion (library routine)
    import torch
    from oracle.precision import round_bf16
    g = np.random.default_rng(0)
    x = np.concatenate([g.normal(size=20000) * 10.0 ** g.integers(-30, 30, 20000),
                        [0.0, -0.0, 1.0, 1.00390625, 1.01171875, 3.0e38, -1e-40]])
    want = torch.from_numpy(x.astype(np.float32)).to(torch.bfloat16).to(torch.float64).numpy()
    assert np.array_equal(round_bf16(x), want)


def test_act_round_only_changes_activations():
    # with act_round="bf16" the layer equals the plain layer on bf16-valued activations:
    # identical when the kappa activations are already bf16-representable (W2 = 0, b2 bf16)
    desc, W, v, e, rp, ci = _rand_problem(15)
    from oracle.precision import round_bf16
    W["W1"] = np.zeros_like(W["W1"])
    W["b1"] = round_bf16(W["b1"])
    W["W2"] = np.zeros_like(W["W2"])
    W["b2"] = round_bf16(W["b2"])
    a = layer.layer_fwd(desc, W, v, e, rp, ci)[0]
    desc.act_round = "bf16"
    b = layer.layer_fwd(desc, W, v, e, rp, ci)[0]
    assert np.array_equal(a, b)


def _ds_grads(P, L, mode, seed=51, dim=2):
    x, gid, attr, r, desc, W, vg = _decomp_case(seed, P, 1, dim)
    G = np.random.default_rng(seed + 1).normal(size=vg.shape)
    l = r * (1 + 2 ** -12)
    _, _, _, ranks = decomp.build_local(x, gid, attr, P, l, r, 8, 5, "diff")
    return decomp.ds_forward_backward(desc, W, ranks, lambda rows: vg[rows], lambda rows: G[rows], L, mode), \
        (x, gid, attr, r, desc, W, vg, G)


def _close(a, b, tol=1e-10):
    return all(np.allclose(a[n], b[n], rtol=tol, atol=tol * max(1.0, np.abs(b[n]).max())) for n in a)


@pytest.mark.parametrize("P,L", [(2, 2), (4, 3)])
def test_ds_reverse_add_gradients_equal_undecomposed(P, L):
    # with REVERSE_ADD (the transpose of the forward halo copy)
    # the decomposed weight gradients equal the single-domain ones for any depth
    g_ds, case = _ds_grads(P, L, decomp.REVERSE_ADD)
    g_1, _ = _ds_grads(1, L, decomp.REVERSE_ADD)
    assert _close(g_ds, g_1)
    # and the single-domain chain written out directly (no partition machinery)
    x, gid, attr, r, desc, W, vg, G = case
    g_plain = decomp.undecomposed_forward_backward(desc, W, x, gid, attr, r, 8, 5, "diff", vg, G, L)
    assert _close(g_plain, g_1)


def test_ds_detach_exact_at_one_layer_only():
    # R16: DETACH drops the halo rows' gradient; it is exact for one layer
    # (Alg. 1 :417 local backprop) and generically not for two
    g1_ds, _ = _ds_grads(4, 1, decomp.DETACH)
    g1_ref, _ = _ds_grads(1, 1, decomp.DETACH)
    assert _close(g1_ds, g1_ref)
    g2_ds, _ = _ds_grads(4, 2, decomp.DETACH)
    g2_ref, _ = _ds_grads(1, 2, decomp.DETACH)
    assert not _close(g2_ds, g2_ref, 1e-6)


def _infer_case(seed=71, n=300, P=4):
    x, gid, attr, r, desc, W, vg = _decomp_case(seed, P, 1, 2)
    return x, attr, r, desc, W, vg


def test_infer_reassemble_single_pass_equals_undecomposed():
    # f4 with s = N and one pass: every node visited once, and the decomposed
    # forward equals the single-domain forward (north_star property), so the
    # reassembled field is exactly the S-MPNN output
    x, attr, r, desc, W, vg = _infer_case()
    n = len(x)
    l = r * (1 + 2 ** -12)
    field, cnt = decomp.infer_reassemble(desc, W, x, attr, 4, l, r, 8, 5, n, [9], vg, 2, "diff")
    assert np.all(cnt == 1)
    ids = sample.sample(n, n, 9).astype(np.int64)
    _, _, _, single = decomp.build_local(x[ids], ids, attr[ids], 1, l, r, 8, 5, "diff")
    ref = decomp.ds_forward(desc, W, single, lambda rows: vg[ids[rows]], 2)[0]
    g = single[0]["local_gid"]
    assert np.array_equal(field[g], ref)


def test_infer_reassemble_counts_and_averages():
    x, attr, r, desc, W, vg = _infer_case(seed=72)
    n = len(x)
    l = r * (1 + 2 ** -12)
    s = n // 3
    seeds = [1, 2, 3]
    field, cnt = decomp.infer_reassemble(desc, W, x, attr, 2, l, r, 8, 5, s, seeds, vg, 1, "diff")
    want = np.zeros(n, np.int64)
    for sd in seeds:
        want[sample.sample(n, s, sd)] += 1
    assert np.array_equal(cnt, want)
    assert np.all(field[cnt == 0] == 0.0)
    # the same pass twice averages to the pass itself (exact in fp64)
    f1, c1 = decomp.infer_reassemble(desc, W, x, attr, 2, l, r, 8, 5, s, [4], vg, 1, "diff")
    f2, c2 = decomp.infer_reassemble(desc, W, x, attr, 2, l, r, 8, 5, s, [4, 4], vg, 1, "diff")
    assert np.array_equal(c2, 2 * c1) and np.array_equal(f1, f2)

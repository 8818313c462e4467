"""GPU parity for a4/a5 (layer forward) and a7 (layer backward) against the
fp64 oracle: normwise-inf relative error <= 1e-5 in F32 mode and <= 2e-2 in
BF16 mode (BASELINE.json north_star), on every output and gradient."""
import numpy as np
import pytest
import torch

from oracle import features, graph, layer, sample
from oracle.layer import LayerDesc
from paper_2402_15106_b200 import synth
from gpu_util import T, N, cuda, hash_rows, nerr

pytestmark = pytest.mark.gpu

TOL = {0: 1e-5, 1: 2e-2}
GNAMES = ("W1", "b1", "W2", "b2", "W3", "b3", "W_root", "b")


@pytest.fixture(scope="module")
def L():
    from paper_2402_15106_b200 import build
    build.build()
    from paper_2402_15106_b200 import _lib
    return _lib


def _problem(n, dim, r, n_e, d_e_mode, d, k, seed, n_dst=None, isolated=0):
    """Oracle-built graph + inputs (nothing comes from the CUDA path)."""
    g = np.random.default_rng(seed)
    x = g.random((n, dim)).astype(np.float32)
    if isolated:
        x[-isolated:] += 50.0 + 10 * np.arange(isolated, dtype=np.float32)[:, None]
    a = g.normal(size=(n, 1)).astype(np.float32)
    gid = g.permutation(10 * n)[:n].astype(np.int64)
    n_dst = n if n_dst is None else n_dst
    rp, col = graph.radius_graph(x, gid, n_dst, r, n_e, seed)
    e = features.edge_features(d_e_mode, x, a, features.dst_of_edges(rp), col)
    d_e = e.shape[1]
    W = synth.weights(d_e, d, d, k, salt=seed)
    v = synth.node_features(n, d, salt=seed)
    G = synth.upstream_grad(n_dst, d, salt=seed)
    return dict(x=x, a=a, gid=gid, rp=rp, col=col, e=e, W=W, v=v, G=G, n_dst=n_dst, n=n, d_e=d_e, d=d, k=k)


def _to_dtype_inputs(p, dtype):
    """BF16 mode: the oracle receives the bf16-rounded v, e, W1, W2, W3, b3, W_root."""
    if dtype == 0:
        return p["v"], p["e"], p["W"]
    W = dict(p["W"])
    for n in ("W1", "W2", "W3", "b3", "W_root"):
        W[n] = synth.round_bf16(W[n])
    return synth.round_bf16(p["v"]), synth.round_bf16(p["e"]), W


def _run_gpu(L, p, dtype, root, act, ranges=None, want_bwd=True, G=None, want_de=True):
    d, k, d_e = p["d"], p["k"], p["d_e"]
    desc = L.make_desc(d_e, d, d, k, dtype, root, act)
    Wd = {n: T(p["W"][n]) for n in GNAMES}
    packed = torch.empty(L.packed_weights_size(desc), dtype=torch.uint8, device=cuda())
    L.pack_weights(desc, Wd, packed)
    n, n_dst = p["n"], p["n_dst"]
    E = len(p["col"])
    if dtype == 0:
        v = T(p["v"])
        e = T(p["e"]) if E else torch.zeros((1, d_e), device=cuda())
    else:
        v = T(p["v"]).to(torch.bfloat16)
        e16 = np.zeros((max(E, 1), 16), np.float32)
        e16[:E, :d_e] = p["e"]
        e = T(e16).to(torch.bfloat16)
    rp = T(p["rp"])
    col = T(p["col"]) if E else torch.zeros(1, dtype=torch.int32, device=cuda())
    out = torch.full((n_dst, d), float("nan"), device=cuda())
    ws = torch.empty(L.layer_workspace_size(desc, n_dst, E), dtype=torch.uint8, device=cuda())
    rph = torch.from_numpy(p["rp"])
    for (a, b) in (ranges or [(0, n_dst)]):
        L.layer_fwd(desc, Wd, packed, v, e, rp, col, n_dst, a, b, out, None, ws, row_ptr_host=rph)
    res = dict(out=N(out))
    if not want_bwd:
        return res
    perm = torch.empty(max(E, 1), dtype=torch.int32, device=cuda())
    cptr = torch.empty(n + 1, dtype=torch.int64, device=cuda())
    L.csc(col[:E], n, perm, cptr)
    gv = torch.zeros((n, d), device=cuda())
    ge = torch.zeros((max(E, 1), d_e), device=cuda())
    grads = {nm: torch.zeros_like(Wd[nm]) for nm in GNAMES}
    bws = torch.empty(L.layer_bwd_workspace_size(desc, n_dst, n, E), dtype=torch.uint8, device=cuda())
    Gt = T(p["G"] if G is None else G)
    L.layer_bwd(desc, Wd, packed, v, e, rp, col, perm, cptr, n_dst, n, 0, n_dst, Gt, gv, ge if want_de else None,
                grads, ws, bws, row_ptr_host=rph)
    torch.cuda.synchronize()
    res.update(dv=N(gv), de=N(ge)[:E] if want_de else None, grads={nm: N(t) for nm, t in grads.items()})
    return res


def _oracle(p, dtype, root, act, rows=None, G=None):
    v, e, W = _to_dtype_inputs(p, dtype)
    desc = LayerDesc(p["d_e"], p["d"], p["d"], p["k"], root, act, "bf16" if dtype == 1 else "none")
    out, _ = layer.layer_fwd(desc, W, v, e, p["rp"], p["col"], rows=rows)
    Gr = p["G"] if G is None else G
    if rows is not None:
        Gr = Gr[rows]
    dv, de, g = layer.layer_bwd(desc, W, v, e, p["rp"], p["col"], Gr, rows=rows)
    return dict(out=out, dv=dv, de=de, grads=g)


def _mask_kinks(p, dtype, root, act, rows=None):
    """BF16 mode: zero the upstream gradient where the oracle's pre-activation
    lies within 2% of its spread from the ReLU kink.  The ReLU decision there is
    a floating-point decision the two precisions may take differently; with G
    zero at those entries the decision has no influence on any gradient."""
    if dtype == 0 or act != 1:
        return
    v, e, W = _to_dtype_inputs(p, dtype)
    desc = LayerDesc(p["d_e"], p["d"], p["d"], p["k"], root, act, "bf16")
    r = np.arange(p["n_dst"]) if rows is None else rows
    _, pre = layer.layer_fwd(desc, W, v, e, p["rp"], p["col"], rows=r)
    G = p["G"].copy()
    sub = G[r]
    sub[np.abs(pre) < 2e-2 * pre.std()] = 0.0
    G[r] = sub
    p["G"] = G


COMBOS = [(2, 1), (1, 0), (0, 1), (0, 0)]  # (root, act): GNO form, paper form, ...


@pytest.mark.parametrize("root,act", COMBOS)
def test_fwd_bwd_f32_tiny(L, root, act):
    # BASELINE configs[0]-sized problem: 64 nodes, r = 0.25, width 16, k = 32
    p = _problem(64, 2, 0.25, 64, "diff", 16, 32, seed=11)
    got = _run_gpu(L, p, 0, root, act)
    ref = _oracle(p, 0, root, act)
    assert nerr(got["out"], ref["out"]) <= TOL[0]
    assert nerr(got["dv"], ref["dv"]) <= TOL[0]
    assert nerr(got["de"], ref["de"]) <= TOL[0]
    for nm in GNAMES:
        if root != 2 and nm == "W_root":
            continue
        assert nerr(got["grads"][nm], ref["grads"][nm]) <= TOL[0], nm


def test_f32_tiles_ragged_and_empty_rows(L):
    # several GEMM tiles with ragged tails, capped rows, isolated (deg 0) rows,
    # n_dst < n_loc (halo-like sources), odd widths
    p = _problem(700, 3, 0.18, 24, "concat", 24, 40, seed=12, n_dst=611, isolated=5)
    p["n_dst"] = 611
    got = _run_gpu(L, p, 0, 2, 1)
    ref = _oracle(p, 0, 2, 1)
    for key in ("out", "dv", "de"):
        assert nerr(got[key], ref[key]) <= TOL[0], key
    for nm in GNAMES:
        assert nerr(got["grads"][nm], ref["grads"][nm]) <= TOL[0], nm


def test_f32_row_ranges_equal_full(L):
    p = _problem(300, 2, 0.15, 32, "diff", 16, 32, seed=13)
    full = _run_gpu(L, p, 0, 2, 1, want_bwd=False)
    split = _run_gpu(L, p, 0, 2, 1, ranges=[(0, 97), (97, 98), (98, 300)], want_bwd=False)
    assert np.array_equal(full["out"], split["out"])


def test_f32_deterministic(L):
    p = _problem(400, 2, 0.12, 32, "diff", 16, 32, seed=14)
    a = _run_gpu(L, p, 0, 2, 1)
    b = _run_gpu(L, p, 0, 2, 1)
    assert np.array_equal(a["out"], b["out"]) and np.array_equal(a["dv"], b["dv"])
    for nm in GNAMES:
        assert np.array_equal(a["grads"][nm], b["grads"][nm])


def _darcy_full(L, dtype, n_rows, want_de=True):
    """configs[1] sizes (d = 64, k = 256, n_e = 64, 16,384 sampled nodes of the
    241^2 grid) on one 4,096-node-ish sub-domain-sized slice: the GPU runs every
    row; the oracle checks sampled rows and the masked-upstream backward."""
    cfg = synth.CONFIGS["darcy"]
    coords, attr = synth.points(cfg)
    ids = sample.sample(len(coords), cfg.s, synth.BASE_SEED + synth.SEED_SAMPLING)
    x, a = coords[ids], attr[ids]
    gid = ids.astype(np.int64)
    # sub-domain sized: destinations = 4096 nodes nearest the lower-left quadrant (all sources kept)
    n = len(x)
    n_dst = 4096
    order = np.lexsort((gid, np.maximum(x[:, 0], x[:, 1])))
    x, a, gid = x[order], a[order], gid[order]
    rows = hash_rows(n_dst, n_rows)
    seedc = synth.BASE_SEED + synth.SEED_CAPPING
    # oracle graph rows (sampled) and full graph for the GPU input: the full
    # CSR is assembled from oracle rows too, so no input comes from the CUDA path
    adj = graph.radius_graph_rows(x, gid, range(n_dst), cfg.r, cfg.n_e, seedc)
    rp = np.zeros(n_dst + 1, np.int64)
    rp[1:] = np.cumsum([len(r_) for r_ in adj])
    col = np.concatenate(adj).astype(np.int32)
    e = features.edge_features("diff", x, a, features.dst_of_edges(rp), col)
    d, k = cfg.d, cfg.k
    W = synth.weights(e.shape[1], d, d, k)
    v = synth.node_features(n, d)
    G = np.zeros((n_dst, d), np.float32)
    G[rows] = synth.upstream_grad(n_dst, d)[rows]
    p = dict(x=x, a=a, gid=gid, rp=rp, col=col, e=e, W=W, v=v, G=G, n_dst=n_dst, n=n, d_e=e.shape[1], d=d, k=k)
    _mask_kinks(p, dtype, 2, 1, rows=rows)
    got = _run_gpu(L, p, dtype, 2, 1, want_de=want_de)
    ref = _oracle(p, dtype, 2, 1, rows=rows)
    assert nerr(got["out"][rows], ref["out"]) <= TOL[dtype]
    assert nerr(got["dv"], ref["dv"]) <= TOL[dtype]
    if want_de:
        assert nerr(got["de"], ref["de"]) <= TOL[dtype]
    for nm in GNAMES:
        assert nerr(got["grads"][nm], ref["grads"][nm]) <= TOL[dtype], nm


def test_f32_darcy_full_size_sampled(L):
    _darcy_full(L, 0, 24)


@pytest.mark.parametrize("d,dim,mode,root,act", [(64, 2, "diff", 2, 1), (32, 3, "concat", 2, 1),
                                                  (64, 2, "diff", 1, 0), (32, 2, "diff", 0, 1)])
def test_fwd_bf16(L, d, dim, mode, root, act):
    # tiles with several rows each, rows straddling tiles (deg 24..40 -> 32..48 slots), isolated rows,
    # n_dst < n_loc; compared with the fp64 oracle on bf16-rounded inputs
    p = _problem(900, dim, 0.09 if dim == 2 else 0.2, 40, mode, d, 256, seed=21 + d, n_dst=850, isolated=3)
    got = _run_gpu(L, p, 1, root, act, want_bwd=False)
    v, e, W = _to_dtype_inputs(p, 1)
    desc = LayerDesc(p["d_e"], d, d, 256, root, act, "bf16")
    ref, _ = layer.layer_fwd(desc, W, v, e, p["rp"], p["col"])
    assert np.isfinite(got["out"]).all()
    assert nerr(got["out"], ref) <= TOL[1]


@pytest.mark.parametrize("d,dim,mode,root,act", [(64, 2, "diff", 2, 1), (32, 3, "concat", 2, 1),
                                                  (64, 2, "diff", 1, 0), (32, 2, "diff", 0, 1)])
def test_fwd_bwd_bf16(L, d, dim, mode, root, act):
    p = _problem(700, dim, 0.1 if dim == 2 else 0.2, 40, mode, d, 256, seed=31 + d, n_dst=650, isolated=3)
    _mask_kinks(p, 1, root, act)
    got = _run_gpu(L, p, 1, root, act)
    ref = _oracle(p, 1, root, act)
    assert nerr(got["out"], ref["out"]) <= TOL[1]
    assert nerr(got["dv"], ref["dv"]) <= TOL[1]
    assert nerr(got["de"], ref["de"]) <= TOL[1]
    for nm in GNAMES:
        if root != 2 and nm == "W_root":
            continue
        assert nerr(got["grads"][nm], ref["grads"][nm]) <= TOL[1], nm


@pytest.mark.parametrize("d,dim,mode,root,act,n", [(64, 2, "diff", 2, 1, 700), (32, 3, "concat", 2, 1, 700),
                                                    (64, 2, "diff", 2, 1, 37)])
def test_fwd_bwd_bf16_no_de(L, d, dim, mode, root, act, n):
    """Without the edge-attribute gradient the library runs the fused edge
    backward (edge_bwd3.cuh: a1 / h in TMEM, kappa bias through the MMA),
    recomputes a1 from e (B4 in dw2.cuh) and fuses B5 and B6 (dz1 stays on
    chip, dW1 accumulated in TMEM); with it, edge_bwd2 writes A1 and GEMMs
    follow.  Both paths meet the oracle bar; the kappa_phi recomputes differ
    (bias through the MMA vs an fp32 add), so a few ReLU decisions at the
    kink may differ between them and only the dense-layer gradients agree to
    fp32 summation order."""
    p = _problem(n, dim, 0.1 if dim == 2 else 0.2, 40, mode, d, 256, seed=41 + d + n, n_dst=n - 50 if n > 100 else n,
                 isolated=3 if n > 100 else 0)
    _mask_kinks(p, 1, root, act)
    got = _run_gpu(L, p, 1, root, act, want_de=False)
    ref = _oracle(p, 1, root, act)
    assert nerr(got["dv"], ref["dv"]) <= TOL[1]
    for nm in GNAMES:
        assert nerr(got["grads"][nm], ref["grads"][nm]) <= TOL[1], nm
    unf = _run_gpu(L, p, 1, root, act, want_de=True)
    # the unfused path (edge_bwd2 + GEMMs, A1 in HBM) against the same oracle
    assert nerr(unf["dv"], ref["dv"]) <= TOL[1]
    for nm in GNAMES:
        assert nerr(unf["grads"][nm], ref["grads"][nm]) <= TOL[1], nm
    # the dense-layer gradients do not depend on kappa_phi's recompute: the
    # two paths give the same values up to fp32 summation order
    for nm in ("W3", "b3", "W_root", "b"):
        assert nerr(got["grads"][nm], unf["grads"][nm]) <= 1e-5, nm


def test_bf16_darcy_full_size_sampled_bwd(L):
    _darcy_full(L, 1, 16)


def test_bf16_darcy_full_size_sampled_bwd_fused_dz1(L):
    # the bench's launch configuration: no edge-attribute gradient -> fused B5 + B6
    _darcy_full(L, 1, 16, want_de=False)


def test_fwd_bf16_darcy_full_size_sampled(L):
    cfg = synth.CONFIGS["darcy"]
    coords, attr = synth.points(cfg)
    ids = sample.sample(len(coords), cfg.s, synth.BASE_SEED + synth.SEED_SAMPLING)
    x, a = coords[ids], attr[ids]
    gid = ids.astype(np.int64)
    n, n_dst = len(x), 4096
    order = np.lexsort((gid, np.maximum(x[:, 0], x[:, 1])))
    x, a, gid = x[order], a[order], gid[order]
    adj = graph.radius_graph_rows(x, gid, range(n_dst), cfg.r, cfg.n_e, synth.BASE_SEED + synth.SEED_CAPPING)
    rp = np.zeros(n_dst + 1, np.int64)
    rp[1:] = np.cumsum([len(r_) for r_ in adj])
    col = np.concatenate(adj).astype(np.int32)
    e = features.edge_features("diff", x, a, features.dst_of_edges(rp), col)
    W = synth.weights(e.shape[1], cfg.d, cfg.d, cfg.k)
    p = dict(x=x, a=a, gid=gid, rp=rp, col=col, e=e, W=W, v=synth.node_features(n, cfg.d), G=None, n_dst=n_dst,
             n=n, d_e=e.shape[1], d=cfg.d, k=cfg.k)
    got = _run_gpu(L, p, 1, 2, 1, want_bwd=False)
    rows = hash_rows(n_dst, 64)
    v, e16, W16 = _to_dtype_inputs(p, 1)
    ref, _ = layer.layer_fwd(LayerDesc(3, cfg.d, cfg.d, cfg.k, 2, 1, "bf16"), W16, v, e16, rp, col, rows=rows)
    assert nerr(got["out"][rows], ref) <= TOL[1]
    # and against the plain fp64 definition (no operand or activation rounding):
    # the BF16 mode's whole rounding budget is inside the same 2e-2 bar
    plain, _ = layer.layer_fwd(LayerDesc(3, cfg.d, cfg.d, cfg.k, 2, 1, "none"), W, p["v"], e, rp, col, rows=rows)
    assert nerr(got["out"][rows], plain) <= TOL[1]


def test_bf16_rows_longer_than_128_edges_are_unsupported(L):
    """The fused BF16 edge kernels tile whole rows of at most 128 edges; a
    longer row is rejected with UNSUPPORTED before any launch (with and
    without the host copy of row_ptr), and the context stays usable."""
    n, d, k = 300, 64, 256
    rp = np.array([0, 129, 131], np.int64)
    col = np.arange(131, dtype=np.int32) % n
    W = synth.weights(3, d, d, k, salt=5)
    desc = L.make_desc(3, d, d, k, L.BF16, L.ROOT_DENSE, L.ACT_RELU)
    Wd = {nm: T(W[nm]) for nm in GNAMES}
    packed = torch.empty(L.packed_weights_size(desc), dtype=torch.uint8, device=cuda())
    L.pack_weights(desc, Wd, packed)
    v = T(synth.node_features(n, d)).to(torch.bfloat16)
    e = torch.zeros((131, 16), dtype=torch.bfloat16, device=cuda())
    out = torch.empty((2, d), device=cuda())
    ws = torch.empty(L.layer_workspace_size(desc, 2, 131), dtype=torch.uint8, device=cuda())
    for host in (torch.from_numpy(rp), None):
        with pytest.raises(L.DsmpnnError) as ei:
            L.layer_fwd(desc, Wd, packed, v, e, T(rp), T(col), 2, 0, 2, out, None, ws, row_ptr_host=host)
        assert ei.value.status == -8
    # row 1 alone (2 edges) is fine
    L.layer_fwd(desc, Wd, packed, v, e, T(rp), T(col), 2, 1, 2, out, None, ws, row_ptr_host=torch.from_numpy(rp))
    torch.cuda.synchronize()
    assert torch.isfinite(out[1]).all()


def test_debug_index_validation_returns_index_error():
    """With DSMPNN_DEBUG set, a CSR with a column index out of range gives
    ERR_INDEX instead of an out-of-bounds read (child process: the switch is
    read once per process)."""
    import os
    import subprocess
    import sys
    code = r'''
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_2402_15106_b200 import _lib as L, synth
n, d, k = 50, 16, 32
W = synth.weights(3, d, d, k, salt=1)
desc = L.make_desc(3, d, d, k, L.F32, L.ROOT_DENSE, L.ACT_RELU)
Wd = {nm: torch.from_numpy(np.ascontiguousarray(W[nm])).cuda() for nm in W}
packed = torch.empty(L.packed_weights_size(desc), dtype=torch.uint8, device="cuda")
L.pack_weights(desc, Wd, packed)
rp = torch.tensor([0, 2, 3], dtype=torch.int64, device="cuda")
col = torch.tensor([1, 7, 10**6], dtype=torch.int32, device="cuda")
v = torch.randn(n, d, device="cuda"); e = torch.zeros(3, 3, device="cuda")
out = torch.empty(2, d, device="cuda")
ws = torch.empty(L.layer_workspace_size(desc, 2, 3), dtype=torch.uint8, device="cuda")
G = torch.randn(2, d, device="cuda"); gv = torch.zeros(n, d, device="cuda")
perm = torch.empty(3, dtype=torch.int32, device="cuda"); cptr = torch.empty(n + 1, dtype=torch.int64, device="cuda")
grads = {nm: torch.zeros_like(t) for nm, t in Wd.items()}
bws = torch.empty(L.layer_bwd_workspace_size(desc, 2, n, 3), dtype=torch.uint8, device="cuda")
try:
    L.layer_bwd(desc, Wd, packed, v, e, rp, col, perm, cptr, 2, n, 0, 2, G, gv, None, grads, ws, bws)
    print("NO_ERROR")
except L.DsmpnnError as ex:
    print("STATUS", ex.status)
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    p = subprocess.run([sys.executable, "-c", code, root], env=dict(os.environ, DSMPNN_DEBUG="1"),
                       capture_output=True, text=True, timeout=300)
    assert "STATUS -3" in p.stdout, p.stdout + p.stderr


@pytest.mark.parametrize("k,d,want_de", [(128, 64, False), (64, 32, False), (100, 64, True)])
def test_fwd_bwd_bf16_kappa_width_below_256(L, k, d, want_de):
    """kappa width k < 256 in BF16 mode: the
    weights are zero-padded to 256 units (dsmpnn_pack_weights), the padded
    units stay exact zeros, and the output and every gradient of width k
    match the fp64 oracle of width k at the north_star's 2e-2 -- on the fused
    backward (no edge-attribute gradient) and on the unfused one."""
    p = _problem(700, 2, 0.1, 40, "diff", d, k, seed=51 + k, n_dst=650, isolated=3)
    _mask_kinks(p, 1, 2, 1)
    got = _run_gpu(L, p, 1, 2, 1, want_de=want_de)
    ref = _oracle(p, 1, 2, 1)
    assert nerr(got["out"], ref["out"]) <= TOL[1]
    assert nerr(got["dv"], ref["dv"]) <= TOL[1]
    if want_de:
        assert nerr(got["de"], ref["de"]) <= TOL[1]
    for nm in GNAMES:
        assert got["grads"][nm].shape == p["W"][nm].shape, nm
        assert nerr(got["grads"][nm], ref["grads"][nm]) <= TOL[1], nm


def test_bf16_kappa_width_above_256_is_unsupported(L):
    desc = L.make_desc(3, 64, 64, 512, L.BF16, L.ROOT_DENSE, L.ACT_RELU)
    with pytest.raises(L.DsmpnnError) as ei:
        L.packed_weights_size(desc)
    assert ei.value.status == -8  # UNSUPPORTED


def test_bf16_bwd_row_ranges_sum_to_full(L):
    """layer_bwd over rows [0, a) plus [a, n_dst) (edges [eb, ee) of each
    range; the B7 scatter then skips the other range's edges) accumulates the
    full-range dv and weight gradients (fused backward, U rows in CSC order)."""
    p = _problem(700, 2, 0.1, 40, "diff", 64, 256, seed=61, n_dst=650, isolated=3)
    d, k, d_e = p["d"], p["k"], p["d_e"]
    desc = L.make_desc(d_e, d, d, k, L.BF16, 2, 1)
    Wd = {n: T(p["W"][n]) for n in GNAMES}
    packed = torch.empty(L.packed_weights_size(desc), dtype=torch.uint8, device=cuda())
    L.pack_weights(desc, Wd, packed)
    n, n_dst, E = p["n"], p["n_dst"], len(p["col"])
    v = T(p["v"]).to(torch.bfloat16)
    e16 = np.zeros((E, 16), np.float32)
    e16[:, :d_e] = p["e"]
    e = T(e16).to(torch.bfloat16)
    rp, col, rph = T(p["rp"]), T(p["col"]), torch.from_numpy(p["rp"])
    out = torch.empty((n_dst, d), device=cuda())
    ws = torch.empty(L.layer_workspace_size(desc, n_dst, E), dtype=torch.uint8, device=cuda())
    L.layer_fwd(desc, Wd, packed, v, e, rp, col, n_dst, 0, n_dst, out, None, ws, row_ptr_host=rph)
    perm = torch.empty(E, dtype=torch.int32, device=cuda())
    cptr = torch.empty(n + 1, dtype=torch.int64, device=cuda())
    L.csc(col, n, perm, cptr)
    bws = torch.empty(L.layer_bwd_workspace_size(desc, n_dst, n, E), dtype=torch.uint8, device=cuda())
    Gt = T(p["G"])
    res = []
    for ranges in ([(0, n_dst)], [(0, 311), (311, n_dst)]):
        gv = torch.zeros((n, d), device=cuda())
        grads = {nm: torch.zeros_like(Wd[nm]) for nm in GNAMES}
        for a, b in ranges:
            L.layer_bwd(desc, Wd, packed, v, e, rp, col, perm, cptr, n_dst, n, a, b, Gt, gv, None, grads, ws, bws,
                        row_ptr_host=rph)
        torch.cuda.synchronize()
        res.append((N(gv), {nm: N(t) for nm, t in grads.items()}))
    assert nerr(res[1][0], res[0][0]) <= 1e-5
    for nm in GNAMES:
        assert nerr(res[1][1][nm], res[0][1][nm]) <= 1e-5, nm

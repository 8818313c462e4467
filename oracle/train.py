"""O9 - the full DS-MPNN hop loop and training step.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md eqs. (i)-(iv) (:39-42) and Alg. 1 (:385-422), per sub-domain:
  k = 1:     v_L = N_e(v^0)                       (i), on every local row
  each hop:  v_res = v_L;  v_L = K_phi(v_L, e) + v_res   (ii) + residual, owned rows
             Comm(v_L)                             (:411, halo rows refreshed)
             v = N_d(v_L)                          (iii), every local row (R26)
             e_ij = v_i - v_j                      (iv), attribute part of e (R25)
  loss:      MSE of v on interior (owned) rows against Y, summed over ranks
  update:    SGD w <- w - eta grad (Alg. 1 :419) or Adam
Readings: R25 the refreshed edge attribute keeps the coordinate part
(x_i - x_j) and replaces the node-attribute part by the decoded difference
(so d_e is unchanged, "R^3" for Darcy); the decoder outputs
n_attr channels.  R26 decoding every local row after the latent refresh
equals decoding then communicating the decoded values (same arithmetic on
the same inputs); received values are detached (R16 DETACH): gradients
reaching halo rows' latent or decoded values are dropped, except at hop 1,
where halo rows' latent values are the local encoder's own outputs.
The conv layer is the "paper form" of R1: identity sigma, identity root
(which is the residual), bias b.  N_e / N_d: 3 Linear layers, ReLU between.
fp64 throughout.
"""
import numpy as np

from . import features, halo, layer
from .layer import LayerDesc, ROOT_IDENTITY, ACT_IDENTITY
from .precision import round_bf16


def mlp_fwd(P, x):
    """3-layer MLP, ReLU after layers 1 and 2.  P = [(W, b)] * 3, W [out, in].
    Returns (y, cache)."""
    h0 = np.asarray(x, np.float64)
    z1 = h0 @ P[0][0].T + P[0][1]
    h1 = np.maximum(z1, 0.0)
    z2 = h1 @ P[1][0].T + P[1][1]
    h2 = np.maximum(z2, 0.0)
    y = h2 @ P[2][0].T + P[2][1]
    return y, (h0, h1, h2)


def mlp_bwd(P, cache, dy):
    """Backward of mlp_fwd: (dx, [(dW, db)] * 3).  ReLU'(0) = 0."""
    h0, h1, h2 = cache
    dy = np.asarray(dy, np.float64)
    g = [None] * 3
    g[2] = (dy.T @ h2, dy.sum(axis=0))
    d2 = (dy @ P[2][0]) * (h2 > 0)
    g[1] = (d2.T @ h1, d2.sum(axis=0))
    d1 = (d2 @ P[1][0]) * (h1 > 0)
    g[0] = (d1.T @ h0, d1.sum(axis=0))
    return d1 @ P[0][0], g


def _refresh(x, u, row_ptr, col_idx):
    """(iv) with R25: e_ij = (x_i - x_j, u_i - u_j) in fp64 (coordinates as given)."""
    dst = features.dst_of_edges(row_ptr)
    ci = np.asarray(col_idx, np.int64)
    x = np.asarray(x, np.float64)
    u = np.asarray(u, np.float64)
    return np.concatenate([x[dst] - x[ci], u[dst] - u[ci]], axis=1)


def conv_desc(d_e, d, k, act_round="none"):
    return LayerDesc(d_e, d, d, k, ROOT_IDENTITY, ACT_IDENTITY, act_round)


def ds_train_grads(params, ranks, v0_rows, Y_rows, hops, dim, n_attr, x_rows, bf16=False):
    """Loss and weight gradients of one DS-MPNN step on the decomposed ranks.

    params: dict enc=[(W,b)]*3, dec=[(W,b)]*3, conv=layer weight dict.
    v0_rows(rows) -> initial node values [x, a] of sampled rows; Y_rows(rows)
    -> targets [n_attr]; x_rows(rows) -> coordinates.  Returns (loss, grads)
    with grads in the same structure (summed over ranks, Alg. 1 :418).
    bf16=True: the BF16 mode's rounding points of the convolution (R18, R27):
    its weights W1, W2, W3, b3, every hop's input v_L and edge attributes e
    are bf16 operands and a1, h are rounded (act_round); the encoder, the
    decoder, the latent values and all arithmetic stay fp64."""
    enc, dec = params["enc"], params["dec"]
    d = enc[2][0].shape[0]
    W = dict(params["conv"])
    W.setdefault("W_root", np.zeros((d, d)))  # identity root: unused
    k = W["W1"].shape[0]
    d_e = dim + n_attr
    desc = conv_desc(d_e, d, k, "bf16" if bf16 else "none")
    rnd = round_bf16 if bf16 else (lambda a: a)
    if bf16:
        for nm in ("W1", "W2", "W3", "b3"):
            W[nm] = round_bf16(W[nm])
    R = len(ranks)
    n_own = [len(q["row_ptr"]) - 1 for q in ranks]
    xs = [np.asarray(x_rows(q["local_rows"]), np.float32) for q in ranks]
    v0 = [np.asarray(v0_rows(q["local_rows"]), np.float64) for q in ranks]
    Y = [np.asarray(Y_rows(q["local_rows"][:n]), np.float64) for q, n in zip(ranks, n_own)]
    # forward, keeping every hop's inputs
    enc_cache, vL, e = [], [], []
    for q in range(R):
        y, cache = mlp_fwd(enc, v0[q])
        enc_cache.append(cache)
        vL.append(y)
        e.append(rnd(ranks[q]["e"]))  # e^0 from the initial values (R21 diff)
    hist = []
    for hop in range(hops):
        vin = [rnd(v) for v in vL]  # the convolution's operand
        outs = [layer.layer_fwd(desc, W, vin[q], e[q], ranks[q]["row_ptr"], ranks[q]["col_idx"])[0]
                for q in range(R)]
        new = []
        for q in range(R):
            nv = vL[q].copy()
            nv[: n_own[q]] = outs[q]
            new.append(nv)
        new = halo.halo_forward(ranks, new)
        dec_out = [mlp_fwd(dec, new[q]) for q in range(R)]
        u = [o[0] for o in dec_out]
        e_next = [rnd(_refresh(xs[q], u[q], ranks[q]["row_ptr"], ranks[q]["col_idx"])) for q in range(R)]
        hist.append(dict(vin=vin, e=e, vout=new, dec_cache=[o[1] for o in dec_out], u=u))
        vL, e = new, e_next
    count = sum(n_own) * n_attr
    u_last = hist[-1]["u"]
    loss = sum(float(((u_last[q][: n_own[q]] - Y[q]) ** 2).sum()) for q in range(R)) / count
    # backward
    gz = lambda P: [(np.zeros_like(Wl), np.zeros_like(bl)) for Wl, bl in P]
    g_enc, g_dec = gz(enc), gz(dec)
    g_conv = {nm: np.zeros_like(np.asarray(W[nm], np.float64)) for nm in ("W1", "b1", "W2", "b2", "W3", "b3", "b")}
    du = [np.zeros_like(u_last[q]) for q in range(R)]
    for q in range(R):
        du[q][: n_own[q]] = 2.0 * (u_last[q][: n_own[q]] - Y[q]) / count
    dvL_in = None
    for hop in reversed(range(hops)):
        H = hist[hop]
        dvout = []
        for q in range(R):
            dd = du[q].copy()
            dd[n_own[q]:] = 0.0  # decoded halo values are received (detached)
            dx, g = mlp_bwd(dec, H["dec_cache"][q], dd)
            for l_ in range(3):
                g_dec[l_] = (g_dec[l_][0] + g[l_][0], g_dec[l_][1] + g[l_][1])
            dvo = dx
            if dvL_in is not None:
                dvo = dvo + dvL_in[q]
            dvout.append(dvo)
        dvL_in, du_prev = [], []
        for q in range(R):
            G = dvout[q][: n_own[q]]
            dv, de, g = layer.layer_bwd(desc, W, H["vin"][q], H["e"][q], ranks[q]["row_ptr"], ranks[q]["col_idx"], G)
            for nm in g_conv:
                g_conv[nm] += g[nm]
            if hop > 0:
                dv[n_own[q]:] = 0.0  # halo latent values of hops > 1 are received (detached)
            dvL_in.append(dv)
            # (iv) e_ij = u_i - u_j on the attribute part: de -> du of the previous hop
            dprev = np.zeros((len(H["vin"][q]), n_attr))
            if hop > 0:
                rp, ci = ranks[q]["row_ptr"], ranks[q]["col_idx"]
                dst = features.dst_of_edges(rp)
                da = de[:, dim:dim + n_attr]
                np.add.at(dprev, dst, da)
                np.add.at(dprev, ci, -da)
            du_prev.append(dprev)
        du = du_prev
    # encoder: every local row (hop-1 halo latent values are local encoder outputs)
    for q in range(R):
        _, g = mlp_bwd(enc, enc_cache[q], dvL_in[q])
        for l_ in range(3):
            g_enc[l_] = (g_enc[l_][0] + g[l_][0], g_enc[l_][1] + g[l_][1])
    return loss, dict(enc=g_enc, dec=g_dec, conv=g_conv)


def sgd(w, g, lr):
    """Alg. 1 :419: w <- w - eta grad."""
    return w - lr * g


def adam(w, g, m, v, step, lr, b1=0.9, b2=0.999, eps=1e-8):
    """Adam, step >= 1: returns (w, m, v)."""
    m = b1 * m + (1 - b1) * g
    v = b2 * v + (1 - b2) * g * g
    mh = m / (1 - b1 ** step)
    vh = v / (1 - b2 ** step)
    return w - lr * mh / (np.sqrt(vh) + eps), m, v

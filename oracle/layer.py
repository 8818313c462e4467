"""O5/O6 - edge-conditioned convolution (Eq. 1) forward and backward, fp64.

PAPER.md:29-32 (§2.1, Eq. 1):
    v_i^l = 1/|E_i| * sum_{j <= n_e} K_phi(e_ij^{l-1}; theta) v_j^{l-1} + b
PAPER.md:40 eq. (ii) (the same on the latent v_L); Alg. 1
(v_res saved before the convolution and added after it); north_star form
sigma(W v_i + mean_j kappa_phi(e_ij) v_j).

Readings:
  R1  sigma in {identity, relu} applied after the sum;
  R2  root term in {none, identity (Alg. 1 residual), dense W v_i};
  R3  |E_i| = post-cap degree of row i; a row with no edges gets a zero message;
  R4  NNConv orientation: K[c][o] = kappa_out[c*d_out + o], m = K^T v_j;
  R5  kappa_phi = Linear(d_e,k) -> ReLU -> Linear(k,k) -> ReLU -> Linear(k, d_in*d_out)
      (PyTorch Linear layout [out, in]);  parity of this architecture with
      the paper is UNPINNED (the paper does not state it), the algebra is pinned;
  R18 ReLU'(0) = 0.

This is the plain definition: the per-edge matrix K_p is materialised and the
messages are summed in CSR (gid-ascending) order.  Work is batched over edges
only to keep numpy fast; nothing is reordered within a row's sum.
"""
from dataclasses import dataclass

import numpy as np

from .precision import round_bf16

ROOT_NONE, ROOT_IDENTITY, ROOT_DENSE = 0, 1, 2
ACT_IDENTITY, ACT_RELU = 0, 1


@dataclass
class LayerDesc:
    d_e: int
    d_in: int
    d_out: int
    k: int
    root: int = ROOT_DENSE
    act: int = ACT_RELU
    act_round: str = "none"   # "bf16": BF16-mode operand rounding of a1, h (oracle/precision.py)


def _w(W, name):
    return np.asarray(W[name], dtype=np.float64)


def kappa(W, e, act_round="none"):
    """kappa_phi on a batch of edge attributes (R5).  Returns (a1, h, Kflat).
    act_round="bf16" rounds the activations a1, h to bf16 (BF16-mode operand
    precision, reading R18)."""
    rnd = round_bf16 if act_round == "bf16" else (lambda x: x)
    e = np.asarray(e, dtype=np.float64)
    z1 = e @ _w(W, "W1").T + _w(W, "b1")
    a1 = rnd(np.maximum(z1, 0.0))
    z2 = a1 @ _w(W, "W2").T + _w(W, "b2")
    h = rnd(np.maximum(z2, 0.0))
    Kflat = h @ _w(W, "W3").T + _w(W, "b3")
    return a1, h, Kflat


def _edge_chunks(p0, p1, chunk):
    a = p0
    while a < p1:
        b = min(p1, a + chunk)
        yield a, b
        a = b


def messages(desc, W, v, e, col_idx, p0, p1):
    """m_p = K_p^T v_j for edges p in [p0, p1), K_p materialised (R4)."""
    _, _, Kflat = kappa(W, e[p0:p1], desc.act_round)
    K = Kflat.reshape(p1 - p0, desc.d_in, desc.d_out)          # K[p, c, o]
    vj = np.asarray(v, dtype=np.float64)[col_idx[p0:p1]]
    return np.einsum("pc,pco->po", vj, K)


def root_term(desc, W, v_i):
    v_i = np.asarray(v_i, dtype=np.float64)
    if desc.root == ROOT_NONE:
        return np.zeros((v_i.shape[0], desc.d_out))
    if desc.root == ROOT_IDENTITY:
        if desc.d_in != desc.d_out:
            raise ValueError("ROOT_IDENTITY needs d_in == d_out")
        return v_i.copy()
    return v_i @ _w(W, "W_root").T


def layer_fwd(desc, W, v, e, row_ptr, col_idx, rows=None, chunk=2048):
    """Return (out, pre) for the requested destination rows (default: all).

    For each row i: agg = (sum_p m_p) / deg_i (0 if deg_i = 0);
    pre = agg + root(v_i) + b;  out = sigma(pre).
    """
    row_ptr = np.asarray(row_ptr, dtype=np.int64)
    col_idx = np.asarray(col_idx, dtype=np.int64)
    n_dst = len(row_ptr) - 1
    rows = np.arange(n_dst) if rows is None else np.asarray(rows, dtype=np.int64)
    agg = np.zeros((len(rows), desc.d_out))
    # group consecutive rows into edge chunks to batch kappa evaluation
    for r0 in range(0, len(rows), 64):
        rr = rows[r0:r0 + 64]
        for t, i in enumerate(rr):
            p0, p1 = int(row_ptr[i]), int(row_ptr[i + 1])
            deg = p1 - p0
            if deg == 0:
                continue
            acc = np.zeros(desc.d_out)
            for a, b in _edge_chunks(p0, p1, chunk):
                m = messages(desc, W, v, e, col_idx, a, b)
                for q in range(b - a):                         # CSR order
                    acc = acc + m[q]
            agg[r0 + t] = acc / deg
    pre = agg + root_term(desc, W, np.asarray(v)[rows]) + _w(W, "b")
    out = np.maximum(pre, 0.0) if desc.act == ACT_RELU else pre
    return out, pre


def layer_bwd(desc, W, v, e, row_ptr, col_idx, G, rows=None, want_de=True):
    """Backward of layer_fwd (the transposes of O5).

    G holds dL/dout for ``rows`` (default all destination rows).  Rows not
    listed contribute nothing (masked upstream gradient).  Returns
    (dv [n_loc x d_in], de [E x d_e] or None, grads dict) where grads hold
    dW1, db1, dW2, db2, dW3, db3, dW_root, db.  Iterates destinations in the
    given order and edges in CSR order.
    """
    row_ptr = np.asarray(row_ptr, dtype=np.int64)
    col_idx = np.asarray(col_idx, dtype=np.int64)
    v = np.asarray(v, dtype=np.float64)
    e64 = np.asarray(e, dtype=np.float64)
    n_dst = len(row_ptr) - 1
    rows = np.arange(n_dst) if rows is None else np.asarray(rows, dtype=np.int64)
    G = np.asarray(G, dtype=np.float64)
    _, pre = layer_fwd(desc, W, v, e, row_ptr, col_idx, rows)
    ghat = G * (pre > 0.0) if desc.act == ACT_RELU else G.copy()

    W1, W2, W3 = _w(W, "W1"), _w(W, "W2"), _w(W, "W3")
    g = {n: np.zeros_like(_w(W, n)) for n in ("W1", "b1", "W2", "b2", "W3", "b3", "W_root", "b")}
    dv = np.zeros_like(v)
    de = np.zeros_like(e64) if want_de else None

    g["b"] += ghat.sum(axis=0)
    vi = v[rows]
    if desc.root == ROOT_DENSE:
        g["W_root"] += ghat.T @ vi
        dv[rows] += ghat @ _w(W, "W_root")
    elif desc.root == ROOT_IDENTITY:
        dv[rows] += ghat

    for t, i in enumerate(rows):
        p0, p1 = int(row_ptr[i]), int(row_ptr[i + 1])
        deg = p1 - p0
        if deg == 0:
            continue
        dm = ghat[t] / deg                                   # d loss / d m_p
        a1, h, Kflat = kappa(W, e64[p0:p1], desc.act_round)
        K = Kflat.reshape(deg, desc.d_in, desc.d_out)
        for q in range(deg):
            p = p0 + q
            j = col_idx[p]
            dv[j] += K[q] @ dm                               # m = K^T v_j
            dK = np.outer(v[j], dm).reshape(-1)              # index c*d_out + o
            g["W3"] += np.outer(dK, h[q])
            g["b3"] += dK
            dh = W3.T @ dK
            dz2 = dh * (h[q] > 0.0)
            g["W2"] += np.outer(dz2, a1[q])
            g["b2"] += dz2
            da1 = W2.T @ dz2
            dz1 = da1 * (a1[q] > 0.0)
            g["W1"] += np.outer(dz1, e64[p])
            g["b1"] += dz1
            if want_de:
                de[p] = W1.T @ dz1
    return dv, de, g


# ---- second formulation, used only by tests to pin the index algebra ---------

def pack_theta(desc, W):
    """Theta~[(k+1)*d_in, d_out]: Theta~[kap*d_in + c, o] = W3[c*d_out + o, kap],
    Theta~[k*d_in + c, o] = b3[c*d_out + o]."""
    k, di, do = desc.k, desc.d_in, desc.d_out
    W3 = _w(W, "W3").reshape(di, do, k)          # [c, o, kap]
    b3 = _w(W, "b3").reshape(di, do)
    T = np.zeros(((k + 1) * di, do))
    T[: k * di] = W3.transpose(2, 0, 1).reshape(k * di, do)
    T[k * di:] = b3
    return T


def messages_contraction(desc, W, v, e, col_idx, p0, p1):
    """m_p = vec(h~_p (x) v_j) . Theta~  (K_p never formed)."""
    _, h, _ = kappa(W, e[p0:p1], desc.act_round)
    ht = np.concatenate([h, np.ones((p1 - p0, 1))], axis=1)
    vj = np.asarray(v, dtype=np.float64)[np.asarray(col_idx)[p0:p1]]
    Z = np.einsum("pk,pc->pkc", ht, vj).reshape(p1 - p0, -1)
    return Z @ pack_theta(desc, W)

"""O8 - GCN layer, the paper's node-based comparison model.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md:70 (§3): "GCN here uses 6 hidden layers with a size of 378";
SPEC.md:249-257: per layer v_i <- act(W . mean_{j in N(i) u {i}} v_j + c), no
edge features, self-inclusion (reading R24 in DESIGN.md: the graph is the
radius graph built as for the MPNN; the mean runs over the row's capped
neighbours plus the node itself).  fp64, written from that definition.
"""
import numpy as np

ACT_IDENTITY, ACT_RELU = 0, 1


def gcn_fwd(W, c, act, v, row_ptr, col_idx):
    """Returns (out [n_dst x d_out], agg [n_dst x d_in]).
    agg_i = (v_i + sum_{p in row i} v_{col p}) / (deg_i + 1);
    out_i = act(W agg_i + c), W in PyTorch [d_out, d_in] layout."""
    v = np.asarray(v, np.float64)
    rp = np.asarray(row_ptr, np.int64)
    ci = np.asarray(col_idx, np.int64)
    n_dst = len(rp) - 1
    agg = np.zeros((n_dst, v.shape[1]))
    for i in range(n_dst):
        nb = ci[rp[i]:rp[i + 1]]
        agg[i] = (v[i] + v[nb].sum(axis=0)) / (len(nb) + 1)
    pre = agg @ np.asarray(W, np.float64).T + np.asarray(c, np.float64)
    out = np.maximum(pre, 0.0) if act == ACT_RELU else pre
    return out, agg


def gcn_bwd(W, c, act, v, row_ptr, col_idx, G):
    """Backward of gcn_fwd for upstream G [n_dst x d_out]: (dv [n_loc x d_in],
    dW, dc).  ReLU'(0) = 0."""
    out, agg = gcn_fwd(W, c, act, v, row_ptr, col_idx)
    W = np.asarray(W, np.float64)
    G = np.asarray(G, np.float64)
    ghat = G * (out > 0.0) if act == ACT_RELU else G
    dW = ghat.T @ agg
    dc = ghat.sum(axis=0)
    dagg = ghat @ W
    rp = np.asarray(row_ptr, np.int64)
    ci = np.asarray(col_idx, np.int64)
    dv = np.zeros(np.asarray(v).shape)
    for i in range(len(rp) - 1):
        nb = ci[rp[i]:rp[i + 1]]
        s = dagg[i] / (len(nb) + 1)
        dv[i] += s
        np.add.at(dv, nb, s)
    return dv, dW, dc

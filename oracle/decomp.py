"""Virtual-rank driver: the decomposed (DS) layer on P sub-domains in one process.

PAPER.md:58-60 (§3) and Alg. 1: decompose the sampled domain,
build each sub-domain's graph over owned centres with neighbours from
owned + overlap nodes, run the convolution per sub-domain and refresh the
overlap from the neighbours' interiors after every hop.  Used by tests to pin
"decomposed with full-width halo == undecomposed" (north_star).
"""
import numpy as np

from . import features, graph, halo, layer, partition, sample
from .precision import round_bf16


def _layer_input(desc, v):
    """The value a layer consumes: in the BF16 mode (act_round="bf16") every
    layer's input v is a bf16 operand (reading R18: the layer
    output is stored as the next layer's bf16 operand), else v itself."""
    return round_bf16(v) if desc.act_round == "bf16" else v


def build_local(coords, gid, attr, nparts, overlap_l, r, n_e, seed, edge_mode):
    """Per-rank local problem: plan + CSR over owned rows + edge features."""
    owner, boxes, internal, ranks = partition.plan(coords, gid, nparts, overlap_l, r)
    for q in ranks:
        rows = q["local_rows"]
        n_own = q["n_deep"] + q["n_near"]
        lc = np.asarray(coords, np.float32)[rows]
        rp, ci = graph.radius_graph(lc, q["local_gid"], n_own, r, n_e, seed)
        q["row_ptr"], q["col_idx"] = rp, ci
        q["e"] = features.edge_features(edge_mode, lc, np.asarray(attr, np.float32)[rows],
                                        features.dst_of_edges(rp), ci)
    return owner, boxes, internal, ranks


def ds_forward(desc, W, ranks, v_global_rows, n_layers):
    """Run n_layers of the layer on every rank with a halo refresh after each.

    v_global_rows: function(rows) -> input features for those sampled rows.
    Returns the per-rank owned outputs of the last layer."""
    vals = [np.asarray(v_global_rows(q["local_rows"]), dtype=np.float64) for q in ranks]
    outs = None
    for _ in range(n_layers):
        vals = [_layer_input(desc, v) for v in vals]
        outs = []
        for q, v in zip(ranks, vals):
            out, _ = layer.layer_fwd(desc, W, v, q["e"], q["row_ptr"], q["col_idx"])
            outs.append(out)
        new_vals = []
        for q, v, o in zip(ranks, vals, outs):
            nv = v.copy()
            nv[: len(o)] = o
            new_vals.append(nv)
        vals = halo.halo_forward(ranks, new_vals)
    return outs


DETACH, REVERSE_ADD = 0, 1


def ds_forward_backward(desc, W, ranks, v_global_rows, G_global_rows, n_layers, mode=DETACH):
    """Decomposed forward (as ds_forward) then backward over n_layers, with the
    halo gradient handled per reading R16 / SURVEY §8(f) f2:

      DETACH       received halo values are constants: the gradient reaching a
                   halo row is dropped (Alg. 1 :417 local backprop);
      REVERSE_ADD  after each layer's backward the halo rows' gradients are
                   added to their owners' rows (halo_reverse_add, q ascending),
                   the transpose of the forward halo copy, so the decomposed
                   gradient equals the undecomposed one.

    G_global_rows(rows) -> dL/dout of the last layer for those sampled rows
    (owned rows are used).  Returns the weight gradients summed over ranks
    (Alg. 1 :418)."""
    vals = [_layer_input(desc, np.asarray(v_global_rows(q["local_rows"]), dtype=np.float64)) for q in ranks]
    acts = [vals]
    for _ in range(n_layers):
        outs = [layer.layer_fwd(desc, W, v, q["e"], q["row_ptr"], q["col_idx"])[0] for q, v in zip(ranks, vals)]
        new_vals = []
        for v, o in zip(vals, outs):
            nv = v.copy()
            nv[: len(o)] = o
            new_vals.append(nv)
        vals = [_layer_input(desc, v) for v in halo.halo_forward(ranks, new_vals)]
        acts.append(vals)
    grads = None
    gouts = [np.asarray(G_global_rows(q["local_rows"][: len(q["row_ptr"]) - 1]), dtype=np.float64) for q in ranks]
    for layer_i in reversed(range(n_layers)):
        dvs = []
        for q, v, g_out in zip(ranks, acts[layer_i], gouts):
            dv, _, g = layer.layer_bwd(desc, W, v, q["e"], q["row_ptr"], q["col_idx"], g_out, want_de=False)
            dvs.append(dv)
            if grads is None:
                grads = {n: np.zeros_like(x) for n, x in g.items()}
            for n in grads:
                grads[n] += g[n]
        if mode == REVERSE_ADD:
            dvs = halo.halo_reverse_add(ranks, dvs)
        gouts = [dv[: len(q["row_ptr"]) - 1] for q, dv in zip(ranks, dvs)]
    return grads


def undecomposed_forward_backward(desc, W, coords, gid, attr, r, n_e, seed, edge_mode, v, G, n_layers):
    """The same L-layer chain on the whole sampled set as one domain (S-MPNN):
    summed weight gradients of sum_i G_i . out_i^(L)."""
    x = np.asarray(coords, np.float32)
    n = len(x)
    rp, ci = graph.radius_graph(x, np.asarray(gid, np.int64), n, r, n_e, seed)
    e = features.edge_features(edge_mode, x, np.asarray(attr, np.float32), features.dst_of_edges(rp), ci)
    acts = [np.asarray(v, np.float64)]
    for _ in range(n_layers):
        acts.append(layer.layer_fwd(desc, W, acts[-1], e, rp, ci)[0])
    g_out = np.asarray(G, np.float64)
    grads = None
    for layer_i in reversed(range(n_layers)):
        dv, _, g = layer.layer_bwd(desc, W, acts[layer_i], e, rp, ci, g_out, want_de=False)
        if grads is None:
            grads = {k: np.zeros_like(x_) for k, x_ in g.items()}
        for k in grads:
            grads[k] += g[k]
        g_out = dv
    return grads


def infer_reassemble(desc, W, coords, attr, nparts, overlap_l, r, n_e, seed_capping, s, seeds, v0_global,
                     n_layers, edge_mode):
    """Inference by sub-domain reassembly: for
    every sampling seed, sample s of the N points, decompose, run the L-layer
    forward with halo refresh (ds_forward) and add every rank's owned-row
    outputs to its global node; the field is the per-node average over the
    passes that visited it (0 where none did).  Returns (field [N x d], count)."""
    coords = np.asarray(coords, np.float32)
    N = len(coords)
    v0_global = np.asarray(v0_global, np.float64)
    acc = np.zeros((N, v0_global.shape[1]))
    cnt = np.zeros(N, np.int64)
    for seed in seeds:
        ids = sample.sample(N, s, seed).astype(np.int64)
        _, _, _, ranks = build_local(coords[ids], ids, np.asarray(attr, np.float32)[ids], nparts, overlap_l, r, n_e,
                                     seed_capping, edge_mode)
        outs = ds_forward(desc, W, ranks, lambda rows: v0_global[ids[rows]], n_layers)
        for q, o in zip(ranks, outs):
            g = q["local_gid"][: len(o)]
            acc[g] += o
            cnt[g] += 1
    field = np.where(cnt[:, None] > 0, acc / np.maximum(cnt, 1)[:, None], 0.0)
    return field, cnt

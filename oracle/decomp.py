"""Virtual-rank driver: the decomposed (DS) layer on P sub-domains in one process.

PAPER.md:58-60 (§3) and Alg. 1: decompose the sampled domain,
build each sub-domain's graph over owned centres with neighbours from
owned + overlap nodes, run the convolution per sub-domain and refresh the
overlap from the neighbours' interiors after every hop.  Used by tests to pin
"decomposed with full-width halo == undecomposed" (north_star).
"""
import numpy as np

from . import features, graph, halo, layer, partition


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

"""O3 - radius graph kernel G_i with random edge cap n_e.

PAPER.md:27 (§2.1): "Graph kernels G_i = (V_i, E_i) are constructed using these
sampled nodes v_i in V_s as centers within a radius rho.  Edge connections
e_ij in E_i are established between node j within a specified radius and the
respective central nodes i.  For edges |E_i| > n_e, n_e edges are further
randomly sampled from |E_i|."   Alg. 1 lines 395-396 (edgeindexcreator, rand).

Readings: R7 fp32 inclusive predicate in a fixed op order, no FMA;
R8 neighbours are sampled nodes only, no self loops; R10 the cap keeps the n_e
smallest (key_edge(seed, gid_i, gid_j), gid_j); R11 rows ordered by gid_j.

This is the plain definition: an all-pairs scan per destination row.
"""
import numpy as np

from .hashing import key_edge


def fp32_within(coords: np.ndarray, i: int, r: float) -> np.ndarray:
    """Boolean mask over all rows j: pred_fp32(x_i, x_j, r) (R7).

    dx_a = fl32(x_i[a] - x_j[a]);  d2 = fl32(fl32(dx_0^2) + fl32(dx_1^2))
    [3-D: d2 = fl32(d2 + fl32(dx_2^2))];  accept iff d2 <= fl32(r*r).
    numpy float32 ufuncs round every operation separately (no contraction).
    """
    x = np.asarray(coords, dtype=np.float32)
    dim = x.shape[1]
    d2 = None
    for a in range(dim):
        dx = x[i, a] - x[:, a]                      # float32 - float32 -> float32
        sq = dx * dx
        d2 = sq if d2 is None else (d2 + sq)
    r32 = np.float32(r)
    return d2 <= (r32 * r32)


def candidates(coords, i: int, r: float) -> np.ndarray:
    """C_i = {j != i : pred_fp32(x_i, x_j, r)} as ascending local indices."""
    m = fp32_within(coords, i, r)
    m[i] = False
    return np.nonzero(m)[0]


def cap_row(cand: np.ndarray, gid: np.ndarray, gi: int, n_e: int, seed: int) -> np.ndarray:
    """Keep the n_e smallest (key_edge(seed, gid_i, gid_j), gid_j) (R10);
    return the kept local indices ordered by gid_j ascending (R11)."""
    if len(cand) > n_e:
        gj = gid[cand].astype(np.int64)
        keys = key_edge(seed, gi, gj)
        order = np.lexsort((gj, keys))
        cand = cand[order[:n_e]]
    return cand[np.argsort(gid[cand], kind="stable")]


def radius_graph_rows(coords, gid, rows, r: float, n_e: int, seed: int):
    """Adjacency of the given destination rows: list of int32 arrays of local
    source indices, each ordered by gid ascending."""
    if r <= 0 or n_e < 1:
        raise ValueError("radius_graph: r must be > 0 and n_e >= 1")
    gid = np.asarray(gid, dtype=np.int64)
    out = []
    for i in rows:
        c = candidates(coords, int(i), r)
        out.append(cap_row(c, gid, int(gid[i]), n_e, seed).astype(np.int32))
    return out


def radius_graph(coords, gid, n_dst: int, r: float, n_e: int, seed: int):
    """CSR by destination for local rows [0, n_dst): (row_ptr int64, col_idx int32)."""
    rows = radius_graph_rows(coords, gid, range(n_dst), r, n_e, seed)
    row_ptr = np.zeros(n_dst + 1, dtype=np.int64)
    row_ptr[1:] = np.cumsum([len(x) for x in rows])
    col = np.concatenate(rows) if rows else np.zeros(0, np.int32)
    return row_ptr, col.astype(np.int32)


def candidate_count(coords, i: int, r: float) -> int:
    return int(len(candidates(coords, i, r)))

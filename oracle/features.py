"""Edge attributes e_ij.

PAPER.md:27 (§2.1): "Edge attributes e_ij^l in this work are derived by
calculating the relative difference between node coordinates and attributes
(v^l) of nodes i and j."  Alg. 1: e <- dv, dv = v_i - v_j.
PAPER.md:82: Darcy attributes (x_i, y_i, a_i) give edge attributes in R^3.
BASELINE.json configs[2]: airfoil edge attribute (x_i, x_j, a_i, a_j).

Reading R21: mode "diff" = (x_i - x_j, a_i - a_j) for Darcy;
mode "concat" = (x_i, x_j, a_i, a_j) for the airfoil and step configs.
Every value is one fp32 operation (or a copy), so the CUDA path reproduces it
bit for bit.
"""
import numpy as np


def edge_features(mode: str, coords, attr, dst_of_edge, col_idx) -> np.ndarray:
    x = np.asarray(coords, dtype=np.float32)
    a = np.asarray(attr, dtype=np.float32)
    i = np.asarray(dst_of_edge, dtype=np.int64)
    j = np.asarray(col_idx, dtype=np.int64)
    if mode == "diff":
        cols = [x[i] - x[j], a[i] - a[j]]
    elif mode == "concat":
        cols = [x[i], x[j], a[i], a[j]]
    else:
        raise ValueError(mode)
    return np.concatenate(cols, axis=1).astype(np.float32)


def dst_of_edges(row_ptr) -> np.ndarray:
    row_ptr = np.asarray(row_ptr, dtype=np.int64)
    return np.repeat(np.arange(len(row_ptr) - 1, dtype=np.int64), np.diff(row_ptr))

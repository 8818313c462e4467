"""O2 - Nystrom node sampling.

PAPER.md:27 (§2.1): "A subset Omega_s of Omega is formed by randomly sampling
nodes, with |V_s| = s."  Alg. 1: ``Omega_s <- rand(Omega)``.
Reading R9: the sample is the min(s, N) ids with the smallest
``(key_node(seed, g), g)``; returned in ascending id order.
"""
import numpy as np

from .hashing import key_node


def sample(n_points: int, s: int, seed: int) -> np.ndarray:
    """Return int32 ids of the sampled nodes, ascending.

    Step by step (R9):
      1. for every global id g in [0, N) form the pair (key_node(seed, g), g);
      2. sort the pairs lexicographically ascending;
      3. keep the first min(s, N);
      4. output their ids in ascending order.
    """
    if s < 1 or n_points < 0:
        raise ValueError("sample: s must be >= 1 and N >= 0")
    g = np.arange(n_points, dtype=np.int64)
    keys = key_node(seed, g)
    order = np.lexsort((g, keys))          # primary: key, secondary: g
    keep = order[: min(s, n_points)]
    return np.sort(g[keep]).astype(np.int32)

"""Helpers shared by the -m gpu parity tests (test infrastructure)."""
import numpy as np
import torch


def cuda():
    return torch.device("cuda:0")


def T(a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.to(cuda())


def N(t):
    return t.detach().float().cpu().numpy() if t.dtype == torch.bfloat16 else t.detach().cpu().numpy()


def nerr(x, ref):
    """normwise-inf relative error max|x - ref| / max|ref|."""
    x = np.asarray(x, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    den = np.max(np.abs(ref)) if ref.size else 0.0
    num = np.max(np.abs(x - ref)) if ref.size else 0.0
    return num / den if den > 0 else num


def hash_rows(n, count, salt=0):
    """Deterministic pseudo-random subset of row ids for sampled checks."""
    g = np.random.default_rng(1000 + salt)
    return np.sort(g.choice(n, size=min(n, count), replace=False))

"""O7 - overlap (halo) update between sub-domains, P virtual ranks in one process.

PAPER.md:60 (§3): "the overlap area of a given domain is updated from the
neighboring domains' interiors".  Alg. 1: v_L <- Comm(i_b, Omega, v_L)
once per hop.  Reading R16: received halo values are detached (gradients of
halo rows are dropped) unless the exact REVERSE_ADD mode is requested.
"""
import numpy as np


def halo_forward(ranks, values):
    """values[q][halo rows owned by p] <- values[p][send(p->q) rows], all q, p."""
    P = len(ranks)
    out = [np.array(v, copy=True) for v in values]
    for q in range(P):
        hq = ranks[q]
        for p in range(P):
            if p == q:
                continue
            a, b = int(hq["halo_ptr"][p]), int(hq["halo_ptr"][p + 1])
            sp = ranks[p]
            s0, s1 = int(sp["send_ptr"][q]), int(sp["send_ptr"][q + 1])
            assert b - a == s1 - s0
            out[q][a:b] = values[p][sp["send_idx"][s0:s1]]
    return out


def halo_reverse_add(ranks, values):
    """values[p][send(p->q) rows] += values[q][matching halo rows], q ascending."""
    P = len(ranks)
    out = [np.array(v, copy=True) for v in values]
    for p in range(P):
        sp = ranks[p]
        for q in range(P):
            if q == p:
                continue
            s0, s1 = int(sp["send_ptr"][q]), int(sp["send_ptr"][q + 1])
            hq = ranks[q]
            a, b = int(hq["halo_ptr"][p]), int(hq["halo_ptr"][p + 1])
            out[p][sp["send_idx"][s0:s1]] += values[q][a:b]
    return out

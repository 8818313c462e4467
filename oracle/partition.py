"""O4 - domain decomposition into n_procs sub-domains with overlap l.

PAPER.md:58 (§3): "dividing Omega into n_procs ... subdomains Omega_r, with each
subdomain featuring an extended overlap of length l ... we set l = r to ensure
that nodes at the edges of any given spatial partition have complete kernels".
PAPER.md:70: "domains are equally partitioned based on their coordinates".
Alg. 1 line 392 (decompose after sampling), line 403 (index i_b).

Readings: R12 median recursive coordinate bisection on the longest
axis, lower median, ties to the lower rank; R13 L-infinity box extension;
R15 a rank computes only owned destinations; near/deep split (R23) so that deep
rows can run before the halo arrives.

The recursion follows SURVEY §8(c) O4 step by step.
"""
import numpy as np


class Degenerate(Exception):
    """RCB split left an empty upper side (all split coordinates tied)."""


def _f32(x):
    return np.float32(x)


def rcb(coords, gid, nparts: int):
    """Return (owner int32[s], boxes float32[P,2,dim], internal bool[P,2,dim]).

    internal[q, 0/1, a] says whether box q's low/high face on axis a was
    created by a split (an internal face) rather than lying on the global
    bounding box.

    RCB(S, p0, P): if P == 1 assign S to p0.  Otherwise ext_a = fl32(max-min)
    over S, a* = argmax (ties -> lowest a); sort S by (x[a*], gid); m =
    ceil(|S|/2); c* = x[a*] of the m-th element; lower = {x[a*] <= c*}, upper =
    rest (empty -> Degenerate); lower box hi[a*] = c*, upper box lo[a*] = c*.
    """
    x = np.asarray(coords, dtype=np.float32)
    gid = np.asarray(gid, dtype=np.int64)
    s, dim = x.shape
    if nparts < 1 or (nparts & (nparts - 1)) != 0 or nparts > s:
        raise ValueError("rcb: nparts must be a power of two <= number of points")
    owner = np.full(s, -1, dtype=np.int32)
    boxes = np.zeros((nparts, 2, dim), dtype=np.float32)
    internal = np.zeros((nparts, 2, dim), dtype=bool)

    def rec(idx, p0, P, lo, hi, ilo, ihi):
        if P == 1:
            owner[idx] = p0
            boxes[p0, 0] = lo
            boxes[p0, 1] = hi
            internal[p0, 0] = ilo
            internal[p0, 1] = ihi
            return
        xs = x[idx]
        ext = xs.max(axis=0) - xs.min(axis=0)          # fp32 subtraction
        a = int(np.argmax(ext))                         # first maximum
        key = xs[:, a] + np.float32(0.0)                # -0.0 -> +0.0
        order = np.lexsort((gid[idx], key))
        m = (len(idx) + 1) // 2
        c = key[order[m - 1]]
        low_mask = key <= c
        lower, upper = idx[low_mask], idx[~low_mask]
        if len(upper) == 0:
            raise Degenerate("rcb: empty upper side")
        hi_l = hi.copy(); hi_l[a] = c
        lo_u = lo.copy(); lo_u[a] = c
        ihi_l = ihi.copy(); ihi_l[a] = True
        ilo_u = ilo.copy(); ilo_u[a] = True
        rec(lower, p0, P // 2, lo, hi_l, ilo, ihi_l)
        rec(upper, p0 + P // 2, P // 2, lo_u, hi, ilo_u, ihi)

    lo0 = x.min(axis=0).astype(np.float32)
    hi0 = x.max(axis=0).astype(np.float32)
    nofaces = np.zeros(dim, dtype=bool)
    rec(np.arange(s), 0, nparts, lo0, hi0, nofaces, nofaces.copy())
    return owner, boxes, internal


def plan(coords, gid, nparts: int, overlap_l: float, radius: float):
    """Full decomposition plan for every rank.

    Returns (owner, boxes, internal, ranks) where ranks[q] is a dict with
      local_rows  int64[n_loc]  indices into the sampled set, local order
                                deep (gid asc) | near (gid asc) | halo (owner asc, gid asc)
      local_gid   int64[n_loc]
      n_deep, n_near, n_halo
      halo_ptr    int64[P+1]    halo rows owned by p are local [halo_ptr[p], halo_ptr[p+1])
      send_ptr    int64[P+1]    send_idx[send_ptr[q]:send_ptr[q+1]] = local rows sent to q
      send_idx    int32[...]    (gid ascending within each q)
    Halo(q) = {j : owner(j) != q, fl32(lo_q - l) <= x_j <= fl32(hi_q + l) all axes}.
    send(p->q) = own(p) ∩ halo(q).  Near(q): owned j with x_j[a] <= fl32(lo_q[a]+t)
    on an internal low face or x_j[a] >= fl32(hi_q[a]-t) on an internal high
    face, t = fl32(max(l, r) * (1 + 2^-10)); a face is internal if it is not on
    the global bounding box (a face created by a split).
    """
    x = np.asarray(coords, dtype=np.float32)
    gid = np.asarray(gid, dtype=np.int64)
    s, dim = x.shape
    if overlap_l < 0 or radius <= 0:
        raise ValueError("plan: l must be >= 0 and r > 0")
    owner, boxes, internal = rcb(x, gid, nparts)
    l32 = _f32(overlap_l)
    t = _f32(_f32(max(_f32(overlap_l), _f32(radius))) * _f32(1.0 + 2.0 ** -10))

    in_ext = np.zeros((nparts, s), dtype=bool)
    for q in range(nparts):
        lo = boxes[q, 0] - l32
        hi = boxes[q, 1] + l32
        in_ext[q] = np.all((x >= lo) & (x <= hi), axis=1)

    ranks = []
    for q in range(nparts):
        own = np.nonzero(owner == q)[0]
        near_mask = np.zeros(len(own), dtype=bool)
        for a in range(dim):
            if internal[q, 0, a]:
                near_mask |= x[own, a] <= boxes[q, 0, a] + t
            if internal[q, 1, a]:
                near_mask |= x[own, a] >= boxes[q, 1, a] - t
        deep = own[~near_mask]
        near = own[near_mask]
        deep = deep[np.argsort(gid[deep], kind="stable")]
        near = near[np.argsort(gid[near], kind="stable")]
        halo_parts = []
        halo_ptr = np.zeros(nparts + 1, dtype=np.int64)
        n_own = len(own)
        halo_ptr[0] = n_own
        for p in range(nparts):
            if p == q:
                h = np.zeros(0, dtype=np.int64)
            else:
                h = np.nonzero((owner == p) & in_ext[q])[0]
                h = h[np.argsort(gid[h], kind="stable")]
            halo_parts.append(h)
            halo_ptr[p + 1] = halo_ptr[p] + len(h)
        local_rows = np.concatenate([deep, near] + halo_parts).astype(np.int64)
        ranks.append(dict(local_rows=local_rows, local_gid=gid[local_rows],
                          n_deep=len(deep), n_near=len(near),
                          n_halo=int(halo_ptr[-1] - n_own), halo_ptr=halo_ptr))

    # send lists: send(p->q) = own(p) ∩ halo(q), as p's local indices, gid ascending
    for p in range(nparts):
        pos = {int(r_): k for k, r_ in enumerate(ranks[p]["local_rows"][: ranks[p]["n_deep"] + ranks[p]["n_near"]])}
        send_ptr = np.zeros(nparts + 1, dtype=np.int64)
        parts = []
        for q in range(nparts):
            hq = ranks[q]
            rows_from_p = hq["local_rows"][hq["halo_ptr"][p]: hq["halo_ptr"][p + 1]]
            idx = np.array([pos[int(r_)] for r_ in rows_from_p], dtype=np.int32)
            parts.append(idx)
            send_ptr[q + 1] = send_ptr[q] + len(idx)
        ranks[p]["send_ptr"] = send_ptr
        ranks[p]["send_idx"] = np.concatenate(parts).astype(np.int32) if parts else np.zeros(0, np.int32)
    return owner, boxes, internal, ranks

"""Pins of oracle parts that round 1 left unpinned:

* oracle/features.py against a hand fixture (sign of v_i - v_j, Alg. 1 :397,
  PAPER.md:27; concat order, reading R21);
* the fp32 radius predicate's operation order (reading R7) on exact grid ties
  (SURVEY §8(c) C.4 "Regression fixture: ... ties accepted in fp32"; H4),
  against an independent emulation of IEEE binary32 rounding written with
  exact rational arithmetic (no numpy float32 arithmetic), so that a predicate
  evaluated in fp64, with the exact radius, or with a different rounding
  sequence fails.
"""
import json
import os
from fractions import Fraction

import numpy as np

from oracle import features, graph


def test_edge_features_hand_fixture(golden_dir):
    fx = json.load(open(os.path.join(golden_dir, "edge_features.json")))
    x = np.array(fx["coords"], np.float32)
    a = np.array(fx["attr"], np.float32)
    dst = features.dst_of_edges(fx["row_ptr"])
    assert dst.tolist() == fx["expected_dst"]
    col = np.array(fx["col_idx"], np.int64)
    assert features.edge_features("diff", x, a, dst, col).tolist() == fx["expected_diff"]
    assert features.edge_features("concat", x, a, dst, col).tolist() == fx["expected_concat"]


def _fl32(q: Fraction) -> Fraction:
    """Round a rational to the nearest IEEE binary32 value, ties to even
    (normal range only; the fixture never leaves it)."""
    if q == 0:
        return Fraction(0)
    s = -1 if q < 0 else 1
    q = abs(q)
    e = 0
    while q >= 2:
        q /= 2
        e += 1
    while q < 1:
        q *= 2
        e -= 1
    m = q * (1 << 23)  # 1 <= q < 2: 24-bit significand
    f = m.numerator // m.denominator
    rem = m - f
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and f % 2 == 1):
        f += 1
    return s * Fraction(f, 1 << 23) * (Fraction(2) ** e)


def _grid(n):
    # R20: x = fl32(col / (n - 1)), y = fl32(row / (n - 1)), gid = row*n + col
    t = [_fl32(Fraction(c, n - 1)) for c in range(n)]
    pts = [(t[c], t[r]) for r in range(n) for c in range(n)]
    return pts, np.array([[float(px), float(py)] for px, py in pts], np.float32)


def _pred_r7(p, q, r32):
    """R7 in exact arithmetic with a binary32 rounding after every operation:
    dx = fl(x_i - x_j), d2 = fl(fl(dx0^2) + fl(dx1^2)), accept iff d2 <= fl(r*r)."""
    dx = _fl32(p[0] - q[0])
    dy = _fl32(p[1] - q[1])
    d2 = _fl32(_fl32(dx * dx) + _fl32(dy * dy))
    return d2 <= _fl32(r32 * r32)


def test_fp32_predicate_on_exact_ties_1d():
    """a 16-point grid at r = 0.2 has 26 ordered pairs at exactly
    three spacings (0.2 in real arithmetic); the fp32 predicate accepts 18 of
    them (the real-number predicate with r = 0.2 would accept all 26)."""
    n = 16
    t = [_fl32(Fraction(c, n - 1)) for c in range(n)]
    x = np.array([[float(v), 0.0] for v in t], np.float32)
    r32 = _fl32(Fraction(1, 5))
    ties = [(i, j) for i in range(n) for j in range(n) if abs(i - j) == 3]
    assert len(ties) == 26
    emu = {(i, j) for i, j in ties if _pred_r7((t[i], Fraction(0)), (t[j], Fraction(0)), r32)}
    got = {(i, j) for i, j in ties if graph.fp32_within(x, i, 0.2)[j]}
    assert got == emu
    assert len(got) == 18


def test_fp32_predicate_op_order_on_2d_ties():
    """26 x 26 grid (spacing 1/25), r = 0.2 = five spacings: offsets (5,0),
    (0,5), (3,4), (4,3) are exact ties in real arithmetic.  The oracle's
    predicate must accept exactly the pairs the binary32 emulation of R7
    accepts, which differ from an fp64 evaluation (with fl32(r)) and from the
    exact-radius predicate; rows 0..3 of the grid as destinations."""
    n = 26
    pts, x = _grid(n)
    r32 = _fl32(Fraction(1, 5))
    N = n * n
    dest = range(4 * n)
    ties = [(i, j) for i in dest for j in range(N)
            if i != j and (i // n - j // n) ** 2 + (i % n - j % n) ** 2 == 25]
    emu = {(i, j) for i, j in ties if _pred_r7(pts[i], pts[j], r32)}
    got = {(i, j) for i, j in ties if graph.fp32_within(x, i, 0.2)[j]}
    assert got == emu
    x64 = x.astype(np.float64)
    f64 = {(i, j) for i, j in ties if ((x64[i] - x64[j]) ** 2).sum() <= float(r32) ** 2}
    exact = {(i, j) for i, j in ties if ((x64[i] - x64[j]) ** 2).sum() <= 0.04}
    assert got != f64 and got != exact  # the fixture separates the candidate readings
    assert 0 < len(got) < len(ties)

"""Pins for oracle O3 (radius graph + cap), R7/R8/R10/R11."""
import numpy as np
from scipy.spatial import cKDTree

from oracle import graph, hashing


def test_collinear_hand_case():
    # x = 0, 0.1, 0.3 with r = 0.15 -> edges {0<->1} only
    c = np.array([[0.0, 0.0], [0.1, 0.0], [0.3, 0.0]], np.float32)
    rp, ci = graph.radius_graph(c, np.arange(3), 3, 0.15, 64, 0)
    assert list(rp) == [0, 1, 2, 2]
    assert list(ci) == [1, 0]


def test_predicate_inclusive():
    # d2 == r^2 exactly representable -> included (R7 "<=")
    c = np.array([[0.0, 0.0], [0.5, 0.0], [0.0, 0.75]], np.float32)
    rp, ci = graph.radius_graph(c, np.arange(3), 3, 0.5, 64, 0)
    assert list(ci[rp[0]:rp[1]]) == [1]


def test_matches_kdtree_library():
    # brute-force O(n^2) against scipy's kd-tree ball query (fp64) on 100+
    # random instances; disagreements only allowed within fp32 rounding of r
    g = np.random.default_rng(0)
    for inst in range(100):
        n = int(g.integers(20, 300))
        dim = 2 + inst % 2
        x = g.random((n, dim)).astype(np.float32)
        r = float(g.uniform(0.05, 0.3))
        tree = cKDTree(x.astype(np.float64))
        for i in range(0, n, max(1, n // 25)):
            mine = set(graph.candidates(x, i, r).tolist())
            lib = set(tree.query_ball_point(x[i].astype(np.float64), r)) - {i}
            for j in mine ^ lib:
                d = np.linalg.norm(x[i].astype(np.float64) - x[j])
                assert abs(d - r) < 1e-6 * max(1.0, r)


def test_pre_cap_symmetry():
    g = np.random.default_rng(1)
    x = g.random((300, 2)).astype(np.float32)
    adj = [set(graph.candidates(x, i, 0.1).tolist()) for i in range(300)]
    for i in range(300):
        for j in adj[i]:
            assert i in adj[j]


def test_cap_rules():
    g = np.random.default_rng(2)
    x = g.random((800, 2)).astype(np.float32)
    gid = np.arange(800) * 3 + 5
    rows = graph.radius_graph_rows(x, gid, range(800), 0.08, 8, seed=21)
    for i, kept in enumerate(rows):
        cand = graph.candidates(x, i, 0.08)
        assert len(kept) == min(len(cand), 8)
        assert set(kept.tolist()) <= set(cand.tolist())
        assert np.all(np.diff(gid[kept]) > 0)                     # R11
        if len(cand) > 8:                                         # R10 brute force
            ks = sorted((hashing.key_edge_int(21, int(gid[i]), int(gid[j])), int(gid[j]), j)
                        for j in cand)
            assert set(kept.tolist()) == {t[2] for t in ks[:8]}


def test_cap_uniformity_monte_carlo():
    # n_e = 1, degree 5, 10^4 seeds -> each neighbour 0.2 +- 0.02
    x = np.array([[0, 0], [0.01, 0], [0, 0.01], [-0.01, 0], [0, -0.01], [0.01, 0.01]],
                 np.float32)
    gid = np.arange(6)
    cnt = np.zeros(6)
    for seed in range(10_000):
        kept = graph.cap_row(graph.candidates(x, 0, 0.05), gid, 0, 1, seed)
        cnt[kept] += 1
    f = cnt[1:] / 10_000
    assert np.all(np.abs(f - 0.2) < 0.02)


def test_expected_degree_closed_form():
    # uniform points in the unit square: E[#candidates] = (N-1)(pi r^2 - 8 r^3/3 + r^4/2)
    g = np.random.default_rng(3)
    N, r = 4000, 0.1
    x = g.random((N, 2)).astype(np.float32)
    counts = [graph.candidate_count(x, i, r) for i in range(0, N, 4)]
    want = (N - 1) * (np.pi * r * r - 8 * r ** 3 / 3 + r ** 4 / 2)
    assert abs(np.mean(counts) - want) / want < 0.02


def test_partition_invariance_of_cap():
    # the cap is keyed by global ids, so relabelling local rows leaves each
    # row's kept gid set unchanged (R10)
    g = np.random.default_rng(4)
    x = g.random((500, 2)).astype(np.float32)
    gid = g.permutation(10_000)[:500]
    perm = g.permutation(500)
    a = graph.radius_graph_rows(x, gid, range(500), 0.12, 6, 9)
    b = graph.radius_graph_rows(x[perm], gid[perm], range(500), 0.12, 6, 9)
    inv = np.argsort(perm)
    for i in range(500):
        assert list(gid[a[i]]) == list(gid[perm][b[inv[i]]])

"""Pins for oracle O4 (decomposition) and O7 (halo), R12/R13/R23."""
import json
import os

import numpy as np
import pytest

from oracle import graph, halo, partition


def _line_fixture(golden_dir):
    with open(os.path.join(golden_dir, "partition_line.json")) as f:
        return json.load(f)


def test_hand_fixture_line(golden_dir):
    fx = _line_fixture(golden_dir)
    x = np.array([[np.float32(v), 0.0] for v in fx["x"]], np.float32)
    gid = np.arange(len(x))
    owner, boxes, internal, ranks = partition.plan(x, gid, fx["P"], fx["l"], fx["r"])
    assert list(owner) == fx["owner"]
    for q in range(2):
        rq = ranks[q]
        nd, nn = rq["n_deep"], rq["n_near"]
        assert list(rq["local_rows"][:nd]) == fx["deep"][q]
        assert list(rq["local_rows"][nd:nd + nn]) == fx["near"][q]
        assert list(rq["local_rows"][nd + nn:]) == fx["halo"][q]
    s01 = ranks[0]["send_idx"][ranks[0]["send_ptr"][1]:ranks[0]["send_ptr"][2]]
    assert list(ranks[0]["local_rows"][s01]) == fx["send"]["0->1"]
    s10 = ranks[1]["send_idx"][ranks[1]["send_ptr"][0]:ranks[1]["send_ptr"][1]]
    assert list(ranks[1]["local_rows"][s10]) == fx["send"]["1->0"]
    assert internal[0, 1, 0] and internal[1, 0, 0] and not internal[0, 0, 0]


def test_identity_partition():
    g = np.random.default_rng(0)
    x = g.random((100, 2)).astype(np.float32)
    owner, boxes, internal, ranks = partition.plan(x, np.arange(100), 1, 0.1, 0.1)
    assert np.all(owner == 0)
    assert ranks[0]["n_halo"] == 0 and ranks[0]["n_near"] == 0
    assert list(ranks[0]["local_rows"]) == list(range(100))
    assert not internal.any()


def test_balanced_median_split():
    # 1000 uniform points, P = 4 -> each count in [230, 270]; median RCB gives 250
    g = np.random.default_rng(1)
    x = g.random((1000, 2)).astype(np.float32)
    owner, _, _ = partition.rcb(x, np.arange(1000), 4)
    assert list(np.bincount(owner)) == [250, 250, 250, 250]


def test_errors():
    x = np.random.default_rng(2).random((10, 2)).astype(np.float32)
    with pytest.raises(ValueError):
        partition.rcb(x, np.arange(10), 3)
    with pytest.raises(ValueError):
        partition.rcb(x, np.arange(10), 16)
    same = np.zeros((8, 2), np.float32)
    with pytest.raises(partition.Degenerate):
        partition.rcb(same, np.arange(8), 2)


def test_split_plane_ties_go_lower():
    # a point exactly on the split plane belongs to the lower rank
    x = np.array([[0.0, 0], [0.5, 0], [0.5, 0.1], [1.0, 0]], np.float32)
    owner, boxes, _ = partition.rcb(x, np.arange(4), 2)
    assert list(owner) == [0, 0, 0, 1]
    assert boxes[0, 1, 0] == np.float32(0.5)


@pytest.mark.parametrize("dim,P", [(2, 4), (3, 8), (2, 8)])
def test_plan_invariants(dim, P):
    g = np.random.default_rng(10 + dim + P)
    n = 1500
    x = g.random((n, dim)).astype(np.float32)
    gid = g.permutation(100_000)[:n]
    r = 0.1
    l = r * (1 + 2 ** -12)
    owner, boxes, internal, ranks = partition.plan(x, gid, P, l, r)
    # disjoint cover
    own_all = np.concatenate([q["local_rows"][: q["n_deep"] + q["n_near"]] for q in ranks])
    assert sorted(own_all.tolist()) == list(range(n))
    for q in range(P):
        rq = ranks[q]
        n_own = rq["n_deep"] + rq["n_near"]
        # exchange-list consistency: send(p->q) = own(p) ∩ ext(q)
        lo = boxes[q, 0] - np.float32(l)
        hi = boxes[q, 1] + np.float32(l)
        ext = np.all((x >= lo) & (x <= hi), axis=1)
        halo_rows = rq["local_rows"][n_own:]
        assert set(halo_rows.tolist()) == set(np.nonzero(ext & (owner != q))[0].tolist())
        for p in range(P):
            hp = rq["local_rows"][rq["halo_ptr"][p]:rq["halo_ptr"][p + 1]]
            assert np.all(owner[hp] == p)
            assert np.all(np.diff(gid[hp]) > 0)
        # halo sufficiency at l = r (1 + 2^-12) and the deep-row invariant
        local = set(rq["local_rows"].tolist())
        deep = set(rq["local_rows"][: rq["n_deep"]].tolist())
        sends = set()
        for p in range(P):
            sends |= set(rq["local_rows"][rq["send_idx"][rq["send_ptr"][p]:rq["send_ptr"][p + 1]]].tolist())
        assert not (deep & sends)
        for i in rq["local_rows"][:n_own][::7]:
            nb = graph.candidates(x, int(i), r)
            assert set(nb.tolist()) <= local
            if i in deep:
                assert np.all(owner[nb] == q)


def test_zero_overlap_halo_only_on_faces():
    # l = 0: the halo holds only points lying exactly on q's closed box (R13)
    g = np.random.default_rng(5)
    x = g.random((400, 2)).astype(np.float32)
    owner, boxes, internal, ranks = partition.plan(x, np.arange(400), 4, 0.0, 0.05)
    for q, rq in enumerate(ranks):
        n_own = rq["n_deep"] + rq["n_near"]
        for j in rq["local_rows"][n_own:]:
            on_face = np.any((x[j] == boxes[q, 0]) | (x[j] == boxes[q, 1]))
            assert on_face


def test_halo_two_rank_hand_trace(golden_dir):
    # SPEC.md:385 two-rank trace: rank 1's halo gets rank 0's rows 0.3, 0.4 and vice versa
    fx = _line_fixture(golden_dir)
    x = np.array([[np.float32(v), 0.0] for v in fx["x"]], np.float32)
    _, _, _, ranks = partition.plan(x, np.arange(8), 2, fx["l"], fx["r"])
    vals = [np.array([[10.0 * r_ + 1] for r_ in q["local_rows"]]) for q in ranks]
    vals[0][4:] = -1
    vals[1][4:] = -1
    out = halo.halo_forward(ranks, vals)
    assert out[0][4:, 0].tolist() == [41.0]
    assert out[1][4:, 0].tolist() == [21.0, 31.0]
    # reverse add: owners accumulate their halo copies (q ascending)
    g = [np.zeros((len(q["local_rows"]), 1)) for q in ranks]
    g[1][4:] = [[1.0], [2.0]]
    g[0][4:] = [[5.0]]
    back = halo.halo_reverse_add(ranks, g)
    loc0 = list(ranks[0]["local_rows"])
    assert back[0][loc0.index(2), 0] == 1.0 and back[0][loc0.index(3), 0] == 2.0
    loc1 = list(ranks[1]["local_rows"])
    assert back[1][loc1.index(4), 0] == 5.0


def test_halo_single_rank_noop():
    x = np.random.default_rng(6).random((50, 2)).astype(np.float32)
    _, _, _, ranks = partition.plan(x, np.arange(50), 1, 0.1, 0.1)
    v = [np.arange(50.0)[:, None]]
    assert np.array_equal(halo.halo_forward(ranks, v)[0], v[0])

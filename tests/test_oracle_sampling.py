"""Pins for oracle O0-O3.  CPU only."""
import itertools
import math
import os

import numpy as np
import pytest

from oracle import sampling as S

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _graph_from_edges(n, edges):
    rows = [[] for _ in range(n)]
    for u, v in edges:
        rows[u].append(v)
    rp = np.zeros(n + 1, dtype=np.int64)
    col = []
    for v in range(n):
        r = sorted(set(rows[v]))
        col += r
        rp[v + 1] = rp[v] + len(r)
    return rp, np.asarray(col, dtype=np.int32)


def _random_graph(n, p, seed):
    rng = np.random.default_rng(seed)
    edges = [(u, v) for u in range(n) for v in range(n) if u != v and rng.random() < p]
    edges += [(v, u) for u, v in edges]
    return _graph_from_edges(n, edges)


# ---------------------------------------------------------------- O0
def test_philox_kat_golden():
    for line in open(os.path.join(GOLD, "philox4x32_kat.txt")):
        if line.startswith("#") or not line.strip():
            continue
        t = line.split()
        rounds = int(t[0])
        ctr = [int(x, 16) for x in t[1:5]]
        key = [int(x, 16) for x in t[5:7]]
        want = [int(x, 16) for x in t[7:11]]
        assert list(S.philox4x32(ctr, key, rounds)) == want


# ---------------------------------------------------------------- O2 Floyd
def test_floyd_worked_example_golden():
    for line in open(os.path.join(GOLD, "floyd_example.txt")):
        if line.startswith("#") or not line.strip():
            continue
        lhs, rhs = line.split("->")
        seed, epoch, g, hop, v, d, k = map(int, lhs.split())
        assert list(S.sample_row(seed, epoch, g, hop, v, d, k)) == list(map(int, rhs.split()))


def test_floyd_worked_example_through_sampler():
    # node 0 with 10 neighbours 1..10, fanout 3, seed 0, epoch 0, g 0 -> positions {3,7,9}
    rp, col = _graph_from_edges(11, [(0, j) for j in range(1, 11)])
    hops = S.neighbor_sample(rp, col, np.array([0]), [3], 0, 0, 0)
    assert list(hops[0]["blk_nbr"]) == [4, 8, 10]


def test_floyd_small_degree_takes_all():
    for d in range(0, 6):
        assert list(S.sample_row(7, 1, 2, 0, 5, d, 5)) == list(range(d))


@pytest.mark.parametrize("d,k", [(5, 2), (6, 3), (4, 1)])
def test_floyd_chi2_uniform_over_subsets(d, k):
    trials = 20000
    subsets = {s: 0 for s in itertools.combinations(range(d), k)}
    for g in range(trials):
        pos = tuple(S.sample_row(11, 0, g, 1, 3, d, k))
        assert pos in subsets                      # brute force: a valid k-subset, ascending
        subsets[pos] += 1
    exp = trials / len(subsets)
    chi2 = sum((c - exp) ** 2 / exp for c in subsets.values())
    dof = len(subsets) - 1
    # p = 0.001 upper quantiles of chi2(dof)
    crit = {3: 16.27, 9: 27.88, 19: 43.82}[dof]
    assert chi2 < crit, (chi2, dof)


# ---------------------------------------------------------------- O1
def test_epoch_perm_and_batching():
    train = np.arange(10, dtype=np.int32)
    p0 = S.epoch_perm(train, 1, 0)
    assert sorted(p0.tolist()) == list(range(10))
    assert np.array_equal(p0, S.epoch_perm(train, 1, 0))
    assert not np.array_equal(p0, S.epoch_perm(train, 1, 1))
    sizes = [len(S.batch_seeds(p0, 4, g)) for g in range(3)]
    assert sizes == [4, 4, 2]
    assert sorted(np.concatenate([S.batch_seeds(p0, 4, g) for g in range(3)]).tolist()) == list(range(10))
    assert len(S.epoch_perm(np.zeros(0, np.int32), 1, 0)) == 0


# ---------------------------------------------------------------- O2 relabel / blocks
def _check_hops(rp, col, seeds, fanouts, hops):
    dst = np.asarray(seeds)
    L = len(fanouts)
    for h, hp in enumerate(hops):
        k = fanouts[L - 1 - h]
        nd, ns = hp["n_dst"], hp["n_src"]
        src = hp["src_ids"]
        assert nd == len(dst) and np.array_equal(src[:nd], dst)            # prefix
        new = src[nd:]
        assert np.all(np.diff(new) > 0)                                    # ascending
        assert not set(new.tolist()) & set(dst.tolist())                   # disjoint
        assert set(src.tolist()) == set(dst.tolist()) | set(hp["blk_nbr"].tolist())
        assert np.array_equal(src[hp["blk_col"]], hp["blk_nbr"])           # relabel map
        brp = hp["blk_rowptr"]
        for i, v in enumerate(dst):
            row = col[rp[v]:rp[v + 1]]
            got = hp["blk_nbr"][brp[i]:brp[i + 1]]
            assert len(got) == min(len(row), k)
            assert set(got.tolist()) <= set(row.tolist())                  # subset of N(v)
            assert len(set(got.tolist())) == len(got)                      # no duplicate edges
            if len(row) <= k:
                assert np.array_equal(got, row)
            pos = np.searchsorted(row, got)
            assert np.all(np.diff(pos) > 0)                                # ascending CSR position
        dst = src                                                          # chaining


@pytest.mark.parametrize("gseed", [0, 1, 2])
def test_neighbor_sample_invariants(gseed):
    rp, col = _random_graph(40, 0.15, gseed)
    seeds = np.array([3, 17, 5, 30], dtype=np.int32)
    fan = [4, 3, 2]
    hops = S.neighbor_sample(rp, col, seeds, fan, 9, 2, 5)
    _check_hops(rp, col, seeds, fan, hops)
    again = S.neighbor_sample(rp, col, seeds, fan, 9, 2, 5)
    for a, b in zip(hops, again):
        for key in ("src_ids", "blk_rowptr", "blk_col", "blk_nbr"):
            assert np.array_equal(a[key], b[key])


def test_degree_zero_seeds():
    rp, col = _graph_from_edges(5, [])
    seeds = np.array([4, 1], dtype=np.int32)
    hops = S.neighbor_sample(rp, col, seeds, [3, 2], 1, 0, 0)
    for hp in hops:
        assert hp["n_edges"] == 0 and np.array_equal(hp["src_ids"], seeds)


def test_star_example():
    # centre + 3 leaves, fanout 3 -> exactly 3 edges into the centre
    rp, col = _graph_from_edges(4, [(0, 1), (0, 2), (0, 3), (1, 0), (2, 0), (3, 0)])
    hops = S.neighbor_sample(rp, col, np.array([0]), [3], 1, 0, 0)
    assert hops[0]["n_edges"] == 3 and sorted(hops[0]["blk_nbr"].tolist()) == [1, 2, 3]


def test_sampled_block_is_member_of_product_set():
    # brute force: every possible block for one seed hop enumerated; the sample is one of them
    rp, col = _graph_from_edges(8, [(0, j) for j in range(1, 7)] + [(1, 2), (1, 3), (1, 4)])
    k = 2
    for g in range(50):
        hop = S.neighbor_sample(rp, col, np.array([0, 1]), [k], 3, 0, g)[0]
        blocks = {(a, b) for a in itertools.combinations(col[rp[0]:rp[1]].tolist(), k)
                  for b in itertools.combinations(col[rp[1]:rp[2]].tolist(), k)}
        got = (tuple(hop["blk_nbr"][0:2].tolist()), tuple(hop["blk_nbr"][2:4].tolist()))
        assert got in blocks


# ---------------------------------------------------------------- O3
def test_shadow_triangle_and_isolated():
    rp, col = _graph_from_edges(4, [(0, 1), (1, 0), (1, 2), (2, 1), (0, 2), (2, 0)])
    hops, blk = S.shadow_sample(rp, col, np.array([0]), [2], 2, 1, 0, 0)
    assert blk["n_src"] == 3 and blk["n_edges"] == 6
    hops, blk = S.shadow_sample(rp, col, np.array([3]), [2, 2], 2, 1, 0, 0)
    assert blk["n_src"] == 1 and blk["n_edges"] == 0


@pytest.mark.parametrize("gseed", [3, 4])
def test_shadow_induced_equals_membership_filter(gseed):
    rp, col = _random_graph(50, 0.1, gseed)
    seeds = np.array([1, 2, 40], dtype=np.int32)
    hops, blk = S.shadow_sample(rp, col, seeds, [3, 2], 3, 5, 1, 0)
    Sset = blk["src_ids"]
    assert np.array_equal(Sset, hops[-1]["src_ids"])
    assert np.array_equal(Sset[:3], seeds)
    member = set(Sset.tolist())
    local = {v: i for i, v in enumerate(Sset.tolist())}
    brute = set()
    for v in range(50):
        for u in col[rp[v]:rp[v + 1]].tolist():
            if u in member and v in member:
                brute.add((local[u], local[v]))
    rows = np.repeat(np.arange(blk["n_dst"]), np.diff(blk["blk_rowptr"]))
    got = set(zip(blk["blk_col"].tolist(), rows.tolist()))
    assert got == brute and len(got) == blk["n_edges"]
    # sampled edges (global ids) are a subset of the induced edges
    ind_global = {(Sset[u], Sset[v]) for u, v in got}
    for hp in hops:
        src = hp["src_ids"]
        r = np.repeat(np.arange(hp["n_dst"]), np.diff(hp["blk_rowptr"]))
        for e in range(hp["n_edges"]):
            assert (hp["blk_nbr"][e], src[r[e]]) in ind_global


def test_epoch_perm_golden():
    """O1 against the hand-derived orders of tests/golden/epoch_perm_example.txt (key64 = w0:w1 of
    Philox tag 1 at the stated counters, sorted ascending).  A swapped word order, a wrong counter
    layout (tag / epoch field) or a descending sort fails here."""
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", "epoch_perm_example.txt")
    words, perms = {}, {}
    for ln in open(path):
        f = ln.split()
        if not f or f[0].startswith("#"):
            continue
        if f[0] == "words":
            words[(int(f[1]), int(f[2]), int(f[3]))] = (int(f[4], 16), int(f[5], 16))
        else:
            perms[(int(f[1]), int(f[2]))] = [int(x) for x in f[4:]]
    for (seed, epoch, v), (w0, w1) in words.items():
        out = S.philox4x32([v, 0, (1 << 28) | ((epoch & 0xFFFFF) << 8), 0], [seed & 0xFFFFFFFF, seed >> 32])
        assert (int(out[0]), int(out[1])) == (w0, w1)
    for (seed, epoch), order in perms.items():
        got = S.epoch_perm(np.arange(6, dtype=np.int32), seed, epoch)
        assert list(got) == order, (epoch, got)

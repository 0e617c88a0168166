"""Pins for the oracle's triangle counting (oracle.tc_count / tc_static / tc_delta; SURVEY §8(f)
NEXT-4).  Tied to: hand examples of SPEC S:457-477 (K3 counted six times, path +
closing edge, fresh triangle, deletions), trace(A^3)/6 by numpy matrix products (an independent
closed form), brute-force triple enumeration, and — for the dynamic inclusion-exclusion identity —
brute-force counts before and after random batches."""
import itertools

import numpy as np
import pytest

import oracle


def _und(n, pairs):
    g = oracle.OracleGraph(n, weighted=False)
    sym = sorted({(u, v) for a, b in pairs for (u, v) in ((a, b), (b, a))})
    if sym:
        s, d = zip(*sym)
        g.insert(s, d)
    return g, sym


def _both(pairs):
    return sorted({(u, v) for a, b in pairs for (u, v) in ((a, b), (b, a))})


def _brute(n, pairs):
    adj = np.zeros((n, n), bool)
    for a, b in pairs:
        if a != b:
            adj[a, b] = adj[b, a] = True
    return sum(1 for i, j, k in itertools.combinations(range(n), 3) if adj[i, j] and adj[j, k] and adj[i, k])


def test_hand_examples():
    k3 = [(0, 1), (1, 2), (0, 2)]
    g, sym = _und(3, k3)
    s, d = zip(*sym)
    assert oracle.tc_count(g, g, s, d) == 6          # S:457 "six times"
    assert oracle.tc_static(g) == 1
    g4, _ = _und(4, list(itertools.combinations(range(4), 2)))
    assert oracle.tc_static(g4) == 4
    tree, _ = _und(6, [(0, 1), (0, 2), (1, 3), (1, 4), (2, 5)])
    assert oracle.tc_static(tree) == 0
    # path 0-1-2, insert {0-2}: s1 = 2, s2 = 0, s3 = 0 -> +1
    after, _ = _und(3, k3)
    upd, bs = _und(3, [(0, 2)])
    s, d = zip(*bs)
    assert oracle.tc_delta(after, upd, s, d, True) == (1, (2, 0, 0))
    # all three edges of a fresh triangle: the S3 term
    upd3, bs3 = _und(3, k3)
    s, d = zip(*bs3)
    assert oracle.tc_delta(after, upd3, s, d, True)[0] == 1
    # deletions: one edge of K3 -> 1; all three -> 1
    after1, _ = _und(3, [(0, 1), (1, 2)])
    s, d = zip(*_both([(0, 2)]))
    assert oracle.tc_delta(after1, _und(3, [(0, 2)])[0], s, d, False)[0] == 1
    empty, _ = _und(3, [])
    s, d = zip(*bs3)
    assert oracle.tc_delta(empty, upd3, s, d, False)[0] == 1


@pytest.mark.parametrize("seed", range(8))
def test_static_vs_trace_and_brute_force(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(5, 40))
    p = float(rng.uniform(0.05, 0.5))
    pairs = [(i, j) for i, j in itertools.combinations(range(n), 2) if rng.random() < p]
    g, _ = _und(n, pairs)
    A = np.zeros((n, n), np.int64)
    for a, b in pairs:
        A[a, b] = A[b, a] = 1
    tr = int(np.trace(A @ A @ A))
    assert tr % 6 == 0
    assert oracle.tc_static(g) == tr // 6 == _brute(n, pairs)


@pytest.mark.parametrize("seed", range(10))
def test_dynamic_identity_vs_brute_force(seed):
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(6, 30))
    allp = list(itertools.combinations(range(n), 2))
    rng.shuffle(allp)
    m = int(rng.integers(n, len(allp) * 2 // 3))
    base = [tuple(x) for x in allp[:m]]
    # insert: a batch of absent edges (often closing fresh triangles among themselves)
    ins = [tuple(x) for x in allp[m:m + int(rng.integers(1, 3 * n))]]
    after, _ = _und(n, base + ins)
    upd, bsym = _und(n, ins)
    s, d = zip(*bsym)
    delta, _ = oracle.tc_delta(after, upd, s, d, True)
    assert delta == _brute(n, base + ins) - _brute(n, base)
    # delete: a batch of present edges
    cur = base + ins
    k = int(rng.integers(1, len(cur)))
    pick = rng.choice(len(cur), k, replace=False)
    dele = [cur[i] for i in pick]
    keep = [cur[i] for i in range(len(cur)) if i not in set(pick.tolist())]
    after2, _ = _und(n, keep)
    upd2, dsym = _und(n, dele)
    s, d = zip(*dsym)
    removed, _ = oracle.tc_delta(after2, upd2, s, d, False)
    assert removed == _brute(n, cur) - _brute(n, keep)

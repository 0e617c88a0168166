"""Pins for the oracle's weakly connected components (orc_wcc):
scipy.sparse.csgraph.connected_components(connection='weak') (an independent library), brute-force
transitive closure of the undirected relation on small graphs, hand examples, and the incremental
property (labels after inserting a batch = labels of the union graph; components never split)."""
import numpy as np
import pytest
from scipy.sparse import csr_matrix
from scipy.sparse.csgraph import connected_components

import oracle


def _g(n, pairs):
    g = oracle.OracleGraph(n, weighted=False)
    if pairs:
        s, d = zip(*pairs)
        g.insert(s, d)
    return g


def _canon(labels):
    """Relabel a component assignment as min-id-of-component."""
    labels = np.asarray(labels)
    out = np.empty(len(labels), np.uint32)
    for c in np.unique(labels):
        idx = np.nonzero(labels == c)[0]
        out[idx] = idx.min()
    return out


def test_hand_examples():
    lab, n = _g(6, [(1, 0), (2, 3), (4, 3)]).wcc()   # direction ignored: 0-1, 2-3-4, 5 alone
    assert lab.tolist() == [0, 0, 2, 2, 2, 5] and n == 3
    lab, n = _g(1, []).wcc()
    assert lab.tolist() == [0] and n == 1


@pytest.mark.parametrize("seed", range(10))
def test_vs_scipy(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(10, 400))
    m = int(rng.integers(0, 2 * n))
    s, d = rng.integers(0, n, m), rng.integers(0, n, m)
    pairs = sorted(set(zip(s.tolist(), d.tolist())))
    lab, k = _g(n, pairs).wcc()
    A = csr_matrix((np.ones(len(pairs)), ([p[0] for p in pairs], [p[1] for p in pairs])), shape=(n, n)) \
        if pairs else csr_matrix((n, n))
    kc, ref = connected_components(A, directed=True, connection="weak")
    assert k == kc and np.array_equal(lab, _canon(ref))


@pytest.mark.parametrize("seed", range(6))
def test_vs_transitive_closure(seed):
    rng = np.random.default_rng(50 + seed)
    n = 12
    pairs = sorted({(int(a), int(b)) for a, b in rng.integers(0, n, (10, 2))})
    R = np.eye(n, dtype=bool)
    for a, b in pairs:
        R[a, b] = R[b, a] = True
    for _ in range(n):
        R = R | ((R.astype(int) @ R.astype(int)) > 0)
    want = np.array([np.nonzero(R[v])[0].min() for v in range(n)], np.uint32)
    assert np.array_equal(_g(n, pairs).wcc()[0], want)


def test_incremental_merges_only():
    rng = np.random.default_rng(9)
    n = 300
    base = sorted({(int(a), int(b)) for a, b in rng.integers(0, n, (250, 2))})
    g = _g(n, base)
    before, _ = g.wcc()
    batch = sorted({(int(a), int(b)) for a, b in rng.integers(0, n, (40, 2))})
    s, d = zip(*batch)
    g.insert(s, d)
    after, _ = g.wcc()
    assert np.array_equal(after, _g(n, sorted(set(base) | set(batch))).wcc()[0])
    # insertion never splits a component and labels only decrease
    assert np.all(after <= before)
    for c in np.unique(before):
        assert len(np.unique(after[before == c])) == 1

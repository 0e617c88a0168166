"""GPU parity of dynamic triangle counting: the Count kernel
Count(G1, G2, edges), the static count and the inclusion-exclusion deltas are bit-exact (integers)
against the oracle (oracle.tc_count / tc_static / tc_delta, pinned in tests/test_oracle_tc.py)."""
import numpy as np
import pytest

import oracle
import synth
from tests.gpu_helpers import cuda

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def sym(s, d):
    """Both orientations, no self-loops, unique (an undirected graph as a directed edge set)."""
    s = np.asarray(s, np.uint64); d = np.asarray(d, np.uint64)
    k = np.unique(np.concatenate([s << np.uint64(32) | d, d << np.uint64(32) | s]))
    a, b = (k >> np.uint64(32)).astype(np.uint32), (k & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    keep = a != b
    return a[keep], b[keep]


def pair(V, s, d, weighted=False, **kw):
    from paper_2305_17813_b200 import Graph
    g = Graph(V, weighted=weighted, degree_hints=synth.degrees(s, V) if len(s) else None, **kw)
    o = oracle.OracleGraph(V, weighted=False)
    if len(s):
        g.insert(cuda(s), cuda(d), cuda(np.ones(len(s), np.uint32)) if weighted else None)
        o.insert(s, d)
    return g, o


def test_k3_and_count_orientations():
    s, d = sym([0, 1, 0], [1, 2, 2])
    g, o = pair(3, s, d)
    assert g.tc_count(g, s, d) == 6 == oracle.tc_count(o, o, s, d)
    assert g.tc_static() == 1


@pytest.mark.parametrize("weighted", [False, True])
def test_random_static_and_count(weighted):
    rng = np.random.default_rng(3)
    V = 300
    m = 4000
    s, d = sym(rng.integers(0, V, m), rng.integers(0, V, m))
    g, o = pair(V, s, d, weighted=weighted)
    assert g.tc_static() == oracle.tc_static(o)
    # Count(G1, G2, edges) with two different graphs and an arbitrary edge list
    s2, d2 = sym(rng.integers(0, V, m), rng.integers(0, V, m))
    g2, o2 = pair(V, s2, d2, weighted=not weighted)
    es, ed = rng.integers(0, V, 5000).astype(np.uint32), rng.integers(0, V, 5000).astype(np.uint32)
    assert g.tc_count(g2, cuda(es), cuda(ed)) == oracle.tc_count(o, o2, es, ed)


@pytest.mark.parametrize("scale,hashing,lf", [(14, True, 0.7), (14, False, 0.7), (13, True, 0.05)])
def test_rmat_dynamic(scale, hashing, lf):
    """R-MAT (hubs with many slab lists, chained pool slabs at lf 0.05): static count, then an
    inserted and a deleted batch: deltas equal the oracle's and the static difference."""
    rs, rd, _ = synth.rmat(scale, 8)
    s, d = sym(rs, rd)
    V = 1 << scale
    key = (s.astype(np.uint64) << np.uint64(32)) | d
    rng = np.random.default_rng(scale)
    # hold out 2000 undirected edges as the insert batch
    und = np.nonzero(s < d)[0]
    held = rng.choice(und, 2000, replace=False)
    hs, hd = sym(s[held], d[held])
    hk = (hs.astype(np.uint64) << np.uint64(32)) | hd
    base = ~np.isin(key, hk)
    g, o = pair(V, s[base], d[base], hashing=hashing, load_factor=lf)
    t0 = g.tc_static()
    assert t0 == oracle.tc_static(o)
    g.insert(cuda(hs), cuda(hd))
    o.insert(hs, hd)
    gu, ou = pair(V, hs, hd)
    added, S = g.tc_delta(gu, cuda(hs), cuda(hd), insert=True)
    oadded, oS = oracle.tc_delta(o, ou, hs, hd, True)
    assert (added, S) == (oadded, oS)
    t1 = g.tc_static()
    assert t1 == oracle.tc_static(o) == t0 + added
    # delete 1500 undirected edges
    und2 = np.nonzero(s < d)[0]
    dl = rng.choice(und2, 1500, replace=False)
    ds, dd = sym(s[dl], d[dl])
    g.delete(cuda(ds), cuda(dd))
    o.delete(ds, dd)
    gd, od = pair(V, ds, dd)
    removed, S = g.tc_delta(gd, cuda(ds), cuda(dd), insert=False)
    assert (removed, S) == oracle.tc_delta(o, od, ds, dd, False)
    assert g.tc_static() == t1 - removed

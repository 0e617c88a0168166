"""Degenerate inputs on the GPU path: empty batches for every batch call, a graph with no edges,
a single vertex, and the source with no out-edges — results equal the oracle's."""
import numpy as np
import pytest

import oracle
import synth
from tests.gpu_helpers import cuda

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
E = np.zeros(0, np.uint32)


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def G(*a, **k):
    from paper_2305_17813_b200 import Graph
    return Graph(*a, **k)


def test_empty_batches_everywhere():
    V = 1024
    s, d, w = synth.uniform(V, 8192)
    g = G(V, degree_hints=synth.degrees(s, V), reverse=True, in_degree_hints=synth.degrees(d, V))
    g.insert(cuda(s), cuda(d), cuda(w))
    o = oracle.OracleGraph(V)
    o.insert(s, d, w)
    sp, bf = g.sssp(0), g.bfs(0)
    pr = g.pagerank()
    c = g.wcc()
    assert g.insert(E, E, E) == 0
    g.trees_incremental([sp, bf], E, E, E)
    c.incremental(E, E)   # incremental WCC follows an insert batch (there is no decremental WCC)
    assert g.delete(E, E) == 0
    g.trees_decremental([sp, bf], E, E)
    f, qw = g.query(E, E)
    assert len(f) == 0
    pr.update()
    assert pr.stats()["iterations"] == 1   # one verification super-step
    assert np.array_equal(sp.nodes(), o.sssp(0)[1]) and np.array_equal(bf.nodes(), o.bfs(0)[1])
    assert np.array_equal(c.labels(), o.wcc()[0])
    assert g.tc_count(g, E, E) == 0


def test_no_edges_and_single_vertex():
    g = G(64)
    t = g.sssp(5)
    node = t.nodes()
    want = np.full(64, oracle.UNREACHED, np.uint64)
    want[5] = 5
    assert np.array_equal(node, want)
    assert g.wcc().components() == 64
    g1 = G(1, reverse=True)
    assert abs(g1.pagerank().values()[0] - 1.0) < 1e-15
    assert g1.sssp(0).nodes().tolist() == [0]


def test_source_without_out_edges():
    V = 256
    rng = np.random.default_rng(3)
    s, d = rng.integers(1, V, 1500).astype(np.uint32), rng.integers(0, V, 1500).astype(np.uint32)
    keep = s != d
    s, d = s[keep], d[keep]
    w = rng.integers(1, 65, len(s)).astype(np.uint32)
    g = G(V, degree_hints=synth.degrees(s, V))
    g.insert(cuda(s), cuda(d), cuda(w))
    o = oracle.OracleGraph(V)
    o.insert(s, d, w)
    t = g.sssp(0)   # vertex 0 has in-edges only
    assert np.array_equal(t.nodes(), o.sssp(0)[1])
    bs, bd, bw = np.array([0], np.uint32), np.array([7], np.uint32), np.array([3], np.uint32)
    g.insert(cuda(bs), cuda(bd), cuda(bw)); o.insert(bs, bd, bw)
    t.incremental(cuda(bs), cuda(bd), cuda(bw))
    assert np.array_equal(t.nodes(), o.sssp(0)[1])
    g.delete(cuda(bs), cuda(bd)); o.delete(bs, bd)
    t.decremental(cuda(bs), cuda(bd))
    assert np.array_equal(t.nodes(), o.sssp(0)[1])

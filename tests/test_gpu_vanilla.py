"""GPU parity of the paper's VANILLA static SSSP / BFS (distances
only, 32-bit atomics) against the oracle's distances (the high halves of its packed nodes,
oracle/meerkat_oracle.c orc_sssp / orc_bfs), bit-exact; and meerkat_tree_distances of the
tree-based variant."""
import json
import os

import numpy as np
import pytest

import oracle
import synth
from tests.gpu_helpers import cuda

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
INF = np.uint32(0xFFFFFFFF)


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def G(*a, **k):
    from paper_2305_17813_b200 import Graph
    return Graph(*a, **k)


def dist_of(node):
    node = np.asarray(node, np.uint64)
    return np.where(node == oracle.UNREACHED, INF, (node >> np.uint64(32)).astype(np.uint32)).astype(np.uint32)


def test_golden_g0(golden_dir):
    J = json.load(open(os.path.join(golden_dir, "g0.json")))
    n, src = J["vertex_n"], J["source"]
    s, d, w = (np.array(c, np.uint32) for c in zip(*J["edges"]))
    g = G(n, degree_hints=synth.degrees(s, n))
    g.insert(s, d, w)
    want_s = np.array([INF if r is None else r[0] for r in J["static_sssp"]], np.uint32)
    want_b = np.array([INF if r is None else r[0] for r in J["static_bfs"]], np.uint32)
    assert np.array_equal(g.sssp_vanilla(src).distances(), want_s)
    assert np.array_equal(g.bfs_vanilla(src).distances(), want_b)
    assert np.array_equal(g.sssp(src).distances(), want_s)
    assert np.array_equal(g.bfs(src).distances(), want_b)


@pytest.mark.parametrize("scale,hashing", [(16, True), (16, False)])
def test_rmat_vanilla_vs_oracle(scale, hashing):
    W = synth.rmat_dynamic(scale, 16, batch=5000, n_ins=1, n_del=1)
    s, d, w = W.base
    V = W.vertex_n
    g = G(V, hashing=hashing, degree_hints=synth.degrees(s, V))
    g.insert(cuda(s), cuda(d), cuda(w))
    o = oracle.OracleGraph(V)
    o.insert(s, d, w)
    vs, vb = g.sssp_vanilla(W.source), g.bfs_vanilla(W.source)
    assert np.array_equal(vs.distances(), dist_of(o.sssp(W.source)[1]))
    assert np.array_equal(vb.distances(), dist_of(o.bfs(W.source)[1]))
    # static only: no dependence tree for the dynamic algorithms
    from paper_2305_17813_b200 import MeerkatError
    (is_, id_, iw), (ds, dd, _) = W.inserts[0], W.deletes[0]
    g.insert(cuda(is_), cuda(id_), cuda(iw))
    with pytest.raises(MeerkatError):
        vs.incremental(cuda(is_), cuda(id_), cuda(iw))
    with pytest.raises(MeerkatError):
        vs.nodes()
    g.delete(cuda(ds), cuda(dd))
    o.insert(is_, id_, iw)
    o.delete(ds, dd)
    vs.recompute(); vb.recompute()
    assert np.array_equal(vs.distances(), dist_of(o.sssp(W.source)[1]))
    assert np.array_equal(vb.distances(), dist_of(o.bfs(W.source)[1]))


def test_unweighted_store_vanilla_bfs():
    s, d, _ = synth.uniform(1024, 8192)
    g = G(1024, weighted=False, degree_hints=synth.degrees(s, 1024))
    g.insert(cuda(s), cuda(d))
    o = oracle.OracleGraph(1024, weighted=False)
    o.insert(s, d)
    assert np.array_equal(g.bfs_vanilla(0).distances(), dist_of(o.bfs(0)[1]))


@pytest.mark.parametrize("hashing", [True, False])
def test_iteration_scheme1_static_equals_scheme2(hashing):
    """The paper's IterationScheme1 (one work item per vertex, its buckets walked in turn by one
    group) gives the same static trees / distances as the <vertex, bucket> items."""
    W = synth.rmat_dynamic(15, 16, batch=1000, n_ins=1, n_del=0)
    s, d, w = W.base
    V = W.vertex_n
    g = G(V, hashing=hashing, degree_hints=synth.degrees(s, V))
    g.insert(cuda(s), cuda(d), cuda(w))
    o = oracle.OracleGraph(V)
    o.insert(s, d, w)
    for mk, ref in ((g.sssp, o.sssp(W.source)[1]), (g.bfs, o.bfs(W.source)[1])):
        t = mk(W.source)
        t.recompute(iteration_scheme=1)
        assert np.array_equal(t.nodes(), ref)
        t.recompute(iteration_scheme=2)
        assert np.array_equal(t.nodes(), ref)
    vt = g.sssp_vanilla(W.source)
    vt.recompute(iteration_scheme=1)
    assert np.array_equal(vt.distances(), dist_of(o.sssp(W.source)[1]))

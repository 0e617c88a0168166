"""Parity at BASELINE config 3's full size (R-MAT scale 24, ~263 M edges, 100 K-edge batches) in
bench.py's launch configuration.  A from-scratch Dijkstra per check would take minutes, so every
tree is verified by the oracle's certificate check (oracle.check_tree: the Bellman equations with
the packed-min parent have exactly one solution when every w >= 1), which covers ALL vertices;
the edge count and a sample of query answers are compared with the oracle's edge set, and the
decremental invalidated set with oracle.invalidated() on the previous (certified) tree."""
import numpy as np
import pytest

import oracle
import synth
from tests.gpu_helpers import cuda

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def workload():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    W = synth.rmat_dynamic(24, 16, batch=100_000, n_ins=1, n_del=1)
    o = oracle.OracleGraph(W.vertex_n)
    o.insert(*W.base)
    return W, o


@pytest.mark.parametrize("reverse", [True, False])
def test_config3_fullsize_certified(workload, reverse):
    from paper_2305_17813_b200 import Graph
    W, o0 = workload
    V, src = W.vertex_n, W.source
    bs, bd, bw = W.base
    g = Graph(V, weighted=True, degree_hints=cuda(np.bincount(bs, minlength=V).astype(np.uint32)),
              reverse=reverse, in_degree_hints=cuda(np.bincount(bd, minlength=V).astype(np.uint32)) if reverse else None)
    assert g.insert(cuda(bs), cuda(bd), cuda(bw)) == o0.num_edges
    t, b = g.sssp(src), g.bfs(src)
    for tree, unit in ((t, False), (b, True)):
        assert o0.check_tree(src, tree.nodes(), unit) == (0, 0xFFFFFFFF)
    # one incremental batch (oracle graph copy advanced alongside)
    o = oracle.OracleGraph(V)
    o.insert(*o0.edges())
    s, d, w = W.inserts[0]
    assert g.insert(cuda(s), cuda(d), cuda(w)) == o.insert(s, d, w)[1]
    t.incremental(cuda(s), cuda(d), cuda(w))
    b.incremental(cuda(s), cuda(d))
    for tree, unit in ((t, False), (b, True)):
        assert o.check_tree(src, tree.nodes(), unit) == (0, 0xFFFFFFFF)
    old_t = t.nodes()
    s, d, _ = W.deletes[0]
    assert g.delete(cuda(s), cuda(d)) == o.delete(s, d)[1]
    t.decremental(cuda(s), cuda(d))
    b.decremental(cuda(s), cuda(d))
    flag, nd = oracle.invalidated(V, src, old_t, s, d)
    st = t.stats()
    assert st["invalidated"] == int(flag.sum()) and st["direct_invalid"] == nd
    assert st["frontier_edges"] == o.dec_frontier_count(old_t, flag)
    for tree, unit in ((t, False), (b, True)):
        assert o.check_tree(src, tree.nodes(), unit) == (0, 0xFFFFFFFF)
    assert g.stats()["edges"] == o.num_edges
    rng = np.random.default_rng(0)
    es, ed, ew = o.edges()
    pick = rng.choice(len(es), 200_000, replace=False)
    qs = np.concatenate([es[pick], rng.integers(0, V, 200_000)]).astype(np.uint32)
    qd = np.concatenate([ed[pick], rng.integers(0, V, 200_000)]).astype(np.uint32)
    f, qw = g.query(cuda(qs), cuda(qd))
    _, ef, eww = o.query(qs, qd)
    assert np.array_equal(f.cpu().numpy(), ef) and np.array_equal(qw.cpu().numpy().view(np.uint32), eww)
    assert g.check()[0] == 0
    g.close()


def test_config4_mixed_batches_certified():
    """BASELINE config 4: power-law R-MAT scale 22, edge factor 24 (~97 M edges, 'LJ/Orkut-shaped'),
    dynamic SSSP + BFS under mixed batches: each round deletes 1% of E then inserts 1% held-out edges
    (SURVEY §8(c) C25); two rounds here, every tree certified by the oracle after every batch."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2305_17813_b200 import Graph
    n1 = 970_000
    W = synth.rmat_dynamic(22, 24, batch=n1, n_ins=2, n_del=2)
    V, src = W.vertex_n, W.source
    bs, bd, bw = W.base
    o = oracle.OracleGraph(V)
    o.insert(bs, bd, bw)
    g = Graph(V, weighted=True, degree_hints=cuda(np.bincount(bs, minlength=V).astype(np.uint32)), reverse=True,
              in_degree_hints=cuda(np.bincount(bd, minlength=V).astype(np.uint32)))
    assert g.insert(cuda(bs), cuda(bd), cuda(bw)) == o.num_edges
    t, b = g.sssp(src), g.bfs(src)
    for r in range(2):
        s, d, _ = W.deletes[r]
        assert g.delete(cuda(s), cuda(d)) == o.delete(s, d)[1]
        t.decremental(cuda(s), cuda(d))
        b.decremental(cuda(s), cuda(d))
        assert o.check_tree(src, t.nodes(), False) == (0, 0xFFFFFFFF)
        assert o.check_tree(src, b.nodes(), True) == (0, 0xFFFFFFFF)
        s, d, w = W.inserts[r]
        assert g.insert(cuda(s), cuda(d), cuda(w)) == o.insert(s, d, w)[1]
        t.incremental(cuda(s), cuda(d), cuda(w))
        b.incremental(cuda(s), cuda(d))
        assert o.check_tree(src, t.nodes(), False) == (0, 0xFFFFFFFF)
        assert o.check_tree(src, b.nodes(), True) == (0, 0xFFFFFFFF)
    assert g.check()[0] == 0 and g.stats()["edges"] == o.num_edges
    g.close()

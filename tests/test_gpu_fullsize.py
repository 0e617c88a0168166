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
    W = synth.rmat_dynamic(24, 16, batch=100_000, n_ins=2, n_del=2)
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


def _tree_checks(o, src, old_nodes, t, b, s, d):
    """Decremental intermediates of both trees of a fused call vs the oracle on the old trees."""
    V = o.V
    for tree, old in ((t, old_nodes[0]), (b, old_nodes[1])):
        flag, nd = oracle.invalidated(V, src, old, s, d)
        st = tree.stats()
        assert st["invalidated"] == int(flag.sum()) and st["direct_invalid"] == nd
        assert st["frontier_edges"] == o.dec_frontier_count(old, flag)


def test_config3_bench_sequence_certified(workload):
    """The exact sequence bench.py times, at BASELINE config 3's full size: in-edge mirror, seeded
    insert (the trees' prologue inside the insert kernel) -> fused trees_incremental -> seeded delete
    -> fused trees_decremental, two batch pairs.  Every tree is certified after every batch, and the
    decremental intermediates of BOTH trees (invalidated set, direct count, valid->invalid frontier)
    are compared with the oracle's on the previous trees."""
    from paper_2305_17813_b200 import Graph
    W, o0 = workload
    V, src = W.vertex_n, W.source
    bs, bd, bw = W.base
    g = Graph(V, weighted=True, load_factor=0.5,   # bench.py's default load factor
              degree_hints=cuda(np.bincount(bs, minlength=V).astype(np.uint32)), reverse=True,
              in_degree_hints=cuda(np.bincount(bd, minlength=V).astype(np.uint32)))
    g.insert(cuda(bs), cuda(bd), cuda(bw), count=False)
    o = oracle.OracleGraph(V)
    o.insert(*o0.edges())
    t, b = g.sssp(src), g.bfs(src)
    for k in range(2):
        s, d, w = (cuda(x) for x in W.inserts[k])
        g.insert(s, d, w, count=False, seed=[t, b])
        g.trees_incremental([t, b], s, d, w)
        o.insert(*W.inserts[k])
        old = (t.nodes(), b.nodes())
        assert o.check_tree(src, old[0], False) == (0, 0xFFFFFFFF), f"sssp after insert {k}"
        assert o.check_tree(src, old[1], True) == (0, 0xFFFFFFFF), f"bfs after insert {k}"
        ds, dd = (cuda(x) for x in W.deletes[k][:2])
        g.delete(ds, dd, count=False, seed=[t, b])
        g.trees_decremental([t, b], ds, dd)
        o.delete(W.deletes[k][0], W.deletes[k][1])
        _tree_checks(o, src, old, t, b, W.deletes[k][0], W.deletes[k][1])
        assert o.check_tree(src, t.nodes(), False) == (0, 0xFFFFFFFF), f"sssp after delete {k}"
        assert o.check_tree(src, b.nodes(), True) == (0, 0xFFFFFFFF), f"bfs after delete {k}"
    g.sync()
    assert g.stats()["edges"] == o.num_edges and g.check()[0] == 0
    g.close()


def test_10m_edge_batches_certified():
    """north_star's upper batch size: 10 M-edge insert and delete batches (the thread-per-edge update
    kernels, with the trees' prologue seeded inside them) on R-MAT scale 23 (~130 M edges), mirror on,
    fused SSSP + BFS; counts vs the oracle, trees certified, decremental intermediates vs the oracle,
    a 1 M query sample element by element."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2305_17813_b200 import Graph
    n = 10_000_000
    W = synth.rmat_dynamic(23, 16, batch=n, n_ins=1, n_del=1)
    V, src = W.vertex_n, W.source
    bs, bd, bw = W.base
    o = oracle.OracleGraph(V)
    o.insert(bs, bd, bw)
    g = Graph(V, weighted=True, degree_hints=cuda(np.bincount(bs, minlength=V).astype(np.uint32)), reverse=True,
              in_degree_hints=cuda(np.bincount(bd, minlength=V).astype(np.uint32)))
    assert g.insert(cuda(bs), cuda(bd), cuda(bw)) == o.num_edges
    t, b = g.sssp(src), g.bfs(src)
    s, d, w = (cuda(x) for x in W.inserts[0])
    assert g.insert(s, d, w, seed=[t, b]) == o.insert(*W.inserts[0])[1]
    g.trees_incremental([t, b], s, d, w)
    old = (t.nodes(), b.nodes())
    assert o.check_tree(src, old[0], False) == (0, 0xFFFFFFFF)
    assert o.check_tree(src, old[1], True) == (0, 0xFFFFFFFF)
    ds, dd = (cuda(x) for x in W.deletes[0][:2])
    assert g.delete(ds, dd, seed=[t, b]) == o.delete(W.deletes[0][0], W.deletes[0][1])[1]
    g.trees_decremental([t, b], ds, dd)
    _tree_checks(o, src, old, t, b, W.deletes[0][0], W.deletes[0][1])
    assert o.check_tree(src, t.nodes(), False) == (0, 0xFFFFFFFF)
    assert o.check_tree(src, b.nodes(), True) == (0, 0xFFFFFFFF)
    rng = np.random.default_rng(1)
    es, ed, ew = o.edges()
    pick = rng.choice(len(es), 500_000, replace=False)
    qs = np.concatenate([es[pick], rng.integers(0, V, 500_000)]).astype(np.uint32)
    qd = np.concatenate([ed[pick], rng.integers(0, V, 500_000)]).astype(np.uint32)
    f, qw = g.query(cuda(qs), cuda(qd))
    _, ef, eww = o.query(qs, qd)
    assert np.array_equal(f.cpu().numpy(), ef) and np.array_equal(qw.cpu().numpy().view(np.uint32), eww)
    assert g.stats()["edges"] == o.num_edges and g.check()[0] == 0
    g.close()

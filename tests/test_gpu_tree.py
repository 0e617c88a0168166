"""GPU parity of batch-dynamic SSSP / BFS against the CPU oracle:
packed <distance, parent> nodes must be bit-exact after every batch; the
decremental intermediates (invalidated set P:144-154, valid->invalid frontier
P:156-164) must equal the oracle's."""
import json
import os

import numpy as np
import pytest

import oracle
import synth
from tests.gpu_helpers import assert_nodes, assert_same_edges, cuda

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def G(*a, **k):
    from paper_2305_17813_b200 import Graph
    return Graph(*a, **k)


def test_golden_g0(golden_dir):
    J = json.load(open(os.path.join(golden_dir, "g0.json")))
    n, src = J["vertex_n"], J["source"]
    s, d, w = (np.array(c, np.uint32) for c in zip(*J["edges"]))
    g = G(n, weighted=True, degree_hints=synth.degrees(s, n))
    g.insert(s, d, w)
    t = g.sssp(src)
    b = g.bfs(src)
    pk = lambda rows: np.array([oracle.UNREACHED if r is None else oracle.pack(*r) for r in rows], np.uint64)
    assert_nodes(t.nodes(), pk(J["static_sssp"]), "static sssp")
    assert_nodes(b.nodes(), pk(J["static_bfs"]), "static bfs")
    o = oracle.OracleGraph(n)
    o.insert(s, d, w)
    for step in J["steps"]:
        es = np.array(step["edges"], np.uint32)
        if step["op"] == "delete":
            g.delete(es[:, 0], es[:, 1])
            o.delete(es[:, 0], es[:, 1])
            t.decremental(es[:, 0], es[:, 1])
            b.decremental(es[:, 0], es[:, 1])
            assert t.invalidated().tolist() == step["invalid"]
            assert t.stats()["frontier_edges"] == len(step["frontier"])
        else:
            g.insert(es[:, 0], es[:, 1], es[:, 2])
            o.insert(es[:, 0], es[:, 1], es[:, 2])
            t.incremental(es[:, 0], es[:, 1], es[:, 2])
            b.incremental(es[:, 0], es[:, 1])
        assert_nodes(t.nodes(), pk(step["sssp"]), step["note"])
        assert_nodes(b.nodes(), o.bfs(src)[1], "bfs " + step["note"])


def _config1_batches(rng, o, V, src, kind):
    """inserts = 56 new + 8 re-inserts with random w;
    deletes = 32 current SSSP-tree edges + 28 random present + 4 absent."""
    es, ed, ew = o.edges()
    if kind == "insert":
        present = set(zip(es.tolist(), ed.tolist()))
        new = []
        while len(new) < 56:
            u, v = int(rng.integers(V)), int(rng.integers(V))
            if u != v and (u, v) not in present:
                new.append((u, v)); present.add((u, v))
        pick = rng.choice(len(es), 8, replace=False)
        re = [(int(es[i]), int(ed[i])) for i in pick]
        pairs = new + re
        w = rng.integers(1, 65, len(pairs)).astype(np.uint32)
        s, d = (np.array(c, np.uint32) for c in zip(*pairs))
        return s, d, w
    _, node = o.sssp(src)
    par = (node & np.uint64(0xFFFFFFFF)).astype(np.int64)
    tree = [(int(par[v]), v) for v in range(V) if v != src and node[v] != oracle.UNREACHED]
    tsel = [tree[i] for i in rng.choice(len(tree), min(32, len(tree)), replace=False)]
    others = [(int(es[i]), int(ed[i])) for i in rng.choice(len(es), 28, replace=False)]
    absent = []
    present = set(zip(es.tolist(), ed.tolist()))
    while len(absent) < 4:
        u, v = int(rng.integers(V)), int(rng.integers(V))
        if (u, v) not in present:
            absent.append((u, v))
    pairs = tsel + others + absent
    s, d = (np.array(c, np.uint32) for c in zip(*pairs))
    return s, d, None


@pytest.mark.parametrize("hashing,reverse", [(True, False), (False, False), (True, True)])
def test_config1_dynamic_sssp_bfs(hashing, reverse):
    """BASELINE config 1: 1K vertices / 8K edges, 4 insert + 4 delete batches of 64, SSSP + BFS from 0."""
    V, src = 1024, 0
    s, d, w = synth.uniform(V, 8192)
    g = G(V, weighted=True, hashing=hashing, degree_hints=synth.degrees(s, V), reverse=reverse,
          in_degree_hints=synth.degrees(d, V))
    o = oracle.OracleGraph(V)
    assert g.insert(cuda(s), cuda(d), cuda(w)) == o.insert(s, d, w)[1]
    t, b = g.sssp(src), g.bfs(src)
    assert_nodes(t.nodes(), o.sssp(src)[1], "static sssp")
    assert_nodes(b.nodes(), o.bfs(src)[1], "static bfs")
    rng = np.random.default_rng(3)
    for step in range(8):
        kind = "insert" if step < 4 else "delete"
        bs, bd, bw = _config1_batches(rng, o, V, src, kind)
        old_s, old_b = o.sssp(src)[1], o.bfs(src)[1]
        if kind == "insert":
            assert g.insert(cuda(bs), cuda(bd), cuda(bw)) == o.insert(bs, bd, bw)[1]
            t.incremental(cuda(bs), cuda(bd), cuda(bw))
            b.incremental(cuda(bs), cuda(bd))
        else:
            assert g.delete(cuda(bs), cuda(bd)) == o.delete(bs, bd)[1]
            t.decremental(cuda(bs), cuda(bd))
            b.decremental(cuda(bs), cuda(bd))
            for tree, old in ((t, old_s), (b, old_b)):
                flag, ndirect = oracle.invalidated(V, src, old, bs, bd)
                st = tree.stats()
                assert tree.invalidated().tolist() == np.nonzero(flag)[0].tolist()
                assert st["direct_invalid"] == ndirect
                assert st["frontier_edges"] == o.dec_frontier_count(old, flag)
        assert_nodes(t.nodes(), o.sssp(src)[1], f"sssp step {step}")
        assert_nodes(b.nodes(), o.bfs(src)[1], f"bfs step {step}")
    assert_same_edges(g, o)


@pytest.mark.parametrize("scale,hashing,lf,reverse", [(14, True, 0.7, False), (14, False, 0.7, False),
                                                       (16, True, 0.5, False), (17, True, 1.0, False),
                                                       (14, True, 0.7, True), (16, False, 0.7, True),
                                                       (17, True, 0.7, True)])
def test_rmat_dynamic_vs_oracle(scale, hashing, lf, reverse):
    """R-MAT (SURVEY §8(d) generator) with held-out inserts and sampled deletes; both trees
    bit-exact after every batch; several tiles, hub vertices, chained slabs; with and
    without the in-edge mirror (decremental frontier by scan vs by in-edges)."""
    W = synth.rmat_dynamic(scale, 16, batch=1000 if scale < 16 else 5000, n_ins=3, n_del=3)
    V, src = W.vertex_n, W.source
    bs, bd, bw = W.base
    g = G(V, weighted=True, hashing=hashing, load_factor=lf, degree_hints=synth.degrees(bs, V), reverse=reverse,
          in_degree_hints=synth.degrees(bd, V))
    o = oracle.OracleGraph(V)
    assert g.insert(cuda(bs), cuda(bd), cuda(bw)) == o.insert(bs, bd, bw)[1]
    t, b = g.sssp(src), g.bfs(src)
    assert_nodes(t.nodes(), o.sssp(src)[1], "static sssp")
    assert_nodes(b.nodes(), o.bfs(src)[1], "static bfs")
    for (s, d, w) in W.inserts:
        assert g.insert(cuda(s), cuda(d), cuda(w)) == o.insert(s, d, w)[1]
        t.incremental(cuda(s), cuda(d), cuda(w))
        b.incremental(cuda(s), cuda(d))
        assert_nodes(t.nodes(), o.sssp(src)[1], "inc sssp")
        assert_nodes(b.nodes(), o.bfs(src)[1], "inc bfs")
    for (s, d, _w) in W.deletes:
        old = o.sssp(src)[1]
        assert g.delete(cuda(s), cuda(d)) == o.delete(s, d)[1]
        t.decremental(cuda(s), cuda(d))
        b.decremental(cuda(s), cuda(d))
        flag, _ = oracle.invalidated(V, src, old, s, d)
        assert t.stats()["invalidated"] == int(flag.sum())
        assert_nodes(t.nodes(), o.sssp(src)[1], "dec sssp")
        assert_nodes(b.nodes(), o.bfs(src)[1], "dec bfs")
    t.recompute()
    assert_nodes(t.nodes(), o.sssp(src)[1], "recompute")
    assert_same_edges(g, o)


def test_unweighted_graph_bfs_and_sssp_rejected():
    from paper_2305_17813_b200 import MeerkatError
    V = 3000
    s, d, _ = synth.uniform(V, 20000, seed_graph=9)
    g = G(V, weighted=False, degree_hints=synth.degrees(s, V), reverse=True)
    o = oracle.OracleGraph(V, weighted=False)
    assert g.insert(s, d) == o.insert(s, d)[1]
    with pytest.raises(MeerkatError):
        g.sssp(0)
    b = g.bfs(5)
    assert_nodes(b.nodes(), o.bfs(5)[1], "static bfs set store")
    rng = np.random.default_rng(0)
    for _ in range(3):
        es, ed, _ = o.edges()
        pick = rng.choice(len(es), 700, replace=False)
        g.delete(es[pick], ed[pick]); o.delete(es[pick], ed[pick])
        b.decremental(es[pick], ed[pick])
        assert_nodes(b.nodes(), o.bfs(5)[1], "dec bfs set store")
        ns = rng.integers(0, V, 500).astype(np.uint32); nd = rng.integers(0, V, 500).astype(np.uint32)
        g.insert(ns, nd); o.insert(ns, nd)
        b.incremental(ns, nd)
        assert_nodes(b.nodes(), o.bfs(5)[1], "inc bfs set store")


def test_ordering_contract_and_edge_cases():
    from paper_2305_17813_b200 import MeerkatError, _lib
    V = 200
    s, d, w = synth.uniform(V, 1500, seed_graph=4)
    g = G(V, weighted=True)
    o = oracle.OracleGraph(V)
    g.insert(s, d, w); o.insert(s, d, w)
    t = g.sssp(199)
    # an update without a matching mutation is refused
    with pytest.raises(MeerkatError) as e:
        t.incremental(s[:1], d[:1], w[:1])
    assert e.value.status == _lib.E_STATE
    # empty batches
    g.insert(s[:0], d[:0], w[:0]); t.incremental(s[:0], d[:0], w[:0])
    g.delete(s[:0], d[:0]); t.decremental(s[:0], d[:0])
    assert_nodes(t.nodes(), o.sssp(199)[1], "empty batches")
    # a mutation not followed by its tree update makes the next one a version mismatch
    g.insert(s[:3], d[:3], w[:3]); o.insert(s[:3], d[:3], w[:3])
    g.delete(s[:3], d[:3]); o.delete(s[:3], d[:3])
    with pytest.raises(MeerkatError):
        t.decremental(s[:3], d[:3])
    t.recompute()
    assert_nodes(t.nodes(), o.sssp(199)[1], "recompute after contract break")
    # self-loops and deletion of the source's own self-loop never invalidate SRC (C4, C12)
    g.insert(np.array([199], np.uint32), np.array([199], np.uint32), np.array([3], np.uint32))
    o.insert(np.array([199], np.uint32), np.array([199], np.uint32), np.array([3], np.uint32))
    t.incremental(np.array([199], np.uint32), np.array([199], np.uint32), np.array([3], np.uint32))
    g.delete(np.array([199], np.uint32), np.array([199], np.uint32))
    o.delete(np.array([199], np.uint32), np.array([199], np.uint32))
    t.decremental(np.array([199], np.uint32), np.array([199], np.uint32))
    assert_nodes(t.nodes(), o.sssp(199)[1], "self loop")


def test_overflow_reported():
    from paper_2305_17813_b200 import MeerkatError, _lib
    big = (1 << 31) - 1
    g = G(4, weighted=True)
    g.insert(np.array([0, 1, 2], np.uint32), np.array([1, 2, 3], np.uint32), np.full(3, big, np.uint32))
    t = g.sssp(0)
    with pytest.raises(MeerkatError) as e:
        g.sync()
    assert e.value.status == _lib.E_OVERFLOW


@pytest.mark.parametrize("reverse,hashing", [(False, True), (True, True), (False, False)])
def test_fused_trees_match_oracle(reverse, hashing):
    """meerkat_trees_incremental / _decremental: SSSP and BFS trees updated by ONE launch (shared
    round barriers, one slab-array stream for both) give the same nodes and intermediates."""
    W = synth.rmat_dynamic(15, 16, batch=2000, n_ins=3, n_del=3)
    V, src = W.vertex_n, W.source
    bs, bd, bw = W.base
    g = G(V, weighted=True, hashing=hashing, degree_hints=synth.degrees(bs, V), reverse=reverse,
          in_degree_hints=synth.degrees(bd, V))
    o = oracle.OracleGraph(V)
    g.insert(cuda(bs), cuda(bd), cuda(bw)); o.insert(bs, bd, bw)
    t, b = g.sssp(src), g.bfs(src)
    for (s, d, w) in W.inserts:
        g.insert(cuda(s), cuda(d), cuda(w)); o.insert(s, d, w)
        g.trees_incremental([t, b], cuda(s), cuda(d), cuda(w))
        assert_nodes(t.nodes(), o.sssp(src)[1], "fused inc sssp")
        assert_nodes(b.nodes(), o.bfs(src)[1], "fused inc bfs")
    for (s, d, _w) in W.deletes:
        old_s, old_b = o.sssp(src)[1], o.bfs(src)[1]
        g.delete(cuda(s), cuda(d)); o.delete(s, d)
        g.trees_decremental([t, b], cuda(s), cuda(d))
        for tree, old in ((t, old_s), (b, old_b)):
            flag, nd = oracle.invalidated(V, src, old, s, d)
            st = tree.stats()
            assert tree.invalidated().tolist() == np.nonzero(flag)[0].tolist()
            assert st["direct_invalid"] == nd
            assert st["frontier_edges"] == o.dec_frontier_count(old, flag)
        assert_nodes(t.nodes(), o.sssp(src)[1], "fused dec sssp")
        assert_nodes(b.nodes(), o.bfs(src)[1], "fused dec bfs")
    # mixing per-tree and fused calls keeps the version contract
    s, d, w = W.inserts[0]
    g.delete(cuda(s), cuda(d)); o.delete(s, d)
    t.decremental(cuda(s), cuda(d))
    b.decremental(cuda(s), cuda(d))
    assert_nodes(t.nodes(), o.sssp(src)[1], "per-tree after fused")


def test_host_batches_staged_once_and_reused():
    """Host (numpy) batches: the tree calls that follow a mutation with the SAME host arrays reuse
    the mutation's staged device copy (api.cu stage_in_reuse); equal arrays at other addresses are
    staged again.  Both paths must give the oracle's trees (fused and per-tree calls)."""
    V = 1024
    s, d, w = synth.uniform(V, 8192)
    g = G(V, weighted=True, degree_hints=synth.degrees(s, V), reverse=True, in_degree_hints=synth.degrees(d, V))
    g.insert(s, d, w)
    o = oracle.OracleGraph(V)
    o.insert(s, d, w)
    sp, bf = g.sssp(0), g.bfs(0)
    rng = np.random.default_rng(21)
    for step in range(6):
        if step % 2 == 0:
            bs = rng.integers(0, V, 200).astype(np.uint32); bd = rng.integers(0, V, 200).astype(np.uint32)
            bw = rng.integers(1, 65, 200).astype(np.uint32)
            g.insert(bs, bd, bw)
            o.insert(bs, bd, bw)
            if step == 2:   # copies at other addresses: staged again
                sp.incremental(bs.copy(), bd.copy(), bw.copy()); bf.incremental(bs.copy(), bd.copy())
            else:
                g.trees_incremental([sp, bf], bs, bd, bw)
        else:
            es, ed, _ = o.edges()
            pick = rng.choice(len(es), 150, replace=False)
            bs, bd = es[pick].copy(), ed[pick].copy()
            g.delete(bs, bd)
            o.delete(bs, bd)
            if step == 3:
                sp.decremental(bs, bd); bf.decremental(bs, bd)
            else:
                g.trees_decremental([sp, bf], bs, bd)
        assert_nodes(sp.nodes(), o.sssp(0)[1], f"sssp step {step}")
        assert_nodes(bf.nodes(), o.bfs(0)[1], f"bfs step {step}")


@pytest.mark.parametrize("reverse,hashing,thread", [(False, True, "0"), (True, True, "0"), (True, True, "1"),
                                                    (False, False, "1")])
def test_batch_trees_match_oracle(reverse, hashing, thread, monkeypatch):
    """meerkat_insert_batch_trees / meerkat_delete_batch_trees: the trees' batch prologue runs
    inside the insert / delete kernel (both kernel kinds); nodes, invalidated sets, direct counts
    and frontier sizes must equal the oracle's, and the mutation counts insert / delete's."""
    monkeypatch.setenv("MEERKAT_THREAD_UPD", thread)
    W = synth.rmat_dynamic(15, 16, batch=2000, n_ins=3, n_del=3)
    V, src = W.vertex_n, W.source
    bs, bd, bw = W.base
    g = G(V, weighted=True, hashing=hashing, degree_hints=synth.degrees(bs, V), reverse=reverse,
          in_degree_hints=synth.degrees(bd, V))
    o = oracle.OracleGraph(V)
    g.insert(cuda(bs), cuda(bd), cuda(bw)); o.insert(bs, bd, bw)
    t, b = g.sssp(src), g.bfs(src)
    for (s, d, w) in W.inserts:
        before = len(o.edges()[0])
        o.insert(s, d, w)
        n_ins = g.insert_trees([t, b], cuda(s), cuda(d), cuda(w))
        assert n_ins == len(o.edges()[0]) - before
        assert_nodes(t.nodes(), o.sssp(src)[1], "batch_trees inc sssp")
        assert_nodes(b.nodes(), o.bfs(src)[1], "batch_trees inc bfs")
    for (s, d, _w) in W.deletes:
        old_s, old_b = o.sssp(src)[1], o.bfs(src)[1]
        before = len(o.edges()[0])
        o.delete(s, d)
        n_del = g.delete_trees([t, b], cuda(s), cuda(d))
        assert n_del == before - len(o.edges()[0])
        for tree, old in ((t, old_s), (b, old_b)):
            flag, nd = oracle.invalidated(V, src, old, s, d)
            st = tree.stats()
            assert tree.invalidated().tolist() == np.nonzero(flag)[0].tolist()
            assert st["direct_invalid"] == nd
            assert st["frontier_edges"] == o.dec_frontier_count(old, flag)
        assert_nodes(t.nodes(), o.sssp(src)[1], "batch_trees dec sssp")
        assert_nodes(b.nodes(), o.bfs(src)[1], "batch_trees dec bfs")
    # a single tree, mixed with the separate calls, keeps the version contract
    s, d, w = W.inserts[1]
    o.delete(s, d)
    g.delete_trees([t], cuda(s), cuda(d))
    b_nodes_stale = b.nodes()
    from paper_2305_17813_b200 import MeerkatError, _lib
    with pytest.raises(MeerkatError) as e:   # b missed the last batch: not current
        g.insert_trees([b], cuda(s), cuda(d), cuda(w))
    assert e.value.status == _lib.E_STATE
    b.decremental(cuda(s), cuda(d))
    assert_nodes(t.nodes(), o.sssp(src)[1], "single-tree delete_trees")
    assert_nodes(b.nodes(), o.bfs(src)[1], "per-tree after batch_trees")
    assert b_nodes_stale.shape == b.nodes().shape


@pytest.mark.parametrize("thread", ["0", "1"])
def test_batch_trees_lazy_heads(thread, monkeypatch):
    """Vertices with degree hint 0 get their head slab lazily (C22b) from the very insert kernel
    that runs the fused prologue: a vertex improved before its head exists is enqueued with the
    LINKING marker and resolved at round 0.  Chains through such vertices must come out exact."""
    monkeypatch.setenv("MEERKAT_THREAD_UPD", thread)
    rng = np.random.default_rng(5)
    V = 4096
    for rep in range(4):
        g = G(V, weighted=True, degree_hints=np.zeros(V, np.uint32), reverse=bool(rep & 1),
              in_degree_hints=np.zeros(V, np.uint32))
        o = oracle.OracleGraph(V)
        s0 = np.array([0], np.uint32); d0 = np.array([1], np.uint32); w0 = np.array([1], np.uint32)
        g.insert(s0, d0, w0); o.insert(s0, d0, w0)
        t, b = g.sssp(0), g.bfs(0)
        # long chains 1 -> p1 -> p2 ... over fresh (headless) vertices plus random extra edges
        perm = rng.permutation(np.arange(2, V)).astype(np.uint32)
        chain = np.concatenate([[1], perm[:1500]]).astype(np.uint32)
        cs, cd = chain[:-1], chain[1:]
        xs = rng.integers(0, V, 3000).astype(np.uint32); xd = rng.integers(0, V, 3000).astype(np.uint32)
        s = np.concatenate([cs, xs]); d = np.concatenate([cd, xd])
        w = rng.integers(1, 9, len(s)).astype(np.uint32)
        order = rng.permutation(len(s))
        s, d, w = s[order], d[order], w[order]
        o.insert(s, d, w)
        g.insert_trees([t, b], cuda(s), cuda(d), cuda(w))
        assert_nodes(t.nodes(), o.sssp(0)[1], f"lazy sssp rep {rep}")
        assert_nodes(b.nodes(), o.bfs(0)[1], f"lazy bfs rep {rep}")
        assert g.check()[0] == 0


def test_seed_contract():
    """insert / delete with seed=trees: the following tree call may name a subset of the seeded
    trees (each later call completes its own seed), never a mix of seeded and unseeded trees; a
    static recompute drops an unused seed (its frontier, counters and V_invalid marks)."""
    from paper_2305_17813_b200 import MeerkatError, _lib
    W = synth.rmat_dynamic(12, 8, batch=300, n_ins=3, n_del=2)
    V, src = W.vertex_n, W.source
    bs, bd, bw = W.base
    g = G(V, weighted=True, degree_hints=synth.degrees(bs, V), reverse=True, in_degree_hints=synth.degrees(bd, V))
    o = oracle.OracleGraph(V)
    g.insert(cuda(bs), cuda(bd), cuda(bw)); o.insert(bs, bd, bw)
    t, b = g.sssp(src), g.bfs(src)
    s, d, w = (cuda(x) for x in W.inserts[0])
    g.insert(s, d, w, seed=[t, b]); o.insert(*W.inserts[0])
    t.incremental(s, d, w)          # each seeded tree completes its own seed
    b.incremental(s, d)
    assert_nodes(t.nodes(), o.sssp(src)[1], "seed split sssp")
    assert_nodes(b.nodes(), o.bfs(src)[1], "seed split bfs")
    s, d = (cuda(x) for x in W.deletes[0][:2])
    g.delete(s, d, seed=[t]); o.delete(*W.deletes[0][:2])
    with pytest.raises(MeerkatError) as e:   # seeded + unseeded in one fused call
        g.trees_decremental([t, b], s, d)
    assert e.value.status == _lib.E_STATE
    with pytest.raises(MeerkatError) as e:   # already seeded
        g.insert(*(cuda(x) for x in W.inserts[1]), seed=[t])
    assert e.value.status == _lib.E_STATE
    g.trees_decremental([t], s, d)
    b.decremental(s, d)
    assert_nodes(t.nodes(), o.sssp(src)[1], "seeded dec sssp")
    assert_nodes(b.nodes(), o.bfs(src)[1], "unseeded dec bfs")
    # an unused seed (the trees never followed this delete), then another mutation: recompute drops it
    s, d = (cuda(x) for x in W.deletes[1][:2])
    g.delete(s, d, seed=[t, b]); o.delete(*W.deletes[1][:2])
    s, d, w = (cuda(x) for x in W.inserts[2])
    g.insert(s, d, w); o.insert(*W.inserts[2])
    t.recompute(); b.recompute()
    assert_nodes(t.nodes(), o.sssp(src)[1], "recompute after unused seed")
    assert_nodes(b.nodes(), o.bfs(src)[1], "recompute after unused seed (bfs)")
    s, d = (cuda(x) for x in W.inserts[2][:2])
    g.delete_trees([t, b], s, d); o.delete(*W.inserts[2][:2])
    assert_nodes(t.nodes(), o.sssp(src)[1], "batch_trees after recompute")
    assert_nodes(b.nodes(), o.bfs(src)[1], "batch_trees after recompute (bfs)")


@pytest.mark.parametrize("reverse", [True, False])
def test_road_like_grid_deep_trees(reverse):
    """SURVEY §8(d)'s road-like stress case (the paper's USAfull regime): a 192 x 192 grid,
    diameter ~380, so the static and dynamic calls run hundreds of frontier rounds (rotating frontier
    slots, stamp epochs, block-0 tail rounds) and deletions invalidate deep subtrees.  The bench's
    sequence (seeded insert / delete + fused trees), then per-tree calls; every node vs the oracle, with
    the invalidated sets, direct and frontier counts of the fused decremental calls."""
    W = synth.grid_dynamic(192, 600, 2, 3)
    V, src = W.vertex_n, W.source
    bs, bd, bw = W.base
    g = G(V, weighted=True, degree_hints=synth.degrees(bs, V), reverse=reverse,
          in_degree_hints=synth.degrees(bd, V), load_factor=0.5)
    o = oracle.OracleGraph(V)
    g.insert(cuda(bs), cuda(bd), cuda(bw)); o.insert(bs, bd, bw)
    t, b = g.sssp(src), g.bfs(src)
    assert_nodes(t.nodes(), o.sssp(src)[1], "grid static sssp")
    assert_nodes(b.nodes(), o.bfs(src)[1], "grid static bfs")
    assert t.stats()["rounds"] > 200
    for (s, d, w) in W.inserts:
        o.insert(s, d, w)
        g.insert_trees([t, b], cuda(s), cuda(d), cuda(w))
        assert_nodes(t.nodes(), o.sssp(src)[1], "grid inc sssp")
        assert_nodes(b.nodes(), o.bfs(src)[1], "grid inc bfs")
    for i, (s, d, _w) in enumerate(W.deletes):
        old_s, old_b = o.sssp(src)[1], o.bfs(src)[1]
        o.delete(s, d)
        if i < 2:
            g.delete_trees([t, b], cuda(s), cuda(d))
            for tree, old in ((t, old_s), (b, old_b)):
                flag, nd = oracle.invalidated(V, src, old, s, d)
                st = tree.stats()
                assert tree.invalidated().tolist() == np.nonzero(flag)[0].tolist()
                assert st["direct_invalid"] == nd
                assert st["frontier_edges"] == o.dec_frontier_count(old, flag)
        else:
            g.delete(cuda(s), cuda(d))
            t.decremental(cuda(s), cuda(d))
            b.decremental(cuda(s), cuda(d))
        assert_nodes(t.nodes(), o.sssp(src)[1], "grid dec sssp")
        assert_nodes(b.nodes(), o.bfs(src)[1], "grid dec bfs")
    assert t.stats()["invalidated"] > 0

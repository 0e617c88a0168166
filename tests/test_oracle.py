"""Pins for the CPU oracle (no GPU).  Each test ties oracle/meerkat_oracle.c to
something other than itself: the worked examples (tests/golden), brute-force
path enumeration, scipy's Dijkstra/BFS (an independent library), the paper's
own dynamic procedure simulated in Python (tests/refsim.py), a Python dict
replay of the store semantics, and invariants of the tree."""
import json
import os
import random

import numpy as np
import pytest

import oracle
from tests import refsim

U = (1 << 64) - 1


def _mk(n, edges, weighted=True):
    g = oracle.OracleGraph(n, weighted)
    if edges:
        s, d, w = zip(*edges)
        st, _ = g.insert(s, d, w)
        assert st == oracle.OK
    return g


def _pairs(node):
    return [None if int(x) == U else [int(x) >> 32, int(x) & 0xFFFFFFFF] for x in node]


# ---------------------------------------------------------------- golden G0

def test_golden_g0(golden_dir):
    G = json.load(open(os.path.join(golden_dir, "g0.json")))
    n, src = G["vertex_n"], G["source"]
    g = _mk(n, G["edges"])
    st, node = g.sssp(src)
    assert st == 0 and _pairs(node) == G["static_sssp"]
    st, bnode = g.bfs(src)
    assert st == 0 and _pairs(bnode) == G["static_bfs"]
    for step in G["steps"]:
        old = node.copy()
        if step["op"] == "delete":
            s, d = zip(*step["edges"])
            g.delete(s, d)
            flag, _ = oracle.invalidated(n, src, old, s, d)
            assert sorted(np.nonzero(flag)[0].tolist()) == step["invalid"]
            assert g.dec_frontier_count(old, flag) == len(step["frontier"])
        else:
            s, d, w = zip(*step["edges"])
            g.insert(s, d, w)
        st, node = g.sssp(src)
        assert _pairs(node) == step["sssp"], step["note"]
        if "packed" in step:
            assert [hex(int(x)) for x in node] == step["packed"]


def test_golden_unreached_sources(golden_dir):
    """Frontier edges start in V_valid only (P:156-158 with P:53-60's V_unreachable): edges from
    unreachable vertices into V_invalid are not counted (tests/golden/g1_unreached.json)."""
    G = json.load(open(os.path.join(golden_dir, "g1_unreached.json")))
    n, src = G["vertex_n"], G["source"]
    g = _mk(n, G["edges"])
    st, node = g.sssp(src)
    assert st == 0 and _pairs(node) == G["static_sssp"]
    for step in G["steps"]:
        old = node.copy()
        s, d = zip(*step["edges"])
        g.delete(s, d)
        flag, _ = oracle.invalidated(n, src, old, s, d)
        assert sorted(np.nonzero(flag)[0].tolist()) == step["invalid"]
        assert g.dec_frontier_count(old, flag) == len(step["frontier"]), step["note"]
        st, node = g.sssp(src)
        assert _pairs(node) == step["sssp"], step["note"]


@pytest.mark.parametrize("seed", range(30))
def test_dec_frontier_count_by_reachability(seed):
    """dec_frontier_count = |{(u, x) in E_new : u in V_valid, x in V_invalid}| with V_valid taken
    as the vertices REACHABLE from SRC in the old graph (a plain graph search over the old edge
    list) that are not invalidated — a route independent of the oracle's packed nodes.
    Sparse random graphs so that unreachable vertices with edges into V_invalid are common."""
    rng = random.Random(1000 + seed)
    n = rng.randint(4, 12)
    E = refsim.random_graph(rng, n, rng.randint(n // 2, 2 * n), 8)
    src = 0
    g = _mk(n, [(u, v, w) for (u, v), w in E.items()])
    _, old = g.sssp(src)
    reach, stack = {src}, [src]
    while stack:
        u = stack.pop()
        for (a, b) in E:
            if a == u and b not in reach:
                reach.add(b)
                stack.append(b)
    batch = rng.sample(sorted(E), rng.randint(1, len(E)))
    g.delete(*zip(*batch))
    for k in batch:
        E.pop(k)
    flag, _ = oracle.invalidated(n, src, old, *zip(*batch))
    want = sum(1 for (u, x) in E if u in reach and not flag[u] and flag[x])
    assert g.dec_frontier_count(old, flag) == want


def test_spec_examples(golden_dir):
    S = json.load(open(os.path.join(golden_dir, "spec_examples.json")))
    c = S["sssp_chain"]
    g = _mk(c["vertex_n"], c["edges"])
    _, node = g.sssp(c["source"])
    d, p = oracle.unpack(node)
    assert d.tolist() == c["dist"] and p.tolist() == c["parent"]
    c = S["sssp_chain_insert"]
    g = _mk(c["vertex_n"], c["edges"])
    s, dd, w = zip(*c["insert"])
    g.insert(s, dd, w)
    _, node = g.sssp(c["source"])
    d, p = oracle.unpack(node)
    assert d.tolist() == c["dist"] and p.tolist() == c["parent"]
    c = S["sssp_isolated_source"]
    g = _mk(c["vertex_n"], c["edges"])
    _, node = g.sssp(c["source"])
    assert all(int(node[v]) == U for v in c["unreached"]) and int(node[c["source"]]) == c["source"]
    c = S["bfs_star"]
    g = _mk(c["vertex_n"], c["edges"])
    _, node = g.bfs(c["source"])
    d, p = oracle.unpack(node)
    assert d.tolist() == c["level"] and p.tolist() == c["parent"]
    c = S["bfs_bridge"]
    g = _mk(c["vertex_n"], c["edges"])
    s, dd = zip(*c["delete"])
    g.delete(s, dd)
    _, node = g.bfs(c["source"])
    assert all(int(node[v]) != U for v in c["reached_after"])
    assert all(int(node[v]) == U for v in c["unreached_after"])


# ---------------------------------------------------------------- brute force

@pytest.mark.parametrize("seed", range(60))
def test_brute_force_paths(seed):
    rng = random.Random(seed)
    n = rng.randint(2, 7)
    m = rng.randint(0, n * (n - 1))
    wmax = rng.choice([1, 2, 3, 64])
    E = refsim.random_graph(rng, n, m, wmax)
    edges = [(u, v, w) for (u, v), w in E.items()]
    g = _mk(n, edges)
    src = rng.randrange(n)
    _, node = g.sssp(src)
    assert [int(x) for x in node] == refsim.brute_force_tree(n, src, edges)
    _, bnode = g.bfs(src)
    assert [int(x) for x in bnode] == refsim.brute_force_tree(n, src, edges, unit=True)


# ---------------------------------------------------------------- scipy (independent library)

@pytest.mark.parametrize("seed", range(4))
def test_scipy_distances(seed):
    from scipy.sparse import csr_matrix
    from scipy.sparse.csgraph import dijkstra, shortest_path
    rng = np.random.default_rng(seed)
    n, m = 400, 3000
    s = rng.integers(0, n, m); d = rng.integers(0, n, m); w = rng.integers(1, 65, m)
    keep = s != d
    s, d, w = s[keep], d[keep], w[keep]
    g = oracle.OracleGraph(n)
    g.insert(s, d, w)
    es, ed, ew = g.edges()
    A = csr_matrix((ew.astype(float), (es, ed)), shape=(n, n))
    ref = dijkstra(A, directed=True, indices=0)
    _, node = g.sssp(0)
    dist, _ = oracle.unpack(node)
    reach = np.isfinite(ref)
    assert np.array_equal(reach, node != oracle.UNREACHED)
    assert np.array_equal(dist[reach], ref[reach].astype(np.int64))
    lv = shortest_path(A, directed=True, unweighted=True, indices=0)
    _, bnode = g.bfs(0)
    bl, _ = oracle.unpack(bnode)
    assert np.array_equal(bl[reach], lv[reach].astype(np.int64))
    # min-weight upsert (C8): the stored weight is the min over duplicate draws
    ref_w = {}
    for a, b, c in zip(s.tolist(), d.tolist(), w.tolist()):
        ref_w[(a, b)] = min(ref_w.get((a, b), 1 << 40), c)
    assert {(a, b): c for a, b, c in zip(es.tolist(), ed.tolist(), ew.tolist())} == ref_w


# ---------------------------------------------------------------- invariants

def _check_invariants(g, src, node, unit):
    es, ed, ew = g.edges()
    dist, par = oracle.unpack(node)
    n = len(node)
    reach = node != oracle.UNREACHED
    assert node[src] == np.uint64(src)
    # tree invariant (BJ): d(v) = d(parent) + w(parent, v), parent is the min tight in-neighbour
    wmap = {(a, b): (1 if unit else c) for a, b, c in zip(es.tolist(), ed.tolist(), ew.tolist())}
    best = {}
    for (a, b), c in wmap.items():
        if reach[a]:
            cand = (int(dist[a]) + c, a)
            if b not in best or cand < best[b]:
                best[b] = cand
    for v in range(n):
        if v == src:
            continue
        if not reach[v]:
            assert v not in best
            continue
        assert (int(dist[v]), int(par[v])) == best[v]
    # arborescence rooted at SRC: every reached vertex's parent chain ends at SRC
    for v in np.nonzero(reach)[0].tolist():
        x, hops = v, 0
        while x != src:
            x = int(par[x]); hops += 1
            assert reach[x] and hops <= n


@pytest.mark.parametrize("seed", range(6))
def test_tree_invariants(seed):
    rng = np.random.default_rng(100 + seed)
    n, m = 300, 1500
    s = rng.integers(0, n, m); d = rng.integers(0, n, m); w = rng.integers(1, 4, m)
    g = oracle.OracleGraph(n)
    g.insert(s, d, w)
    _, node = g.sssp(0)
    _check_invariants(g, 0, node, unit=False)
    _, bnode = g.bfs(0)
    _check_invariants(g, 0, bnode, unit=True)


@pytest.mark.parametrize("seed", range(4))
def test_unit_weights_sssp_equals_bfs(seed):
    rng = np.random.default_rng(seed)
    n, m = 500, 2500
    s = rng.integers(0, n, m); d = rng.integers(0, n, m)
    g = oracle.OracleGraph(n)
    g.insert(s, d, np.ones(m, np.uint32))
    _, a = g.sssp(3)
    _, b = g.bfs(3)
    _, c = g.sssp(3, unit=True)
    assert np.array_equal(a, b) and np.array_equal(b, c)


def test_weight_scaling_invariance():
    """scaling all weights by k scales distances by k, parents unchanged."""
    rng = np.random.default_rng(7)
    n, m = 300, 2000
    s = rng.integers(0, n, m); d = rng.integers(0, n, m); w = rng.integers(1, 5, m)
    g1 = oracle.OracleGraph(n); g1.insert(s, d, w)
    g3 = oracle.OracleGraph(n); g3.insert(s, d, 3 * w)
    _, a = g1.sssp(0)
    _, b = g3.sssp(0)
    da, pa = oracle.unpack(a); db, pb = oracle.unpack(b)
    r = a != oracle.UNREACHED
    assert np.array_equal(r, b != oracle.UNREACHED)
    assert np.array_equal(pa[r], pb[r]) and np.array_equal(3 * da[r], db[r])


# ---------------------------------------------------------------- the method reaches the definition

@pytest.mark.parametrize("seed", range(40))
def test_paper_method_simulation_matches_oracle(seed):
    """The paper's dynamic procedure, run in random order,
    lands on the oracle's from-scratch result after every batch."""
    rng = random.Random(seed)
    n = rng.randint(3, 10)
    wmax = rng.choice([1, 2, 3, 64])
    unit = rng.random() < 0.3
    E = refsim.random_graph(rng, n, rng.randint(1, n * (n - 1) // 2), wmax)
    src = 0
    g = _mk(n, [(u, v, w) for (u, v), w in E.items()])
    node = refsim.simulate_static(n, src, E, unit, rng)
    _, ref = (g.bfs(src) if unit else g.sssp(src))
    assert node == [int(x) for x in ref]
    for _ in range(6):
        if rng.random() < 0.5 and E:
            batch = rng.sample(sorted(E), rng.randint(1, len(E)))
            batch += [(rng.randrange(n), rng.randrange(n)) for _ in range(2)]   # absent deletes (C11)
            g.delete(*zip(*batch))
            old = list(node)
            for k in batch:
                E.pop(k, None)
            node, inval = refsim.simulate_decremental(node, src, E, batch, unit, rng)
            flag, _ = oracle.invalidated(n, src, np.array(old, np.uint64), *zip(*batch))
            assert [bool(x) for x in flag] == inval
        else:
            batch = []
            for _ in range(rng.randint(1, 4)):
                u, v = rng.randrange(n), rng.randrange(n)
                if u != v:
                    batch.append((u, v, rng.randint(1, wmax)))
            if not batch:
                continue
            g.insert(*zip(*batch))
            for (u, v, w) in batch:
                E[(u, v)] = min(E.get((u, v), w), w)
            node = refsim.simulate_incremental(node, src, E, batch, unit, rng)
        _, ref = (g.bfs(src) if unit else g.sssp(src))
        assert node == [int(x) for x in ref]


# ---------------------------------------------------------------- store semantics

@pytest.mark.parametrize("seed", range(8))
def test_store_vs_dict_replay(seed):
    rng = random.Random(seed)
    n = rng.choice([5, 40, 300])
    g = oracle.OracleGraph(n)
    ref = refsim.dict_store()
    for _ in range(30):
        k = rng.randint(0, 60)
        if rng.random() < 0.6:
            b = [(rng.randrange(n), rng.randrange(n), rng.randint(1, 9)) for _ in range(k)]
            st, c = g.insert(*zip(*b)) if b else (0, 0)
            assert c == ref.insert(b)
        else:
            keys = list(ref.e)
            b = [rng.choice(keys) if keys and rng.random() < 0.7 else (rng.randrange(n), rng.randrange(n))
                 for _ in range(k)]
            st, c = g.delete(*zip(*b)) if b else (0, 0)
            assert c == ref.delete(b)
        qs = [(rng.randrange(n), rng.randrange(n)) for _ in range(20)] + list(ref.e)[:20]
        st, found, w = g.query(*zip(*qs))
        assert found.tolist() == [int(q in ref.e) for q in qs]
        assert w.tolist() == [ref.e.get(q, 0) for q in qs]
        es, ed, ew = g.edges()
        assert dict(zip(zip(es.tolist(), ed.tolist()), ew.tolist())) == ref.e


def test_store_idempotence_and_latest_weight():
    g = oracle.OracleGraph(4)
    assert g.insert([0, 1], [1, 0], [5, 6]) == (0, 2)
    assert g.insert([0, 1], [1, 0], [5, 6]) == (0, 0)            # re-insert -> 0
    assert g.delete([2], [3]) == (0, 0)                           # delete absent -> 0 (C11)
    assert g.delete([0], [1]) == (0, 1)
    assert g.insert([0], [1], [9]) == (0, 1)                      # insert∘delete∘insert -> latest
    assert g.query([0], [1])[2].tolist() == [9]
    assert g.insert([0], [1], [4]) == (0, 0)                      # min-weight upsert (C8)
    assert g.query([0], [1])[2].tolist() == [4]


def test_validation_errors():
    g = oracle.OracleGraph(4)
    st, c = g.insert([0, 9, 1], [1, 1, 2], [1, 1, 0])
    assert st == oracle.E_VERTEX_RANGE and c == 1                # id >= V skipped; w = 0 skipped (C6)
    st, c = g.insert([1], [2], [1 << 31])
    assert st == oracle.E_WEIGHT and c == 0
    st, found, w = g.query([0, 7], [1, 1])
    assert st == oracle.E_VERTEX_RANGE and found.tolist() == [1, 0]


# ---------------------------------------------------------------- certificate checker

@pytest.mark.parametrize("seed", range(5))
def test_check_tree_accepts_truth_rejects_corruption(seed):
    """Fault injection: any single corrupted node must be detected."""
    rng = np.random.default_rng(seed)
    n, m = 200, 900
    s = rng.integers(0, n, m); d = rng.integers(0, n, m); w = rng.integers(1, 10, m)
    g = oracle.OracleGraph(n)
    g.insert(s, d, w)
    for unit in (False, True):
        _, node = (g.bfs(0) if unit else g.sssp(0))
        assert g.check_tree(0, node, unit) == (0, 0xFFFFFFFF)
        for trial in range(20):
            bad = node.copy()
            v = int(rng.integers(0, n))
            kind = trial % 4
            if kind == 0:
                bad[v] = np.uint64(int(bad[v]) ^ 1) if int(bad[v]) != U else np.uint64(5 << 32)
            elif kind == 1:
                bad[v] = np.uint64(U) if int(bad[v]) != U else np.uint64(0)
            elif kind == 2:
                bad[v] = np.uint64((int(bad[v]) + (1 << 32)) % (1 << 64))
            else:
                bad[v] = np.uint64(max(int(bad[v]) - (1 << 32), 0)) if int(bad[v]) != U else np.uint64(1 << 32)
            if np.array_equal(bad, node):
                continue
            nbad, fb = g.check_tree(0, bad, unit)
            assert nbad >= 1


def test_overflow_flagged():
    """C5: a distance reaching 2^32-1 is reported as OVERFLOW."""
    g = oracle.OracleGraph(4)
    big = (1 << 31) - 1
    g.insert([0, 1, 2], [1, 2, 3], [big, big, big])
    st, node = g.sssp(0)
    assert st == oracle.E_OVERFLOW

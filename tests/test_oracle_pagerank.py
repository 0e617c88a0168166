"""Pins for the oracle's PageRank (oracle/meerkat_oracle.c orc_pagerank; SURVEY §8(f) NEXT-1,
P:825-904, Eq. (1), d and eps P:1559-1560, teleport reading C27).  Each test ties it
to something other than itself: a hand-computed super-step (tests/golden/pr_example.json), the
closed forms of SPEC S:444-445, the exact fixpoint from a dense linear solve (numpy.linalg,
an independent library), mass conservation of the Google matrix, the contraction bound of the
stopping rule, and the warm-start property of the dynamic variant."""
import json
import os

import numpy as np
import pytest

import oracle

D = 0.85


def _graph(n, edges):
    g = oracle.OracleGraph(n, weighted=True)
    if edges:
        s, t = zip(*edges)
        st, _ = g.insert(s, t, [1] * len(s))
        assert st == oracle.OK
    return g


def _random_edges(rng, n, m, self_loops=True):
    e = set()
    while len(e) < m:
        u, v = int(rng.integers(n)), int(rng.integers(n))
        if u == v and not self_loops:
            continue
        e.add((u, v))
    return sorted(e)


def _closed_form(n, edges, d=D):
    """Exact fixpoint of Eq. (1) with the teleport term: x = (1-d)/N + d (A x), A the column-
    stochastic matrix (A[v,u] = 1/out[u] for u->v; A[v,z] = 1/N for out[z] = 0), by a dense solve."""
    out = np.zeros(n)
    for u, _ in edges:
        out[u] += 1
    A = np.zeros((n, n))
    for u, v in edges:
        A[v, u] += 1.0 / out[u]
    for z in range(n):
        if out[z] == 0:
            A[:, z] += 1.0 / n
    return np.linalg.solve(np.eye(n) - d * A, np.full(n, (1 - d) / n))


def test_hand_computed_super_step(golden_dir):
    G = json.load(open(os.path.join(golden_dir, "pr_example.json")))
    g = _graph(G["vertex_n"], G["edges"])
    st, pr, it, delta = g.pagerank(d=G["d"], eps=1e-9, max_iter=1)
    assert st == oracle.OK and it == 1
    want = np.array(G["pr1_num"], dtype=np.float64) / G["pr1_den"]
    assert np.allclose(pr, want, rtol=0, atol=1e-15)
    assert delta == pytest.approx(G["delta1_num"] / G["delta1_den"], abs=1e-15)


def test_two_cycle_and_isolated_vertex():
    # 2-cycle -> [0.5, 0.5] exactly (symmetry; one verification super-step)
    st, pr, it, delta = _graph(2, [(0, 1), (1, 0)]).pagerank()
    assert st == oracle.OK and list(pr) == [0.5, 0.5] and it == 1 and delta == 0.0
    # a single isolated vertex -> 1.0 via the teleport term: (1-d) + d*1 = 1
    st, pr, it, _ = _graph(1, []).pagerank()
    assert st == oracle.OK and pr[0] == pytest.approx(1.0, abs=1e-15)


@pytest.mark.parametrize("seed", range(12))
def test_fixpoint_equals_dense_solve(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(2, 48))
    m = int(rng.integers(1, min(n * n, 4 * n) + 1))
    edges = _random_edges(rng, n, m)
    st, pr, it, delta = _graph(n, edges).pagerank(eps=1e-14, max_iter=20000)
    assert st == oracle.OK and delta <= 1e-14
    x = _closed_form(n, edges)
    assert np.abs(pr - x).sum() <= 1e-11


@pytest.mark.parametrize("seed", range(6))
def test_mass_conserved_every_super_step(seed):
    # the teleport term makes the iteration matrix column-stochastic: sum(PR_i) = 1 for every i
    rng = np.random.default_rng(100 + seed)
    n = 64
    edges = _random_edges(rng, n, 160, self_loops=False)
    g = _graph(n, edges)
    for k in range(1, 12):
        _, pr, it, _ = g.pagerank(eps=1e-300, max_iter=k)
        assert it == k and abs(pr.sum() - 1.0) <= 1e-13


@pytest.mark.parametrize("seed", range(6))
def test_stopping_rule_and_contraction_bound(seed):
    rng = np.random.default_rng(200 + seed)
    n = 80
    edges = _random_edges(rng, n, 300)
    g = _graph(n, edges)
    eps = 1e-5   # the paper's error margin
    _, pr, k, delta = g.pagerank(eps=eps, max_iter=1000)
    assert delta <= eps and k >= 2
    _, _, k1, delta1 = g.pagerank(eps=eps, max_iter=k - 1)   # one super-step fewer: not yet converged
    assert k1 == k - 1 and delta1 > eps
    # L1 contraction by d: ||x_k - x*|| <= d/(1-d) * ||x_k - x_{k-1}||
    x = _closed_form(n, edges)
    assert np.abs(pr - x).sum() <= D / (1 - D) * delta * (1 + 1e-9)


def test_warm_start_dynamic():
    rng = np.random.default_rng(7)
    n = 200
    edges = _random_edges(rng, n, 900, self_loops=False)
    g = _graph(n, edges)
    _, pr0, _, _ = g.pagerank(eps=1e-12, max_iter=10000)
    # unchanged graph: one verification super-step, vector unchanged within eps
    _, pr1, it, delta = g.pagerank(eps=1e-5, pr=pr0)
    assert it == 1 and delta <= 1e-5 and np.abs(pr1 - pr0).sum() <= 1e-5
    # insert a batch, then warm- and cold-started runs land within 10 eps of each other and of
    # the new fixpoint
    extra = [e for e in _random_edges(rng, n, 60, self_loops=False) if e not in set(edges)]
    s, t = zip(*extra)
    g.insert(s, t, [1] * len(s))
    _, warm, kw, _ = g.pagerank(eps=1e-5, pr=pr0)
    _, cold, kc, _ = g.pagerank(eps=1e-5)
    x = _closed_form(n, sorted(set(edges) | set(extra)))
    assert np.abs(warm - cold).sum() <= 1e-4 and np.abs(warm - x).sum() <= 1e-4
    assert kw < kc   # the warm start is the paper's source of dynamic speedup


def test_invalid_arguments():
    g = _graph(3, [(0, 1)])
    for d, eps, mi in [(0.0, 1e-5, 10), (1.0, 1e-5, 10), (0.85, 0.0, 10), (0.85, 1e-5, 0)]:
        st, _, _, _ = g.pagerank(d=d, eps=eps, max_iter=mi)
        assert st == oracle.E_INVALID_ARG

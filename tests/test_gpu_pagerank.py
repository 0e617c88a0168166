"""GPU parity of static and dynamic PageRank (Eq. (1)
P:834-836, teleport reading C27) against the CPU oracle (oracle/meerkat_oracle.c orc_pagerank,
pinned in tests/test_oracle_pagerank.py).  Bar (BASELINE.json north_star): relative L1
sum|gpu - oracle| / sum|oracle| <= 1e-6, with the same number of super-steps (both sides
compute in double precision; only the summation order of the in-edge sums differs, ~1e-16
relative, so the stopping decision delta <= eps lands on the same super-step)."""
import json
import os

import numpy as np
import pytest

import oracle
import synth
from tests.gpu_helpers import cuda

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

TOL = 1e-6
D, EPS = 0.85, 1e-5


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def G(*a, **k):
    from paper_2305_17813_b200 import Graph
    k.setdefault("reverse", True)
    return Graph(*a, **k)


def rel_l1(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).sum() / np.abs(np.asarray(b)).sum())


def _pair(n, s, d, w=None, weighted=True, **kw):
    s = np.asarray(s, np.uint32); d = np.asarray(d, np.uint32)
    if w is None:
        w = np.ones(len(s), np.uint32)
    g = G(n, weighted=weighted, degree_hints=synth.degrees(s, n) if len(s) else None,
          in_degree_hints=synth.degrees(d, n) if len(d) else None, **kw)
    if len(s):
        g.insert(cuda(s), cuda(d), cuda(w) if weighted else None)
    o = oracle.OracleGraph(n, weighted=True)
    if len(s):
        o.insert(s, d, w)
    return g, o


def _check(p, o, pr_prev=None, what=""):
    st, ref, it, delta = o.pagerank(D, EPS, 1000, pr=pr_prev)
    assert st == oracle.OK
    got = p.values()
    s = p.stats()
    assert s["iterations"] == it, (what, s["iterations"], it, s["delta"], delta)
    e = rel_l1(got, ref)
    assert e <= TOL, (what, e)
    return ref


def test_closed_forms_and_hand_example(golden_dir):
    # S:444 2-cycle -> [0.5, 0.5]; S:445 isolated vertex -> [1.0]
    g, _ = _pair(2, [0, 1], [1, 0])
    p = g.pagerank(D, EPS)
    assert np.allclose(p.values(), [0.5, 0.5], atol=1e-15) and p.stats()["iterations"] == 1
    g1, _ = _pair(1, [], [])
    assert abs(g1.pagerank(D, EPS).values()[0] - 1.0) <= 1e-15
    # first super-step of the hand-computed example (tests/golden/pr_example.json)
    J = json.load(open(os.path.join(golden_dir, "pr_example.json")))
    s, d = zip(*J["edges"])
    g3, _ = _pair(J["vertex_n"], s, d)
    p3 = g3.pagerank(J["d"], 1e-9, max_iter=1)
    want = np.array(J["pr1_num"], np.float64) / J["pr1_den"]
    assert np.allclose(p3.values(), want, rtol=0, atol=1e-15)
    assert abs(p3.stats()["delta"] - J["delta1_num"] / J["delta1_den"]) <= 1e-15


def test_requires_in_edge_mirror_and_valid_args():
    from paper_2305_17813_b200 import MeerkatError
    g = G(8, reverse=False)
    with pytest.raises(MeerkatError):
        g.pagerank()
    g2 = G(8)
    for d, e, m in [(0.0, 1e-5, 10), (1.0, 1e-5, 10), (0.85, 0.0, 10), (0.85, 1e-5, 0)]:
        with pytest.raises(MeerkatError):
            g2.pagerank(d, e, m)


@pytest.mark.parametrize("weighted", [True, False])
def test_config1_static_and_dynamic(weighted):
    """BASELINE config 1 graph (uniform 1K / 8K), 4 insert + 4 delete batches of 64 edges; after
    each batch the dynamic (warm-started) run is compared with the oracle warm-started from its own
    previous vector."""
    V = 1024
    s, d, w = synth.uniform(V, 8192)
    g, o = _pair(V, s, d, w, weighted=weighted)
    p = g.pagerank(D, EPS)
    ref = _check(p, o, None, "static")
    rng = np.random.default_rng(5)
    es, ed, ew = o.edges()
    for b in range(8):
        if b < 4:
            bs = rng.integers(0, V, 64).astype(np.uint32); bd = rng.integers(0, V, 64).astype(np.uint32)
            bw = rng.integers(1, 65, 64).astype(np.uint32)
            g.insert(cuda(bs), cuda(bd), cuda(bw) if weighted else None)
            o.insert(bs, bd, bw)
        else:
            es, ed, _ = o.edges()
            pick = rng.choice(len(es), 64, replace=False)
            g.delete(cuda(es[pick]), cuda(ed[pick]))
            o.delete(es[pick], ed[pick])
        p.update()
        assert p.stats()["warm"] == 1
        ref = _check(p, o, ref, f"batch {b}")
    p.recompute()
    _check(p, o, None, "recompute")


@pytest.mark.parametrize("scale,hashing,lf", [(16, True, 0.7), (16, False, 0.7), (14, True, 0.05)])
def test_rmat_parity(scale, hashing, lf):
    """R-MAT (several thousand slabs: multi-bucket hubs whose slab runs are combined, pool chains
    at lf 0.05, one list per vertex without hashing), static + dynamic after a mixed batch."""
    W = synth.rmat_dynamic(scale, 16, batch=2000, n_ins=1, n_del=1)
    s, d, w = W.base
    g, o = _pair(W.vertex_n, s, d, w, hashing=hashing, load_factor=lf)
    assert g.check()[0] == 0
    p = g.pagerank(D, EPS)
    ref = _check(p, o, None, "static")
    (is_, id_, iw), (ds, dd, _) = W.inserts[0], W.deletes[0]
    g.insert(cuda(is_), cuda(id_), cuda(iw)); o.insert(is_, id_, iw)
    g.delete(cuda(ds), cuda(dd)); o.delete(ds, dd)
    assert g.check()[0] == 0   # includes the degree table
    p.update()
    _check(p, o, ref, "dynamic")


def test_scale20_parity():
    """BASELINE config 2 graph (R-MAT scale 20, 16 M edges) static + one 100K-edge insert batch."""
    W = synth.rmat_dynamic(20, 16, batch=100_000, n_ins=1, n_del=0)
    s, d, w = W.base
    g, o = _pair(W.vertex_n, s, d, w)
    p = g.pagerank(D, EPS)
    ref = _check(p, o, None, "static")
    is_, id_, iw = W.inserts[0]
    g.insert(cuda(is_), cuda(id_), cuda(iw)); o.insert(is_, id_, iw)
    p.update()
    _check(p, o, ref, "dynamic")


@pytest.mark.slow
def test_scale24_fixpoint_property():
    """BASELINE config 3 size (R-MAT scale 24, 263 M edges): mass conservation and, on a seeded
    sample of 2,000 vertices, the Eq. (1) residual |PR[v] - ((1-d)/N + d sum PR[u]/out[u] +
    d Z/N)| — the sampled residuals sum to at most ||x_k - F(x_k)||_1 <= d * delta."""
    W = synth.rmat_dynamic(24, 16, batch=100_000, n_ins=1, n_del=0)
    s, d, w = W.base
    V = W.vertex_n
    g = G(V, degree_hints=synth.degrees(s, V), in_degree_hints=synth.degrees(d, V))
    g.insert(cuda(s), cuda(d), cuda(w))
    p = g.pagerank(D, EPS)
    pr = p.values()
    st = p.stats()
    assert st["delta"] <= EPS and abs(pr.sum() - 1.0) <= 1e-9
    out = np.bincount(s, minlength=V).astype(np.float64)
    Z = pr[out == 0].sum()
    rng = np.random.default_rng(11)
    sample = np.unique(np.concatenate([rng.choice(V, 2000, replace=False), [W.source]]))
    mask = np.isin(d, sample)
    acc = np.zeros(V)
    np.add.at(acc, d[mask], pr[s[mask]] / out[s[mask]])
    resid = np.abs(pr[sample] - ((1 - D) / V + D * acc[sample] + D * Z / V))
    assert resid.sum() <= D * st["delta"] * (1 + 1e-6)

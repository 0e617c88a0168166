"""GPU parity of the slab store against the CPU oracle:
edge sets, insert/delete counts and query answers must be bit-exact — for both update-kernel
kinds (group-cooperative and thread-per-edge, store.cu thread_upd)."""
import json
import os

import numpy as np
import pytest

import oracle
import synth
from tests.gpu_helpers import assert_same_edges, cuda

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.fixture(autouse=True, params=["group", "thread"])
def update_kernel(request, monkeypatch):
    """Every store test runs with both update-kernel kinds: 8-lane groups (small batches) and
    thread-per-edge (large batches), forced via MEERKAT_THREAD_UPD (read at each launch)."""
    monkeypatch.setenv("MEERKAT_THREAD_UPD", "1" if request.param == "thread" else "0")
    return request.param


def G(*a, **k):
    from paper_2305_17813_b200 import Graph
    return Graph(*a, **k)


def test_arena_shape(golden_dir):
    """S:63 / S:149 / S:151 worked examples and S:617's single-arena size rule."""
    A = json.load(open(os.path.join(golden_dir, "spec_examples.json")))["arena"]
    g = G(3, weighted=False, load_factor=A["set"]["lf"], degree_hints=np.array(A["set"]["hints"], np.uint32))
    st = g.stats()
    assert st["head_slabs"] == A["set"]["total"] and st["buckets"] == A["set"]["total"]
    g = G(1, weighted=True, load_factor=A["map"]["lf"], degree_hints=np.array(A["map"]["hints"], np.uint32))
    assert g.stats()["head_slabs"] == A["map"]["total"]
    rng = np.random.default_rng(5)
    for _ in range(10):
        hints = rng.integers(0, 400, 300).astype(np.uint32)
        lf = float(rng.choice([0.3, 0.6, 0.7, 1.0]))
        for weighted in (False, True):
            cap = 15 if weighted else 31
            g = G(300, weighted=weighted, load_factor=lf, degree_hints=hints)
            lfc = float(np.float32(lf))
            expect = sum(int(np.ceil(h / (lfc * cap))) for h in hints.tolist() if h > 0)
            assert g.stats()["head_slabs"] == expect
            assert g.stats()["buckets"] == expect + int((hints == 0).sum())
    g = G(300, weighted=True, hashing=False, degree_hints=hints)
    assert g.stats()["head_slabs"] == int((hints > 0).sum())


def test_spill_32_keys(golden_dir):
    """32 distinct keys -> 31 in the head slab and 1 in a newly chained slab (set store)."""
    g = G(64, weighted=False, hashing=False, pool_slabs=16)
    n = g.insert(np.zeros(32, np.uint32), np.arange(1, 33, dtype=np.uint32))
    assert n == 32
    st = g.stats()
    assert st["head_slabs"] == 64 and st["pool_used"] == 1
    s, d, _ = g.export_edges()
    assert s.tolist() == [0] * 32 and d.tolist() == list(range(1, 33))


@pytest.mark.parametrize("weighted", [True, False])
@pytest.mark.parametrize("hints", ["none", "zero", "degree"])
@pytest.mark.parametrize("hashing", [True, False])
def test_random_batches_vs_oracle(weighted, hints, hashing):
    rng = np.random.default_rng(100 * int(weighted) + 10 * ["none", "zero", "degree"].index(hints) + int(hashing))
    V = 700
    base = synth.rmat(10, 8, seed_graph=11)
    if hints == "none":
        h = None
    elif hints == "zero":
        h = np.zeros(V, np.uint32)
    else:
        h = synth.degrees(base[0], 1024)[:V]
    g = G(V, weighted=weighted, hashing=hashing, load_factor=0.7, degree_hints=h, pool_slabs=1 << 15)
    o = oracle.OracleGraph(V, weighted)
    for it in range(24):
        kind = rng.random()
        n = int(rng.choice([0, 1, 7, 33, 500, 3000]))
        if kind < 0.55:
            s = rng.integers(0, V, n).astype(np.uint32)
            d = rng.integers(0, V, n).astype(np.uint32)
            if n > 10:   # duplicates and hub rows within one batch
                s[: n // 5] = s[0]
                d[n // 5: n // 4] = d[0]
                s[n // 4: n // 3] = s[n // 4]
                d[n // 4: n // 3] = d[n // 4]
            w = rng.integers(1, 65, n).astype(np.uint32) if weighted else None
            exp = o.insert(s, d, w)[1]
            got = g.insert(cuda(s), cuda(d), cuda(w) if weighted else None)
            assert got == exp, (it, got, exp)
        elif kind < 0.9:
            es, ed, _ = o.edges()
            k = min(n, len(es))
            pick = rng.choice(len(es), k, replace=False) if k else np.array([], int)
            s = np.concatenate([es[pick], rng.integers(0, V, n - k).astype(np.uint32)]).astype(np.uint32)
            d = np.concatenate([ed[pick], rng.integers(0, V, n - k).astype(np.uint32)]).astype(np.uint32)
            if n > 4:
                s[-2:] = s[:2]; d[-2:] = d[:2]   # duplicate deletes (C11)
            exp = o.delete(s, d)[1]
            got = g.delete(cuda(s), cuda(d))
            assert got == exp, (it, got, exp)
        else:
            es, ed, ew = o.edges()
            s = np.concatenate([es[: n // 2], rng.integers(0, V, n - n // 2)]).astype(np.uint32)
            d = np.concatenate([ed[: n // 2], rng.integers(0, V, n - n // 2)]).astype(np.uint32)
            _, ef, eww = o.query(s, d)
            f, w = g.query(cuda(s), cuda(d))
            assert np.array_equal(f.cpu().numpy(), ef)
            assert np.array_equal(w.cpu().numpy().view(np.uint32), eww)
    assert_same_edges(g, o)
    assert g.stats()["edges"] == o.num_edges


def test_hub_link_races():
    """Thousands of concurrent inserts into one slab list (hashing off): exact count, no duplicate,
    chain links under contention (C9, H8)."""
    V = 20000
    g = G(V, weighted=True, hashing=False, pool_slabs=1 << 16)
    o = oracle.OracleGraph(V)
    rng = np.random.default_rng(1)
    for rep in range(3):
        d = rng.integers(0, V, 40000).astype(np.uint32)
        s = np.full_like(d, 7)
        w = rng.integers(1, 65, len(d)).astype(np.uint32)
        assert g.insert(cuda(s), cuda(d), cuda(w)) == o.insert(s, d, w)[1]
    assert_same_edges(g, o)
    st = g.stats()
    assert st["pool_used"] >= o.num_edges // 15 - 1


def test_host_pointers_equal_device_pointers():
    V = 500
    s, d, w = synth.uniform(V, 4000, seed_graph=3)
    g1 = G(V, weighted=True)
    g2 = G(V, weighted=True)
    assert g1.insert(s, d, w) == g2.insert(cuda(s), cuda(d), cuda(w))
    f1, w1 = g1.query(s, d)
    f2, w2 = g2.query(cuda(s), cuda(d))
    assert np.array_equal(f1, f2.cpu().numpy()) and np.array_equal(w1, w2.cpu().numpy().view(np.uint32))
    a, b = g1.export_edges(), g2.export_edges()
    assert all(np.array_equal(x, y) for x, y in zip(a, b))


def test_invalid_edges_skipped_and_reported():
    from paper_2305_17813_b200 import _lib
    V = 10
    g = G(V, weighted=True)
    o = oracle.OracleGraph(V)
    s = np.array([0, 11, 2, 3], np.uint32); d = np.array([1, 1, 99, 4], np.uint32); w = np.array([1, 1, 1, 0], np.uint32)
    st, n = g.insert(s, d, w, raise_on_error=False)
    ost, on = o.insert(s, d, w)
    assert st == _lib.E_VERTEX_RANGE == ost and n == on == 1
    st, n = g.insert(np.array([4], np.uint32), np.array([5], np.uint32), np.array([1 << 31], np.uint32),
                     raise_on_error=False)
    assert st == _lib.E_WEIGHT and n == 0
    st, f, w = g.query(np.array([0, 20], np.uint32), np.array([1, 1], np.uint32), raise_on_error=False)
    assert st == _lib.E_VERTEX_RANGE and f.tolist() == [1, 0]
    assert_same_edges(g, o)
    g.sync()   # error was reported and cleared


def test_pool_exhaustion_reports_capacity():
    from paper_2305_17813_b200 import _lib
    # one arena head + 2 pool slabs: at most 93 keys for vertex 0.  Under exhaustion a slab lost
    # to a link race is cleared and never reachable, and which inserts still find a free cell
    # depends on timing: only the head (31) is guaranteed.  Placed edges are kept and counted.
    d = np.arange(4, 400, dtype=np.uint32)
    g = G(500, weighted=False, hashing=False, pool_slabs=2)
    st, n = g.insert(np.zeros(len(d), np.uint32), d, raise_on_error=False)
    assert st == _lib.E_CAPACITY
    s, dd, _ = g.export_edges()
    assert 31 <= n <= 93 and len(dd) == n and len(np.unique(dd)) == n and set(dd.tolist()) <= set(d.tolist())
    assert g.stats()["pool_used"] == 2
    assert g.stats()["edges"] == n


@pytest.mark.parametrize("hashing", [True, False])
def test_fresh_draw_stress_with_fsck(hashing):
    """Large batches of fresh R-MAT draws (duplicates, self-loops, hub rows, vertices whose head slab is
    created lazily by racing groups) then deletes, with the structural check after every kernel and the
    edge set / counts against the oracle.  Regression test for a group-divergence race on lazy heads."""
    scale = 16
    s, d, w = synth.rmat(scale, 16)
    V = 1 << scale
    g = G(V, weighted=True, hashing=hashing, degree_hints=synth.degrees(s, V))
    o = oracle.OracleGraph(V)
    assert g.insert(cuda(s), cuda(d), cuda(w)) == o.insert(s, d, w)[1]
    assert g.check()[0] == 0
    for r in range(4):
        fs, fd, fw = synth.rmat_draws(scale, 200000, r * 200000, 11, scramble_seed=11)
        assert g.insert(cuda(fs), cuda(fd), cuda(fw)) == o.insert(fs, fd, fw)[1]
        assert g.check()[0] == 0, g.check()
        pick = synth.sample_distinct(len(s), 100000, 100 + r)
        assert g.delete(cuda(s[pick]), cuda(d[pick])) == o.delete(s[pick], d[pick])[1]
        assert g.check()[0] == 0, g.check()
    assert_same_edges(g, o)

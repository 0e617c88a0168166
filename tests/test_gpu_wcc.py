"""GPU parity of static and incremental WCC (P:905-912, P:381-395,
P:486-493): canonical labels (smallest id of the component) bit-exact against the oracle
(orc_wcc, pinned in tests/test_oracle_wcc.py) after the static build and after every batch."""
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


def G(*a, **k):
    from paper_2305_17813_b200 import Graph
    return Graph(*a, **k)


def test_hand_example():
    g = G(6, weighted=False)
    g.insert(np.array([1, 2, 4], np.uint32), np.array([0, 3, 3], np.uint32))
    c = g.wcc()
    assert c.labels().tolist() == [0, 0, 2, 2, 2, 5] and c.components() == 3
    g.insert(np.array([5], np.uint32), np.array([4], np.uint32))
    c.incremental(np.array([5], np.uint32), np.array([4], np.uint32))
    assert c.labels().tolist() == [0, 0, 2, 2, 2, 2] and c.components() == 2


@pytest.mark.parametrize("weighted,hashing", [(False, True), (True, True), (False, False)])
def test_sparse_random_incremental(weighted, hashing):
    """Sparse uniform graph (many components), 6 insert batches."""
    rng = np.random.default_rng(2)
    V = 20000
    s, d = rng.integers(0, V, 12000).astype(np.uint32), rng.integers(0, V, 12000).astype(np.uint32)
    w = np.ones(len(s), np.uint32)
    g = G(V, weighted=weighted, hashing=hashing, degree_hints=synth.degrees(s, V))
    g.insert(cuda(s), cuda(d), cuda(w) if weighted else None)
    o = oracle.OracleGraph(V, weighted=False)
    o.insert(s, d)
    c = g.wcc()
    lab, k = o.wcc()
    assert np.array_equal(c.labels(), lab) and c.components() == k
    for b in range(6):
        bs, bd = rng.integers(0, V, 2000).astype(np.uint32), rng.integers(0, V, 2000).astype(np.uint32)
        g.insert(cuda(bs), cuda(bd), cuda(np.ones(2000, np.uint32)) if weighted else None)
        o.insert(bs, bd)
        c.incremental(cuda(bs), cuda(bd))
        lab, k = o.wcc()
        assert np.array_equal(c.labels(), lab), b
        assert c.components() == k
    c.recompute()
    assert np.array_equal(c.labels(), o.wcc()[0])


@pytest.mark.parametrize("scale", [16, 20])
def test_rmat(scale):
    W = synth.rmat_dynamic(scale, 16, batch=10000, n_ins=2, n_del=0)
    s, d, w = W.base
    V = W.vertex_n
    g = G(V, degree_hints=synth.degrees(s, V))
    g.insert(cuda(s), cuda(d), cuda(w))
    o = oracle.OracleGraph(V)
    o.insert(s, d, w)
    c = g.wcc()
    assert np.array_equal(c.labels(), o.wcc()[0])
    for b in range(2):
        bs, bd, bw = W.inserts[b]
        g.insert(cuda(bs), cuda(bd), cuda(bw))
        o.insert(bs, bd, bw)
        c.incremental(cuda(bs), cuda(bd))
        assert np.array_equal(c.labels(), o.wcc()[0])


@pytest.mark.parametrize("kernel", ["group", "thread"])
@pytest.mark.parametrize("weighted,hashing,lf", [(False, True, 0.7), (True, True, 0.3), (False, False, 0.7)])
def test_update_iterator_incremental(kernel, weighted, hashing, lf, monkeypatch):
    """The paper's UpdateIterator path: with update tracking, unioning the edges of the
    slab lists written since the last call (from their first updated cell on) gives the oracle's
    labels; both update-kernel kinds record the placements; tracking resets after every call."""
    monkeypatch.setenv("MEERKAT_THREAD_UPD", "1" if kernel == "thread" else "0")
    rng = np.random.default_rng(31)
    V = 20000
    s, d = rng.integers(0, V, 12000).astype(np.uint32), rng.integers(0, V, 12000).astype(np.uint32)
    hints = synth.degrees(s, V)
    hints[: V // 4] = 0   # lazily headed lists too
    g = G(V, weighted=weighted, hashing=hashing, load_factor=lf, degree_hints=hints, update_tracking=True)
    one = lambda n: cuda(np.ones(n, np.uint32)) if weighted else None
    g.insert(cuda(s), cuda(d), one(len(s)))
    o = oracle.OracleGraph(V, weighted=False)
    o.insert(s, d)
    c = g.wcc()
    c.incremental_tracked()   # consumes the tracking of the bulk insert (already reflected)
    assert np.array_equal(c.labels(), o.wcc()[0])
    for b in range(5):
        n = 3000
        bs, bd = rng.integers(0, V, n).astype(np.uint32), rng.integers(0, V, n).astype(np.uint32)
        g.insert(cuda(bs), cuda(bd), one(n))
        o.insert(bs, bd)
        c.incremental_tracked()
        lab, k = o.wcc()
        assert np.array_equal(c.labels(), lab), b
        assert c.components() == k
    assert g.check()[0] == 0


def test_tracking_required():
    from paper_2305_17813_b200 import MeerkatError
    g = G(100, weighted=False)
    g.insert(np.array([1], np.uint32), np.array([2], np.uint32))
    c = g.wcc()
    with pytest.raises(MeerkatError):
        c.incremental_tracked()

"""GPU tests of the ordering contract (meerkat.h; "the graph object G undergoes modifications
through the application of an insertion/deletion edge batch; the incremental/decremental SSSP algorithm
re-computes"): a tree call must get exactly the batch the last mutation applied.  Host checks (version,
kind, n) fail at once; a same-size batch with different edges is caught on the device by the batch
fingerprint before the tree is touched, reported as MEERKAT_E_STATE by the next synchronising call, and
leaves the tree stale until a static recompute.  A permutation of the applied batch is the same batch
(set semantics) and is accepted."""
import numpy as np
import pytest

import oracle
import synth
from tests.gpu_helpers import assert_nodes, cuda

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _setup(reverse=False):
    from paper_2305_17813_b200 import Graph
    V = 1024
    s, d, w = synth.uniform(V, 8192)
    g = Graph(V, weighted=True, degree_hints=synth.degrees(s, V), reverse=reverse,
              in_degree_hints=synth.degrees(d, V) if reverse else None)
    o = oracle.OracleGraph(V)
    g.insert(cuda(s), cuda(d), cuda(w))
    o.insert(s, d, w)
    return g, o, V


def _fresh_batch(o, V, rng, n=64):
    es, ed, _ = o.edges()
    have = set(zip(es.tolist(), ed.tolist()))
    out = []
    while len(out) < n:
        a, b = int(rng.integers(0, V)), int(rng.integers(0, V))
        if a != b and (a, b) not in have:
            have.add((a, b))
            out.append((a, b))
    bs, bd = (np.array(c, np.uint32) for c in zip(*out))
    return bs, bd, rng.integers(1, 65, n).astype(np.uint32)


def _state_error(fn):
    from paper_2305_17813_b200._lib import E_STATE, MeerkatError
    with pytest.raises(MeerkatError) as ei:
        fn()
    assert ei.value.status == E_STATE, ei.value


@pytest.mark.parametrize("reverse", [False, True])
def test_wrong_batch_refused_on_device_and_tree_untouched(reverse):
    g, o, V = _setup(reverse)
    sp, bf = g.sssp(0), g.bfs(0)
    rng = np.random.default_rng(1)
    bs, bd, bw = _fresh_batch(o, V, rng)
    g.insert(cuda(bs), cuda(bd), cuda(bw))
    o.insert(bs, bd, bw)
    before_s, before_b = sp.nodes(), bf.nodes()
    # same size, different edges: the host checks pass, the kernel's fingerprint does not
    xs, xd, xw = _fresh_batch(o, V, rng)
    g.trees_incremental([sp, bf], cuda(xs), cuda(xd), cuda(xw))
    _state_error(g.sync)
    assert np.array_equal(sp.nodes(), before_s) and np.array_equal(bf.nodes(), before_b)
    # different weights only: the SSSP fingerprint includes them
    g2, o2, _ = _setup(reverse)
    t2 = g2.sssp(0)
    g2.insert(cuda(bs), cuda(bd), cuda(bw))
    g2.trees_incremental([t2], cuda(bs), cuda(bd), cuda(bw + 1))
    _state_error(g2.sync)
    # a stale tree refuses the next dynamic call too, until a static recompute
    ds, dd = bs[:16], bd[:16]
    g.delete(cuda(ds), cuda(dd))
    o.delete(ds, dd)
    g.trees_decremental([sp, bf], cuda(ds), cuda(dd))
    _state_error(g.sync)
    sp.recompute(); bf.recompute()
    assert_nodes(sp.nodes(), o.sssp(0)[1], "sssp after recompute")
    assert_nodes(bf.nodes(), o.bfs(0)[1], "bfs after recompute")
    # and dynamic calls work again afterwards
    bs, bd, bw = _fresh_batch(o, V, rng)
    g.insert(cuda(bs), cuda(bd), cuda(bw)); o.insert(bs, bd, bw)
    g.trees_incremental([sp, bf], cuda(bs), cuda(bd), cuda(bw))
    g.sync()
    assert_nodes(sp.nodes(), o.sssp(0)[1], "sssp"); assert_nodes(bf.nodes(), o.bfs(0)[1], "bfs")
    g.close(); g2.close()


def test_permuted_batch_is_the_same_batch():
    g, o, V = _setup()
    sp, bf = g.sssp(0), g.bfs(0)
    rng = np.random.default_rng(2)
    bs, bd, bw = _fresh_batch(o, V, rng)
    g.insert(cuda(bs), cuda(bd), cuda(bw)); o.insert(bs, bd, bw)
    p = rng.permutation(len(bs))
    g.trees_incremental([sp, bf], cuda(bs[p]), cuda(bd[p]), cuda(bw[p]))
    g.sync()
    assert_nodes(sp.nodes(), o.sssp(0)[1], "sssp"); assert_nodes(bf.nodes(), o.bfs(0)[1], "bfs")
    es, ed, _ = o.edges()
    pick = rng.choice(len(es), 48, replace=False)
    ds, dd = es[pick], ed[pick]
    g.delete(cuda(ds), cuda(dd)); o.delete(ds, dd)
    q = rng.permutation(len(ds))
    g.trees_decremental([sp, bf], cuda(ds[q]), cuda(dd[q]))   # delete fingerprint: (src, dst) only
    g.sync()
    assert_nodes(sp.nodes(), o.sssp(0)[1], "sssp"); assert_nodes(bf.nodes(), o.bfs(0)[1], "bfs")
    g.close()


def test_host_checks_size_kind_version():
    g, o, V = _setup()
    sp = g.sssp(0)
    rng = np.random.default_rng(3)
    bs, bd, bw = _fresh_batch(o, V, rng)
    g.insert(cuda(bs), cuda(bd), cuda(bw))
    # truncated batch: refused on the host, nothing launched
    _state_error(lambda: sp.incremental(cuda(bs[:-1]), cuda(bd[:-1]), cuda(bw[:-1])))
    # wrong kind
    _state_error(lambda: sp.decremental(cuda(bs), cuda(bd)))
    sp.incremental(cuda(bs), cuda(bd), cuda(bw))
    g.sync()
    # a second call with the same batch: the tree is already current
    _state_error(lambda: sp.incremental(cuda(bs), cuda(bd), cuda(bw)))
    # seeded calls: the batch prologue ran on the applied batch; only n is checked
    o.insert(bs, bd, bw)
    es, ed, _ = o.edges()
    ds, dd = es[:32], ed[:32]
    g.delete(cuda(ds), cuda(dd), seed=[sp]); o.delete(ds, dd)
    _state_error(lambda: sp.decremental(cuda(ds[:-1]), cuda(dd[:-1])))
    sp.decremental(cuda(ds), cuda(dd))
    g.sync()
    assert_nodes(sp.nodes(), o.sssp(0)[1], "sssp")
    g.close()


def test_wcc_incremental_checks():
    from paper_2305_17813_b200 import Graph
    V = 512
    s, d, w = synth.uniform(V, 2048)
    g = Graph(V, weighted=True, degree_hints=synth.degrees(s, V))
    g.insert(cuda(s), cuda(d), cuda(w))
    c = g.wcc()
    g.delete(cuda(s[:10]), cuda(d[:10]))
    _state_error(lambda: c.incremental(cuda(s[:10]), cuda(d[:10])))
    c.recompute()
    g.insert(cuda(s[:10]), cuda(d[:10]), cuda(w[:10]))
    _state_error(lambda: c.incremental(cuda(s[:9]), cuda(d[:9])))
    c.incremental(cuda(s[:10]), cuda(d[:10]))
    g.close()


def test_counters_async_and_latency_probe():
    """meerkat_counters_async: the cumulative insert / delete counters copied on the graph's stream
    (no synchronisation) equal the synchronous counts; meerkat_probe_latency returns plausible,
    positive latencies on the graph's device."""
    g, o, V = _setup()
    rng = np.random.default_rng(4)
    bs, bd, bw = _fresh_batch(o, V, rng)
    out = torch.zeros(3, dtype=torch.int64).pin_memory()
    n0 = g.stats()["edges"]
    g.insert(cuda(bs), cuda(bd), cuda(bw), count=False)
    g.delete(cuda(bs[:10]), cuda(bd[:10]), count=False)
    g.counters_async(out)
    torch.cuda.synchronize()
    ins, dele, pool = (int(x) for x in out.tolist())
    assert ins - dele == n0 + len(bs) - 10 == g.stats()["edges"]
    dev = torch.zeros(3, dtype=torch.int64, device="cuda")
    g.counters_async(dev)
    assert dev.cpu().tolist() == out.tolist()
    lat = g.probe_latency()
    assert 0 < lat["l2_load_ns"] < lat["dram_load_ns"] < 5000 and 0 < lat["grid_sync_us"] < 100
    assert lat["grid_blocks"] > 0
    g.close()

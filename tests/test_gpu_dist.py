"""Vertex-partitioned (multi-GPU) path against the oracle.

The box has one GPU, so world_size 2 and 3 run as separate processes sharing
cuda:0 and exchanging through host memory (gloo); the partition logic, the
phase kernels, routing and termination are the ones NCCL drives on 8 GPUs.
world_size 1 runs through NCCL.  Every result must be bit-identical to the
oracle (edge set, counts, query answers, SSSP and BFS nodes after every batch)."""
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, backend, scale, q):
    import torch.distributed as dist
    try:
        torch.cuda.set_device(0)
        kw = {"device_id": torch.device("cuda", 0)} if backend == "nccl" else {}
        dist.init_process_group(backend, init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=ws, **kw)
        import oracle
        import synth
        from paper_2305_17813_b200.dist import DistGraph
        W = synth.rmat_dynamic(scale, 16, batch=500, n_ins=2, n_del=2)
        V, src = W.vertex_n, W.source
        bs, bd, bw = W.base
        # each rank brings a different slice of every batch (routing must gather them)
        sl = lambda a: a[rank::ws]
        g = DistGraph(V, degree_hints=synth.degrees(bs, V), device=torch.device("cuda", 0))
        o = oracle.OracleGraph(V)
        n = g.insert(sl(bs), sl(bd), sl(bw))
        assert n == o.insert(bs, bd, bw)[1], "bulk insert count"
        t, b = g.sssp(src), g.bfs(src)
        errs = []

        def check(tag):
            gs, gb = t.nodes(), b.nodes()
            if rank == 0:
                rs, rb = o.sssp(src)[1], o.bfs(src)[1]
                if not np.array_equal(gs, rs):
                    errs.append(f"{tag} sssp: {int((gs != rs).sum())} mismatches")
                if not np.array_equal(gb, rb):
                    errs.append(f"{tag} bfs: {int((gb != rb).sum())} mismatches")

        check("static")
        for i, (s, d, w) in enumerate(W.inserts):
            n = g.insert(sl(s), sl(d), sl(w))
            assert n == o.insert(s, d, w)[1]
            if i % 2 == 0:   # fused lock-step update of both trees (DistGraph.trees_incremental)
                g.trees_incremental([t, b], sl(s), sl(d), sl(w))
            else:
                t.incremental(sl(s), sl(d), sl(w))
                b.incremental(sl(s), sl(d))
            check(f"inc{i}")
        for i, (s, d, _w) in enumerate(W.deletes):
            n = g.delete(sl(s), sl(d))
            assert n == o.delete(s, d)[1]
            if i % 2 == 0:
                g.trees_decremental([t, b], sl(s), sl(d))
            else:
                t.decremental(sl(s), sl(d))
                b.decremental(sl(s), sl(d))
            check(f"dec{i}")
        # queries in the caller's order, across partitions
        es, ed, ew = o.edges()
        rng = np.random.default_rng(rank)
        qs = np.concatenate([es[:300], rng.integers(0, V, 300)]).astype(np.uint32)
        qd = np.concatenate([ed[:300], rng.integers(0, V, 300)]).astype(np.uint32)
        f, qw = g.query(qs, qd)
        _, ef, eww = o.query(qs, qd)
        if not (np.array_equal(f.cpu().numpy(), ef) and np.array_equal(qw.cpu().numpy().view(np.uint32), eww)):
            errs.append("query answers")
        gs, gd, gw = g.export_edges()
        if rank == 0 and not (np.array_equal(gs, es) and np.array_equal(gd, ed) and np.array_equal(gw, ew)):
            errs.append("edge set")
        q.put((rank, errs))
    except Exception:  # pragma: no cover
        import traceback
        q.put((rank, [traceback.format_exc()]))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


@pytest.mark.parametrize("ws,backend,scale", [(1, "nccl", 12), (2, "gloo", 12), (3, "gloo", 13), (4, "gloo", 12),
                                             (8, "gloo", 12)])
def test_partitioned_dynamic_sssp_bfs(ws, backend, scale):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, ws, port, backend, scale, q)) for r in range(ws)]
    for p in ps:
        p.start()
    res = [q.get(timeout=600) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    for r, errs in res:
        assert not errs, f"rank {r}: {errs}"

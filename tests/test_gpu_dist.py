"""Vertex-partitioned (multi-GPU) path against the oracle.

The box has one GPU, so world_size 2..8 run as separate processes sharing
cuda:0 whose library exchanges through host memory (the gloo host transport);
routing, the exchange units, the device-side phase changes and termination are
the ones the NCCL transport drives on 8 GPUs.  world_size 1 runs with the
library's own NCCL communicator.  Every result must be bit-identical to the
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


def _worker(rank, ws, port, backend, scale, reverse, pairs, q, units=False):
    import os
    import torch.distributed as dist
    if units:   # one exchange unit per phase at world size 1: the P > 1 protocol and host pipeline
        os.environ["MEERKAT_PART_UNITS"] = "1"
    if units == "nccl_self":   # ... with the rank's own blocks and segments through ncclSend / ncclRecv
        os.environ["MEERKAT_PART_NCCL_SELF"] = "1"
    try:
        torch.cuda.set_device(0)
        kw = {"device_id": torch.device("cuda", 0)} if backend == "nccl" else {}
        dist.init_process_group(backend, init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=ws, **kw)
        import oracle
        import synth
        from paper_2305_17813_b200.dist import DistGraph
        if isinstance(scale, str):   # "grid<side>": the road-like stress case (deep trees, many units)
            W = synth.grid_dynamic(int(scale[4:]), 500, 2, 2)
        else:
            W = synth.rmat_dynamic(scale, 16, batch=500, n_ins=2, n_del=2)
        V, src = W.vertex_n, W.source
        bs, bd, bw = W.base
        # each rank brings a different slice of every batch (the library routes them)
        sl = lambda a: a[rank::ws]
        g = DistGraph(V, degree_hints=synth.degrees(bs, V), in_degree_hints=synth.degrees(bd, V) if reverse else None,
                      reverse=reverse, device=torch.device("cuda", 0), exchange_pairs=pairs)
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
            if i % 2 == 0:   # fused lock-step update of both trees
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
            st = t.stats()
            if (ws > 1 or units) and st["exchanges"] < 2:
                errs.append(f"dec{i}: {st['exchanges']} exchanges")
        # queries in the caller's order, across partitions
        es, ed, ew = o.edges()
        rng = np.random.default_rng(rank)
        qs = np.concatenate([es[:300], rng.integers(0, V, 300)]).astype(np.uint32)
        qd = np.concatenate([ed[:300], rng.integers(0, V, 300)]).astype(np.uint32)
        f, qw = g.query(qs, qd)
        _, ef, eww = o.query(qs, qd)
        if not (np.array_equal(np.asarray(f), ef) and np.array_equal(np.asarray(qw).view(np.uint32), eww)):
            errs.append("query answers")
        gs, gd, gw = g.export_edges()
        if rank == 0 and not (np.array_equal(gs, es) and np.array_equal(gd, ed) and np.array_equal(gw, ew)):
            errs.append("edge set")
        # static recompute equals the maintained trees
        before = t.nodes()
        t.recompute()
        after = t.nodes()   # collective: every rank calls it
        if rank == 0 and not np.array_equal(before, after):
            errs.append("recompute")
        # ordering contract: a different batch than the last mutation's -- on one rank only -- is refused
        # on every rank before any tree is touched; the right batch is then accepted
        from paper_2305_17813_b200._lib import MeerkatError
        s, d, w = W.inserts[0]
        s, d, w = s[:60] ^ 1, d[:60], w[:60]   # edges not in the graph (ids flipped in the low bit)
        g.insert(sl(s), sl(d), sl(w))
        o.insert(s, d, w)
        wrong = (sl(s[::-1]), sl(d), sl(w)) if rank == 0 else (sl(s), sl(d), sl(w))
        try:
            t.incremental(*wrong)
            errs.append("wrong batch accepted")
        except MeerkatError as e:
            if "STATE" not in str(e):
                errs.append(f"wrong batch: {e}")
        t.incremental(sl(s), sl(d), sl(w))
        gs = t.nodes()
        if rank == 0 and not np.array_equal(gs, o.sssp(src)[1]):
            errs.append("after a refused batch")
        q.put((rank, errs))
    except Exception:  # pragma: no cover
        import traceback
        q.put((rank, [traceback.format_exc()]))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


# world_size, backend, R-MAT scale, in-edge mirror (pull frontier) or the paper's scan, messages
# per peer per exchange (small values force carry-over across exchanges)
@pytest.mark.parametrize("ws,backend,scale,reverse,pairs", [
    (1, "nccl", 12, False, 0), (1, "nccl", 12, True, 0), (2, "gloo", 12, False, 0), (2, "gloo", 12, True, 0),
    (3, "gloo", 13, True, 0), (4, "gloo", 12, False, 0), (4, "gloo", 12, True, 64), (8, "gloo", 12, True, 0),
    (8, "gloo", 12, False, 32), (3, "gloo", "grid64", True, 0), (2, "gloo", "grid64", False, 0)])
def test_partitioned_dynamic_sssp_bfs(ws, backend, scale, reverse, pairs):
    _run(ws, backend, scale, reverse, pairs)


@pytest.mark.parametrize("reverse,self_nccl", [(True, False), (False, False), (True, True)])
def test_partitioned_nccl_unit_pipeline(reverse, self_nccl):
    """World size 1 through the library's NCCL communicator with one exchange unit per phase
    (MEERKAT_PART_UNITS=1): the pipelined host loop (units launched PIPE ahead, mode words read from
    mapped memory) and the device-side phase changes of P > 1, on one GPU; with self_nccl
    (MEERKAT_PART_NCCL_SELF=1) every own segment and unit block also moves through ncclSend / ncclRecv
    to the rank itself, so the NCCL calls of the P > 1 path run with real data."""
    _run(1, "nccl", 12, reverse, 0, units="nccl_self" if self_nccl else True)


def _run(ws, backend, scale, reverse, pairs, units=False):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, ws, port, backend, scale, reverse, pairs, q, units))
          for r in range(ws)]
    for p in ps:
        p.start()
    res = [q.get(timeout=900) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    for r, errs in res:
        assert not errs, f"rank {r}: {errs}"

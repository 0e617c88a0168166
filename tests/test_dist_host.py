"""Host-side logic of the multi-GPU path on CPU (gloo, world_size 2): the
variable-size exchanges, the all-gather of invalid sets, the frontier-size
all-reduce and the owner / interleave arithmetic."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, q):
    try:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=ws)
        from paper_2305_17813_b200.dist import Transport
        tp = Transport(None, torch.device("cpu"))
        assert tp.staged and tp.ws == ws and tp.rank == rank
        # alltoallv: rank r sends (r+1)*(d+1) rows of 2 values to rank d, value = 100*r + d
        counts = [(rank + 1) * (d + 1) for d in range(ws)]
        send = torch.cat([torch.full(((rank + 1) * (d + 1) * 2,), 100 * rank + d, dtype=torch.int64) for d in range(ws)])
        recv, rc = tp.alltoallv(send, counts, elem=2)
        assert rc == [(s + 1) * (rank + 1) for s in range(ws)]
        exp = torch.cat([torch.full(((s + 1) * (rank + 1) * 2,), 100 * s + rank, dtype=torch.int64) for s in range(ws)])
        assert torch.equal(recv, exp)
        # known counts (no count exchange)
        rk = tp.alltoallv_known(send, counts, [(s + 1) * (rank + 1) for s in range(ws)], elem=2)
        assert torch.equal(rk, exp)
        # empty exchange
        recv, rc = tp.alltoallv(torch.empty(0, dtype=torch.int64), [0] * ws, elem=2)
        assert recv.numel() == 0 and rc == [0] * ws
        # all-gather of different lengths
        parts = tp.allgather_var(torch.arange(rank * 3, dtype=torch.int32))
        assert [p.tolist() for p in parts] == [list(range(r * 3)) for r in range(ws)]
        assert tp.allreduce_sum(rank + 1) == ws * (ws + 1) // 2
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def test_transport_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    for r, msg in res:
        assert msg == "ok", msg


def test_owner_and_interleave():
    from paper_2305_17813_b200.dist import interleave, local_count, owner_of
    V, ws = 23, 4
    v = np.arange(V)
    own = owner_of(v, ws)
    assert sorted(np.bincount(own).tolist()) == sorted(local_count(V, ws, r) for r in range(ws))
    parts = [v[r::ws].astype(np.uint64) * 10 for r in range(ws)]
    assert interleave(parts, ws, V).tolist() == (v * 10).tolist()
    assert sum(local_count(V, ws, r) for r in range(ws)) == V

#!/usr/bin/env python
"""Large-batch update kernels (GPU diagnostics, not a test): R-MAT --scale graph with the in-edge mirror,
one insert and one delete batch of --batch edges (thread-per-edge kernels), optionally seeding a BFS
tree; CUDA-event times and the store counters.  Used with ncu to profile k_insert_t / k_delete_t.

    python tools/big_batch.py [--scale 24] [--batch 10000000] [--seed-bfs]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=24)
    ap.add_argument("--batch", type=int, default=10_000_000)
    ap.add_argument("--seed-bfs", action="store_true")
    ap.add_argument("--weighted", action="store_true")
    a = ap.parse_args()
    import torch
    import synth
    from paper_2305_17813_b200 import Graph
    W = synth.rmat_dynamic(a.scale, 16, batch=a.batch, n_ins=1, n_del=1)
    s, d, w = W.base
    V = W.vertex_n
    T = lambda x: torch.from_numpy(np.ascontiguousarray(x, np.uint32).view(np.int32)).cuda()
    stream = torch.cuda.current_stream()
    g = Graph(V, weighted=a.weighted, degree_hints=T(synth.degrees(s, V)), in_degree_hints=T(synth.degrees(d, V)),
              reverse=True, stream=stream)
    g.insert(T(s), T(d), T(w) if a.weighted else None, count=False)
    bf = g.bfs(W.source) if a.seed_bfs else None
    st0 = g.stats()
    ev = lambda: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    bs, bd, bw = (T(x) for x in W.inserts[0])
    e0, e1 = ev()
    torch.cuda.synchronize()
    e0.record(stream)
    g.insert(bs, bd, bw if a.weighted else None, count=False, seed=[bf] if bf else None)
    e1.record(stream); e1.synchronize()
    t_ins = e0.elapsed_time(e1)
    if bf:
        g.trees_incremental([bf], bs, bd)
    st1 = g.stats()
    ds, dd = (T(x) for x in W.deletes[0][:2])
    e0, e1 = ev()
    torch.cuda.synchronize()
    e0.record(stream)
    g.delete(ds, dd, count=False, seed=[bf] if bf else None)
    e1.record(stream); e1.synchronize()
    t_del = e0.elapsed_time(e1)
    if bf:
        g.trees_decremental([bf], ds, dd)
    g.sync()
    print(json.dumps({"scale": a.scale, "batch": a.batch, "insert_ms": t_ins, "delete_ms": t_del,
                      "insert_edges_per_s": a.batch / (t_ins / 1e3), "delete_edges_per_s": a.batch / (t_del / 1e3),
                      "pool_slabs_taken": st1["pool_used"] - st0["pool_used"],
                      "in_pool_slabs_taken": st1["in_pool_used"] - st0["in_pool_used"]}))
    g.close()


if __name__ == "__main__":
    main()

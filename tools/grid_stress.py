#!/usr/bin/env python
"""Road-like stress case of SURVEY §8(d) (not a BASELINE config): a side x side grid with 4 out-edges per
vertex (diameter ~2*side), static SSSP / BFS and 10K-edge incremental / decremental batches through the
bench's sequence (seeded insert / delete + fused trees, in-edge mirror), timed with CUDA events; the
BFS tree of the first and last batch certified against the oracle when --check.

    python tools/grid_stress.py [--side 2048] [--batch 10000] [--check]
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
    ap.add_argument("--side", type=int, default=2048)
    ap.add_argument("--batch", type=int, default=10_000)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--check", action="store_true")
    a = ap.parse_args()
    import torch
    import synth
    from paper_2305_17813_b200 import Graph
    W = synth.grid_dynamic(a.side, a.batch, a.steps, a.steps)
    V, src = W.vertex_n, W.source
    T = lambda x: torch.from_numpy(np.ascontiguousarray(x, np.uint32).view(np.int32)).cuda()
    s, d, w = W.base
    st = torch.cuda.current_stream()
    g = Graph(V, degree_hints=T(synth.degrees(s, V)), in_degree_hints=T(synth.degrees(d, V)), reverse=True,
              load_factor=0.5, stream=st)
    g.insert(T(s), T(d), T(w), count=False)
    ev = lambda: torch.cuda.Event(enable_timing=True)
    res = {"side": a.side, "vertices": V, "edges": int(len(s)), "batch": a.batch}
    e0, e1 = ev(), ev()
    e0.record(st); sp = g.sssp(src); e1.record(st); e1.synchronize()
    res["static_sssp_ms"] = e0.elapsed_time(e1)
    e0.record(st); bf = g.bfs(src); e1.record(st); e1.synchronize()
    res["static_bfs_ms"] = e0.elapsed_time(e1)
    res["static_rounds"] = {"sssp": sp.stats()["rounds"], "bfs": bf.stats()["rounds"]}
    calls = {"insert": [], "trees_inc": [], "delete": [], "trees_dec": []}
    dec = []
    for k in range(a.steps):
        (si, di, wi), (sd, dd, _) = W.inserts[k], W.deletes[k]
        si, di, wi, sd, dd = T(si), T(di), T(wi), T(sd), T(dd)
        es = [ev() for _ in range(5)]
        es[0].record(st)
        g.insert(si, di, wi, count=False, seed=[sp, bf]); es[1].record(st)
        g.trees_incremental([sp, bf], si, di, wi); es[2].record(st)
        g.delete(sd, dd, count=False, seed=[sp, bf]); es[3].record(st)
        g.trees_decremental([sp, bf], sd, dd); es[4].record(st)
        es[4].synchronize()
        for j, n in enumerate(calls):
            calls[n].append(es[j].elapsed_time(es[j + 1]))
        x = sp.stats()
        dec.append({"invalidated_sssp": x["invalidated"], "propagate_rounds": x["propagate_rounds"],
                    "relax_rounds": x["rounds"], "frontier_edges": x["frontier_edges"]})
    res["per_call_ms"] = {n: float(np.median(v)) for n, v in calls.items()}
    res["decremental"] = dec
    if a.check:
        import oracle
        o = oracle.OracleGraph(V)
        o.insert(*W.base)
        for k in range(a.steps):
            o.insert(*W.inserts[k]); o.delete(*W.deletes[k][:2])
        res["bfs_last_batch_ok"] = bool(np.array_equal(bf.nodes(), o.bfs(src)[1]))
    print(json.dumps(res))


if __name__ == "__main__":
    main()

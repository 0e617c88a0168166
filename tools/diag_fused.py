#!/usr/bin/env python
"""Device timeline of the fused, seeded tree calls bench.py times (GPU diagnostics, not a test).

Builds the config-3 workload (R-MAT scale 24, in-edge mirror), runs a few steps of the bench sequence
(seeded insert -> trees_incremental -> seeded delete -> trees_decremental) and prints, per tree call,
every interval between grid barriers in us with the frontier items of that round (0 = a non-round
phase: batch prologue, pull-frontier enqueue, ...), the call's counters, and the measured latency probe.

    python tools/diag_fused.py [--scale 24] [--steps 3]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=24)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--batch", type=int, default=100_000)
    a = ap.parse_args()
    import torch
    import synth
    from paper_2305_17813_b200 import Graph
    W = synth.rmat_dynamic(a.scale, 16, batch=a.batch, n_ins=a.steps, n_del=a.steps)
    s, d, w = W.base
    V = W.vertex_n
    T = lambda x: torch.from_numpy(np.ascontiguousarray(x, np.uint32).view(np.int32)).cuda()
    g = Graph(V, degree_hints=T(synth.degrees(s, V)), in_degree_hints=T(synth.degrees(d, V)), reverse=True,
              stream=torch.cuda.current_stream())
    g.insert(T(s), T(d), T(w), count=False)
    sp, bf = g.sssp(W.source), g.bfs(W.source)
    print("probe", {k: round(v, 3) if isinstance(v, float) else v for k, v in g.probe_latency().items()})
    fmt = lambda tl: " ".join(f"{us:.1f}" + (f"[{n}]" if n else "") for us, n in tl)
    for i in range(a.steps):
        bs, bd, bw = (T(x) for x in W.inserts[i])
        g.insert(bs, bd, bw, count=False, seed=[sp, bf])
        g.trees_incremental([sp, bf], bs, bd, bw)
        torch.cuda.synchronize()
        tl, st = sp.timeline(items=True), sp.stats()
        print(f"step {i} trees_inc: {sum(x for x, _ in tl):.1f} us, rounds {st['rounds']} items {st['items']} "
              f"slabs {st['slabs_read']} improved {st['improved']}\n   {fmt(tl)}")
        ds, dd = (T(x) for x in W.deletes[i][:2])
        g.delete(ds, dd, count=False, seed=[sp, bf])
        g.trees_decremental([sp, bf], ds, dd)
        torch.cuda.synchronize()
        tl, st, st2 = sp.timeline(items=True), sp.stats(), bf.stats()
        print(f"step {i} trees_dec: {sum(x for x, _ in tl):.1f} us, prop {st['propagate_rounds']} rounds "
              f"{st['rounds']} items {st['items']} slabs {st['slabs_read']} improved {st['improved']} "
              f"invalid sssp/bfs {st['invalidated']}/{st2['invalidated']} frontier {st['frontier_edges']}/"
              f"{st2['frontier_edges']}\n   {fmt(tl)}")
    g.close()


if __name__ == "__main__":
    main()

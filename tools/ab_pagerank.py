#!/usr/bin/env python
"""PageRank timing on the config-3 graph (GPU; A/B of library builds via MEERKAT_SO_PATH, not a test):
static run (cold start) and a dynamic run after a 100 K-edge insert batch; CUDA events, L2 flushed.

    MEERKAT_SO_PATH=... python tools/ab_pagerank.py [--scale 24] [--reps 3]
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
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    import torch
    import synth
    from paper_2305_17813_b200 import Graph
    W = synth.rmat_dynamic(a.scale, 16, batch=100_000, n_ins=1, n_del=0)
    s, d, w = W.base
    V = W.vertex_n
    T = lambda x: torch.from_numpy(np.ascontiguousarray(x, np.uint32).view(np.int32)).cuda()
    stream = torch.cuda.current_stream()
    g = Graph(V, degree_hints=T(synth.degrees(s, V)), in_degree_hints=T(synth.degrees(d, V)), reverse=True,
              stream=stream)
    g.insert(T(s), T(d), T(w), count=False)
    p = g.pagerank(0.85, 1e-5, 1000)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ev = lambda: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    st = []
    for _ in range(a.reps):
        flush.zero_()
        e0, e1 = ev()
        e0.record(stream); p.recompute(); e1.record(stream); e1.synchronize()
        st.append(e0.elapsed_time(e1))
    stats = p.stats()
    bs, bd, bw = (T(x) for x in W.inserts[0])
    g.insert(bs, bd, bw, count=False)
    flush.zero_()
    e0, e1 = ev()
    e0.record(stream); p.update(); e1.record(stream); e1.synchronize()
    inc = e0.elapsed_time(e1)
    out = {"so": os.environ.get("MEERKAT_SO_PATH", "default"), "static_ms": st, "iterations": stats["iterations"],
           "ms_per_iteration": float(np.median(st)) / stats["iterations"], "alg_bytes": stats["alg_bytes"],
           "GBps_alg": stats["alg_bytes"] / (float(np.median(st)) * 1e-3) / 1e9, "incremental_ms": inc,
           "values_sum": float(p.values().sum())}
    print(json.dumps(out))
    g.close()


if __name__ == "__main__":
    main()

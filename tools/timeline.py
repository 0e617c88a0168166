#!/usr/bin/env python
"""Per-round device timeline of the tree kernels on the bench workload (GPU)."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2305_17813_b200 import Graph  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=24)
ap.add_argument("--batch", type=int, default=100000)
ap.add_argument("--frontier", default="reverse")
ap.add_argument("--steps", type=int, default=3)
a = ap.parse_args()
W = synth.rmat_dynamic(a.scale, 16, batch=a.batch, n_ins=a.steps + 1, n_del=a.steps + 1)
V = W.vertex_n
dev = torch.device("cuda:0")
T = lambda x: torch.from_numpy(np.ascontiguousarray(x, np.uint32).view(np.int32)).to(dev)
bs, bd, bw = W.base
rev = a.frontier == "reverse"
g = Graph(V, degree_hints=T(np.bincount(bs, minlength=V).astype(np.uint32)), reverse=rev,
          in_degree_hints=T(np.bincount(bd, minlength=V).astype(np.uint32)) if rev else None)
g.insert(T(bs), T(bd), T(bw))
sp, bf = g.sssp(W.source), g.bfs(W.source)
fmt = lambda xs: " ".join(f"{x:.1f}" for x in xs)
print("static sssp", fmt(sp.timeline()))
st = torch.cuda.current_stream()


def timed(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    fn()
    e1.record(st)
    e1.synchronize()
    return 1e3 * e0.elapsed_time(e1)


for i in range(a.steps + 1):
    s, d, w = (T(x) for x in W.inserts[i])
    g.insert(s, d, w, count=False)
    ev1 = timed(lambda: sp.incremental(s, d, w)); t1 = sp.timeline()
    ev2 = timed(lambda: bf.incremental(s, d)); t2 = bf.timeline()
    s, d = (T(x) for x in W.deletes[i][:2])
    g.delete(s, d, count=False)
    ev3 = timed(lambda: sp.decremental(s, d)); t3 = sp.timeline(); st3 = sp.stats()
    ev4 = timed(lambda: bf.decremental(s, d)); t4 = bf.timeline()
    if i:
        print(f"step {i}: sssp_inc event {ev1:.1f} us, in-kernel {sum(t1):.1f} us: {fmt(t1)}")
        print(f"        bfs_inc  event {ev2:.1f} us, in-kernel {sum(t2):.1f} us: {fmt(t2)}")
        print(f"        sssp_dec event {ev3:.1f} us, in-kernel {sum(t3):.1f} us (prop {st3['propagate_rounds']}, "
              f"relax {st3['rounds']}): {fmt(t3)}")
        print(f"        bfs_dec  event {ev4:.1f} us, in-kernel {sum(t4):.1f} us: {fmt(t4)}")

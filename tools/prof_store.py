#!/usr/bin/env python
"""Config-2 store kernels in isolation (for ncu): R-MAT scale 20 graph, then one batch each of
insert (fresh draws), delete (present edges) and query, at --batch edges."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2305_17813_b200 import Graph  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=20)
ap.add_argument("--batch", type=int, default=1000000)
ap.add_argument("--no-hashing", action="store_true")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
dev = torch.device("cuda:0")
T = lambda x: torch.from_numpy(np.ascontiguousarray(x, np.uint32).view(np.int32)).to(dev)
s, d, w = synth.rmat(a.scale, 16)
V = 1 << a.scale
g = Graph(V, hashing=not a.no_hashing, degree_hints=T(np.bincount(s, minlength=V).astype(np.uint32)))
g.insert(T(s), T(d), T(w))
for r in range(a.reps):
    fs, fd, fw = synth.rmat_draws(a.scale, a.batch, r * a.batch, 11, scramble_seed=11)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ins = (T(fs), T(fd), T(fw))
    torch.cuda.synchronize()
    e0.record(); n = g.insert(*ins); e1.record(); e1.synchronize()
    pick = synth.sample_distinct(len(s), a.batch, 100 + r)
    ds, dd = T(s[pick]), T(d[pick])
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record(); m = g.delete(ds, dd); e3.record(); e3.synchronize()
    print(f"rep {r}: insert {e0.elapsed_time(e1):.3f} ms ({n} new), delete {e2.elapsed_time(e3):.3f} ms ({m})",
          g.stats())

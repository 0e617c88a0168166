#!/usr/bin/env python
"""Concurrency stress of the slab store: repeated large fresh-draw insert / present-edge delete
batches on R-MAT, with meerkat_check (structural fsck) after every kernel and the edge set
compared with the oracle at the end."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2305_17813_b200 import Graph  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=18)
ap.add_argument("--batch", type=int, default=300000)
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--no-hashing", action="store_true")
ap.add_argument("--oracle", action="store_true")
a = ap.parse_args()
dev = torch.device("cuda:0")
T = lambda x: torch.from_numpy(np.ascontiguousarray(x, np.uint32).view(np.int32)).to(dev)
s, d, w = synth.rmat(a.scale, 16)
V = 1 << a.scale
g = Graph(V, hashing=not a.no_hashing, degree_hints=T(np.bincount(s, minlength=V).astype(np.uint32)))
o = None
if a.oracle:
    import oracle
    o = oracle.OracleGraph(V)
    o.insert(s, d, w)
g.insert(T(s), T(d), T(w))
print("bulk", g.check(), flush=True)
for r in range(a.reps):
    fs, fd, fw = synth.rmat_draws(a.scale, a.batch, r * a.batch, 11, scramble_seed=11)
    n = g.insert(T(fs), T(fd), T(fw))
    c = g.check()
    print(f"rep {r} insert {n} check {c}", flush=True)
    if o is not None:
        assert n == o.insert(fs, fd, fw)[1]
    if c[0]:
        sys.exit(1)
    pick = synth.sample_distinct(len(s), a.batch, 100 + r)
    m = g.delete(T(s[pick]), T(d[pick]))
    c = g.check()
    print(f"rep {r} delete {m} check {c}", flush=True)
    if o is not None:
        assert m == o.delete(s[pick], d[pick])[1]
    if c[0]:
        sys.exit(1)
if o is not None:
    gs, gd, gw = g.export_edges()
    es, ed, ew = o.edges()
    print("edge set equal:", np.array_equal(gs, es) and np.array_equal(gd, ed) and np.array_equal(gw, ew))

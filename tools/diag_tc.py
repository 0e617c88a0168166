"""TC static timing repeatability (GPU): build the symmetrised scale-20 R-MAT graph, run tc_static 4x."""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch, synth
from paper_2305_17813_b200 import Graph
T = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.uint32).view(np.int32)).cuda()
rs, rd, _ = synth.rmat(20, 16)
k = np.unique(np.concatenate([(rs.astype(np.uint64) << np.uint64(32)) | rd, (rd.astype(np.uint64) << np.uint64(32)) | rs]))
s, d = (k >> np.uint64(32)).astype(np.uint32), (k & np.uint64(0xFFFFFFFF)).astype(np.uint32)
keep = s != d; s, d = s[keep], d[keep]
V = 1 << 20
for hashing in (True, False):
    g = Graph(V, weighted=False, hashing=hashing, degree_hints=T(np.bincount(s, minlength=V).astype(np.uint32)))
    g.insert(T(s), T(d)); g.sync()
    for r in range(4):
        t0 = time.perf_counter(); tri = g.tc_static(); dt = time.perf_counter() - t0
        print(f"hashing={hashing} run {r}: {tri} triangles {1e3*dt:.1f} ms")
    # count over the exported edge list sorted by (src, dst) vs shuffled
    es, ed, _ = g.export_edges()
    for name, perm in (("sorted", np.arange(len(es))), ("shuffled", np.random.default_rng(0).permutation(len(es)))):
        torch.cuda.synchronize(); t0 = time.perf_counter(); c = g.tc_count(g, T(es[perm]), T(ed[perm])); dt = time.perf_counter() - t0
        print(f"  count {name}: {c} in {1e3*dt:.1f} ms")
    g.close()

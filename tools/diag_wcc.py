"""Debug helper: compare GPU WCC labels with the oracle on a sparse random graph."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle, synth
from tests.gpu_helpers import cuda
from paper_2305_17813_b200 import Graph
rng = np.random.default_rng(2)
V = 20000
s, d = rng.integers(0, V, 12000).astype(np.uint32), rng.integers(0, V, 12000).astype(np.uint32)
for hashing in (True, False):
    g = Graph(V, weighted=False, hashing=hashing, degree_hints=synth.degrees(s, V))
    g.insert(cuda(s), cuda(d))
    o = oracle.OracleGraph(V, weighted=False); o.insert(s, d)
    c = g.wcc(); lab = c.labels(); ref, k = o.wcc()
    bad = np.nonzero(lab != ref)[0]
    print("hashing", hashing, "mismatch", len(bad), "gpu comps", len(np.unique(lab)), "oracle", k)
    print(" edges inconsistent:", int((lab[s] != lab[d]).sum()), " label>v:", int((lab > np.arange(V)).sum()),
          " non-root labels:", int((lab[lab] != lab).sum()))
    print(" first bad:", [(int(v), int(lab[v]), int(ref[v])) for v in bad[:5]])
    es, ed, _ = g.export_edges(); os_, od, _ = o.edges()
    print(" export edges equal:", len(es) == len(os_) and np.array_equal(es, os_) and np.array_equal(ed, od))
    print(" stats", g.stats())

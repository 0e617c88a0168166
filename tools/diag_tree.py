#!/usr/bin/env python
"""Where does a latency-bound tree call spend its rounds?  (GPU; diagnostics only, not a test.)

Builds the bench workload (R-MAT scale 24 by default, in-edge mirror), then for a few batch pairs
runs the per-tree SSSP incremental / decremental calls and prints, per call: the device timeline
(us between grid barriers), tree statistics, and the bucket (slab-list) counts of the vertices whose
node changed / that were invalidated — the enqueue and expansion work of hubs.

    python tools/diag_tree.py [--scale 24] [--batches 3]
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
    ap.add_argument("--batches", type=int, default=3)
    ap.add_argument("--batch", type=int, default=100_000)
    a = ap.parse_args()
    import torch
    import synth
    from paper_2305_17813_b200 import Graph
    W = synth.rmat_dynamic(a.scale, 16, batch=a.batch, n_ins=a.batches, n_del=a.batches)
    s, d, w = W.base
    V = W.vertex_n
    T = lambda x: torch.from_numpy(np.ascontiguousarray(x, np.uint32).view(np.int32)).cuda()
    outdeg = synth.degrees(s, V)
    indeg = synth.degrees(d, V)
    g = Graph(V, degree_hints=T(outdeg), in_degree_hints=T(indeg), reverse=True)
    g.insert(T(s), T(d), T(w))
    sp = g.sssp(W.source)
    bk_out = np.maximum(1, np.ceil(outdeg / (0.7 * 15))).astype(np.int64)
    bk_in = np.maximum(1, np.ceil(indeg / (0.7 * 15))).astype(np.int64)

    def show(name, changed, bk):
        b = bk[changed]
        top = np.sort(b)[::-1][:8]
        print(f"  {name}: {len(changed)} vertices, buckets sum {int(b.sum())}, top {top.tolist()}")

    for i in range(a.batches):
        n0 = sp.nodes()
        bs, bd, bw = W.inserts[i]
        g.insert(T(bs), T(bd), T(bw), count=False)
        sp.incremental(T(bs), T(bd), T(bw))
        torch.cuda.synchronize()
        n1 = sp.nodes()
        st = sp.stats()
        tl = sp.timeline()
        print(f"batch {i} sssp_inc: rounds {st['rounds']} items {st['items']} slabs {st['slabs_read']} "
              f"improved {st['improved']} timeline {[round(x, 1) for x in tl]}")
        show("changed", np.nonzero(n0 != n1)[0], bk_out)
        ds, dd, _ = W.deletes[i]
        g.delete(T(ds), T(dd), count=False)
        sp.decremental(T(ds), T(dd))
        torch.cuda.synchronize()
        n2 = sp.nodes()
        st = sp.stats()
        tl = sp.timeline()
        inv = sp.invalidated()
        print(f"batch {i} sssp_dec: prop {st['propagate_rounds']} rounds {st['rounds']} items {st['items']} "
              f"slabs {st['slabs_read']} improved {st['improved']} frontier {st['frontier_edges']} "
              f"timeline {[round(x, 1) for x in tl]}")
        show("invalidated (out buckets)", inv, bk_out)
        show("invalidated (in buckets)", inv, bk_in)
        show("changed", np.nonzero(n1 != n2)[0], bk_out)


if __name__ == "__main__":
    main()

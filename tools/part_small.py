#!/usr/bin/env python
"""Small single-process run of the partitioned engine (world size 1, gloo host transport) against the
oracle, for compute-sanitizer: routed insert / delete / query, static + fused / per-tree dynamic SSSP and
BFS, mirror (pull) and scan frontiers.  MEERKAT_PART_UNITS=1 runs one exchange unit per phase.

    python tools/part_small.py [--scale 10] [--reverse 0|1]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=10)
    ap.add_argument("--reverse", type=int, default=1)
    a = ap.parse_args()
    import torch
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29561")
    dist.init_process_group("gloo", rank=0, world_size=1)
    import oracle
    import synth
    from paper_2305_17813_b200.dist import DistGraph
    W = synth.rmat_dynamic(a.scale, 16, batch=200, n_ins=2, n_del=2)
    V, src = W.vertex_n, W.source
    bs, bd, bw = W.base
    g = DistGraph(V, degree_hints=synth.degrees(bs, V), in_degree_hints=synth.degrees(bd, V) if a.reverse else None,
                  reverse=bool(a.reverse), device=torch.device("cuda", 0), transport="host")
    o = oracle.OracleGraph(V)
    assert g.insert(bs, bd, bw) == o.insert(bs, bd, bw)[1]
    t, b = g.sssp(src), g.bfs(src)
    bad = []
    chk = lambda tag: bad.extend([f"{tag} sssp"] if not np.array_equal(t.nodes(), o.sssp(src)[1]) else []) or \
        bad.extend([f"{tag} bfs"] if not np.array_equal(b.nodes(), o.bfs(src)[1]) else [])
    chk("static")
    for i, (s, d, w) in enumerate(W.inserts):
        assert g.insert(s, d, w) == o.insert(s, d, w)[1]
        g.trees_incremental([t, b], s, d, w)
        chk(f"inc{i}")
    for i, (s, d, _w) in enumerate(W.deletes):
        assert g.delete(s, d) == o.delete(s, d)[1]
        if i % 2:
            g.trees_decremental([t, b], s, d)
        else:
            t.decremental(s, d)
            b.decremental(s, d)
        chk(f"dec{i}")
    es, ed, _ = o.edges()
    f, _w = g.query(es[:100], ed[:100])
    if not np.asarray(f).all():
        bad.append("query")
    print("part_small", "OK" if not bad else bad, flush=True)
    dist.destroy_process_group()
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""BASELINE config 5 on ONE B200: "Twitter-shaped R-MAT scale-26 (~1B edges) ...: 10M-edge update
batches plus BFS recompute" (BASELINE.json configs[4]).  The 8-GPU vertex partition
cannot run on a one-GPU box; the whole graph fits one B200's 180 GB (store + in-edge mirror ~40 GB).

Per batch: a 10 M-edge insert (thread-per-edge kernels, BFS prologue seeded inside) + incremental BFS,
a 10 M-edge delete + decremental BFS; then a static BFS recompute.  CUDA events on the graph's stream.
Parity: the oracle follows every batch on the host; the BFS tree is certified (oracle.check_tree, the
Bellman certificate over ALL vertices) after the FIRST and the LAST batch, and the edge count is compared
after every batch (a from-scratch BFS per batch would take minutes at this size).

    python tools/config5.py [--scale 26] [--batch 10000000] [--batches 2] [--json-out F]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--scale", type=int, default=26)
    p.add_argument("--ef", type=int, default=16)
    p.add_argument("--batch", type=int, default=10_000_000)
    p.add_argument("--batches", type=int, default=2, help="insert batches and delete batches (each)")
    p.add_argument("--no-oracle", action="store_true")
    p.add_argument("--json-out", default=None)
    a = p.parse_args()
    import torch
    import oracle
    import synth
    from paper_2305_17813_b200 import Graph
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev)
    T = lambda x: torch.from_numpy(np.ascontiguousarray(x, np.uint32).view(np.int32)).to(dev)
    t0 = time.time()
    W = synth.rmat_dynamic(a.scale, a.ef, batch=a.batch, n_ins=a.batches, n_del=a.batches)
    gen_s = time.time() - t0
    V, src = W.vertex_n, W.source
    bs, bd, _ = W.base
    n_base = len(bs)
    o = None
    orc_s = 0.0
    if not a.no_oracle:
        t0 = time.time()
        o = oracle.OracleGraph(V, weighted=False)
        o.insert(bs, bd)
        orc_s += time.time() - t0
    g = Graph(V, weighted=False, degree_hints=T(np.bincount(bs, minlength=V).astype(np.uint32)), reverse=True,
              in_degree_hints=T(np.bincount(bd, minlength=V).astype(np.uint32)), device=0, stream=stream)
    ev = lambda: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    e0, e1 = ev()
    ts, td = T(bs), T(bd)
    e0.record(stream)
    n_ins = g.insert(ts, td)
    e1.record(stream)
    e1.synchronize()
    bulk_ms = e0.elapsed_time(e1)
    del ts, td
    torch.cuda.empty_cache()
    if o is not None:
        assert n_ins == o.num_edges, (n_ins, o.num_edges)
    bf = g.bfs(src)
    torch.cuda.synchronize()
    per = {"insert": [], "bfs_inc": [], "delete": [], "bfs_dec": []}
    certified = []

    def certify(tag):
        nonlocal orc_s
        if o is None:
            return
        t = time.time()
        st = o.check_tree(src, bf.nodes(), True)
        orc_s += time.time() - t
        assert st == (0, 0xFFFFFFFF), (tag, st)
        certified.append(tag)

    order = [("ins", i) for i in range(a.batches)] + [("del", i) for i in range(a.batches)]
    for j, (kind, i) in enumerate(order):
        x, y, _ = W.inserts[i] if kind == "ins" else W.deletes[i]
        s, d = T(x), T(y)
        (a0, a1), (b0, b1) = ev(), ev()
        a0.record(stream)
        if kind == "ins":
            g.insert(s, d, count=False, seed=[bf])
        else:
            g.delete(s, d, count=False, seed=[bf])
        a1.record(stream)
        b0.record(stream)
        if kind == "ins":
            g.trees_incremental([bf], s, d)
        else:
            g.trees_decremental([bf], s, d)
        b1.record(stream)
        b1.synchronize()
        per["insert" if kind == "ins" else "delete"].append(a0.elapsed_time(a1))
        per["bfs_inc" if kind == "ins" else "bfs_dec"].append(b0.elapsed_time(b1))
        if o is not None:
            t = time.time()
            (o.insert(x, y) if kind == "ins" else o.delete(x, y))
            orc_s += time.time() - t
            g.sync()
            assert g.stats()["edges"] == o.num_edges, (kind, i)
        if j == 0 or j == len(order) - 1:
            certify(f"{kind}{i}")
    e0, e1 = ev()
    e0.record(stream)
    bf.recompute()
    e1.record(stream)
    e1.synchronize()
    static_ms = e0.elapsed_time(e1)
    if o is not None:
        t = time.time()
        assert o.check_tree(src, bf.nodes(), True) == (0, 0xFFFFFFFF)
        orc_s += time.time() - t
        certified.append("static")
    st = g.stats()
    mean = {k: float(np.mean(v)) for k, v in per.items()}
    peak = 6556.8
    try:
        peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        pass
    # SURVEY §8(d) per-edge bytes for a set store (4-B keys): batch 8 + vmeta 8 + 128 x 1.04 slabs + CAS 4,
    # for the out store and the in-edge mirror, + the BFS prologue (node reads / atomicMin, 16 / 8 B)
    alg = {"insert": a.batch * (2 * (8 + 8 + 133 + 4) + 16), "delete": a.batch * (2 * (8 + 8 + 133 + 4) + 8)}
    out = {
        "workload": f"rmat-s{a.scale}-ef{a.ef} (BASELINE config 5, one B200), {n_base} base edges, "
                    f"{a.batch}-edge insert / delete batches, BFS (set store + in-edge mirror)",
        "vertices": V, "base_edges": n_base, "batch": a.batch, "batches_each": a.batches,
        "bulk_build": {"ms": bulk_ms, "edges_per_s": n_base / (bulk_ms / 1e3)},
        "per_batch_ms": mean,
        "insert_edges_per_s": a.batch / (mean["insert"] / 1e3),
        "delete_edges_per_s": a.batch / (mean["delete"] / 1e3),
        "update_edges_per_s": 2 * a.batch / ((mean["insert"] + mean["delete"]) / 1e3),
        "bfs_ms_per_batch": {"incremental": mean["bfs_inc"], "decremental": mean["bfs_dec"]},
        "static_bfs_ms": static_ms,
        "roofline": {k: {"bound": "hbm", "alg_bytes_per_launch": alg[k],
                         "achieved": alg[k] / (mean[k] * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": alg[k] / (mean[k] * 1e-3) / 1e9 / peak} for k in ("insert", "delete")},
        "slab_index_headroom": {"slabs": int(st["head_slabs"] + st["pool_capacity"]),
                                "in_slabs": int(st.get("in_head_slabs", 0)), "limit": 0xFFFFFFF0},
        "bytes_device": int(st["bytes_device"]),
        "parity": {"certified_after": certified, "edge_count_checked_every_batch": o is not None,
                   "method": "oracle.check_tree (Bellman certificate over all vertices) + live-edge count"},
        "generate_s": gen_s, "oracle_s": orc_s,
    }
    print(json.dumps(out), flush=True)
    if a.json_out:
        with open(a.json_out, "w") as f:
            json.dump(out, f, indent=1)
    g.close()


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Benchmark of the Meerkat hot path on B200 (BASELINE.json metric:
"edge updates/sec (insert+delete) and dynamic-SSSP ms/batch").

Workload (BASELINE config 3): R-MAT scale 24, edge factor 16,
Graph500 initiator, scrambled ids, w ~ U{1..64}; the base graph is E minus the
held-out insert batches; the source is R-MAT's hub.  One STEP = the whole hot
path over one batch pair:

    insert_batch(100K held-out edges) -> sssp_incremental -> bfs_incremental
    delete_batch(100K present edges)  -> sssp_decremental -> bfs_decremental

value = 200K edge updates / device time of the step (inputs resident in HBM),
with per-call times reported beside it.  The decremental valid->invalid
frontier is read from an in-edge mirror store by default (--frontier reverse);
the paper's full slab scan (--frontier scan) is timed too and reported under
"alt" (--no-compare skips it).  L2 is flushed (256 MiB write) between
timed steps, outside the timed intervals.  `e2e` repeats the step through the
C ABI with pinned HOST batch arrays (staged by the library inside each call)
and reads the insert/delete counts back to the host.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "edge updates/sec (insert+delete) and dynamic-SSSP ms/batch at 1/2/4/8 B200"
BATCH_SEED_BASE = 3


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--scale", type=int, default=24)
    p.add_argument("--ef", type=int, default=16)
    p.add_argument("--batch", type=int, default=100_000)
    p.add_argument("--lf", type=float, default=0.5,
                   help="load factor of the slab stores (SURVEY C22: a performance knob the paper leaves open; 0.5 measured best for the config-3 step, DESIGN.md §10)")
    p.add_argument("--in-lf", type=float, default=0.0,
                   help="load factor of the in-edge mirror (0 = --lf); the mirror is only walked (pull frontier)")
    p.add_argument("--no-hashing", action="store_true")
    p.add_argument("--seed", action=argparse.BooleanOptionalAction, default=True,
                   help="with --fused, the insert / delete kernels seed the tree calls (batch prologue "
                        "inside the mutation kernel: meerkat_*_batch_trees)")
    p.add_argument("--fused", action=argparse.BooleanOptionalAction, default=True,
                   help="update the SSSP and BFS trees with one fused launch per batch (meerkat_trees_*)")
    p.add_argument("--per-tree", action=argparse.BooleanOptionalAction, default=True,
                   help="with --fused, also time per-tree calls for the SSSP / BFS split")
    p.add_argument("--compare", action=argparse.BooleanOptionalAction, default=True,
                   help="also time the other decremental-frontier mode (reported under 'alt')")
    p.add_argument("--frontier", choices=["scan", "reverse"], default="reverse",
                   help="decremental valid->invalid frontier: stream every slab (paper, P:156-164) or "
                        "read the in-edges of V_invalid from an in-edge mirror store")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--l2-flush", action=argparse.BooleanOptionalAction, default=True,
                   help="write a 256 MiB buffer between timed steps (default); --no-l2-flush relies on the "
                        "inputs (the 12.7 GB store) being larger than L2 instead")
    p.add_argument("--wcc", action=argparse.BooleanOptionalAction, default=True,
                   help="also time static and incremental WCC on the workload graph (SURVEY §8(f) NEXT-3)")
    p.add_argument("--tc", action=argparse.BooleanOptionalAction, default=True,
                   help="also time triangle counting on a symmetrised R-MAT (--tc-scale) graph (NEXT-4)")
    p.add_argument("--tc-scale", type=int, default=20)
    p.add_argument("--config4", action=argparse.BooleanOptionalAction, default=True,
                   help="also time BASELINE config 4 (R-MAT scale 22, ef 24, mixed 1%%-of-E delete / insert rounds)")
    p.add_argument("--pagerank", action=argparse.BooleanOptionalAction, default=True,
                   help="also time static and dynamic PageRank on the same graph (SURVEY §8(f) NEXT-1; "
                        "needs the in-edge mirror, i.e. --frontier reverse)")
    p.add_argument("--hashing-ab", action=argparse.BooleanOptionalAction, default=True,
                   help="also time the step, the static recomputes and the config-2 sweep with hashing OFF (one "
                        "slab list per vertex; the paper's traversal trade-off, P:2282-2286) -> hashing_ab")
    p.add_argument("--probe", action=argparse.BooleanOptionalAction, default=True,
                   help="measure DRAM / L2 / atomic latency and the grid-barrier cost on the device and report the "
                        "tree calls' latency floor (latency_floor)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-scale", type=int, default=20, help="R-MAT scale of the oracle's bounded sample")
    p.add_argument("--cpu-steps", type=int, default=8,
                   help="oracle steps in the cpu_baseline sample (~1.2 s each at scale 20: a 10-s bounded sample)")
    p.add_argument("--json-out", default=None)
    p.add_argument("--sweep", action=argparse.BooleanOptionalAction, default=True,
                   help="also run the config-2 insert/delete/query batch-size sweep (reported under store_sweep)")
    p.add_argument("--sweep-scale", type=int, default=20)
    p.add_argument("--partitioned", action="store_true",
                   help="use the vertex-partitioned multi-GPU path even at --gpus 1 (NCCL, world size 1)")
    return p.parse_args()


# ------------------------------------------------------------------ distributed plumbing

def dist_init(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "ours" and (ws > 1 or args.partitioned):   # the reference arm needs no process group
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        if not dist.is_initialized():
            if ws == 1:
                os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
                os.environ.setdefault("MASTER_PORT", "29533")
                os.environ.setdefault("RANK", "0")
                os.environ.setdefault("WORLD_SIZE", "1")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return ws, rank, local


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def allreduce_max(x, ws):
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def allreduce_sum(x, ws):
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


# ------------------------------------------------------------------ clocks

_SAMPLER = r"""
import sys, time, pynvml
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(int(sys.argv[1]))
print("max", pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM), flush=True)
while True:
    try:
        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
        try:
            rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
        except Exception:
            rs = -1   # reasons unavailable: the clock is still recorded
        print(sm, rs, flush=True)
    except Exception:
        pass
    time.sleep(0.002)
"""


class ClockSampler:
    """SM clock and clock-event (throttle) reasons sampled every ~2 ms via NVML by a separate
    process (no GIL contention with the timed loop) during the timed region."""
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap",
               0x80: "hw_power_brake_slowdown"}

    def __init__(self, device):
        idx = device
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        if vis:
            try:
                idx = int(vis.split(",")[device])
            except (ValueError, IndexError):
                pass
        self.idx = idx
        self.proc = None
        self.lines = []
        self.n0 = 0

    def start(self):
        import subprocess
        try:
            self.proc = subprocess.Popen([sys.executable, "-c", _SAMPLER, str(self.idx)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=lambda: self.lines.extend(self.proc.stdout), daemon=True)
            self.t.start()
            t0 = time.time()
            while len(self.lines) < 2 and time.time() - t0 < 20:   # wait until samples arrive ("max" + one)
                time.sleep(0.01)
            self.n0 = len(self.lines)   # samples from here on are the timed region's
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml sampler unavailable"]}
        t0 = time.time()
        # a timed region shorter than the sampling period still gets the sample that ends it
        while len(self.lines) <= self.n0 and time.time() - t0 < 2:
            time.sleep(0.002)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        mx, sm, reasons = None, [], set()
        for i, ln in enumerate(self.lines):
            p = ln.split()
            if p and p[0] == "max":
                mx = int(p[1])
            elif len(p) == 2 and i >= self.n0:
                sm.append(int(p[0]))
                rs = int(p[1])
                if rs < 0:
                    reasons.add("reasons unavailable")
                else:
                    reasons |= {n for bit, n in self.REASONS.items() if rs & bit}
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ workload

def make_workload(args, n_batches, rank=0):
    import synth
    t0 = time.time()
    W = synth.rmat_dynamic(args.scale, args.ef, batch=args.batch, n_ins=n_batches, n_del=n_batches,
                           seed_batch=BATCH_SEED_BASE + 1000 * rank)
    return W, time.time() - t0


def workload_config(args, V, n_base, source, ws=1):
    """The `config` object of the JSON line (shared by both arms)."""
    return {"workload": f"rmat-s{args.scale}-ef{args.ef} dynamic SSSP+BFS, {args.batch}-edge insert+delete "
                        f"batches (BASELINE config 3)",
            "vertices": V, "edges": n_base, "batch": args.batch, "source": source,
            "hashing": not args.no_hashing, "load_factor": args.lf, "in_load_factor": args.in_lf or args.lf,
            "decremental_frontier": args.frontier,
            "tree_updates": ("fused SSSP+BFS (meerkat_trees_*)" if args.fused else "per tree")
                            + (", seeded by the insert / delete kernels" if args.fused and args.seed else ""),
            "parallelism": "single GPU" if ws == 1 else f"{ws} independent replicas",
            "l2": ("flushed between timed steps (256 MiB write, outside the intervals); store > L2" if args.l2_flush
                   else "not flushed: inputs larger than L2 (store > L2), batches back to back")}


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def cpu_baseline(args, steps):
    """The oracle as it stands, on a bounded sample of the same workload recipe (R-MAT at
    --cpu-scale, same generator, same batch size): per step it applies an insert batch and a
    delete batch and recomputes SSSP + BFS from scratch after each (the oracle has no dynamic
    algorithm).  Timed per part: apply, SSSP and BFS seconds per batch."""
    import oracle
    import synth
    W = synth.rmat_dynamic(args.cpu_scale, args.ef, batch=args.batch, n_ins=steps, n_del=steps,
                           seed_batch=BATCH_SEED_BASE)
    o = oracle.OracleGraph(W.vertex_n)
    o.insert(*W.base)
    n_base = int(len(W.base[0]))
    parts = {"apply_insert": [], "apply_delete": [], "sssp": [], "bfs": []}
    clock = time.perf_counter

    def timed(key, fn):
        t = clock(); fn(); parts[key].append(clock() - t)
    t0 = clock()
    for i in range(steps):
        timed("apply_insert", lambda: o.insert(*W.inserts[i])); timed("sssp", lambda: o.sssp(W.source))
        timed("bfs", lambda: o.bfs(W.source))
        timed("apply_delete", lambda: o.delete(W.deletes[i][0], W.deletes[i][1]))
        timed("sssp", lambda: o.sssp(W.source)); timed("bfs", lambda: o.bfs(W.source))
    dt = clock() - t0
    return {"value": 2 * args.batch * steps / dt, "unit": "edges/s", "cores": 1, "kind": "oracle",
            "host_cores": os.cpu_count(), "cpu_model": cpu_model(), "oracle_threads": 1,
            "per_batch_s": {k: float(np.median(v)) for k, v in parts.items()},
            "sample_scale": args.cpu_scale, "sample_vertices": int(W.vertex_n), "sample_edges": n_base,
            "sample": (f"oracle (single-threaded C) on R-MAT scale {args.cpu_scale} ef {args.ef} "
                       f"({W.vertex_n} vertices, {n_base} edges; the workload's recipe at "
                       f"1/{2 ** max(0, args.scale - args.cpu_scale)} of its vertices), "
                       f"{steps} step(s) of insert {args.batch} + delete {args.batch} edges, each followed by "
                       f"from-scratch SSSP + BFS; {dt:.1f} s"),
            "seconds": dt}


def run_reference(args, ws, rank):
    if rank != 0:
        return
    t_all = time.time()
    for _ in range(args.warmup):
        pass   # the oracle has no warm state worth warming; bounded sample only
    cb = cpu_baseline(args, max(1, min(args.steps, args.cpu_steps)))
    # the line's config describes what was TIMED: the oracle sample at --cpu-scale (the full workload
    # our arm runs is named in sample_of); at --cpu-scale == --scale the two are the same workload
    cfg = workload_config(args, cb["sample_vertices"], cb["sample_edges"], 0)
    cfg["workload"] = cfg["workload"].replace(f"rmat-s{args.scale}-", f"rmat-s{args.cpu_scale}-")
    if args.cpu_scale != args.scale:
        cfg["workload"] += f" -- bounded oracle sample at scale {args.cpu_scale}"
        cfg["sample_of"] = workload_config(args, 1 << args.scale, None, 0)["workload"]
    cfg["parallelism"] = "one host thread (the oracle)"
    cfg["tree_updates"] = "from-scratch SSSP (Dijkstra) + BFS after every batch (the oracle has no dynamic algorithm)"
    for k in ("decremental_frontier", "l2"):
        cfg.pop(k, None)
    line = {"metric": METRIC, "value": cb["value"], "unit": "edges/s", "n_gpus": 0, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * cb["seconds"] / max(1, min(args.steps, args.cpu_steps)),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "impl": "reference",
            "config": cfg,
            "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample", "host_cores", "cpu_model",
                                                "oracle_threads", "per_batch_s")},
            "e2e": {"value": cb["value"], "unit": "edges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "wall_s": time.time() - t_all}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm

def build(args, W, frontier, dev, local, stream, T):
    """Graph + SSSP/BFS trees for workload W (not timed, except the bulk build as its own datum)."""
    import torch
    from paper_2305_17813_b200 import Graph
    V = W.vertex_n
    bs, bd, bw = W.base
    hints = np.bincount(bs, minlength=V).astype(np.uint32)
    rev = frontier == "reverse"
    ihints = np.bincount(bd, minlength=V).astype(np.uint32) if rev else None
    g = Graph(V, weighted=True, hashing=not args.no_hashing, load_factor=args.lf, degree_hints=T(hints),
              device=local, stream=stream, reverse=rev, in_degree_hints=T(ihints) if rev else None,
              in_load_factor=args.in_lf)
    base_t = (T(bs), T(bd), T(bw))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    n_base = g.insert(*base_t)
    e1.record(stream)
    torch.cuda.synchronize()
    bulk_ms = e0.elapsed_time(e1)
    del base_t
    sp = g.sssp(W.source)
    bf = g.bfs(W.source)
    torch.cuda.synchronize()
    return g, sp, bf, int(n_base), bulk_ms


NAMES = ["insert", "sssp_inc", "bfs_inc", "delete", "sssp_dec", "bfs_dec"]
NAMES_FUSED = ["insert", "trees_inc", "delete", "trees_dec"]


def one_step(g, sp, bf, ins, dels, evs, stream, fused=False, seed=False, after_inc=None):
    """The hot path over one batch pair: mutate, then update both trees.  fused: one
    launch updates the SSSP and the BFS tree together (meerkat_trees_*); seed: the trees' batch
    prologue runs inside the insert / delete kernel (meerkat_*_batch_trees).  after_inc (untimed
    warm-up only): called between the incremental and the delete half, e.g. to read tree counters."""
    s, d, w = ins
    if fused:
        trees = [sp, bf] if seed else None
        evs[0].record(stream)
        g.insert(s, d, w, count=False, seed=trees)
        evs[1].record(stream)
        g.trees_incremental([sp, bf], s, d, w)
        evs[2].record(stream)
        if after_inc:
            after_inc()
        s, d = dels
        g.delete(s, d, count=False, seed=trees)
        evs[3].record(stream)
        g.trees_decremental([sp, bf], s, d)
        evs[4].record(stream)
        return
    evs[0].record(stream)
    g.insert(s, d, w, count=False)
    evs[1].record(stream)
    sp.incremental(s, d, w)
    evs[2].record(stream)
    bf.incremental(s, d)
    evs[3].record(stream)
    s, d = dels
    g.delete(s, d, count=False)
    evs[4].record(stream)
    sp.decremental(s, d)
    evs[5].record(stream)
    bf.decremental(s, d)
    evs[6].record(stream)


def measure(args, ws, W, frontier, dev, local, stream, T, flush, K, Wm, clocks=None, fused=True):
    import torch
    seed = fused and getattr(args, "seed", False)
    g, sp, bf, n_base, bulk_ms = build(args, W, frontier, dev, local, stream, T)
    ins = [tuple(T(x) for x in b) for b in W.inserts]
    dels = [tuple(T(x) for x in b[:2]) for b in W.deletes]
    names = NAMES_FUSED if fused else NAMES
    ev = lambda: [torch.cuda.Event(enable_timing=True) for _ in range(len(names) + 1)]
    inc_stats = []   # counters of a fused incremental call (last warm-up step): its rounds for the latency floor
    for i in range(Wm):
        grab = (lambda: inc_stats.append(sp.stats())) if (fused and i == Wm - 1) else None
        one_step(g, sp, bf, ins[i], dels[i], ev(), stream, fused, seed, after_inc=grab)
        flush.zero_()
    torch.cuda.synchronize()
    g.sync()
    st0 = g.stats()
    per_call = {n: [] for n in names}
    tstats = {("trees_dec" if fused else "sssp_dec"): [], "bfs_dec": []}
    if clocks:
        clocks.start()
    barrier(ws)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push(f"timed_{frontier}")   # ncu --nvtx --nvtx-include "timed_<mode>/" selects these
    total_ms = 0.0
    for k in range(K):
        i = Wm + k
        evs = ev()
        one_step(g, sp, bf, ins[i], dels[i], evs, stream, fused, seed)
        evs[-1].synchronize()
        for j, n in enumerate(names):
            per_call[n].append(evs[j].elapsed_time(evs[j + 1]))
        total_ms += evs[0].elapsed_time(evs[-1])
        s1, s2 = sp.stats(), bf.stats()   # device counters of the last call, read outside the intervals
        if fused:   # one launch: per-call counters are shared, frontier edges (16 B each) per tree
            s1 = dict(s1, alg_bytes=s1["alg_bytes"] + 16 * s2["frontier_edges"])
            tstats["trees_dec"].append(s1)
        else:
            tstats["sssp_dec"].append(s1)
        tstats["bfs_dec"].append(s2)
        flush.zero_()
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    barrier(ws)
    clk = clocks.stop() if clocks else None
    g.sync()
    st1 = g.stats()
    total_ms = allreduce_max(total_ms, ws)
    # static recompute on the final graph: the s_b^n baseline
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    static = {}
    for name, t in (("sssp", sp), ("bfs", bf)):
        flush.zero_()
        a.record(stream)
        t.recompute()
        b.record(stream)
        b.synchronize()
        static[name] = a.elapsed_time(b)
    # the paper's IterationScheme1 (one work item per vertex) for the static recompute
    scheme1 = {}
    if fused:
        for name, t in (("sssp", sp), ("bfs", bf)):
            flush.zero_()
            a.record(stream)
            t.recompute(iteration_scheme=1)
            b.record(stream)
            b.synchronize()
            scheme1[name] = a.elapsed_time(b)
    # the paper's vanilla variant (distances only, 32-bit atomics) on the same graph:
    # the tree-based overhead of P:2313-2317 (17.2% BFS, ~14% SSSP on its GPU)
    vanilla = {}
    if fused:
        for name, mk in (("sssp", g.sssp_vanilla), ("bfs", g.bfs_vanilla)):
            vt = mk(W.source)
            flush.zero_()
            a.record(stream)
            vt.recompute()
            b.record(stream)
            b.synchronize()
            vanilla[name] = a.elapsed_time(b)
            vt.close()
    mean = {n: float(np.mean(v)) for n, v in per_call.items()}
    res = {
        "frontier": frontier, "fused": fused, "K": K, "total_ms": total_ms, "ms_per_step": total_ms / K, "mean": mean,
        "per_call": per_call, "tstats": tstats, "clocks": clk, "n_base": n_base, "bulk_ms": bulk_ms,
        "launches": int(st1["kernel_launches"] - st0["kernel_launches"]), "static_ms": static,
        "inc_stats": inc_stats[-1] if inc_stats else None,
        "vanilla_ms": vanilla, "scheme1_ms": scheme1,
        "store": {k: g.stats()[k] for k in ("head_slabs", "buckets", "pool_used", "bytes_device")},
    }
    return res, (g, sp, bf)


def roofline_of(res, peak, peak_src, traffic_file):
    mean = res["mean"]
    dom = max(mean, key=mean.get)
    if dom not in res["tstats"]:
        return {"bound": "hbm", "kernel": dom, "achieved": None, "peak": peak, "unit": "GB/s", "frac": None,
                "traffic": None}
    ab = float(np.mean([s["alg_bytes"] for s in res["tstats"][dom]]))
    ach = ab / (mean[dom] * 1e-3) / 1e9
    traffic, l2hit = None, None
    try:
        tj = json.load(open(traffic_file))
        traffic = tj.get(f"{res['frontier']}/{dom}")
        l2hit = tj.get("l2_hit_rate", {}).get(f"{res['frontier']}/{dom}")
    except Exception:
        pass
    return {"bound": "hbm", "kernel": f"k_tree_dec ({dom}, {res['frontier']} frontier{', fused SSSP+BFS' if res['fused'] else ''})",
            "achieved": ach,
            "peak": peak, "unit": "GB/s", "frac": ach / peak, "traffic": traffic, "alg_bytes_per_launch": ab,
            "traffic_frac": (traffic / (mean[dom] * 1e-3) / 1e9 / peak) if traffic else None,
            "l2_hit_rate_pct": l2hit, "peak_source": peak_src}


def update_roofline(res, args, peak, peak_src, traffic_file, n_stores, n_trees):
    """HBM roofline of the seeding insert / delete kernels: SURVEY §8(d)'s per-edge bytes per store
    (insert 161 B, delete 157 B: batch + vmeta + 128 x 1.04 slabs + CAS) for the out store and the
    in-edge mirror, plus the fused tree prologue per edge and tree (insert: node[u] + atomicMin
    node[v] = 16 B; delete: node[v] = 8 B)."""
    out = {}
    try:
        tj = json.load(open(traffic_file))
    except Exception:
        tj = {}
    for name, per_store, per_tree in (("insert", 161, 16), ("delete", 157, 8)):
        ms = res["mean"][name]
        ab = args.batch * (n_stores * per_store + n_trees * per_tree)
        ach = ab / (ms * 1e-3) / 1e9
        traffic = tj.get(f"{res['frontier']}/{name}")
        out[name] = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                     "alg_bytes_per_launch": ab, "traffic": traffic,
                     "traffic_over_alg": (traffic / ab) if traffic else None, "peak_source": peak_src}
    return out


def latency_floor(lat, res):
    """Floor of the latency-bound tree calls from measured device latencies (meerkat_probe_latency):
    every grid-synchronised phase costs one grid barrier plus its dependent chain -- item fetch (L2),
    slab load (DRAM), packed atomicMin on node[x] (DRAM atomic), stamp atomicExch + vmeta (DRAM
    atomic), warp enqueue (L2 atomic) -- so floor = phases x (grid_sync + l2 + dram + 2 x dram_atomic
    + l2).  Phases: incremental = relax rounds; decremental = propagation rounds + 2 (pull-frontier
    enqueue, pull) + relax rounds (the last tail rounds run on block barriers, so this overstates
    them slightly)."""
    if not lat:
        return None
    chain_us = (2 * lat["l2_load_ns"] + lat["dram_load_ns"] + 2 * lat["dram_atomic_ns"]) / 1e3
    phase_us = lat["grid_sync_us"] + chain_us
    out = {"probe": lat, "phase_us": phase_us, "chain_us": chain_us}
    dec = res["tstats"].get("trees_dec") or []
    if dec:
        ph = float(np.mean([s["rounds"] + s["propagate_rounds"] + 2 for s in dec]))
        out["trees_dec"] = {"phases": ph, "floor_us": ph * phase_us, "measured_us": 1e3 * res["mean"]["trees_dec"]}
    if res.get("inc_stats"):
        ph = float(res["inc_stats"]["rounds"])
        out["trees_inc"] = {"phases": ph, "floor_us": ph * phase_us, "measured_us": 1e3 * res["mean"]["trees_inc"]}
    return out


def tree_detail(res):
    return {n: {k: float(np.mean([s[k] for s in v])) for k in
                ("rounds", "propagate_rounds", "invalidated", "frontier_edges", "scan_slabs", "slabs_read",
                 "alg_bytes")} for n, v in res["tstats"].items() if v}


def store_sweep(args, dev, stream):
    """BASELINE config 2: R-MAT scale 20, batch insert / delete / query at
    1K..1M edges per batch.  Inserts are fresh R-MAT draws (graph seed 11, duplicates and
    self-loops kept as drawn), deletes are sampled present edges, queries are 50% present /
    50% absent.  Median device time of `reps` batches per point; algorithmic bytes per edge
    161 / 157 / 154 B."""
    import torch
    import synth
    from paper_2305_17813_b200 import Graph
    scale, reps = args.sweep_scale, 5
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.uint32).view(np.int32)).to(dev)
    s, d, w = synth.rmat(scale, 16)
    V = 1 << scale
    g = Graph(V, weighted=True, hashing=not args.no_hashing, load_factor=args.lf,
              degree_hints=T(np.bincount(s, minlength=V).astype(np.uint32)), device=dev.index or 0, stream=stream)
    g.insert(T(s), T(d), T(w), count=False)
    g.sync()
    sizes = [1000, 10000, 100000, 1000000]
    need = sum(sizes) * reps
    dels = synth.sample_distinct(len(s), need, 17)
    fresh = synth.rmat_draws(scale, need, 0, 11)
    rng = np.random.default_rng(5)
    out, di, fi = {}, 0, 0
    ev = lambda: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    for b in sizes:
        t_ins, t_del, t_q = [], [], []
        for r in range(reps):
            ins = tuple(T(x[fi:fi + b]) for x in fresh)
            fi += b
            dl = dels[di:di + b]
            di += b
            ds, dd = T(s[dl]), T(d[dl])
            half = b // 2
            qs = T(np.concatenate([s[rng.integers(0, len(s), half)], rng.integers(0, V, b - half)]))
            qd = T(np.concatenate([d[rng.integers(0, len(s), half)], rng.integers(0, V, b - half)]))
            qs2 = torch.cat([ds[:0], qs])
            torch.cuda.synchronize()
            for lst, fn in ((t_ins, lambda: g.insert(*ins, count=False)),
                            (t_del, lambda: g.delete(ds, dd, count=False)),
                            (t_q, lambda: g.query(qs2, qd))):
                e0, e1 = ev()
                e0.record(stream)
                fn()
                e1.record(stream)
                e1.synchronize()
                lst.append(e0.elapsed_time(e1))
        med = lambda x: float(np.median(x))
        out[str(b)] = {"insert_edges_per_s": b / (med(t_ins) / 1e3), "delete_edges_per_s": b / (med(t_del) / 1e3),
                       "query_edges_per_s": b / (med(t_q) / 1e3),
                       "insert_GBps_alg": 161 * b / (med(t_ins) / 1e3) / 1e9,
                       "delete_GBps_alg": 157 * b / (med(t_del) / 1e3) / 1e9,
                       "query_GBps_alg": 154 * b / (med(t_q) / 1e3) / 1e9,
                       "ms": {"insert": med(t_ins), "delete": med(t_del), "query": med(t_q)}}
    g.sync()
    g.close()
    return {"workload": f"rmat-s{scale}-ef16 (BASELINE config 2), {len(s)} edges, hashing "
                        f"{'off' if args.no_hashing else 'on'} lf {args.lf}", "by_batch": out}


def measure_pagerank(g, W, T, stream, flush, peak, peak_src):
    """PageRank on the workload graph (d = 0.85, error margin 1e-5): static (cold start,
    the s_b^n baseline), then dynamic (warm start) after a 100K-edge insert batch and
    after the matching delete batch.  One persistent launch per run; CUDA events on the graph's stream."""
    import torch
    p = g.pagerank(0.85, 1e-5, 1000)          # allocation + a first static run (untimed)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def timed(fn):
        flush.zero_()
        a.record(stream)
        fn()
        b.record(stream)
        b.synchronize()
        return a.elapsed_time(b), p.stats()

    st_ms, st = timed(p.recompute)
    s, d, w = W.deletes[0]                      # deleted in warm-up step 0: absent now
    g.insert(T(s), T(d), T(w), count=False)
    inc_ms, inc = timed(p.update)
    g.delete(T(s), T(d), count=False)
    dec_ms, dec = timed(p.update)
    p.close()
    ach = st["alg_bytes"] / (st_ms * 1e-3) / 1e9
    traffic = l2hit = None
    try:
        tj = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        traffic, l2hit = tj.get("pagerank/static"), tj.get("l2_hit_rate", {}).get("pagerank/static")
    except Exception:
        pass
    return {"damping": 0.85, "error_margin": 1e-5, "dtype": "f64",
            "static_ms": st_ms, "static_iterations": st["iterations"],
            "incremental_ms": inc_ms, "incremental_iterations": inc["iterations"],
            "decremental_ms": dec_ms, "decremental_iterations": dec["iterations"],
            "batch": int(len(s)),
            "per_iteration": {"slabs": st["slabs"], "in_edges": st["in_edges"], "atomics": st["atomics"],
                              "ms": st_ms / max(1, st["iterations"])},
            "roofline": {"bound": "hbm", "kernel": "k_pagerank (static run)", "achieved": ach, "peak": peak,
                         "unit": "GB/s", "frac": ach / peak, "alg_bytes_per_launch": st["alg_bytes"],
                         "traffic": traffic, "l2_hit_rate_pct": l2hit,
                         "traffic_frac": (traffic / (st_ms * 1e-3) / 1e9 / peak) if traffic else None,
                         "peak_source": peak_src}}


def measure_wcc(g, W, T, stream, flush):
    """WCC on the workload graph: static (MinHooking + union + compression) and
    incremental after a 100K-edge insert batch (union of the batch + compression)."""
    import torch
    c = g.wcc()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def timed(fn):
        flush.zero_()
        a.record(stream)
        fn()
        b.record(stream)
        b.synchronize()
        return a.elapsed_time(b)

    st_ms = timed(c.recompute)
    s, d, w = W.deletes[0]                      # absent at this point (see measure_pagerank)
    g.insert(T(s), T(d), T(w), count=False)
    ts, td = T(s), T(d)
    inc_ms = timed(lambda: c.incremental(ts, td))
    comps = c.components()
    g.delete(ts, td, count=False)
    c.close()
    return {"static_ms": st_ms, "incremental_ms": inc_ms, "batch": int(len(s)), "components": comps}


def measure_config4(args, dev, stream, flush, rounds=4):
    """BASELINE config 4 (reading C25): R-MAT scale 22, edge factor 24 ('LJ/Orkut-shaped',
    ~97 M edges); each round deletes 1% of E (970 K edges) and runs the fused decremental SSSP + BFS
    update, then inserts 970 K held-out edges and runs the fused incremental update.  One warm-up
    round, then `rounds` timed rounds (CUDA events on the graph's stream, L2 flushed between calls)."""
    import torch
    import synth
    from paper_2305_17813_b200 import Graph
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.uint32).view(np.int32)).to(dev)
    n1 = 970_000
    W = synth.rmat_dynamic(22, 24, batch=n1, n_ins=rounds + 1, n_del=rounds + 1)
    V = W.vertex_n
    bs, bd, bw = W.base
    g = Graph(V, weighted=True, degree_hints=T(np.bincount(bs, minlength=V).astype(np.uint32)), reverse=True,
              in_degree_hints=T(np.bincount(bd, minlength=V).astype(np.uint32)), device=dev.index or 0, stream=stream)
    g.insert(T(bs), T(bd), T(bw), count=False)
    sp, bf = g.sssp(W.source), g.bfs(W.source)
    ev = lambda: [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    names = ["delete", "trees_dec", "insert", "trees_inc"]
    per = {n: [] for n in names}
    for r in range(rounds + 1):
        ds, dd = T(W.deletes[r][0]), T(W.deletes[r][1])
        is_, id_, iw = (T(x) for x in W.inserts[r])
        e = ev()
        flush.zero_()
        e[0].record(stream); g.delete(ds, dd, count=False); e[1].record(stream)
        g.trees_decremental([sp, bf], ds, dd); e[2].record(stream)
        flush.zero_()   # (between calls; the flush is not inside any interval below)
        e[2].synchronize()
        e2 = ev()
        e2[0].record(stream); g.insert(is_, id_, iw, count=False); e2[1].record(stream)
        g.trees_incremental([sp, bf], is_, id_, iw); e2[2].record(stream)
        e2[2].synchronize()
        if r == 0:
            continue
        per["delete"].append(e[0].elapsed_time(e[1])); per["trees_dec"].append(e[1].elapsed_time(e[2]))
        per["insert"].append(e2[0].elapsed_time(e2[1])); per["trees_inc"].append(e2[1].elapsed_time(e2[2]))
    mean = {n: float(np.mean(v)) for n, v in per.items()}
    out = {"workload": f"rmat-s22-ef24 (BASELINE config 4), {len(bs)} base edges, {n1}-edge delete + insert rounds",
           "rounds": rounds, "per_call_ms": mean,
           "round_ms": sum(mean.values()),
           "update_edges_per_s": 2 * n1 / ((mean["delete"] + mean["insert"]) / 1e3),
           "sssp_bfs_fused_ms_per_batch": {"decremental": mean["trees_dec"], "incremental": mean["trees_inc"]}}
    g.close()
    return out


def measure_tc(args, dev, stream):
    """Triangle counting on a symmetrised R-MAT graph (both orientations stored, set store): the static
    count and the dynamic deltas of a 10K-undirected-edge insert and delete batch
    (inclusion-exclusion, three Count launches each)."""
    import torch
    import synth
    from paper_2305_17813_b200 import Graph
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.uint32).view(np.int32)).to(dev)
    rs, rd, _ = synth.rmat(args.tc_scale, 16)
    k = np.unique(np.concatenate([(rs.astype(np.uint64) << np.uint64(32)) | rd,
                                  (rd.astype(np.uint64) << np.uint64(32)) | rs]))
    s, d = (k >> np.uint64(32)).astype(np.uint32), (k & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    keep = s != d
    s, d = s[keep], d[keep]
    V = 1 << args.tc_scale
    rng = np.random.default_rng(7)
    und = np.nonzero(s < d)[0]
    pick = rng.choice(und, 10_000, replace=False)
    bs = np.concatenate([s[pick], d[pick]]); bd = np.concatenate([d[pick], s[pick]])
    g = Graph(V, weighted=False, degree_hints=T(np.bincount(s, minlength=V).astype(np.uint32)), device=dev.index or 0,
              stream=stream)
    g.insert(T(s), T(d), count=False)
    gu = Graph(V, weighted=False, device=dev.index or 0, stream=stream)
    gu.insert(T(bs), T(bd), count=False)
    g.sync(); gu.sync()
    def timed(fn, reps=5):   # the counts do not mutate: CUDA events on the graph's stream around each
        ev, wall, r = [], [], None   # (synchronising) call, median of 5; host wall clock beside it
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            a.record(stream); r = fn(); b.record(stream)
            b.synchronize()
            wall.append(1e3 * (time.perf_counter() - t0)); ev.append(a.elapsed_time(b))
        return r, float(np.median(ev)), [float(min(ev)), float(max(ev))], float(np.median(wall))
    tri, st_ms, st_rng, st_wall = timed(g.tc_static)
    g.delete(T(bs), T(bd), count=False)
    g.sync()
    (removed, _), dec_ms, dec_rng, dec_wall = timed(lambda: g.tc_delta(gu, T(bs), T(bd), insert=False))
    g.insert(T(bs), T(bd), count=False)
    g.sync()
    (added, S), inc_ms, inc_rng, inc_wall = timed(lambda: g.tc_delta(gu, T(bs), T(bd), insert=True))
    out = {"graph": f"rmat-s{args.tc_scale}-ef16 symmetrised, {len(s)} directed edges", "triangles": tri,
           "static_ms": st_ms, "batch_undirected": 10_000, "incremental_ms": inc_ms, "added": added,
           "decremental_ms": dec_ms, "removed": removed, "S": S,
           "min_max_ms": {"static": st_rng, "incremental": inc_rng, "decremental": dec_rng},
           "wall_ms": {"static": st_wall, "incremental": inc_wall, "decremental": dec_wall},
           "timing": "CUDA events on the graph's stream around each call (a call synchronises once for its plan "
                     "scan's host read-back, inside the interval), median of 5; wall_ms = host clock"}
    g.close(); gu.close()
    return out


def run_ours(args, ws, rank, local):
    import torch

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    K, Wm = args.steps, args.warmup
    W, gen_s = make_workload(args, K + Wm, rank)
    V = W.vertex_n
    stream = torch.cuda.current_stream(dev)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.uint32).view(np.int32)).to(dev)
    flush = torch.empty((256 << 20) if args.l2_flush else 1, dtype=torch.uint8, device=dev)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak = peaks.get("hbm_gbs") or 6650.0
    peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)" if peaks.get("hbm_gbs") else "fallback (B200_PROFILING.md)"
    traffic_file = os.path.join(ROOT, "profiles", "traffic.json")

    res, (g, sp, bf) = measure(args, ws, W, args.frontier, dev, local, stream, T, flush, K, Wm,
                               clocks=ClockSampler(local), fused=args.fused)
    edges = 2 * args.batch * K * ws
    value = edges / (res["total_ms"] / 1e3)
    mean = res["mean"]

    # ---------------- e2e through the C ABI with pinned host buffers
    e2e = None
    if not args.no_e2e:
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.uint32).view(np.int32)).pin_memory()
        hi = [tuple(pin(x) for x in b) for b in W.inserts[Wm:Wm + K]]
        hd = [tuple(pin(x) for x in b[:2]) for b in W.deletes[Wm:Wm + K]]
        # the timed steps already applied these batches: undo them (not timed), then replay from host memory
        for k in reversed(range(K)):
            g.insert(*[T(x) for x in W.deletes[Wm + k]], count=False)
            g.delete(*[T(x) for x in W.inserts[Wm + k][:2]], count=False)
        sp.recompute(); bf.recompute()
        g.sync()
        e_ms = 0.0
        barrier(ws)
        for k in range(K):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            s, d, w = hi[k]
            seed = [sp, bf] if (args.fused and args.seed) else None
            g.insert(s, d, w, count=True, seed=seed)   # H2D staged inside the call, count read back (D2H)
            if args.fused:
                g.trees_incremental([sp, bf], s, d, w)
            else:
                sp.incremental(s, d, w)
                bf.incremental(s, d)
            s, d = hd[k]
            g.delete(s, d, count=True, seed=seed)
            if args.fused:
                g.trees_decremental([sp, bf], s, d)
            else:
                sp.decremental(s, d)
                bf.decremental(s, d)
            b.record(stream)
            b.synchronize()
            e_ms += a.elapsed_time(b)
            flush.zero_()
        e_ms = allreduce_max(e_ms, ws)
        n = args.batch
        e2e_sync = {"value": edges / (e_ms / 1e3), "unit": "edges/s",
                    # src, dst, w of the insert batch and src, dst of the delete batch; the tree calls that
                    # follow with the same host arrays reuse the staged copies (api.cu stage_in_reuse)
                    "h2d_bytes_per_step": n * 4 * (3 + 2),
                    "d2h_bytes_per_step": 2 * 64,
                    "ms_per_step": e_ms / K,
                    "how": "each step timed alone: the library stages the pinned host batches inside each call "
                           "and the insert / delete counts are read back synchronously (L2 flushed between steps)"}
        # pipelined: the next step's batches move host -> device on a copy stream while this step
        # computes (two device slots); each step's result -- the cumulative insert / delete counters --
        # is copied device -> host without stalling (meerkat_counters_async); one synchronisation at the end
        for k in reversed(range(K)):   # undo the synchronous run's batches again (not timed)
            g.insert(*[T(x) for x in W.deletes[Wm + k]], count=False)
            g.delete(*[T(x) for x in W.inserts[Wm + k][:2]], count=False)
        sp.recompute(); bf.recompute()
        g.sync()
        cs = torch.cuda.Stream(dev)
        # one pinned buffer per step holding the step's five arrays (insert src, dst, w; delete src, dst)
        # and one device slot per parity: ONE copy per step (five separate copies cost more host time
        # than the device spends on a step when the host is slow)
        hb = [torch.cat([*hi[k], *hd[k]]).pin_memory() for k in range(K)]
        dbuf = [torch.empty(5 * n, dtype=torch.int32, device=dev) for _ in range(2)]
        slots = [([dbuf[i][j * n:(j + 1) * n] for j in range(3)], [dbuf[i][j * n:(j + 1) * n] for j in (3, 4)])
                 for i in range(2)]
        ready = [torch.cuda.Event() for _ in range(2)]
        freed = [torch.cuda.Event() for _ in range(2)]
        ctr = torch.zeros((K, 3), dtype=torch.int64).pin_memory()

        def h2d(k):
            sl = k % 2
            with torch.cuda.stream(cs):
                if k >= 2:
                    cs.wait_event(freed[sl])   # step k - 2 is done with this slot
                dbuf[sl].copy_(hb[k], non_blocking=True)
                ready[sl].record(cs)
        torch.cuda.synchronize()
        barrier(ws)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        t_host = time.perf_counter()
        h2d(0)
        seed = [sp, bf] if (args.fused and args.seed) else None
        for k in range(K):
            sl = k % 2
            if k + 1 < K:
                h2d(k + 1)
            stream.wait_event(ready[sl])
            s, d, w = slots[sl][0]
            g.insert(s, d, w, count=False, seed=seed)
            if args.fused:
                g.trees_incremental([sp, bf], s, d, w)
            else:
                sp.incremental(s, d, w); bf.incremental(s, d)
            s, d = slots[sl][1]
            g.delete(s, d, count=False, seed=seed)
            if args.fused:
                g.trees_decremental([sp, bf], s, d)
            else:
                sp.decremental(s, d); bf.decremental(s, d)
            g.counters_async(ctr[k])
            freed[sl].record(stream)
        b.record(stream)
        host_ms = (time.perf_counter() - t_host) * 1e3   # the host's enqueue time for the K steps
        b.synchronize()
        p_ms = allreduce_max(a.elapsed_time(b), ws)
        st_end = g.stats()
        live = [int(r[0] - r[1]) for r in ctr.tolist()]
        e2e = {"value": edges / (p_ms / 1e3), "unit": "edges/s",
               "h2d_bytes_per_step": n * 4 * (3 + 2),   # src, dst, w of the insert batch; src, dst of the delete
               "d2h_bytes_per_step": 3 * 8,             # the cumulative counters after the step
               "ms_per_step": p_ms / K,
               "how": "the K steps back to back through the public API (Graph on CUDA tensors): each step's "
                      "batches copied from pinned host memory (one buffer per step) on a copy stream while the "
                      "previous step computes (two device slots, events), each step's counters copied back with "
                      "meerkat_counters_async; one synchronisation at the end; no L2 flush (store > L2)",
               "host_enqueue_ms_per_step": host_ms / K,
               "result_check": {"live_edges_after_last_step": live[-1], "stats_edges": st_end["edges"],
                                "ok": live[-1] == st_end["edges"]},
               "synchronous": e2e_sync}
    lat = g.probe_latency() if args.probe else None
    pagerank = None
    if args.pagerank and args.frontier == "reverse" and ws == 1:
        pagerank = measure_pagerank(g, W, T, stream, flush, peak, peak_src)
    wcc = measure_wcc(g, W, T, stream, flush) if args.wcc and ws == 1 else None
    g.close()
    del g, sp, bf
    torch.cuda.empty_cache()

    # ---------------- the paper's own decremental frontier (full slab scan) for comparison
    # ---------------- per-tree calls (unfused) for the SSSP / BFS split of the same step
    per_tree = None
    if args.fused and args.per_tree:
        r1, objs = measure(args, ws, W, args.frontier, dev, local, stream, T, flush, K, Wm, fused=False)
        objs[0].close()
        del objs
        per_tree = r1["mean"]

    alt = None
    if args.compare:
        other = "scan" if args.frontier == "reverse" else "reverse"
        r2, objs = measure(args, ws, W, other, dev, local, stream, T, flush, K, Wm, fused=args.fused)
        objs[0].close()
        del objs
        alt = {"decremental_frontier": other, "value": edges / (r2["total_ms"] / 1e3),
               "ms_per_step": r2["ms_per_step"], "per_call_ms": r2["mean"],
               "roofline": roofline_of(r2, peak, peak_src, traffic_file), "tree_calls": tree_detail(r2)}

    sweep = store_sweep(args, dev, stream) if args.sweep and ws == 1 else None

    # ---------------- hashing off vs on (hashing disabled ran BFS / SSSP 9-11% faster on the
    # paper's GPU): the same step and static recomputes on a store with one slab list per vertex
    hashing_ab = None
    if args.hashing_ab and not args.no_hashing and ws == 1:
        import copy
        a_off = copy.copy(args)
        a_off.no_hashing = True
        r3, objs = measure(a_off, ws, W, args.frontier, dev, local, stream, T, flush, K, Wm, fused=args.fused)
        objs[0].close()
        del objs
        sw_off = store_sweep(a_off, dev, stream) if args.sweep else None
        on = {"ms_per_step": res["ms_per_step"], "per_call_ms": mean, "static_ms": res["static_ms"],
              "vanilla_static_ms": res["vanilla_ms"], "store": res["store"]}
        off = {"ms_per_step": r3["ms_per_step"], "per_call_ms": r3["mean"], "static_ms": r3["static_ms"],
               "vanilla_static_ms": r3["vanilla_ms"], "store": r3["store"],
               "tree_calls": tree_detail(r3)}
        faster = lambda x_on, x_off: x_on / x_off - 1   # > 0: hashing off is faster by that fraction
        hashing_ab = {
            "on": on, "off": off,
            "off_faster_by": {
                "step": faster(on["ms_per_step"], off["ms_per_step"]),
                **{f"call_{k}": faster(on["per_call_ms"][k], off["per_call_ms"][k]) for k in on["per_call_ms"]},
                **{f"static_{k}": faster(on["static_ms"][k], off["static_ms"][k]) for k in on["static_ms"]},
                **{f"vanilla_static_{k}": faster(on["vanilla_static_ms"][k], off["vanilla_static_ms"][k])
                   for k in (on["vanilla_static_ms"] or {})}},
            "config2_sweep_off": sw_off,
            "paper": "hashing disabled: BFS vanilla / tree 10.78% / 9.1% faster, SSSP vanilla / tree 9.9% / 11% faster "
                     "on average (RTX 2080 Ti, 7 graphs; P:2282-2286)"}
    tc = measure_tc(args, dev, stream) if args.tc and ws == 1 else None
    config4 = measure_config4(args, dev, stream, flush) if args.config4 and ws == 1 else None

    cb = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cb = cpu_baseline(args, args.cpu_steps)
        cb = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample", "host_cores", "cpu_model",
                                 "oracle_threads", "per_batch_s")}

    split = mean if not args.fused else per_tree
    dyn = {"sssp": split["sssp_inc"] + split["sssp_dec"], "bfs": split["bfs_inc"] + split["bfs_dec"]} if split else None
    line = {
        "metric": METRIC, "value": value, "unit": "edges/s", "n_gpus": ws, "steps": K, "warmup": Wm,
        "ms_per_step": res["ms_per_step"], "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u64", "data": "synthetic",
        "config": workload_config(args, V, res["n_base"], W.source, ws),
        "update_edges_per_s": 2 * args.batch / ((mean["insert"] + mean["delete"]) / 1e3),
        "insert_edges_per_s": args.batch / (mean["insert"] / 1e3),
        "delete_edges_per_s": args.batch / (mean["delete"] / 1e3),
        "sssp_bfs_fused_ms_per_batch": ({"incremental": mean["trees_inc"], "decremental": mean["trees_dec"]}
                                        if args.fused else None),
        "sssp_ms_per_batch": ({"incremental": split["sssp_inc"], "decremental": split["sssp_dec"],
                               "measured": "per-tree calls, separate run" if args.fused else "in the timed steps"}
                              if split else None),
        "bfs_ms_per_batch": ({"incremental": split["bfs_inc"], "decremental": split["bfs_dec"]} if split else None),
        "per_call_ms": mean,
        "per_call_ms_p50_p95": {n: [float(np.percentile(v, 50)), float(np.percentile(v, 95))]
                                for n, v in res["per_call"].items()},
        "static_recompute_ms": res["static_ms"],
        "vanilla_static_ms": res["vanilla_ms"] or None,
        "iteration_scheme1_static_ms": res["scheme1_ms"] or None,
        "tree_overhead_vs_vanilla": ({k: res["static_ms"][k] / res["vanilla_ms"][k] - 1 for k in res["vanilla_ms"]}
                                     if res["vanilla_ms"] else None),
        "self_relative_speedup": ({k: res["static_ms"][k] / (dyn[k] / 2) for k in dyn} if dyn else None),
        "bulk_build": {"edges": res["n_base"], "ms": res["bulk_ms"], "edges_per_s": res["n_base"] / (res["bulk_ms"] / 1e3)},
        "tree_calls": tree_detail(res),
        "roofline": roofline_of(res, peak, peak_src, traffic_file),
        "update_roofline": update_roofline(res, args, peak, peak_src, traffic_file,
                                           2 if args.frontier == "reverse" else 1, 2 if args.fused else 0),
        "latency_floor": latency_floor(lat, res),
        "hashing_ab": hashing_ab,
        "cpu_baseline": cb,
        "e2e": e2e,
        "gpu_launches": res["launches"],
        "clocks": res["clocks"],
        "store": res["store"],
        "alt": alt,
        "store_sweep": sweep,
        "pagerank": pagerank,
        "wcc": wcc,
        "tc": tc,
        "config4": config4,
        "generate_s": gen_s,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
        if args.json_out:
            with open(args.json_out, "w") as f:
                json.dump(line, f, indent=1)


def run_dist(args, ws, rank, local):
    """Vertex-partitioned path: the SAME config-3 graph split over `ws` GPUs by the
    library's placement (owner = mix(v) mod ws); every rank brings 1/ws of each batch and the library
    routes it (one all-to-all-v); tree updates run as device-driven exchange units over the library's
    NCCL communicator (a fixed-size all-to-all per unit) -> strong scaling."""
    import torch
    from paper_2305_17813_b200.dist import DistGraph

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    K, Wm = args.steps, args.warmup
    W, gen_s = make_workload(args, K + Wm, 0)
    V = W.vertex_n
    stream = torch.cuda.current_stream(dev)
    sl = lambda a: np.ascontiguousarray(a[rank::ws])
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.uint32).view(np.int32)).to(dev)
    bs, bd, bw = W.base
    reverse = args.frontier == "reverse"
    g = DistGraph(V, hashing=not args.no_hashing, load_factor=args.lf,
                  degree_hints=np.bincount(bs, minlength=V).astype(np.uint32),
                  in_degree_hints=np.bincount(bd, minlength=V).astype(np.uint32) if reverse else None,
                  reverse=reverse, device=dev, stream=stream)
    barrier(ws)
    t0 = time.time()
    n_base = g.insert(T(sl(bs)), T(sl(bd)), T(sl(bw)))
    sp, bf = g.sssp(W.source), g.bfs(W.source)
    build_s = time.time() - t0
    ins = [tuple(T(sl(x)) for x in b) for b in W.inserts]
    dels = [tuple(T(sl(x)) for x in b[:2]) for b in W.deletes]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    names = NAMES_FUSED   # SSSP + BFS in lock step: one exchange per round for both trees
    for i in range(Wm):
        one_step(g, sp, bf, ins[i], dels[i], [torch.cuda.Event(enable_timing=True) for _ in range(len(names) + 1)],
                 stream, fused=True)
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    per_call = {n: [] for n in names}
    total_ms = 0.0
    dec_bytes = []
    exchanges = []
    l0 = g.stats()["kernel_launches"]
    for k in range(K):
        flush.zero_()
        torch.cuda.synchronize()
        barrier(ws)
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(len(names) + 1)]
        one_step(g, sp, bf, ins[Wm + k], dels[Wm + k], evs, stream, fused=True)
        evs[-1].synchronize()
        step_ms = allreduce_max(evs[0].elapsed_time(evs[-1]), ws)
        total_ms += step_ms
        for j, n in enumerate(names):
            per_call[n].append(allreduce_max(evs[j].elapsed_time(evs[j + 1]), ws))
        # algorithmic bytes of the decremental call on this rank (both trees), read outside the interval
        dec_bytes.append(sp.stats()["alg_bytes"] + bf.stats()["alg_bytes"])
        exchanges.append(sp.stats()["exchanges"])
    launches = g.stats()["kernel_launches"] - l0
    clk = clocks.stop()
    mean = {n: float(np.mean(v)) for n, v in per_call.items()}
    edges = 2 * args.batch * K
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak = peaks.get("hbm_gbs") or 6650.0
    tot_bytes = allreduce_sum(float(np.mean(dec_bytes)), ws)   # all ranks' bytes of one call
    ach = tot_bytes / (mean["trees_dec"] * 1e-3) / 1e9
    roofline = {"bound": "hbm", "kernel": "fused decremental update, all exchange units (partitioned)",
                "achieved": ach, "peak": peak * ws, "unit": "GB/s", "frac": ach / (peak * ws),
                "traffic": None, "alg_bytes_per_launch": tot_bytes,
                "peak_source": ("measured (MEASURED_PEAKS.json hbm_gbs) x " if peaks.get("hbm_gbs") else
                                "fallback (B200_PROFILING.md) x ") + f"{ws} GPUs"}
    # e2e: the same fused step from pinned HOST batches through the public API (DistGraph), counts read
    # back; the timed batches are undone first (not timed) and the trees recomputed
    e2e = None
    if not args.no_e2e:
        for k in reversed(range(K)):
            s, d, w = W.deletes[Wm + k]
            g.insert(T(sl(s)), T(sl(d)), T(sl(w)), count=False)
            s, d, _ = W.inserts[Wm + k]
            g.delete(T(sl(s)), T(sl(d)), count=False)
        sp.recompute(); bf.recompute()
        torch.cuda.synchronize()
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(sl(a), np.uint32).view(np.int32)).pin_memory()
        hi = [tuple(pin(x) for x in W.inserts[Wm + k]) for k in range(K)]
        hd = [tuple(pin(x) for x in W.deletes[Wm + k][:2]) for k in range(K)]
        e_ms = 0.0
        for k in range(K):
            barrier(ws)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            s, d, w = hi[k]
            g.insert(s, d, w, count=True)                # H2D inside, all-reduced count read back
            g.trees_incremental([sp, bf], s, d, w)
            s, d = hd[k]
            g.delete(s, d, count=True)
            g.trees_decremental([sp, bf], s, d)
            b.record(stream)
            b.synchronize()
            e_ms += allreduce_max(a.elapsed_time(b), ws)
            flush.zero_()
        e2e = {"value": edges / (e_ms / 1e3), "unit": "edges/s",
               "h2d_bytes_per_step": args.batch * 4 * (3 + 3 + 2 + 2), "d2h_bytes_per_step": 2 * 8 * ws,
               "ms_per_step": e_ms / K}
    line = {
        "metric": METRIC, "value": edges / (total_ms / 1e3), "unit": "edges/s", "n_gpus": ws, "steps": K,
        "warmup": Wm, "ms_per_step": total_ms / K, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": f"rmat-s{args.scale}-ef{args.ef} dynamic SSSP+BFS, {args.batch}-edge insert+delete "
                               f"batches (BASELINE config 3)", "vertices": V, "edges": int(n_base),
                   "batch": args.batch, "source": W.source, "hashing": not args.no_hashing,
                   "load_factor": args.lf,
                   "decremental_frontier": "in-edge mirror, pull requests to owner(u)" if reverse else
                   "scan (per partition, invalid sets exchanged)",
                   "parallelism": f"vertex-partitioned over {ws} GPUs (owner = mix(v) mod {ws}), library NCCL "
                                  f"communicator, one fixed-size all-to-all per exchange unit",
                   "l2": "flushed before every timed step; store > L2"},
        "update_edges_per_s": 2 * args.batch / ((mean["insert"] + mean["delete"]) / 1e3),
        "sssp_bfs_fused_ms_per_batch": {"incremental": mean["trees_inc"], "decremental": mean["trees_dec"]},
        "per_call_ms": mean, "build_s": build_s, "roofline": roofline, "cpu_baseline": None,
        "e2e": e2e, "gpu_launches": allreduce_sum(float(launches), ws), "clocks": clk, "generate_s": gen_s,
        "exchanges_per_decremental_call": float(np.mean(exchanges)) if exchanges else None,
        "note": "device-driven exchange units (the host reads a mode word PIPE units behind); timings are max "
                "over ranks",
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
        if args.json_out:
            with open(args.json_out, "w") as f:
                f.write(json.dumps(line) + "\n")


def self_launch(n):
    """`python bench.py --gpus N` outside torchrun: start the N ranks ourselves (one process per GPU,
    127.0.0.1 rendezvous) exactly as the driver's torchrun command would."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    os.execv(sys.executable, cmd)


def main():
    args = parse()
    ws_env = int(os.environ.get("WORLD_SIZE", "1"))
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        self_launch(args.gpus)
    if args.gpus != ws_env and args.impl == "ours":
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws_env}: launch one rank per GPU "
                 f"(torchrun --nproc-per-node {args.gpus}) or omit WORLD_SIZE to let bench.py start them")
    if ws_env > 1:   # N generator processes on one host: split the cores
        os.environ.setdefault("OMP_NUM_THREADS", str(max(1, (os.cpu_count() or 8) // ws_env)))
    ws, rank, local = dist_init(args)
    if args.impl == "reference":
        run_reference(args, ws, rank)
    elif ws > 1 or args.partitioned:
        run_dist(args, ws, rank, local)
    else:
        run_ours(args, ws, rank, local)
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

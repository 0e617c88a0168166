#!/usr/bin/env python
"""Where does a partitioned (multi-GPU path) step spend its time?  World size 1 through NCCL on one
GPU: host wall time of every phase call and every exchange, per fused tree update.  GPU only.
    python tools/diag_dist.py [--scale 24]"""
import argparse, os, sys, time
from collections import defaultdict
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=24)
    a = ap.parse_args()
    import torch
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29533")
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    import synth
    from paper_2305_17813_b200 import dist as D
    W = synth.rmat_dynamic(a.scale, 16, batch=100_000, n_ins=3, n_del=3)
    V = W.vertex_n
    T = lambda x: torch.from_numpy(np.ascontiguousarray(x, np.uint32).view(np.int32)).cuda()
    bs, bd, bw = W.base
    g = D.DistGraph(V, degree_hints=np.bincount(bs, minlength=V).astype(np.uint32), device=torch.device("cuda", 0))
    g.insert(T(bs), T(bd), T(bw))
    sp, bf = g.sssp(W.source), g.bfs(W.source)
    acc = defaultdict(float); cnt = defaultdict(int)
    orig_phase, orig_ex = D.DistTree._phase, D.DistGraph._exchange_apply

    def phase(self, ph, *x, **k):
        t0 = time.perf_counter(); r = orig_phase(self, ph, *x, **k)
        acc[f"phase{ph}"] += time.perf_counter() - t0; cnt[f"phase{ph}"] += 1
        return r

    def ex(self, *x, **k):
        t0 = time.perf_counter(); r = orig_ex(self, *x, **k)
        acc["exchange"] += time.perf_counter() - t0; cnt["exchange"] += 1
        return r
    D.DistTree._phase, D.DistGraph._exchange_apply = phase, ex
    for i in range(3):
        acc.clear(); cnt.clear()
        s, d, w = (T(x) for x in W.inserts[i])
        g.insert(s, d, w, count=False); torch.cuda.synchronize()
        t0 = time.perf_counter(); g.trees_incremental([sp, bf], s, d, w); torch.cuda.synchronize()
        ti = time.perf_counter() - t0
        inc = dict(acc); ic = dict(cnt); acc.clear(); cnt.clear()
        s, d = T(W.deletes[i][0]), T(W.deletes[i][1])
        g.delete(s, d, count=False); torch.cuda.synchronize()
        t0 = time.perf_counter(); g.trees_decremental([sp, bf], s, d); torch.cuda.synchronize()
        td = time.perf_counter() - t0
        print(f"batch {i}: inc {1e3*ti:.2f} ms {{" + ", ".join(f"{k}: {1e3*v:.2f} ms/{ic[k]}" for k, v in inc.items()) + "}")
        print(f"         dec {1e3*td:.2f} ms {{" + ", ".join(f"{k}: {1e3*v:.2f} ms/{cnt[k]}" for k, v in acc.items()) + "}")
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

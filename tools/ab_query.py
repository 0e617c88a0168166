"""A/B of the query kernels (group-cooperative vs thread-per-edge) on R-MAT scale 20 (config 2):
median device time of 5 batches per size; parity of the answers between the two.  GPU only.
    python tools/ab_query.py   (runs both variants in subprocesses)"""
import os, subprocess, sys, json
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run():
    import torch, synth
    from paper_2305_17813_b200 import Graph
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.uint32).view(np.int32)).cuda()
    s, d, w = synth.rmat(20, 16)
    V = 1 << 20
    g = Graph(V, degree_hints=T(np.bincount(s, minlength=V).astype(np.uint32)))
    g.insert(T(s), T(d), T(w))
    rng = np.random.default_rng(5)
    out = {}
    for b in (1000, 10000, 100000, 1000000):
        half = b // 2
        qs = T(np.concatenate([s[rng.integers(0, len(s), half)], rng.integers(0, V, b - half)]))
        qd = T(np.concatenate([d[rng.integers(0, len(s), half)], rng.integers(0, V, b - half)]))
        ts = []
        for r in range(7):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); f, ww = g.query(qs, qd); e1.record(); e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        out[b] = {"ms": float(np.median(ts[2:])), "found": int(f.sum().item()), "wsum": int(ww.sum().item())}
    print(json.dumps(out))


if __name__ == "__main__":
    if len(sys.argv) > 1:
        run()
    else:
        for v in ("0", "1"):
            env = dict(os.environ, MEERKAT_THREAD_QUERY=v)
            r = subprocess.run([sys.executable, __file__, "x"], env=env, capture_output=True, text=True)
            print("thread" if v == "1" else "group", r.stdout.strip(), r.stderr[-500:])

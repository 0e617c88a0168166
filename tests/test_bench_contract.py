"""bench.py's JSON-line contract on the CPU: the reference arm (--impl reference times the oracle,
the one arm that runs without a GPU) prints exactly one JSON line with the keys the driver reads,
a `config` describing the oracle sample it timed (and the workload it samples), and the cpu_baseline /
e2e objects."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1", "--warmup", "1",
           "--scale", "12", "--cpu-scale", "11", "--cpu-steps", "1", "--batch", "500"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "edges/s"
    # the config describes what was timed (the scale-11 sample), and names the workload it samples
    assert d["config"]["workload"].startswith("rmat-s11-ef16") and d["config"]["batch"] == 500
    assert d["config"]["sample_of"].startswith("rmat-s12-ef16")
    assert d["config"]["vertices"] == 1 << 11 and d["config"]["edges"] > 0
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] == 1 and cb["value"] == d["value"] and "sample" in cb
    assert cb["host_cores"] >= 1 and cb["cpu_model"] and cb["oracle_threads"] == 1
    assert set(cb["per_batch_s"]) == {"apply_insert", "apply_delete", "sssp", "bfs"}
    assert d["e2e"] == {"value": d["value"], "unit": "edges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_gpus_flag_self_launches_ranks():
    """`bench.py --gpus 2` outside torchrun starts the two ranks itself (127.0.0.1 rendezvous); for the
    reference arm rank 0 alone prints the line and the other rank exits 0 without work."""
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2", "--steps", "1",
           "--warmup", "1", "--scale", "12", "--cpu-scale", "11", "--cpu-steps", "1", "--batch", "500"]
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1 and json.loads(lines[0])["impl"] == "reference"


def test_gpus_flag_mismatch_fails():
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1", "--warmup", "1"]
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode != 0 and "WORLD_SIZE" in (r.stderr + r.stdout)

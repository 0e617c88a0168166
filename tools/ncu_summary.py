#!/usr/bin/env python
"""Summarise ncu artefacts for profiles/ (runs here, no GPU needed).

  python tools/ncu_summary.py rep  <file.ncu-rep> [top]   # key raw metrics + per-source-line stall/inst shares
  python tools/ncu_summary.py list <launches.csv>         # per-kernel launch count, total and share of time
"""
import csv
import subprocess
import sys
from collections import defaultdict

RAW = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
       "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
       "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum", "launch__registers_per_thread",
       "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
       "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]


def rep(path, top=25):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        for w in RAW:
            if w in hdr:
                i = hdr.index(w)
                print(f"  {w:62s} {vals[i]} {units[i]}")
        rd = float(vals[hdr.index("dram__bytes_read.sum")]) if "dram__bytes_read.sum" in hdr else 0
        print()
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    cur, hdr, agg = None, None, {}
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 8 or not r[0]:
            continue
        try:
            samp, inst = float(r[4] or 0), float(r[7] or 0)
        except ValueError:
            continue
        k = (cur, int(r[0]))
        a = agg.setdefault(k, [0.0, 0.0, r[1]])
        a[0] += samp
        a[1] += inst
    ts = sum(v[0] for v in agg.values()) or 1
    ti = sum(v[1] for v in agg.values()) or 1
    print(f"source lines by warp-stall samples (total samples {ts:.0f}, instructions {ti:.0f}):")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"  {k[0]}:{k[1]:<5d} stall {100 * v[0] / ts:5.1f}%  inst {100 * v[1] / ti:5.1f}%  {v[2].strip()[:100]}")


def launches(path):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    ki, mi, ui, vi = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0]
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1e-3)
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", "")) * scale
    tot = sum(v[1] for v in agg.values()) or 1
    print(f"{'kernel':60s} {'launches':>8s} {'total us':>12s} {'mean us':>10s} {'share':>7s}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k[:60]:60s} {v[0]:8d} {v[1]:12.1f} {v[1] / v[0]:10.1f} {100 * v[1] / tot:6.1f}%")


if __name__ == "__main__":
    if sys.argv[1] == "rep":
        rep(sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 25)
    else:
        launches(sys.argv[2])

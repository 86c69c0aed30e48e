#!/usr/bin/env python
"""Summarize ncu reports (gpurun_out/*.ncu-rep, launches.csv) into profiles/.

    python scripts/ncu_summary.py --round r01 [--dir gpurun_out]

Writes profiles/ncu_summary.json (per kernel: duration, DRAM bytes per launch,
throughput %, registers, occupancy) and profiles/<round>_launches.txt (the
launch list of the bench command aggregated per kernel, with time shares).
"""
import argparse
import csv
import glob
import io
import json
import os
import re
import subprocess
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_peak",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct_of_peak",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__shared_mem_per_block_dynamic": "dyn_smem",
    "lts__t_bytes.sum": "l2_bytes",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0,
         "nsecond": 1e-9, "second": 1.0}


def short(name: str) -> str:
    m = re.search(r"(\w+_kernel)", name)
    return m.group(1) if m else name.split("(")[0]


def parse_rep(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        rec = {"kernel": r[hdr.index("Kernel Name")], "report": os.path.basename(path)}
        for m, key in METRICS.items():
            if m not in hdr:
                continue
            i = hdr.index(m)
            val = r[i].replace(",", "")
            try:
                v = float(val)
            except ValueError:
                continue
            u = units[i]
            if key in ("dram_read", "dram_write", "l2_bytes"):
                v *= SCALE.get(u, 1)
            if key == "duration":
                v *= SCALE.get(u, 1e-9)
            rec[key] = v
        if "dram_read" in rec and "dram_write" in rec:
            rec["dram_bytes_per_launch"] = rec["dram_read"] + rec["dram_write"]
            rec["dram_gbs"] = rec["dram_bytes_per_launch"] / rec["duration"] / 1e9
        res.append(rec)
    return res


def parse_launches(path):
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.reader(io.StringIO(text[start:])))
    hdr = rows[0]
    ki, mi, vi, ui = (hdr.index("Kernel Name"), hdr.index("Metric Name"),
                      hdr.index("Metric Value"), hdr.index("Metric Unit"))
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        t = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1e-9)
        agg[short(r[ki]) if "tdkv" in r[ki] or "_kernel" in r[ki] else r[ki][:60]][0] += 1
        agg[short(r[ki]) if "tdkv" in r[ki] or "_kernel" in r[ki] else r[ki][:60]][1] += t
    total = sum(v[1] for v in agg.values())
    lines = [f"{'kernel':60s} {'launches':>9s} {'total_ms':>10s} {'share':>7s}"]
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"{k:60s} {n:9d} {t * 1e3:10.3f} {t / total:7.1%}")
    return "\n".join(lines)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", default="r01")
    ap.add_argument("--dir", default=os.path.join(ROOT, "gpurun_out"))
    args = ap.parse_args()
    prof = os.path.join(ROOT, "profiles")
    os.makedirs(prof, exist_ok=True)
    summary_path = os.path.join(prof, "ncu_summary.json")
    summary = json.load(open(summary_path)) if os.path.exists(summary_path) else {}
    for rep in sorted(glob.glob(os.path.join(args.dir, "*.ncu-rep"))):
        for rec in parse_rep(rep):
            rec["round"] = args.round
            # one entry per (kernel, capture): the same kernel is captured on
            # several workloads (e.g. K1 at C1 / C2 / C3 and as the family restore)
            name = os.path.splitext(os.path.basename(rep))[0]
            summary[f"{short(rec['kernel'])}@{name}"] = rec
    with open(summary_path, "w") as f:
        json.dump(summary, f, indent=1, sort_keys=True)
    launches = os.path.join(args.dir, "launches.csv")
    if os.path.exists(launches):
        with open(os.path.join(prof, f"{args.round}_launches.txt"), "w") as f:
            f.write(parse_launches(launches) + "\n")
    print(json.dumps({k: {kk: v.get(kk) for kk in ("duration", "dram_bytes_per_launch",
                                                   "dram_gbs", "dram_pct_of_peak", "registers")}
                      for k, v in summary.items()}, indent=1))


if __name__ == "__main__":
    main()

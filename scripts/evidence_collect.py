#!/usr/bin/env python
"""Copy the evidence of a `scripts/gpu_evidence.sh` (+ `gpu_sanitize.sh`) run from
gpurun_out/ into profiles/ (bench lines, codec sweep, HBM probe, pytest tail,
sanitizer summaries, ncu summary and text exports) and print the headline
numbers.

    python scripts/evidence_collect.py --round r01
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")


def last_json(path):
    with open(path) as f:
        lines = [l for l in f.read().splitlines() if l.startswith("{")]
    return json.loads(lines[-1])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", default="r01")
    r = ap.parse_args().round
    # r01: the default bench line was C2; from r02 the default is C3
    default = "c2" if r == "r01" else "c3"
    for src, dst in (("bench.log", default), ("bench_c1.log", "c1"), ("bench_c2.log", "c2"),
                     ("bench_c3.log", "c3"), ("bench_c4.log", "c4"), ("bench_c5.log", "c5"),
                     ("bench_ref.log", "ref")):
        if not os.path.exists(os.path.join(OUT, src)):
            continue
        d = last_json(os.path.join(OUT, src))
        with open(os.path.join(PROF, f"{r}_bench_{dst}.json"), "w") as f:
            json.dump(d, f, indent=1)
        if dst == "c4" and "codec_sweep" in d:
            with open(os.path.join(PROF, f"{r}_codec_sweep_c4.json"), "w") as f:
                json.dump({"config": d["config"], "codec_sweep": d["codec_sweep"]}, f, indent=1)
    with open(os.path.join(OUT, "hbm_probe.json")) as f, \
            open(os.path.join(PROF, f"{r}_hbm_probe.json"), "w") as g:
        g.write(f.read())
    with open(os.path.join(OUT, "pytest_gpu.log")) as f, \
            open(os.path.join(PROF, f"{r}_pytest_gpu.txt"), "w") as g:
        g.writelines(f.readlines()[-12:])
    lines = ["# compute-sanitizer over the GPU parity tests (scripts/gpu_sanitize.sh) at HEAD"]
    for tool in ("memcheck", "racecheck", "synccheck"):
        path = os.path.join(OUT, f"sanitize_{tool}.log")
        if os.path.exists(path):
            with open(path) as f:
                keep = [l.rstrip() for l in f if "passed" in l or "failed" in l or "SUMMARY" in l]
            lines += [f"## {tool}"] + keep[-2:]
    if not os.path.exists(os.path.join(PROF, f"{r}_sanitizers.txt")):
        with open(os.path.join(PROF, f"{r}_sanitizers.txt"), "w") as f:
            f.write("\n".join(lines) + "\n")
    for script in ("ncu_summary.py", "ncu_export.py"):
        subprocess.run([sys.executable, os.path.join(ROOT, "scripts", script), "--round", r],
                       check=True, stdout=subprocess.DEVNULL)
    d = json.load(open(os.path.join(PROF, f"{r}_bench_{default}.json")))
    print(default, d["value"], d["roofline"]["frac"], d["e2e"]["value"], d["codec"]["encode_gbs"],
          d["codec"]["decode_gbs"], d["selection"]["device_ms"], d["recovery"]["speedup"])


if __name__ == "__main__":
    main()

# per-kernel device time of GPU collective_recover on configs[0] (run under gpurun)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --print-units base --log-file gpurun_out/rec_launches.csv python scripts/recovery_profile.py > /dev/null 2>&1
python - <<'PY'
import csv, collections, re
lines = open("gpurun_out/rec_launches.csv").read().splitlines()
rows = list(csv.reader(lines[next(i for i, l in enumerate(lines) if l.startswith('"ID"')):]))
h = rows[0]
ik, iv = h.index("Kernel Name"), h.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    if len(r) <= iv: continue
    try: v = float(r[iv].replace(",", ""))
    except ValueError: continue
    m = re.search(r"(\w+_kernel)", r[ik]); k = m.group(1) if m else r[ik][:40]
    agg[k][0] += 1; agg[k][1] += v
tot = sum(v for _, v in agg.values())
print("device ms per collective_recover", tot / 7 / 1e6)
for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1])[:14]:
    print(f"{k:40s} {n:6d} {v/7/1e6:9.3f} ms/call {100*v/tot:5.1f}%")
PY

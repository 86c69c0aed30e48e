# family restore breakdown (C2/C3 codec family): A/B timing + per-kernel launch durations
OUT=gpurun_out
mkdir -p $OUT
for sh in c2 c3; do RESTORE_SHAPE=$sh timeout 300 python scripts/restore_ab.py > $OUT/restore_ab_$sh.txt 2>&1; echo $sh; cat $OUT/restore_ab_$sh.txt; done
RESTORE_SHAPE=c2 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --print-units base \
  -k regex:"collect_kernel|overlay_rows_kernel|rope_table" --log-file $OUT/restore_launches.csv python scripts/restore_ab.py > /dev/null 2>&1; echo ncu=$?
python - <<'PY'
import csv, collections, re
lines = open("gpurun_out/restore_launches.csv").read().splitlines()
rows = list(csv.reader(lines[next(i for i, l in enumerate(lines) if l.startswith('"ID"')):]))
h = rows[0]
ik, im, iv = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
agg = collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows[1:]:
    if len(r) <= iv: continue
    m = re.search(r"(\w+_kernel)", r[ik]); k = m.group(1) if m else r[ik][:40]
    try: agg[k][r[im]].append(float(r[iv].replace(",", "")))
    except ValueError: pass
for k, d in agg.items():
    t = d["gpu__time_duration.sum"]
    print(k, "launches", len(t), "median us", sorted(t)[len(t)//2] / 1e3,
          "dram GB", (sorted(d["dram__bytes_read.sum"])[len(t)//2] + sorted(d["dram__bytes_write.sum"])[len(t)//2]) / 1e9)
PY

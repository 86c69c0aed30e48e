# the reference-contract drop-in (host numpy contexts): parity tests + the C1 bench line's `dropin`
OUT=gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "align_cached or collector or skeleton" 2>&1 | tail -2
timeout 600 python bench.py --config c1 --steps 50 > $OUT/bench_c1.log 2>&1; echo c1=$?
python - <<'P'
import json
for l in open("gpurun_out/bench_c1.log"):
    if l.startswith("{"): d=json.loads(l); print(d.get("dropin")); print(d["value"], d["roofline"]["frac"])
P

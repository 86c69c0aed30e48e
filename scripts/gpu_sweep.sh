# K1 tile-budget sweep + ncu of the current K1 (run under gpurun)
set -x
OUT=gpurun_out
for b in 32768 65536 98304; do
  TDKV_TILE_SMEM=$b timeout 300 python bench.py --steps 20 --warmup 3 --no-codec --no-e2e --no-cpu > $OUT/sweep_$b.log 2>&1
  python -c "import json;d=json.loads(open('$OUT/sweep_$b.log').read().strip().splitlines()[-1]);print($b, d['value'], d['roofline']['frac'])"
done
timeout 600 python bench.py --steps 10 --warmup 3 --no-codec --no-cpu > $OUT/bench_e2e.log 2>&1
tail -1 $OUT/bench_e2e.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['e2e'])"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:collect_kernel -s 2 -c 1 \
  -o $OUT/k1_collect -f python bench.py --profile --steps 3 --warmup 1 > $OUT/k1.log 2>&1
echo k1=$?

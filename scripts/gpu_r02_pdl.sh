# r02: full GPU suite + C1/C2/C3 bench lines + PDL / auto-graph A/B on C1 (one GPU)
OUT=gpurun_out
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo pytest=$?
tail -5 $OUT/pytest_gpu.log
for cfg in c1 c2; do
  timeout 600 python bench.py --config $cfg --no-cpu > $OUT/bench_$cfg.json 2> $OUT/bench_$cfg.err; echo bench_$cfg=$?
done
for v in "TDKV_PDL=0" "TDKV_ROUND_GRAPHS=0" "TDKV_PDL=0 TDKV_ROUND_GRAPHS=0"; do
  env $v timeout 600 python bench.py --config c1 --no-cpu --no-codec --no-e2e > "$OUT/bench_c1_$(echo $v | tr ' =' '__').json" 2>&1; echo "c1 $v"=$?
done
timeout 900 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err; echo bench=$?

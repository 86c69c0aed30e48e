# everything the round's evidence needs, in one box call (run under gpurun)
set -x
OUT=gpurun_out
bash scripts/gpu_check.sh
bash scripts/gpu_configs.sh
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/launches.csv python bench.py --steps 3 --warmup 1 --no-cpu --no-e2e > $OUT/launches_bench.log 2>&1
echo launches=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:collect_kernel -s 2 -c 1 \
  -o $OUT/k1_collect -f python bench.py --profile --steps 3 --warmup 1 > $OUT/k1.log 2>&1; echo k1=$?

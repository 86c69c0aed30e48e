# ncu evidence for the bench kernels (run under gpurun; one GPU)
set -x
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo smoke=$?
# 1) launch list of the bench command (cold, serialized: compare shares)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/launches.csv python bench.py --steps 3 --warmup 1 --no-cpu --no-e2e > $OUT/launches_bench.log 2>&1
echo launches=$?
# 2) full sets of the top kernels
timeout 900 ncu --set full --clock-control none --import-source on -k regex:collect_kernel -s 2 -c 1 \
  -o $OUT/k1_collect -f python bench.py --profile --steps 3 --warmup 1 > $OUT/k1.log 2>&1
echo k1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"diff_compare|diff_compact" -s 2 -c 2 \
  -o $OUT/k2_codec -f python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > $OUT/k2.log 2>&1
echo k2=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rows_kernel -s 1 -c 1 \
  -o $OUT/k3_rows -f python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > $OUT/k3.log 2>&1
echo k3=$?
ls -la $OUT

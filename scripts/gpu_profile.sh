# ncu evidence for every kernel family (run under gpurun; one GPU)
set -x
OUT=gpurun_out
rm -f $OUT/*.ncu-rep
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/launches.csv python bench.py --steps 3 --warmup 1 --no-cpu --no-e2e > $OUT/launches_bench.log 2>&1
echo launches=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:collect_kernel -s 2 -c 1 \
  -o $OUT/k1_collect -f python bench.py --profile --steps 3 --warmup 1 > $OUT/k1.log 2>&1; echo k1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"diff_encode" -s 2 -c 1 \
  -o $OUT/k2_codec -f python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > $OUT/k2.log 2>&1; echo k2=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rows_tma_kernel -s 2 -c 1 \
  -o $OUT/k3_rows -f python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > $OUT/k3.log 2>&1; echo k3=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"keydiff_kernel|select_kernel" -s 2 -c 2 \
  -o $OUT/k4_select -f python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > $OUT/k4.log 2>&1; echo k4=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_" -s 1 -c 2 \
  -o $OUT/k5_gemm -f python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > $OUT/k5.log 2>&1; echo k5=$?
ls -la $OUT

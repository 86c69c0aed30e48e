# r02: new GPU tests, default bench (C3), C3 ncu captures (one GPU)
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_t3.py tests/test_gpu_dist.py tests/test_gpu_bf16_codec.py -x -q > $OUT/pytest_new.log 2>&1; echo pytest_new=$?
tail -15 $OUT/pytest_new.log
timeout 900 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err; echo bench=$?
tail -c 600 $OUT/bench_default.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:collect_kernel -s 2 -c 1 \
  -o $OUT/k1_collect_c3 -f python bench.py --profile --config c3 --steps 3 --warmup 1 > $OUT/k1_c3.log 2>&1; echo k1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"diff_encode" -s 2 -c 1 \
  -o $OUT/k2_codec_c3 -f python bench.py --config c3 --steps 1 --warmup 1 --no-cpu --no-e2e > $OUT/k2_c3.log 2>&1; echo k2=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rows_tma_kernel -s 2 -c 1 \
  -o $OUT/k3_rows_c3 -f python bench.py --config c3 --steps 1 --warmup 1 --no-cpu --no-e2e > $OUT/k3_c3.log 2>&1; echo k3=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/launches_c3.csv python bench.py --steps 3 --warmup 1 --no-cpu --no-e2e > $OUT/launches_c3.log 2>&1; echo launches=$?
ls -la $OUT

# r02: GPU suite + family-order A/B for K2/K3 + DRAM bytes per launch (one GPU)
OUT=gpurun_out
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo pytest=$?
tail -5 $OUT/pytest_gpu.log
for mode in family legacy; do
  if [ $mode = legacy ]; then export TDKV_ENCODE_ORDER=pair TDKV_RESTORE_ORDER=job; fi
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > $OUT/bench_c2_$mode.json 2> $OUT/bench_c2_$mode.err; echo bench_$mode=$?
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum \
    --clock-control none -k regex:"diff_encode|rows_tma" -c 6 --csv --log-file $OUT/ncu_codec_$mode.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > $OUT/ncu_codec_$mode.log 2>&1; echo ncu_$mode=$?
done
unset TDKV_ENCODE_ORDER TDKV_RESTORE_ORDER

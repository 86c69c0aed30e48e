OUT=gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:diff_encode -s 2 -c 1 \
  -o $OUT/k2_codec_c3 -f python bench.py --config c3 --steps 1 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1; echo k2c3=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:diff_encode -s 2 -c 1 \
  -o $OUT/k2_codec_c2 -f python bench.py --config c2 --steps 1 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1; echo k2c2=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rows_tma -s 2 -c 1 \
  -o $OUT/k3_rows_c3 -f env RESTORE_SHAPE=c3 python scripts/restore_ab.py > /dev/null 2>&1; echo k3c3=$?

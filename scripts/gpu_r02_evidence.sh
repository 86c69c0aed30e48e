# round-2 evidence pass on one B200 (run under gpurun): parity, bench lines of every config + the
# reference arm, the default bench command's launch list, one ncu --set full capture per kernel
OUT=gpurun_out
mkdir -p $OUT
rm -f $OUT/*.ncu-rep
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo smoke=$?; tail -1 $OUT/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 $OUT/pytest_gpu.log
timeout 300 python scripts/hbm_probe.py > $OUT/hbm_probe.json 2>&1
timeout 600 python bench.py > $OUT/bench.log 2>&1; echo bench=$?
timeout 600 python bench.py --config c1 --steps 50 > $OUT/bench_c1.log 2>&1; echo c1=$?
timeout 600 python bench.py --config c2 > $OUT/bench_c2.log 2>&1; echo c2=$?
timeout 900 python bench.py --config c4 --no-cpu --codec-mirrors 32 --codec-sweep > $OUT/bench_c4.log 2>&1; echo c4=$?
timeout 900 python bench.py --config c5 --steps 3 --no-cpu --no-codec > $OUT/bench_c5.log 2>&1; echo c5=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref.log 2>&1; echo ref=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/launches.csv python bench.py --steps 3 --warmup 1 --no-cpu --no-e2e > $OUT/launches_bench.log 2>&1; echo launches=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:collect_kernel -s 2 -c 1 \
  -o $OUT/k1_collect_c3 -f python bench.py --profile --steps 3 --warmup 1 > $OUT/k1_c3.log 2>&1; echo k1_c3=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:collect_kernel -s 2 -c 1 \
  -o $OUT/k1_collect_c2 -f python bench.py --config c2 --profile --steps 3 --warmup 1 > $OUT/k1_c2.log 2>&1; echo k1_c2=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:collect_kernel -s 5 -c 1 \
  -o $OUT/k1_collect_c1 -f python scripts/c1_probe.py c1 3 > $OUT/k1_c1.log 2>&1; echo k1_c1=$?
RESTORE_SHAPE=c2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:collect_kernel -s 3 -c 1 \
  -o $OUT/k1_family_restore_c2 -f python scripts/restore_ab.py > $OUT/k1_rest.log 2>&1; echo k1_rest=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:diff_encode -s 2 -c 1 \
  -o $OUT/k2_codec_c2 -f python bench.py --config c2 --steps 1 --warmup 1 --no-cpu --no-e2e > $OUT/k2.log 2>&1; echo k2=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attention_tc -s 3 -c 1 \
  -o $OUT/k5_attention_tc -f python scripts/recovery_profile.py > $OUT/k5_attn.log 2>&1; echo k5_attn=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"keydiff_kernel|select_kernel" -s 2 -c 2 \
  -o $OUT/k4_select -f python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > $OUT/k4.log 2>&1; echo k4=$?
RESTORE_SHAPE=c3 timeout 900 ncu --set full --clock-control none --import-source on -k regex:rows_tma -s 3 -c 1 \
  -o $OUT/k3_rows_restore_c3 -f python scripts/restore_ab.py > $OUT/k3_c3.log 2>&1; echo k3_c3=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:diff_encode -s 2 -c 1 \
  -o $OUT/k2_codec_c3 -f python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > $OUT/k2_c3.log 2>&1; echo k2_c3=$?
bash scripts/gpu_recovery_launches.sh > $OUT/recovery_launches.txt 2>&1
ls -la $OUT

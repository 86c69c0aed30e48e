OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_recompute.py tests/test_gpu_pic.py tests/test_gpu_t3.py -x -q > $OUT/pytest_attn.log 2>&1; echo pytest=$?
tail -8 $OUT/pytest_attn.log
for v in 1 0; do TDKV_ATTN_BLOCK=$v timeout 600 python scripts/recovery_ab.py > $OUT/recovery_attn$v.json 2>&1; echo rec$v=$?; done
for v in "TDKV_PDL=1" "TDKV_PDL=0" "TDKV_PDL=1 TDKV_ROUND_GRAPHS=0" "TDKV_PDL=0 TDKV_ROUND_GRAPHS=0" "TDKV_PDL=1"; do
  env $v timeout 600 python bench.py --config c2 --steps 20 --no-cpu --no-codec --no-e2e > "$OUT/ab_c2_$(echo $v | tr ' =' '__').json" 2>&1; echo "c2 $v"=$?
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_recovery.csv python scripts/recovery_ab.py > $OUT/launches_recovery.log 2>&1; echo ncu=$?

# family restore: per-warp job rotation; L2 prefetch A/B; C1 K1 ncu capture (graphs off)
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_family_restore.py tests/test_gpu_bf16_codec.py -x -q > $OUT/pytest_family.log 2>&1; echo pytest=$?
tail -3 $OUT/pytest_family.log
for v in "TDKV_OVL_PREFETCH=1" "TDKV_OVL_PREFETCH=0" "TDKV_RESTORE_FAMILY=0"; do env $v timeout 300 python scripts/restore_ab.py > $OUT/restore_ab.txt 2>&1; echo "$v"; cat $OUT/restore_ab.txt; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:collect_kernel -s 3 -c 1 -o $OUT/k1fam_c2c python scripts/restore_ab.py > $OUT/ncu_fam.log 2>&1; echo ncu_fam=$?
TDKV_ROUND_GRAPHS=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:collect_kernel -s 5 -c 1 -o $OUT/k1_c1 python bench.py --config c1 --steps 5 --warmup 3 --no-cpu --no-codec --no-e2e > $OUT/ncu_c1.log 2>&1; echo ncu_c1=$?
timeout 600 python bench.py --config c2 --no-cpu --no-e2e > $OUT/fam_c2.json 2> $OUT/fam_c2.err; echo c2=$?

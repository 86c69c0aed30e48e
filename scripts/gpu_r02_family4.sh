# family restore: K1 skips payload tiles and queues them; overlay pass moves them
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_family_restore.py tests/test_gpu_bf16_codec.py tests/test_gpu_wire.py -x -q > $OUT/pytest_family.log 2>&1; echo pytest=$?
tail -3 $OUT/pytest_family.log
for v in "TDKV_RESTORE_FAMILY=1" "TDKV_RESTORE_FAMILY=0"; do env $v timeout 300 python scripts/restore_ab.py > $OUT/restore_ab.txt 2>&1; echo "$v"; cat $OUT/restore_ab.txt; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"collect_kernel|overlay_rows" -s 6 -c 4 python scripts/restore_ab.py > $OUT/ncu_fam4.log 2>&1; echo ncu=$?
grep -E "collect_kernel|overlay_rows|duration|bytes" $OUT/ncu_fam4.log | head -30

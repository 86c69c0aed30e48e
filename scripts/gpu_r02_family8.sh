OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_family_restore.py tests/test_gpu_bf16_codec.py -x -q > $OUT/pytest_family.log 2>&1; echo pytest=$?
tail -2 $OUT/pytest_family.log
for sh in c3 c2; do for v in 1 0; do RESTORE_SHAPE=$sh TDKV_RESTORE_FAMILY=$v timeout 300 python scripts/restore_ab.py > $OUT/restore_ab.txt 2>&1; echo "$sh fam=$v"; head -2 $OUT/restore_ab.txt; done; done

OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_family_restore.py -x -q > $OUT/pytest_family.log 2>&1; echo pytest=$?
tail -2 $OUT/pytest_family.log
for c in c3 c2; do
  for v in 1 0; do TDKV_RESTORE_FAMILY=$v timeout 600 python bench.py --config $c --no-cpu --no-e2e > $OUT/fam_${c}_$v.json 2> $OUT/fam_${c}_$v.err; echo "$c fam=$v"=$?; done
done

# family restore after templating the overlay (collector registers restored) + L2 prefetch of payload rows
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_family_restore.py tests/test_gpu_bf16_codec.py tests/test_gpu_wire.py tests/test_gpu_parity.py -x -q > $OUT/pytest_family.log 2>&1; echo pytest=$?
tail -5 $OUT/pytest_family.log
for c in c3 c2; do
  for v in 1 0; do TDKV_RESTORE_FAMILY=$v timeout 600 python bench.py --config $c --no-cpu --no-e2e > $OUT/fam_${c}_$v.json 2> $OUT/fam_${c}_$v.err; echo "$c fam=$v"=$?; done
done
for v in 1 0; do TDKV_RESTORE_FAMILY=$v timeout 300 python scripts/restore_ab.py > $OUT/restore_ab_$v.txt 2>&1; echo rab$v=$?; cat $OUT/restore_ab_$v.txt; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:collect_kernel -s 3 -c 1 -o $OUT/k1fam_c2b python scripts/restore_ab.py > $OUT/ncu_fam.log 2>&1; echo ncu_fam=$?

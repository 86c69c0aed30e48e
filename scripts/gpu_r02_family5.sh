# family restore (K1 + overlay pass): GPU suite, codec numbers at C2/C3 (both restore forms), ncu
OUT=gpurun_out
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 $OUT/pytest_gpu.log
for c in c3 c2; do
  for v in 1 0; do TDKV_RESTORE_FAMILY=$v timeout 600 python bench.py --config $c --no-cpu --no-e2e > $OUT/fam_${c}_$v.json 2> $OUT/fam_${c}_$v.err; echo "$c fam=$v"=$?; done
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"collect_kernel|overlay_rows" -s 6 -c 2 -o $OUT/k1fam_c2 python scripts/restore_ab.py > $OUT/ncu_fam.log 2>&1; echo ncu_fam=$?

# K1 instruction-count A/B under gpurun: C1 probe, C2/C3 collector lines, collector parity tests
OUT=gpurun_out
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_family_restore.py -x -q > $OUT/pytest_k1.log 2>&1; echo pytest=$?; tail -2 $OUT/pytest_k1.log
: > $OUT/c1_probe.txt
for v in "X=1" "TDKV_PLAN_ITEMS=296"; do
  echo "$v $(env $v timeout 300 python scripts/c1_probe.py c1 50 2>&1 | tail -1)" >> $OUT/c1_probe.txt
done
cat $OUT/c1_probe.txt
for c in c2 c3; do timeout 600 python bench.py --config $c --steps 20 --no-cpu --no-codec --no-e2e > $OUT/k1_$c.json 2>&1; echo $c=$?; tail -1 $OUT/k1_$c.json | cut -c1-300; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:collect_kernel -s 5 -c 1 \
  -o $OUT/c1_collect -f python scripts/c1_probe.py c1 3 > $OUT/c1_ncu.log 2>&1; echo ncu=$?

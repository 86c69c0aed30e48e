# A/B: the paired (two units per thread, staged cos/sin rows) loop for interleaved rounds
# (TDKV_K1_PAIRED=1, default) vs one unit per thread (0); whole GPU suite first
OUT=gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo pytest=$?; tail -1 $OUT/pytest_gpu.log
line() { python -c "
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'): d=json.loads(l); print(sys.argv[2], d['value'], d['roofline']['frac'], d['ms_per_step'])" $1 $2; }
for rep in 1 2; do
  for pr in 0 1; do
    for c in c3 c2 c4 c5; do
      TDKV_K1_PAIRED=$pr timeout 600 python bench.py --config $c --steps 5 --no-cpu --no-codec --no-e2e > $OUT/b_${c}_${pr}.log 2>&1
      line $OUT/b_${c}_${pr}.log "paired=$pr $c"
    done
    TDKV_FUSE_TABLE=0 TDKV_K1_PAIRED=$pr timeout 600 python bench.py --config c1 --agents 64 --steps 20 --no-cpu --no-codec --no-e2e > $OUT/b_c1x_${pr}.log 2>&1
    line $OUT/b_c1x_${pr}.log "paired=$pr c1-64agents-f32-K0table"
  done
done

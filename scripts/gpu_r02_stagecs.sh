# A/B: K0 rows staged in shared memory per job group for interleaved rounds (TDKV_K1_STAGE_CS)
OUT=gpurun_out
TDKV_K1_STAGE_CS=1 timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_family_restore.py -q -x 2>&1 | tail -1
line() { python -c "
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'): d=json.loads(l); print(sys.argv[2], d['value'], d['roofline']['frac'], d['ms_per_step'])" $1 $2; }
for rep in 1 2; do
for st in 0 1; do
  for c in c3 c2 c4; do
    TDKV_K1_STAGE_CS=$st timeout 600 python bench.py --config $c --no-cpu --no-codec --no-e2e > $OUT/b_${c}_${st}.log 2>&1
    line $OUT/b_${c}_${st}.log "stage=$st $c"
  done
  RESTORE_SHAPE=c2 TDKV_K1_STAGE_CS=$st timeout 600 python scripts/restore_ab.py 2>&1 | tail -2
done
done

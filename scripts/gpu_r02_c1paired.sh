# A/B: C1 (float32, fused table) with the paired loop (TDKV_K1_PAIRED=2) vs the fused one-unit loop
OUT=gpurun_out
TDKV_K1_PAIRED=2 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
for rep in 1 2; do
  for pr in 1 2; do
    TDKV_K1_PAIRED=$pr timeout 300 python bench.py --config c1 --steps 50 --no-cpu --no-codec --no-e2e > $OUT/c1_$pr.log 2>&1
    python -c "
import json
for l in open('$OUT/c1_$pr.log'):
    if l.startswith('{'): d=json.loads(l); print('paired=$pr', d['value'], d['roofline']['frac'], d['cold_round']['frac'])"
  done
done

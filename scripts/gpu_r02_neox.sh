# rotate-half collector: parity tests + C3 / C2 bench lines with --rope-style neox
OUT=gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "neox or fused_table" 2>&1 | tail -1
for c in c3 c2; do
  timeout 600 python bench.py --config $c --rope-style neox --no-cpu --no-codec --no-e2e > $OUT/bench_neox_$c.log 2>&1
  python -c "
import json
for l in open('$OUT/bench_neox_$c.log'):
    if l.startswith('{'): d=json.loads(l); print('$c', d['value'], d['roofline']['frac'])"
done

# same-box A/B: interleaved vs rotate-half collector rounds (C3, C2), alternating
OUT=gpurun_out
line() { python -c "
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'): d=json.loads(l); print(sys.argv[2], d['value'], d['roofline']['frac'], d['ms_per_step'])" $1 $2; }
for rep in 1 2; do
  for st in interleaved neox; do
    for c in c3 c2; do
      timeout 600 python bench.py --config $c --rope-style $st --no-cpu --no-codec --no-e2e > $OUT/b_${c}_${st}.log 2>&1
      line $OUT/b_${c}_${st}.log "$st $c"
    done
  done
done

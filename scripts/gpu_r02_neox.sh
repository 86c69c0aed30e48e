# rotate-half (neox) collector vs the reference's interleaved pairs, collector line only
for cfg in c3 c2 c1; do for st in interleaved neox interleaved neox; do
  echo "$cfg $st $(timeout 600 python bench.py --config $cfg --rope-style $st --steps 20 --no-cpu --no-codec --no-e2e 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["frac"])')"
done; done

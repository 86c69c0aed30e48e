# one item per CTA for the large (K0-table) rounds too? A/B at C2 / C3 / C4
for cfg in c3 c2 c4; do for v in "TDKV_K1_SINGLE=1" "TDKV_K1_SINGLE=2" "TDKV_K1_SINGLE=1" "TDKV_K1_SINGLE=2"; do
  echo "$cfg $v $(env $v timeout 600 python bench.py --config $cfg --steps 20 --no-cpu --no-codec --no-e2e 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["frac"])')"
done; done

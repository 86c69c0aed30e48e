# K1 tile-size A/B at C3 / C2 (collector line only)
for cfg in c3 c2; do for v in 32768 65536 32768 65536; do
  echo "$cfg TILE_SMEM=$v $(TDKV_TILE_SMEM=$v timeout 600 python bench.py --config $cfg --steps 20 --no-cpu --no-codec --no-e2e 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["frac"], d.get("graph",{}).get("value"))')"
done; done

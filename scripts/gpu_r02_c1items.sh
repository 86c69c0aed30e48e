# C1 (cold) work-item granularity / tile size A/B
OUT=gpurun_out
mkdir -p $OUT
for v in "X=1" "TDKV_TILE_SMEM=65536" "TDKV_TILE_SMEM=16384" "TDKV_TILE_SMEM=65536 TDKV_PLAN_ITEMS=1200" "TDKV_COLLECT_V_BULK=0"; do
  env $v timeout 300 python bench.py --config c1 --steps 50 --no-cpu --no-codec --no-e2e > $OUT/c1i.json 2>&1; echo "$v $(python -c "import json;d=json.loads(open('$OUT/c1i.json').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['roofline']['frac'],d['graph']['ms_per_step'])")"
done
for c in c2 c3; do timeout 300 python bench.py --config $c --no-cpu --no-codec --no-e2e > $OUT/c1i.json 2>&1; echo "$c $(python -c "import json;d=json.loads(open('$OUT/c1i.json').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['roofline']['frac'])")"; done

OUT=gpurun_out
mkdir -p $OUT
for v in 0 1 0 1; do TDKV_ATTN_TC=$v timeout 600 python scripts/recovery_ab.py > $OUT/recovery_tc$v.json 2>&1; python -c "import json;d=json.loads(open('$OUT/recovery_tc$v.json').read().strip().splitlines()[-1]);print('tc=$v', d['grouped_ms'],d['grouped_ms_min'],d['serial_ms'],d['speedup'], [(r['agents'], r['grouped_ms']) for r in d['group_size_sweep']])"; done

# tensor-core attention: parity (recompute, recovery pipeline, T3 rounds) + recovery timing A/B + launch list
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_recompute.py tests/test_gpu_pic.py tests/test_gpu_t3.py -x -q > $OUT/pytest_attn.log 2>&1; echo pytest=$?
tail -15 $OUT/pytest_attn.log
for v in 1 0; do TDKV_ATTN_TC=$v timeout 600 python scripts/recovery_ab.py > $OUT/recovery_tc$v.json 2>&1; echo tc$v=$?; python -c "import json;d=json.loads(open('$OUT/recovery_tc$v.json').read().strip().splitlines()[-1]);print(d['grouped_ms'],d['serial_ms'],d['speedup'])"; done
bash scripts/gpu_recovery_launches.sh

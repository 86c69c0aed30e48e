# 3xTF32 GEMM over pre-split operands: parity, recovery A/B, launch breakdown, GEMM rate
OUT=gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_recompute.py tests/test_gpu_pic.py tests/test_gpu_t3.py -x -q > $OUT/pytest_presplit.log 2>&1; echo pytest=$?; tail -3 $OUT/pytest_presplit.log
for v in 1 0 1 0; do TDKV_GEMM_PRESPLIT=$v timeout 600 python scripts/recovery_ab.py > $OUT/recovery_ps$v.json 2>&1; python -c "import json;d=json.loads(open('$OUT/recovery_ps$v.json').read().strip().splitlines()[-1]);print('presplit=$v', d['grouped_ms'],d['grouped_ms_min'],d['serial_ms'],d['speedup'], [(r['agents'], r['grouped_ms']) for r in d['group_size_sweep']])"; done
bash scripts/gpu_recovery_launches.sh
timeout 300 python -c "
import json,sys,types
sys.path.insert(0,'.')
import torch, bench
dev=torch.device('cuda',0)
print(json.dumps(bench.recompute_bench(dev, types.SimpleNamespace(steps=5)), indent=0)[:1500])
"

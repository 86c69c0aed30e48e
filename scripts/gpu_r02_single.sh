# small-round K1: one item per 128-thread CTA (dynamic row buffers: 8 CTAs/SM) vs persistent
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_family_restore.py -x -q 2>&1 | tail -2
for v in 1 0 1 0; do echo "single=$v $(TDKV_K1_SINGLE=$v timeout 600 python bench.py --config c1 --steps 50 --no-cpu --no-codec --no-e2e 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["frac"], d["cold_round"]["frac"])')"; done
for c in c2 c3; do echo "$c $(timeout 600 python bench.py --config $c --steps 20 --no-cpu --no-codec --no-e2e 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["frac"])')"; done

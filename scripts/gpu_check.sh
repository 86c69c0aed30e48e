# parity + bench on one B200 (run under gpurun)
set -x
OUT=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -x -q -s > $OUT/pytest_gpu.log 2>&1; echo pytest=$?
tail -30 $OUT/pytest_gpu.log
timeout 300 python scripts/hbm_probe.py > $OUT/hbm_probe.json 2>&1; cat $OUT/hbm_probe.json
timeout 600 python bench.py --steps 10 --warmup 3 ${BENCH_ARGS:-} > $OUT/bench.log 2>&1; echo bench=$?
tail -5 $OUT/bench.log

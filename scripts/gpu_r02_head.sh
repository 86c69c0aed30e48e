# HEAD check on one B200 (run under gpurun): smoke, GPU suite, default bench, C1/C2 lines, reference arm
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo smoke=$?; tail -2 $OUT/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo pytest=$?
tail -8 $OUT/pytest_gpu.log
timeout 600 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err; echo bench=$?
for c in c1 c2; do timeout 600 python bench.py --config $c > $OUT/bench_$c.json 2> $OUT/bench_$c.err; echo bench_$c=$?; done
timeout 600 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo ref=$?

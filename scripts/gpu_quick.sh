# quick iteration on one B200 (run under gpurun): build, the given tests, a bench line
set -x
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest ${TESTS:-tests} -m gpu -x -q > $OUT/pytest_quick.log 2>&1; echo pytest=$?
tail -15 $OUT/pytest_quick.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e ${BENCH_ARGS:-} > $OUT/bench_quick.log 2>&1; echo bench=$?
tail -1 $OUT/bench_quick.log

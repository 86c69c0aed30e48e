# bench lines for the other BASELINE configs + the reference arm (run under gpurun)
set -x
OUT=gpurun_out
timeout 300 python bench.py --config c1 --steps 20 --warmup 3 --no-cpu > $OUT/bench_c1.log 2>&1; tail -1 $OUT/bench_c1.log | cut -c1-600
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu --codec-mirrors 24 > $OUT/bench_c3.log 2>&1; tail -1 $OUT/bench_c3.log | cut -c1-600
timeout 900 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu --codec-mirrors 32 --codec-sweep > $OUT/bench_c4.log 2>&1; tail -3 $OUT/bench_c4.log | cut -c1-600
timeout 900 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu --no-codec > $OUT/bench_c5.log 2>&1; tail -1 $OUT/bench_c5.log | cut -c1-600
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref.log 2>&1; tail -2 $OUT/bench_ref.log
nproc; free -g | head -2

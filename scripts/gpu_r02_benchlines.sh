# bench lines only (every config + the reference arm), for profiles/r02_bench_*.json
OUT=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python bench.py > $OUT/bench.log 2>&1; echo bench=$?
timeout 600 python bench.py --config c1 --steps 50 > $OUT/bench_c1.log 2>&1; echo c1=$?
timeout 600 python bench.py --config c2 > $OUT/bench_c2.log 2>&1; echo c2=$?
timeout 900 python bench.py --config c4 --no-cpu --codec-mirrors 32 --codec-sweep > $OUT/bench_c4.log 2>&1; echo c4=$?
timeout 900 python bench.py --config c5 --steps 3 --no-cpu --no-codec > $OUT/bench_c5.log 2>&1; echo c5=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref.log 2>&1; echo ref=$?

set -x
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_dist.py tests/test_gpu_parity.py -x -q > $OUT/pytest_dist.log 2>&1; echo pytest=$?
tail -30 $OUT/pytest_dist.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --dist-backend gloo --exchange p2p --no-codec --no-e2e --no-cpu > $OUT/bench_p2p.log 2>&1; echo p2p=$?
tail -3 $OUT/bench_p2p.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > $OUT/bench_codec.log 2>&1; echo bench=$?
tail -2 $OUT/bench_codec.log

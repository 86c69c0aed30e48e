set -x
timeout 600 python -m pytest tests/test_gpu_dist.py -x -q 2>&1 | tail -3
timeout 900 python bench.py --config c5 --steps 3 --warmup 3 --no-codec --no-cpu > gpurun_out/b_c5.log 2>&1; echo c5=$?
timeout 900 python bench.py --config c3 --steps 5 --warmup 3 --no-codec --no-cpu > gpurun_out/b_c3.log 2>&1; echo c3=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --config c3 --dist-backend gloo --steps 3 --warmup 3 --no-codec --no-cpu --no-e2e > gpurun_out/b_c3_n2_gloo.log 2>&1; echo c3n2=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --dist-backend gloo --steps 3 --warmup 3 --no-codec --no-cpu --no-e2e > gpurun_out/b_c2_n2_gloo.log 2>&1; echo c2n2=$?

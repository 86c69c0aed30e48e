# the N>1 bench path with two ranks sharing the one GPU (gloo; NCCL needs distinct GPUs)
OUT=gpurun_out
for cfg in c3 c2; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus 2 --config $cfg --steps 3 --warmup 3 --dist-backend gloo --no-cpu > $OUT/mr_$cfg.log 2>&1; echo "$cfg rc=$?"
  grep '^{' $OUT/mr_$cfg.log | tail -1 | cut -c1-400
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 \
  bench.py --gpus 2 --config c2 --steps 3 --warmup 3 --dist-backend gloo --exchange p2p --no-cpu --no-codec > $OUT/mr_p2p.log 2>&1; echo "p2p rc=$?"
grep '^{' $OUT/mr_p2p.log | tail -1 | cut -c1-400
tail -5 $OUT/mr_p2p.log

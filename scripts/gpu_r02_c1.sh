OUT=gpurun_out
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo pytest=$?
tail -5 $OUT/pytest_gpu.log
for v in "TDKV_FUSE_TABLE=auto" "TDKV_FUSE_TABLE=0" "TDKV_ROUND_GRAPHS=0" "TDKV_FUSE_TABLE=auto"; do
  env $v timeout 600 python bench.py --config c1 --steps 50 --no-cpu --no-codec > "$OUT/ab_c1_$(echo $v | tr ' =' '__').json" 2>&1; echo "c1 $v"=$?
done
timeout 600 python bench.py --config c2 --steps 20 --no-cpu --no-codec --no-e2e > $OUT/ab_c2.json 2>&1; echo c2=$?

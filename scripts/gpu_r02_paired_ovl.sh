# A/B: the paired loop in the family restore's collector round (TDKV_K1_PAIRED=1 default vs 0)
OUT=gpurun_out
timeout 600 python -m pytest tests/test_gpu_family_restore.py tests/test_gpu_t3.py tests/test_gpu_bf16_codec.py -q -x 2>&1 | tail -1
for rep in 1 2; do
  for pr in 0 1; do
    for sh in c2 c3; do
      echo "paired=$pr $sh"; RESTORE_SHAPE=$sh TDKV_K1_PAIRED=$pr timeout 600 python scripts/restore_ab.py 2>&1 | grep "family model"
    done
  done
done

# A/B: K3 consumers with two units per thread per row (TDKV_K3_PAIRED=1) vs one (0)
OUT=gpurun_out
TDKV_K3_PAIRED=1 timeout 600 python -m pytest tests/test_gpu_family_restore.py tests/test_gpu_parity.py tests/test_gpu_bf16_codec.py tests/test_gpu_t3.py -q -x 2>&1 | tail -1
for rep in 1 2; do
  for pr in 0 1; do
    echo "k3paired=$pr c3"; RESTORE_SHAPE=c3 TDKV_K3_PAIRED=$pr timeout 600 python scripts/restore_ab.py 2>&1 | grep "family model"
    echo "k3paired=$pr c2 per-mirror K3"; TDKV_RESTORE_FAMILY=0 TDKV_K3_PAIRED=$pr timeout 600 python scripts/restore_ab.py 2>&1 | grep "family model"
  done
done

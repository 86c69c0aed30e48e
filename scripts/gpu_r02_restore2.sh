# family restore: overlay inside K1 vs separate, parity + A/B
OUT=gpurun_out
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_family_restore.py tests/test_gpu_bf16_codec.py tests/test_gpu_t3.py -x -q > $OUT/pytest_rest.log 2>&1; echo pytest=$?; tail -2 $OUT/pytest_rest.log
TDKV_OVERLAY_SEPARATE=1 timeout 600 python -m pytest tests/test_gpu_family_restore.py -x -q > $OUT/pytest_rest_sep.log 2>&1; echo pytest_sep=$?; tail -1 $OUT/pytest_rest_sep.log
for sh in c2 c3; do for v in 0 1 0; do echo "$sh separate=$v"; RESTORE_SHAPE=$sh TDKV_OVERLAY_SEPARATE=$v timeout 300 python scripts/restore_ab.py 2>&1 | tail -2 | head -1; done; done

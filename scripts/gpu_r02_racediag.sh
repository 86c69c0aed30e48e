OUT=gpurun_out
T=tests/test_gpu_family_restore.py
for v in 0 1; do
  TDKV_OVERLAY_SEPARATE=$v timeout 600 compute-sanitizer --tool memcheck python -m pytest $T -x -q > $OUT/diag_mem_sep$v.log 2>&1; echo "memcheck separate=$v rc=$?"; grep -E "passed|failed" $OUT/diag_mem_sep$v.log | tail -2
done
TDKV_RESTORE_FAMILY=0 timeout 600 compute-sanitizer --tool memcheck python -m pytest $T -x -q > $OUT/diag_mem_k3.log 2>&1; echo "memcheck k3only rc=$?"; grep -E "passed|failed" $OUT/diag_mem_k3.log | tail -2
for i in 1 2 3; do timeout 300 python -m pytest $T -x -q 2>&1 | tail -1; done
CUDA_LAUNCH_BLOCKING=1 timeout 300 python -m pytest $T -x -q 2>&1 | tail -1

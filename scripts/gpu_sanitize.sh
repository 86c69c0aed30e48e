# compute-sanitizer passes over the GPU parity tests (run under gpurun)
OUT=gpurun_out
export PYTHONDONTWRITEBYTECODE=1
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
    python -m pytest tests/test_gpu_parity.py tests/test_gpu_select.py tests/test_gpu_gemm.py tests/test_gpu_recompute.py tests/test_gpu_wire.py tests/test_gpu_pic.py tests/test_gpu_bf16_codec.py tests/test_gpu_family_restore.py tests/test_gpu_t3.py \
    -x -q -k "not full_size" > $OUT/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|passed|failed" $OUT/sanitize_$tool.log | tail -3
done

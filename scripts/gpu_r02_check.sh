# HEAD check: smoke, the whole GPU suite, memcheck over the host-transfer paths (wire staging,
# pinned direct H2D, chunked host-context read-back)
OUT=gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo smoke=$?; tail -1 $OUT/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 $OUT/pytest_gpu.log
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest -q -x \
  tests/test_gpu_wire.py "tests/test_gpu_parity.py::test_align_cached_host_contexts_chunked_readback" \
  "tests/test_gpu_parity.py::test_align_cached_dropin_matches_reference_goldens" > $OUT/memcheck_host.log 2>&1
echo memcheck=$?; tail -3 $OUT/memcheck_host.log

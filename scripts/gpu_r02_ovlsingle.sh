# family restore (K1 with the overlay) in the one-item form vs persistent (TDKV_K1_SINGLE=0)
timeout 900 python -m pytest tests/test_gpu_family_restore.py tests/test_gpu_parity.py tests/test_gpu_t3.py tests/test_gpu_bf16_codec.py -x -q 2>&1 | tail -1
for sh in c2 c3; do for v in 1 0 1 0; do echo "$sh single=$v $(TDKV_K1_SINGLE=$v RESTORE_SHAPE=$sh timeout 300 python scripts/restore_ab.py 2>&1 | grep 'family model')"; done; done
for sh in c3; do for v in 1; do echo "$sh family=1 single=$v $(TDKV_RESTORE_FAMILY=1 TDKV_K1_SINGLE=$v RESTORE_SHAPE=$sh timeout 300 python scripts/restore_ab.py 2>&1 | grep 'family model')"; done; done

# K3 (rows_tma) consumer-count A/B: C3 family restore (K3 form) and C2 per-mirror K3 (family off)
for sh in c3 c2; do for lib in "" scratch_ab/libtdkv_r128.so scratch_ab/libtdkv_r64.so "" scratch_ab/libtdkv_r128.so scratch_ab/libtdkv_r64.so; do
  echo "$sh lib=${lib:-intree} $(TDKV_LIBRARY=$lib TDKV_RESTORE_FAMILY=0 RESTORE_SHAPE=$sh timeout 300 python scripts/restore_ab.py 2>&1 | grep 'family model')"
done; done

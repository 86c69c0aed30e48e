# C3 codec host-side diagnostics (run under gpurun): submission cost of the family restore and encode
OUT=gpurun_out
mkdir -p $OUT
RESTORE_SHAPE=c3 timeout 300 python scripts/restore_ab.py > $OUT/c3_restore_ab.txt 2>&1; echo ab=$?
RESTORE_SHAPE=c3 TDKV_RESTORE_FAMILY=1 timeout 300 python scripts/restore_ab.py > $OUT/c3_restore_ab_fam.txt 2>&1; echo abf=$?
RESTORE_SHAPE=c3 timeout 300 python scripts/restore_host_profile.py > $OUT/c3_restore_host.txt 2>&1; echo rh=$?
ENCODE_SHAPE=c3 timeout 300 python scripts/encode_host_profile.py > $OUT/c3_encode_host.txt 2>&1; echo eh=$?
RESTORE_SHAPE=c3 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/c3_restore_launches.csv python scripts/restore_ab.py > /dev/null 2>&1; echo ncu=$?

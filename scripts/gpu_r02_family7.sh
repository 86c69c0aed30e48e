OUT=gpurun_out
mkdir -p $OUT
for sh in c3 c2; do for v in 1 0; do RESTORE_SHAPE=$sh TDKV_RESTORE_FAMILY=$v timeout 300 python scripts/restore_ab.py > $OUT/restore_ab.txt 2>&1; echo "$sh fam=$v"; head -1 $OUT/restore_ab.txt; done; done
RESTORE_SHAPE=c3 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"collect_kernel|overlay_rows|rows_tma|rope_table" -s 8 -c 6 python scripts/restore_ab.py > $OUT/ncu_fam_c3.log 2>&1; echo ncu=$?
grep -E "collect_kernel|overlay_rows|rows_tma|rope_table|duration|bytes" $OUT/ncu_fam_c3.log | head -40
RESTORE_SHAPE=c3 TDKV_RESTORE_FAMILY=0 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"rows_tma" -s 4 -c 1 python scripts/restore_ab.py > $OUT/ncu_k3_c3.log 2>&1; echo ncu=$?
grep -E "rows_tma|duration|bytes" $OUT/ncu_k3_c3.log | head -10

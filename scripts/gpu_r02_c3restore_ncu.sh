OUT=gpurun_out
RESTORE_SHAPE=c3 TDKV_RESTORE_FAMILY=auto timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --print-units base \
  -k regex:"rows_tma|collect_kernel" -c 6 python scripts/restore_ab.py 2>/dev/null | grep -E "rows_tma|collect_kernel" | awk -F'","' '{print $5, $(NF-2), $NF}' | cut -c1-200
RESTORE_SHAPE=c3 TDKV_RESTORE_FAMILY=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --print-units base \
  -k regex:"rows_tma|collect_kernel" -c 6 python scripts/restore_ab.py 2>/dev/null | grep -E "rows_tma|collect_kernel" | awk -F'","' '{print $5, $(NF-2), $NF}' | cut -c1-200

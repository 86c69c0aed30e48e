timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --print-units base \
  -k regex:diff_encode -c 3 python bench.py --config c3 --steps 1 --warmup 1 --no-cpu --no-e2e 2>/dev/null | grep diff_encode | awk -F'","' '{print $(NF-2), $NF}'

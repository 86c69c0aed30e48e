OUT=gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:collect_kernel -s 5 -c 1 -o $OUT/k1_c1_single -f python scripts/c1_probe.py c1 3 > /dev/null 2>&1; echo ncu=$?
timeout 300 python scripts/c1_probe.py c1 50 | tail -1

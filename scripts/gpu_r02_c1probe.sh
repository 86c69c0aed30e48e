# C1 collector A/B under gpurun: plan items, tile rows, fused table, L2 states; one ncu capture
OUT=gpurun_out
mkdir -p $OUT
: > $OUT/c1_probe.txt
for v in "X=1" "TDKV_PLAN_ITEMS=1184" "TDKV_PLAN_ITEMS=2368" "TDKV_PLAN_ITEMS=4736" "TDKV_TILE_SMEM=16384" "TDKV_TILE_SMEM=65536" "TDKV_FUSE_TABLE=0" "TDKV_TILE_SMEM=16384 TDKV_PLAN_ITEMS=2368"; do
  echo "$v $(env $v timeout 300 python scripts/c1_probe.py c1 50 2>&1 | tail -1)" >> $OUT/c1_probe.txt
done
cat $OUT/c1_probe.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:collect_kernel -s 5 -c 1 \
  -o $OUT/c1_collect -f python scripts/c1_probe.py c1 3 > $OUT/c1_ncu.log 2>&1; echo ncu=$?

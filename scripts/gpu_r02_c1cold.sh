# C1 timed cold (L2 flushed between rounds): tile-size / fused-table / PDL A/B; recovery attention A/B
OUT=gpurun_out
mkdir -p $OUT
for v in "X=1" "TDKV_TILE_SMEM=16384" "TDKV_TILE_SMEM=65536" "TDKV_FUSE_TABLE=0" "TDKV_PDL=1" "TDKV_ROUND_GRAPHS=0"; do
  env $v timeout 300 python bench.py --config c1 --steps 50 --no-cpu --no-codec --no-e2e > "$OUT/c1cold_$(echo $v | tr ' =' '__').json" 2>&1; echo "c1 $v"=$?
done
for v in 1 0; do TDKV_ATTN_BLOCK=$v timeout 600 python scripts/recovery_ab.py > $OUT/recovery_attn$v.json 2>&1; echo rec$v=$?; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_recovery.csv python scripts/recovery_ab.py > $OUT/launches_recovery.log 2>&1; echo ncu=$?

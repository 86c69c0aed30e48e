# K3 tile size / ring depth A/B (TDKV_ROWS_SMEM budget, TDKV_ROWS_STAGES) at C3 family and C2 per-mirror
for sh in c3 c2; do for v in "X=1" "TDKV_ROWS_SMEM=36864" "TDKV_ROWS_SMEM=36864 TDKV_ROWS_STAGES=3" "TDKV_ROWS_SMEM=18432" "TDKV_ROWS_SMEM=18432 TDKV_ROWS_STAGES=4" "X=1"; do
  echo "$sh $v $(env $v TDKV_RESTORE_FAMILY=0 RESTORE_SHAPE=$sh timeout 300 python scripts/restore_ab.py 2>&1 | grep 'family model')"
done; done

# where the family restore (K1 + overlay, paired loop) overtakes per-mirror K3: C3 (24 mirrors)
# and smaller C2-shaped families, TDKV_RESTORE_FAMILY=1 (always family) vs 0 (always K3)
OUT=gpurun_out
for rep in 1 2; do
  for fm in 0 1; do
    echo "family=$fm c3 (24 mirrors)"; RESTORE_SHAPE=c3 TDKV_RESTORE_FAMILY=$fm timeout 600 python scripts/restore_ab.py 2>&1 | grep "family model"
    for P in 8 16; do
      echo "family=$fm c2 $P mirrors"; RESTORE_MIRRORS=$P TDKV_RESTORE_FAMILY=$fm timeout 600 python scripts/restore_ab.py 2>&1 | grep "family model"
    done
  done
done

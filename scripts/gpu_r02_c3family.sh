# C3 codec family (24 mirrors): family K1 (overlay inside) vs per-mirror K3, alternating
for v in 1 auto 1 auto; do echo "family=$v $(RESTORE_SHAPE=c3 TDKV_RESTORE_FAMILY=$v timeout 300 python scripts/restore_ab.py 2>&1 | grep 'family model')"; done
for v in 1 auto; do echo "c2 family=$v $(RESTORE_SHAPE=c2 TDKV_RESTORE_FAMILY=$v timeout 300 python scripts/restore_ab.py 2>&1 | grep 'family model')"; done

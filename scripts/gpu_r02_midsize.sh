# mid-size rounds (< 1 GB: fused table + one item per CTA) vs the persistent K0+K1 form
for a in "c2 3" "c3 30" "c1 64" "c1 32"; do set -- $a; for v in "X=1" "TDKV_FUSE_TABLE=0" "TDKV_K1_SINGLE=0"; do
  echo "$1 agents=$2 $v $(env $v timeout 600 python bench.py --config $1 --agents $2 --steps 20 --no-cpu --no-codec --no-e2e 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["frac"], d["roofline"]["algorithmic_bytes_per_launch"])')"
done; done

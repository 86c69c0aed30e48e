# same-box A/B of the collector line: in-tree build vs scratch_ab/libtdkv_head.so
for cfg in c2 c3; do for lib in "" scratch_ab/libtdkv_head.so "" scratch_ab/libtdkv_head.so; do
  echo "$cfg lib=${lib:-intree} $(TDKV_LIBRARY=$lib timeout 600 python bench.py --config $cfg --steps 20 --no-cpu --no-codec --no-e2e 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["frac"])')"
done; done

# K2 A/B: CTA size and loads in flight per thread (C2 family encode, then C3)
for cfg in c2 c3; do for lib in scratch_ab/libtdkv_t128u3.so scratch_ab/libtdkv_t128u4.so scratch_ab/libtdkv_t64u3.so scratch_ab/libtdkv_t64u4.so; do
  echo "$cfg lib=$lib $(TDKV_LIBRARY=$lib timeout 600 python bench.py --config $cfg --steps 5 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); c=d["codec"]; print(c["family_model"]["encode_device_gbs"], c["family_model"]["encode_device_frac"], c["encode_ms_per_family"])')"
done; done

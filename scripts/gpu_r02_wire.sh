# wire format host staging: GPU wire tests + the C2 bench line's codec wire numbers
OUT=gpurun_out
timeout 300 python -m pytest tests/test_gpu_wire.py -q -x 2>&1 | tail -2
timeout 600 python bench.py --config c2 > $OUT/bench_c2.log 2>&1; echo c2=$?
python - <<'P'
import json
for l in open("gpurun_out/bench_c2.log"):
    if l.startswith("{"):
        d=json.loads(l); c=d["codec"]
        print(d["value"], d["roofline"]["frac"], c["wire_pack_gbs"], c["wire_unpack_gbs"], c["wire_unpack_pageable_gbs"], c["family_model"])
P

"""Recovery sub-benchmark alone (bench.recovery_bench): grouped vs serial
recovery of a BASELINE configs[0] round.  For A/B runs of the attention
kernels (TDKV_ATTN_BLOCK=0/1) under gpurun."""
import json
import os
import sys
from types import SimpleNamespace

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
print(json.dumps(bench.recovery_bench(dev, SimpleNamespace(steps=10))))

"""Host time per phase of the grouped recovery (configs[0], 8 agents), with a
device sync after each phase so each is host + its own device work
(diagnostic, under gpurun)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2604_03143_b200 import pic, rounds  # noqa: E402
from paper_2604_03143_b200.collector import collect_into_contexts  # noqa: E402
from paper_2604_03143_b200.recompute import ToyModel  # noqa: E402


class _Pic:
    recompute_fraction = 0.15
    check_layer = 1


dev = torch.device("cuda", 0)
w = rounds.toy_weights(2, 8, 64, 1024, seed=0)
members = rounds.toy_round(w, seed=1, device=dev)
group = rounds.ToyGroup(members)
model = ToyModel.of(w, dev)
T = {"skeletons": [], "collect": [], "probe_select": [], "refresh": [], "tail": [], "total": []}
for it in range(13):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ctx = pic._skeletons(w, group.members, dev)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    collect_into_contexts(group.members, ctx, model.rope_base, None)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    sel = pic.probe_and_select(w, group.members, ctx, _Pic, None)
    torch.cuda.synchronize(); t3 = time.perf_counter()
    pic.refresh_many(w, group.members, ctx, [i for i, _ in sel], None)
    torch.cuda.synchronize(); t4 = time.perf_counter()
    pic.collective_recover(w, group, _Pic)
    torch.cuda.synchronize(); t5 = time.perf_counter()
    if it >= 3:
        for k, v in zip(("skeletons", "collect", "probe_select", "refresh", "total"),
                        (t1 - t0, t2 - t1, t3 - t2, t4 - t3, t5 - t4)):
            T[k].append(v)
print({k: round(float(np.median(v)) * 1e3, 3) for k, v in T.items() if v}, "ms")

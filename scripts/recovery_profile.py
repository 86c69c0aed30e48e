"""Host profile of GPU collective_recover on BASELINE configs[0] (diagnostic)."""
import cProfile
import pstats
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2604_03143_b200 import pic, rounds  # noqa: E402
from paper_2604_03143_b200.ledger import CostLedger  # noqa: E402


class _Pic:
    recompute_fraction = 0.15
    check_layer = 1


w = rounds.toy_weights(2, 8, 64, 1024, seed=0)
members = rounds.toy_round(w, seed=1, device=torch.device("cuda", 0))
group = rounds.ToyGroup(members)
pic.collective_recover(w, group, _Pic, CostLedger(2))
torch.cuda.synchronize()
t0 = time.perf_counter()
pic.collective_recover(w, group, _Pic, CostLedger(2))
torch.cuda.synchronize()
print("grouped ms", (time.perf_counter() - t0) * 1e3)
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    pic.collective_recover(w, group, _Pic, CostLedger(2))
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(45)

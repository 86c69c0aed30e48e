"""cProfile of the grouped recovery (configs[0], 8 agents): which host
functions the ~4 ms round spends its time in (diagnostic, under gpurun)."""
import cProfile
import pstats
import sys

import torch

sys.path.insert(0, ".")
from paper_2604_03143_b200 import pic, rounds  # noqa: E402
from paper_2604_03143_b200.recompute import ToyModel  # noqa: E402


class _Pic:
    recompute_fraction = 0.15
    check_layer = 1


dev = torch.device("cuda", 0)
w = rounds.toy_weights(2, 8, 64, 1024, seed=0)
members = rounds.toy_round(w, seed=1, device=dev)
group = rounds.ToyGroup(members)
ToyModel.of(w, dev)
for _ in range(5):
    pic.collective_recover(w, group, _Pic)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    pic.collective_recover(w, group, _Pic)
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
st.sort_stats("cumtime").print_stats(40)

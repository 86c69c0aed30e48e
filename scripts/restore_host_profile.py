"""Host-side profile of fused_restore_many at the C2 codec family (49 mirrors;
diagnostic, run under gpurun): where the ~1 ms of submission goes."""
import cProfile
import os
import pstats
import sys

os.environ.setdefault("RESTORE_SHAPE", "c2")
sys.argv = [sys.argv[0]]
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import restore_ab as ab  # noqa: E402  (builds the family and times it once)
import torch  # noqa: E402

pr = cProfile.Profile()
pr.enable()
for _ in range(10):
    ab.tk.fused_restore_many(ab.handles, ab.spans, ab.pool, ab.maps, 10000.0)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("cumulative").print_stats(30)

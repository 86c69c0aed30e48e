"""Where the family restore's time goes between back-to-back calls at the
C3 codec family (diagnostic, run under gpurun): CUDA events around every
tdkv launch inside 6 back-to-back fused_restore_many calls, against events
around the whole loop."""
import os
import sys

import numpy as np
import torch

os.environ.setdefault("RESTORE_SHAPE", "c3")
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import restore_ab as ab  # noqa: E402
from paper_2604_03143_b200 import _lib  # noqa: E402

marks = []
_call = _lib.call


def timed_call(name, *args):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    r = _call(name, *args)
    b.record()
    marks.append((name, a, b))
    return r


_lib.call = timed_call
for rep in range(3):
    marks.clear()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(6):
        ab.tk.fused_restore_many(ab.handles, ab.spans, ab.pool, ab.maps, 10000.0)
    e.record()
    torch.cuda.synchronize()
    tot = s.elapsed_time(e) / 6
    per = {}
    for name, a, b in marks:
        per.setdefault(name, []).append(a.elapsed_time(b))
    gaps = [marks[i][1].elapsed_time(marks[i + 1][1]) - marks[i][1].elapsed_time(marks[i][2])
            for i in range(len(marks) - 1)]
    print("loop ms per call", round(tot, 4), {k: round(float(np.mean(v)), 4) for k, v in per.items()},
          "gaps ms", [round(g, 4) for g in gaps])

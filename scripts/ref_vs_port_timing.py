"""Build-container check that the oracle port times like the reference itself.

Runs roundkv.pic.align_cached (+ the _skeleton V copy + PagedPool.write_rows)
from /root/reference and oracle.roundkv_port.collect_into_pool on the same
inputs (2 agents of the C2 round, f32), single thread, best of 3.
Not used on the GPU box (the reference tree is not there).
"""
import sys
import time
from types import SimpleNamespace

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ".")
from roundkv.core import LayeredKv  # noqa: E402
from roundkv.paged_pool import PagedPool, SlotMap  # noqa: E402
from roundkv.pic import align_cached  # noqa: E402

from oracle import roundkv_port as port  # noqa: E402
from paper_2604_03143_b200 import rounds  # noqa: E402

spec = rounds.CONFIGS["c2"].scaled(num_agents=2)
mk, mv = rounds.master_planes_host(spec)
T, L, H, D = spec.tokens_per_agent, spec.num_layers, spec.num_heads, spec.head_dim
src = rounds.source_offsets(spec)
segs = [LayeredKv(mk[:, s * 256:(s + 1) * 256].copy(), mv[:, s * 256:(s + 1) * 256].copy(),
                  np.arange(src[s], src[s] + 256)) for s in range(spec.num_segments)]


class _Hit:
    def __init__(self, kv, target_idx, delta):
        self.kv, self.target_idx, self.delta = kv, target_idx, delta

    def __len__(self):
        return int(self.target_idx.size)


def reference_once():
    members, contexts = [], []
    for a in range(spec.num_agents):
        starts = rounds.segment_starts(spec, a)
        hits = []
        for s in range(spec.num_segments):
            tgt = np.arange(starts[s], starts[s] + 256)
            hits.append(_Hit(segs[s], tgt, tgt - segs[s].positions))
        members.append(SimpleNamespace(hits=hits))
        contexts.append((np.zeros((L, T, H, D), np.float32), np.zeros((L, T, H, D), np.float32)))
    pool = PagedPool(spec.num_agents * T, L, H, D, debug=False)
    maps = [pool.allocate(T, a) for a in range(spec.num_agents)]
    t0 = time.perf_counter()
    for m, c in zip(members, contexts):
        for h in m.hits:
            c[1][:, h.target_idx] = h.kv.v
    align_cached(members, contexts, 10000.0)
    for m, c, sm in zip(members, contexts, maps):
        sl = SlotMap(0, sm.slots[np.concatenate([h.target_idx for h in m.hits])])
        idx = np.concatenate([h.target_idx for h in m.hits])
        for layer in range(L):
            pool.write_rows(sl, layer, c[0][layer][idx], c[1][layer][idx])
    return time.perf_counter() - t0


def port_once():
    t0 = time.perf_counter()
    import bench
    bench._cpu_collect_agents(spec, range(spec.num_agents), mk, mv)
    return time.perf_counter() - t0


r = min(reference_once() for _ in range(3))
p = min(port_once() for _ in range(3))
b = spec.collector_bytes(spec.num_agents)
print(f"reference {r:.2f} s ({b / r / 1e9:.3f} GB/s)  port {p:.2f} s ({b / p / 1e9:.3f} GB/s)")

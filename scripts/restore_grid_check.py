"""Fused restore (K3 and the family form) against the oracle at several
grid limits: persistent kernels with few CTAs cycle their smem rings many
times (diagnostic, run under gpurun)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2604_03143_b200 as tk  # noqa: E402
from paper_2604_03143_b200 import restore as rs  # noqa: E402
import test_gpu_family_restore as t  # noqa: E402

rs._FAMILY_MIN = 1
L, T, H, D = 2, 150, 4, 128
for bs in (8, 16, 32):
    rng = np.random.default_rng(bs)
    mk, mv, mirrors, hints = t._family_host(rng, L, T, H, D, 5, bs)
    pos = np.arange(T, dtype=np.int64)
    entry = tk.MasterEntry(0, tk.LayeredKv(mk, mv, pos), pin_count=5)
    diffs = [tk.encode_diff(entry.kv, tk.LayeredKv(k, v, pos), h, tk.CacheBlockConfig(bs))
             for (k, v), h in zip(mirrors, hints)]
    handles = [tk.MirrorHandle(0, i + 1, entry, d) for i, d in enumerate(diffs)]
    spans = [tk.PositionSpan.shifted(pos, 3 + i) for i in range(5)]
    layers = [[(ld.indices, ld.k_blocks, ld.v_indices, ld.v_blocks) for ld in d.layers]
              for d in diffs]
    for fam in (False, True):
        rs._FAMILY_K1 = fam
        for gl in (0, 1, 2, 3, 5, 16, 64):
            pool = t._pool_f32(8 * T, L, H, D)
            maps = [pool.allocate(T, i) for i in range(5)]
            tk.fused_restore_many(handles, spans, pool, maps, 10000.0, grid_limit=gl)
            torch.cuda.synchronize()
            bad = []
            for i in range(5):
                mkk, mvv = mirrors[i]
                wk, wv = t._oracle_pool(mk, mv, None, bs, spans[i], maps[i].slots, pool.capacity) \
                    if False else (None, None)
                # oracle: the mirror's own dense planes, rotated
                want_k = np.stack([tk_rope for tk_rope in [None]]) if False else None
                gk, gv = t._read(pool, maps[i])
                from oracle import roundkv_port as ref
                ek = np.stack([ref.rope_apply(mkk[l], np.full(T, 3 + i)) for l in range(L)])
                nk = int((np.abs(gk - ek) > 1e-5).sum())
                nv = int((gv != mvv).sum())
                if nk or nv:
                    bad.append((i, nk, nv))
            print(f"bs={bs} family={fam} grid_limit={gl}: {'ok' if not bad else bad}", flush=True)

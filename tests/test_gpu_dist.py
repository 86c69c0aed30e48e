"""Multi-rank collector on the GPU: torchrun with 2 ranks (gloo when the box
has a single GPU, nccl otherwise) running scripts/dist_check.py."""
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_rank_broadcast_collect(tmp_path):
    """Two ranks collect their agent shards after the master broadcast; each
    rank's pool equals a single-process collect (inside dist_check), and the
    union of the ranks' rows equals the CPU oracle's collector (bf16 keys
    within 1e-2 of the oracle on the bf16-rounded masters, values bit for
    bit) -- anchored on the oracle, not only on the product itself."""
    import numpy as np
    from paper_2604_03143_b200 import rounds
    from oracle import roundkv_port as ref
    backend = "nccl" if torch.cuda.device_count() >= 2 else "gloo"
    env = dict(os.environ, TDKV_DIST_BACKEND=backend, TDKV_DIST_DUMP=str(tmp_path))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "scripts", "dist_check.py")]
    res = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    assert "dist_check ok" in res.stdout
    spec = rounds.CONFIGS["c2"].scaled(num_layers=5, num_agents=9, num_segments=3, hist_len=11)
    mk, mv = rounds.master_planes_host(spec)
    mk = torch.from_numpy(mk).bfloat16().float().numpy()      # what the ranks hold
    mv = torch.from_numpy(mv).bfloat16().float().numpy()
    seen = []
    for r in range(2):
        d = np.load(tmp_path / f"rank{r}.npz")
        off = 0
        for a, slots in zip(d["agents"], d["slots"]):
            seen.append(int(a))
            for j in rounds.agent_jobs(spec, int(a), slots):
                n = len(j.dst_rows)
                r0 = j.segment * spec.seg_len
                for layer in range(spec.num_layers):
                    want = ref.rope_apply(mk[layer, r0:r0 + spec.seg_len], j.delta)
                    got = d["k"][layer, off:off + n]
                    assert np.abs(got - want).max() <= 1e-2 * max(1.0, np.abs(want).max())
                    assert np.array_equal(d["v"][layer, off:off + n], mv[layer, r0:r0 + n])
                off += n
    assert sorted(seen) == list(range(spec.num_agents))      # the shards cover every agent

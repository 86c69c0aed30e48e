"""GPU parity of K4 (check-layer key diff + top-k + deviation) against the
reference's own probe_and_select outputs (tests/golden) and the oracle."""
import numpy as np
import pytest
import torch

import paper_2604_03143_b200 as tk
from helpers import load_golden, load_npz
from oracle import roundkv_port as ref
from paper_2604_03143_b200 import select as sel

pytestmark = pytest.mark.gpu
G = load_golden()
DEV = torch.device("cuda", 0)


def test_selection_matches_reference_probe_and_select():
    meta = G["collector"]["selection"]
    z = load_npz("collector.npz")
    led = tk.CostLedger(2)
    out = sel.batched_selection(z["sel_fresh"], z["sel_cached"], meta["counts"],
                                meta["fraction"], ledger=led)
    assert led.selection_passes == 1
    for m, (imp, dev) in enumerate(out):
        assert imp.tolist() == meta["important_rel"][m]
        assert abs(dev - meta["deviation"][m]) <= 1e-5 * max(1.0, abs(meta["deviation"][m]))
    assert sel.select_master({m: d for m, (_, d) in enumerate(out)}) == meta["master"]
    mags = sel.key_diff(z["sel_fresh"], z["sel_cached"])
    assert np.abs(mags - z["sel_mags"]).max() <= 1e-6


def test_known_answers():
    fresh = np.zeros((3, 2, 4), np.float32)
    cached = np.zeros((3, 2, 4), np.float32)
    cached[1, 0, 0], cached[1, 1, 0] = 3.0, 4.0
    assert sel.key_diff(fresh, cached).tolist() == [0.0, 5.0, 0.0]
    mags = np.array([0.0, 3.0, 3.0, 1.0, 0.0, 2.0], np.float32)
    assert sel.select_important(mags, 3).tolist() == [1, 2, 5]
    assert sel.select_important(mags, 10).tolist() == [1, 2, 3, 5]
    assert sel.select_important(mags, 0).tolist() == []
    assert sel.select_important(np.array([5.0, 5.0, 5.0, 1.0], np.float32), 2).tolist() == [0, 1]
    assert sel.recompute_budget(0.15, 20) == 3 and sel.recompute_budget(0.15, 21) == 4
    with pytest.raises(ValueError):
        sel.key_diff(np.zeros((2, 2, 4), np.float32), np.zeros((3, 2, 4), np.float32))


@pytest.mark.parametrize("n_members,count", [(1, 1), (3, 37), (8, 4096), (2, 16384)])
def test_random_members_against_oracle(n_members, count):
    rng = np.random.default_rng(count)
    R = n_members * count
    fresh = rng.standard_normal((R, 4, 32)).astype(np.float32)
    cached = fresh.copy()
    # a third of the rows identical (zero magnitude -> never selected)
    moved = rng.random(R) > 0.33
    cached[moved] += rng.standard_normal((int(moved.sum()), 4, 32)).astype(np.float32) * 0.1
    out = sel.batched_selection(fresh, cached, [count] * n_members, 0.15)
    mags = ref.key_diff(fresh, cached)
    for m, (imp, dev) in enumerate(out):
        mm = mags[m * count:(m + 1) * count]
        want = ref.select_important(mm, ref.recompute_budget(0.15, count))
        assert imp.tolist() == want.tolist()
        assert abs(dev - float(mm.sum())) <= 1e-5 * max(1.0, float(mm.sum()))


def test_cached_rows_from_the_pool():
    """The cached keys are read straight from a pool plane by slot."""
    rng = np.random.default_rng(9)
    pool = torch.from_numpy(rng.standard_normal((500, 2, 16)).astype(np.float32)).to(DEV)
    slots = rng.choice(500, 120, replace=False)
    fresh = pool[torch.from_numpy(slots).to(DEV)].clone()
    fresh[::3] += 0.5
    out = sel.batched_selection(fresh, pool, [50, 70], 0.2, cached_rows=slots)
    dense = pool[torch.from_numpy(slots).to(DEV)]
    want = sel.batched_selection(fresh, dense, [50, 70], 0.2)
    for (a, da), (b, db) in zip(out, want):
        assert a.tolist() == b.tolist() and da == db


def test_bf16_keys():
    rng = np.random.default_rng(4)
    f = torch.from_numpy(rng.standard_normal((300, 4, 128)).astype(np.float32)).to(DEV).bfloat16()
    c = (f.float() + 0.05 * torch.randn_like(f.float())).bfloat16()
    out = sel.batched_selection(f, c, [100, 200], 0.15)
    mags = ref.key_diff(f.float().cpu().numpy(), c.float().cpu().numpy())
    for (imp, dev), (lo, n) in zip(out, [(0, 100), (100, 200)]):
        mm = mags[lo:lo + n]
        assert imp.tolist() == ref.select_important(mm, ref.recompute_budget(0.15, n)).tolist()


def test_ragged_members_and_repeated_passes():
    """Ragged members incl. empty ones and members of one row, ties, zero
    rows, repeated passes: every member's important set and deviation equal
    the oracle's."""
    rng = np.random.default_rng(7)
    counts = [0, 1, 63, 64, 65, 700, 0, 4096, 5, 129]
    R = sum(counts)
    fresh = rng.standard_normal((R, 2, 64)).astype(np.float32)
    cached = fresh.copy()
    moved = rng.random(R) > 0.4
    cached[moved] += np.round(rng.standard_normal((int(moved.sum()), 2, 64)) * 4) / 4
    f = torch.from_numpy(fresh).to(DEV)
    c = torch.from_numpy(cached).to(DEV)
    mags = ref.key_diff(fresh, cached)
    off = np.concatenate([[0], np.cumsum(counts)])
    for _ in range(3):
        out = sel.batched_selection(f, c, counts, 0.2)
        for m, (imp, dv) in enumerate(out):
            mm = mags[off[m]:off[m + 1]]
            want = ref.select_important(mm, ref.recompute_budget(0.2, counts[m])) if counts[m] \
                else np.zeros(0, np.int64)
            assert imp.tolist() == want.tolist(), m
            assert abs(dv - float(mm.sum())) <= 1e-5 * max(1.0, abs(float(mm.sum())))

"""Seeded input generators shared by the CPU and GPU parity tests.

The random streams match the ones the reference tests draw
(``pkg/tests/conftest.py:54-73``) and ``tests/golden/make_golden.py``, so
the golden digests recorded from the reference apply to these inputs.
"""
from __future__ import annotations

import hashlib
import json
import os
from dataclasses import dataclass

import numpy as np

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_golden() -> dict:
    with open(os.path.join(GOLDEN_DIR, "golden.json")) as f:
        return json.load(f)


def load_npz(name: str):
    return np.load(os.path.join(GOLDEN_DIR, name))


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode() + str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def random_planes(rng, t, layers=4, heads=2, dim=8, start=0):
    shape = (layers, t, heads, dim)
    k = rng.standard_normal(shape).astype(np.float32)
    v = rng.standard_normal(shape).astype(np.float32)
    return k, v, np.arange(start, start + t, dtype=np.int64)


def perturb(rng, k, v, block_size, block_ids):
    """Mirror = master with whole blocks re-drawn in every layer."""
    t = k.shape[1]
    mk, mv = k.copy(), v.copy()
    hints = []
    for b in block_ids:
        lo, hi = b * block_size, min(b * block_size + block_size, t)
        mk[:, lo:hi] = rng.standard_normal(mk[:, lo:hi].shape).astype(np.float32)
        mv[:, lo:hi] = rng.standard_normal(mv[:, lo:hi].shape).astype(np.float32)
        hints.extend(range(lo, hi))
    return mk, mv, np.asarray(sorted(hints), dtype=np.int64)


@dataclass
class CodecTrial:
    block_size: int
    master_k: np.ndarray
    master_v: np.ndarray
    positions: np.ndarray
    mirror_k: np.ndarray
    mirror_v: np.ndarray
    hints: np.ndarray


def codec_trials(n=1000):
    """The acceptance-C04 trial stream (pkg/tests/test_acceptance.py:186-228)."""
    rng = np.random.default_rng(0xD1FF)
    for _ in range(n):
        bs = int(rng.choice([8, 16, 32]))
        t = int(rng.integers(1, 180))
        layers = int(rng.integers(1, 4))
        heads = int(rng.integers(1, 3))
        dim = 2 * int(rng.integers(1, 5))
        start = int(rng.integers(0, 40))
        k, v, pos = random_planes(rng, t, layers, heads, dim, start)
        mk, mv = k.copy(), v.copy()
        nb = -(-t // bs)
        count = int(rng.integers(0, nb + 1))
        chosen = rng.choice(nb, size=count, replace=False)
        hints = []
        for b in sorted(int(b) for b in chosen):
            lo, hi = b * bs, min(b * bs + bs, t)
            hints.extend(range(lo, hi))
            mode = int(rng.integers(0, 4))
            row = int(rng.integers(lo, hi))
            if mode == 0:
                mk[:, lo:hi] += 1.0
            elif mode == 1:
                mv[:, lo:hi] -= 1.0
            elif mode == 2:
                mk[:, row] = rng.standard_normal(mk[:, row].shape).astype(np.float32)
        yield CodecTrial(bs, k, v, pos, mk, mv, np.asarray(hints, dtype=np.int64))


@dataclass
class RestoreTrial:
    block_size: int
    master_k: np.ndarray
    master_v: np.ndarray
    positions: np.ndarray
    mirror_k: np.ndarray
    mirror_v: np.ndarray
    hints: np.ndarray
    delta: int


def restore_trials(n=200):
    """The acceptance-C05 trial stream (pkg/tests/test_acceptance.py:231-279)."""
    rng = np.random.default_rng(0xF05E)
    bs = 16
    for _ in range(n):
        t = int(rng.integers(8, 90))
        start = int(rng.integers(0, 60))
        delta = int(rng.integers(-start, 80))
        k, v, pos = random_planes(rng, t, 3, 2, 8, start)
        nb = -(-t // bs)
        count = int(rng.integers(0, min(nb, 3) + 1))
        chosen = sorted(int(b) for b in rng.choice(nb, count, replace=False))
        mk, mv, hints = perturb(rng, k, v, bs, chosen)
        yield RestoreTrial(bs, k, v, pos, mk, mv, hints, delta)


def replay_segment_index(make_index, entry_factory, ops):
    """Replay the reference's recorded segment-index stream (golden.json
    'segment_index') on ``make_index(budget, is_pinned, on_evict)`` and check
    every recorded outcome; ``entry_factory(tok, nbytes, ref)`` builds an
    entry for a 1-token segment."""
    import hashlib

    class Ref:
        def __init__(self):
            self.pinned = False

    def digest(tok):
        return hashlib.blake2b(np.asarray([tok], dtype="<u4").tobytes(), digest_size=16).digest()

    made, label, evicted = [], {}, []
    idx = make_index(2000, lambda r: r.pinned, lambda e: evicted.append(label[id(e)]))
    for step, op in enumerate(ops):
        if op["op"] == "insert":
            e = entry_factory(op["tok"], op["nbytes"], Ref())
            label[id(e)] = len(made)
            made.append(e)
            idx.insert(e)
        elif op["op"] == "lookup":
            hit = idx.lookup(digest(op["tok"]))
            assert (-1 if hit is None else label[id(hit)]) == op["hit"], step
        elif op["op"] == "pin":
            made[op["label"]].kv_ref.pinned = not made[op["label"]].kv_ref.pinned
        elif op["op"] == "remove":
            raised = False
            try:
                idx.remove(made[op["label"]])
            except Exception:                     # the pinned-entry error of each API
                raised = True
            assert raised == op["raised"], step
        else:
            assert idx.evict_to_budget(op["budget"]) == op["n"], step
        assert evicted == op["evicted"], step
        assert idx.total_bytes == op["total"] and len(idx) == op["len"], step
        assert [label[id(e)] for e in idx.entries()] == op["lru"], step


# soundness-violation magnitudes with NaN / inf / signed zeros outside the
# hints; the same cases as tests/golden/make_golden.py VIOLATION_CASES:
# (plane, index, value or None = +2.5, edit the master instead of the mirror)
VIOLATION_CASES = {
    "nan_k": [("k", (0, 100, 0, 0), float("nan"), False)],
    "nan_v_and_k": [("v", (0, 100, 0, 0), float("nan"), False), ("k", (0, 101, 1, 3), None, False)],
    "nan_both_v": [("v", (2, 99, 1, 1), float("nan"), False), ("v", (2, 99, 1, 1), float("nan"), True)],
    "neg_inf_k": [("k", (3, 127, 0, 7), float("-inf"), False)],
    "signed_zero": [("k", (1, 110, 1, 2), 0.0, True), ("k", (1, 110, 1, 2), -0.0, False)],
}


def violation_case(case):
    """(master k, master v, mirror k, mirror v, hints) of a special case."""
    rng = np.random.default_rng(24)
    k, v, _ = random_planes(rng, 128)
    mk, mv, hints = perturb(rng, k, v, 32, [1])
    planes = {("k", True): k, ("v", True): v, ("k", False): mk, ("v", False): mv}
    for plane, idx, value, on_master in VIOLATION_CASES[case]:
        arr = planes[(plane, on_master)]
        arr[idx] = value if value is not None else arr[idx] + np.float32(2.5)
    return k, v, mk, mv, hints

"""Native round planning (tdkv_plan_offsets, host C++) against its numpy
restatement, record for record: the stable segment order of the jobs, one
delta per job, the (tile, job-chunk) units and the plan totals.  Host only --
no GPU needed."""
import math

import numpy as np
import pytest

import paper_2604_03143_b200 as tk
from paper_2604_03143_b200 import _lib
from paper_2604_03143_b200 import collector as col


@pytest.fixture(scope="module", autouse=True)
def _built():
    tk.build_library()


def _plan_numpy(seg_row0, seg_len, segments, dst_off, job_delta, L, tile_rows, target_items):
    """The numpy planning the native call replaced (collector._build_units
    plus the stable job sort)."""
    segments = np.asarray(segments, np.int64)
    J = segments.size
    if J == 0:
        return (np.zeros(0, _lib.COLLECT_UNIT), np.zeros(0, _lib.COLLECT_JOB),
                np.zeros(0, np.int64), False, 0, 0)
    order = np.argsort(segments, kind="stable")
    seg_o = segments[order]
    jobs = np.zeros(J, dtype=_lib.COLLECT_JOB)
    jobs["dst_off"] = np.asarray(dst_off, np.int64)[order]
    jobs["seg_row0"] = np.asarray(seg_row0, np.int64)[seg_o]
    jobs["tbl_row"] = np.arange(J)
    useg, first, njobs = np.unique(seg_o, return_index=True, return_counts=True)
    n_s = np.asarray(seg_len, np.int64)[useg]
    r0_s = np.asarray(seg_row0, np.int64)[useg]
    nt = (n_s + tile_rows - 1) // tile_rows
    tile_seg = np.repeat(np.arange(useg.size), nt)
    starts = np.concatenate([[0], np.cumsum(nt)[:-1]])
    tile_i = np.arange(int(nt.sum())) - np.repeat(starts, nt)
    base = max(1, L * tile_seg.size)
    nchunk = min(int(njobs.max()), max(1, math.ceil(target_items / base)))
    per = np.maximum(1, -(-njobs // nchunk))
    nc = -(-njobs // per)
    nc_t = nc[tile_seg]
    unit_tile = np.repeat(np.arange(tile_seg.size), nc_t)
    cstart = np.concatenate([[0], np.cumsum(nc_t)[:-1]]) if nc_t.size else np.zeros(0, np.int64)
    unit_c = np.arange(int(nc_t.sum())) - np.repeat(cstart, nc_t)
    us = tile_seg[unit_tile]
    units = np.zeros(unit_tile.size, dtype=_lib.COLLECT_UNIT)
    units["row0"] = r0_s[us] + tile_i[unit_tile] * tile_rows
    units["nrows"] = np.minimum(tile_rows, n_s[us] - tile_i[unit_tile] * tile_rows)
    jb = first[us] + unit_c * per[us]
    units["job_begin"] = jb
    units["job_end"] = np.minimum(jb + per[us], first[us] + njobs[us])
    deltas = np.asarray(job_delta, np.int64)[order]
    total = int(np.asarray(seg_len, np.int64)[segments].sum())
    return units, jobs, deltas, bool(deltas.any()), total, int(n_s.sum())


def _case(rng, n_seg, n_jobs, zero_len=False):
    seg_len = rng.integers(0 if zero_len else 1, 90, n_seg)
    seg_row0 = np.concatenate([[0], np.cumsum(seg_len)[:-1]])
    segments = rng.integers(0, n_seg, n_jobs)
    dst_off = rng.integers(0, 1 << 40, n_jobs)
    delta = rng.integers(-500, 5000, n_jobs) * (rng.random(n_jobs) < 0.8)
    return seg_row0, seg_len, segments, dst_off, delta


@pytest.mark.parametrize("seed", range(12))
def test_native_plan_equals_numpy(seed):
    rng = np.random.default_rng(seed)
    n_seg = int(rng.integers(1, 300))
    n_jobs = int(rng.integers(1, 7000))
    args = _case(rng, n_seg, n_jobs, zero_len=seed % 3 == 0)
    L = int(rng.choice([1, 2, 28, 48]))
    tile = int(rng.choice([1, 4, 8, 16, 32]))
    target = int(rng.choice([1, 64, 592, 100000]))
    got = col.plan_host_offsets(*args, L, tile, target)
    units, jobs, deltas, rotate, total, master = _plan_numpy(*args, L, tile, target)
    assert np.array_equal(got.units, units)
    assert np.array_equal(got.jobs, jobs)
    assert np.array_equal(got.deltas, deltas)
    assert (got.rotate, got.rows_written, got.master_rows) == (rotate, total, master)


def test_native_plan_c3_round_shape():
    """The C3 round: 10 sessions x 25 shared segments of 20 rows, 250 agents
    each reading its session's 25 segments."""
    S = 250
    seg_len = np.full(S, 20, np.int64)
    seg_row0 = np.arange(S, dtype=np.int64) * 20
    segs = np.concatenate([np.arange(s * 25, (s + 1) * 25) for s in range(10) for _ in range(25)])
    dst_off = np.arange(segs.size, dtype=np.int64) * 20
    delta = np.random.default_rng(0).integers(0, 700, segs.size)
    for tile in (8, 16):
        got = col.plan_host_offsets(seg_row0, seg_len, segs, dst_off, delta, 48, tile, 592)
        want = _plan_numpy(seg_row0, seg_len, segs, dst_off, delta, 48, tile, 592)
        assert np.array_equal(got.units, want[0]) and np.array_equal(got.jobs, want[1])
        assert got.rows_written == 250 * 25 * 20 and got.master_rows == S * 20


def test_native_plan_empty_and_errors():
    z = np.zeros(0, np.int64)
    p = col.plan_host_offsets(np.array([0]), np.array([4]), z, z, z, 2, 8)
    assert p.units.size == 0 and p.jobs.size == 0 and not p.rotate and p.rows_written == 0
    with pytest.raises(ValueError):       # a job naming a segment the arena lacks
        col.plan_host_offsets(np.array([0]), np.array([4]), np.array([1]), np.array([0]),
                              np.array([0]), 2, 8)
    with pytest.raises(ValueError):       # one delta per job
        col.plan_host_offsets(np.array([0]), np.array([4]), np.array([0]), np.array([0]),
                              np.array([0, 1]), 2, 8)

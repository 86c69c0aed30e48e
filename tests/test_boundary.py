"""CPU-side checks of the drop-in boundary: the C-ABI library loads and
exports every symbol include/tdkv.h declares, descriptor layouts match the
header, host-side planning (allocator policy, collect plan tiling) matches
the reference, and the product package never imports the oracle."""
import ast
import os
import re

import numpy as np
import pytest

from helpers import load_golden
from oracle import roundkv_port as ref

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2604_03143_b200")


def _header_functions():
    text = open(os.path.join(ROOT, "include", "tdkv.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int32_t|int64_t|const char\*|void\*?)\s+(tdkv_\w+)\s*\(",
                                 text, re.M)))


def test_library_exports_every_header_symbol():
    from paper_2604_03143_b200 import _lib
    _lib.build_library()
    lib = _lib.load()
    declared = _header_functions()
    assert declared, "no functions parsed from tdkv.h"
    assert set(declared) == set(_lib.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), name
    assert _lib.version() == (1 << 16)
    assert _lib.launch_count() >= 0


def test_descriptor_layouts_match_header():
    from paper_2604_03143_b200 import _lib
    text = open(os.path.join(ROOT, "include", "tdkv.h")).read()
    for struct, dt in [("tdkv_collect_job", _lib.COLLECT_JOB),
                       ("tdkv_collect_unit", _lib.COLLECT_UNIT),
                       ("tdkv_diff_pair", _lib.DIFF_PAIR), ("tdkv_diff_out", _lib.DIFF_OUT),
                       ("tdkv_wire_seg", _lib.WIRE_SEG),
                       ("tdkv_rows_job", _lib.ROWS_JOB),
                       ("tdkv_collect_overlay", _lib.COLLECT_OVERLAY)]:
        body = re.search(r"typedef struct \{([^{}]*)\}\s*" + struct + ";", text).group(1)
        # field count and total size (pointers / int64 = 8 B, int32 = 4 B)
        sizes = []
        for line in body.strip().splitlines():
            line = line.split("/*")[0].strip()
            if not line:
                continue
            sizes.append(8 if ("*" in line or "int64_t" in line) else 4)
        assert sum(sizes) == dt.itemsize, struct
        assert len(sizes) == len(dt.names), struct


def test_allocator_policy_matches_reference_stream():
    from paper_2604_03143_b200.paged_pool import choose_slots
    free = np.ones(256, bool)
    live = {}
    for op in load_golden()["allocator"]:
        if op["op"] == "alloc":
            got = choose_slots(free, op["n"], 32)
            assert got.tolist() == op["slots"]
            free[got] = False
            live[op["serial"]] = got
        elif op["op"] == "free":
            free[live.pop(op["serial"])] = True


def test_allocator_randomized_against_oracle():
    from paper_2604_03143_b200.paged_pool import choose_slots
    rng = np.random.default_rng(5)
    for cap, bs in [(100, 32), (257, 16), (64, 8), (1000, 32)]:
        free_a = np.ones(cap, bool)
        live = []
        for step in range(300):
            if live and rng.random() < 0.4:
                m = live.pop(int(rng.integers(len(live))))
                free_a[m] = True
                continue
            n = int(rng.integers(1, cap // 4))
            if n > free_a.sum():
                continue
            want = ref.allocate_slots(free_a.copy(), n, bs)
            got = choose_slots(free_a, n, bs)
            assert got.tolist() == want.tolist()
            free_a[got] = False
            live.append(got)


def test_product_never_imports_oracle():
    for dirpath, _, files in os.walk(PKG):
        for f in files:
            if not f.endswith(".py"):
                continue
            tree = ast.parse(open(os.path.join(dirpath, f)).read())
            for node in ast.walk(tree):
                if isinstance(node, ast.Import):
                    assert all(not a.name.startswith("oracle") for a in node.names), f
                if isinstance(node, ast.ImportFrom):
                    assert not (node.module or "").startswith("oracle"), f


def test_wire_size_formula_matches_serialization():
    from paper_2604_03143_b200.diffstore import BlockSparseDiff, LayerDiff, serialize_diff, wire_nbytes
    rng = np.random.default_rng(3)
    layers = []
    for c in (0, 2, 1):
        idx = np.sort(rng.choice(5, c, replace=False))
        kb = rng.standard_normal((c, 8, 2, 4)).astype(np.float32)
        layers.append(LayerDiff(idx, kb, kb.copy()))
    diff = BlockSparseDiff(3, 8, 2, 4, 37, layers)
    assert wire_nbytes(diff) == len(serialize_diff(diff))
    want = ref.serialize([ref.DiffLayer(l.indices, l.k_blocks, l.v_blocks) for l in layers],
                         8, 2, 4, 37)
    assert serialize_diff(diff) == want


def test_deserialize_rejects_malformed_like_reference():
    from paper_2604_03143_b200.diffstore import MalformedDiffError, deserialize_diff
    rng = np.random.default_rng(41)
    k = rng.standard_normal((4, 64, 2, 8)).astype(np.float32)
    v = rng.standard_normal((4, 64, 2, 8)).astype(np.float32)
    mk, mv = k.copy(), v.copy()
    mk[:, :32] += 1
    wire = ref.serialize(ref.encode_diff(k, v, mk, mv, np.arange(32), 32), 32, 2, 8, 64)
    back = deserialize_diff(wire)
    assert back.changed_blocks_per_layer == [1, 1, 1, 1]
    for bad, what in [(b"XXXX" + wire[4:], "magic"), (wire[:4] + b"\xff\x00" + wire[6:], "version"),
                      (wire[:10], "truncated"), (wire[:-6], "truncated"),
                      (wire + b"\x00", "trailing"), (b"", "truncated")]:
        with pytest.raises(MalformedDiffError, match=what):
            deserialize_diff(bad)


def test_offset_planning_matches_row_planning():
    from paper_2604_03143_b200 import rounds
    from paper_2604_03143_b200.collector import plan_host, plan_host_offsets
    spec = rounds.CONFIGS["c2"].scaled(num_agents=7)
    T = spec.tokens_per_agent
    spec = spec.scaled(sessions=2)
    starts = np.stack([rounds.segment_starts(spec, a) for a in range(7)])
    slots = np.random.default_rng(0).permutation(7 * T).reshape(7, T)
    base = np.arange(7) * T
    segs, dst_off, jd = rounds.round_offsets(spec, range(7), base)
    rows = (starts[:, :, None] + np.arange(spec.seg_len)).reshape(7, -1)
    dst = np.take_along_axis(slots, rows, axis=1).reshape(-1)
    dl = np.repeat(jd, spec.seg_len)
    seg_row0 = np.arange(spec.total_segments) * spec.seg_len
    seg_len = np.full(spec.total_segments, spec.seg_len)
    a = plan_host(seg_row0, seg_len, segs, dst, dl, spec.num_layers, 8)
    b = plan_host_offsets(seg_row0, seg_len, segs, dst_off, jd, spec.num_layers, 8)
    assert np.array_equal(a.units, b.units)
    assert np.array_equal(a.jobs["seg_row0"], b.jobs["seg_row0"])
    assert np.array_equal(a.jobs["tbl_row"], b.jobs["tbl_row"])
    assert (a.jobs["tbl_stride"] == 0).all() and np.array_equal(a.deltas, b.deltas)
    flat = slots.reshape(-1)
    for j in range(a.jobs.size):
        n = spec.seg_len
        assert np.array_equal(a.dst_rows[a.jobs["dst_off"][j]:a.jobs["dst_off"][j] + n],
                              flat[b.jobs["dst_off"][j]:b.jobs["dst_off"][j] + n])
    assert a.rows_written == b.rows_written and a.master_rows == b.master_rows


def test_native_allocator_matches_reference_policy():
    """tdkv_alloc_* (host C++) against the reference's recorded allocator
    stream and the oracle policy under random alloc/free churn."""
    from paper_2604_03143_b200.paged_pool import OutOfSlotsError, SlotAllocator
    a = SlotAllocator(256, 32)
    live = {}
    for op in load_golden()["allocator"]:
        if op["op"] == "alloc":
            got = a.take(op["n"])
            assert got.tolist() == op["slots"]
            live[op["serial"]] = got
        elif op["op"] == "free":
            a.release(live.pop(op["serial"]))
    rng = np.random.default_rng(9)
    for cap, bs in [(1000, 32), (777, 16), (64, 64)]:
        al = SlotAllocator(cap, bs)
        free = np.ones(cap, bool)
        held = []
        for _ in range(400):
            if held and rng.random() < 0.45:
                m = held.pop(int(rng.integers(len(held))))
                al.release(m)
                free[m] = True
                continue
            n = int(rng.integers(1, max(2, cap // 5)))
            if n > free.sum():
                with pytest.raises(OutOfSlotsError):
                    al.take(n)
                continue
            want = ref.allocate_slots(free, n, bs)
            got = al.take(n)
            assert got.tolist() == want.tolist()
            held.append(got)
        assert al.free_count == int(free.sum())
    with pytest.raises(ValueError, match="not allocated"):
        al.release(np.array([0, 0]))


def test_c_abi_rejects_bad_arguments_without_a_gpu():
    """Argument validation happens before any CUDA call: the status codes and
    messages are observable on a CPU-only host."""
    import ctypes
    from paper_2604_03143_b200 import _lib
    lib = _lib.load()
    null = ctypes.c_void_p(0)
    rc = lib.tdkv_collect(null, null, 0, null, 1, 8, null, null, null, 0, null, null, 0,
                          2, 2, 7, 0, 0, null)
    assert rc == 1 and b"geometry" in lib.tdkv_last_error()
    rc = lib.tdkv_collect(null, null, 0, null, 1, 8, null, null, null, 0, null, null, 0,
                          2, 2, 8, 0, 0, null)
    assert rc == 1 and b"null pointer" in lib.tdkv_last_error()
    rc = lib.tdkv_collect(null, null, 0, null, 1, 64, null, null, null, 0, null, null, 0,
                          2, 2, 8, 0, 0, null)
    assert rc == 1 and b"max_rows" in lib.tdkv_last_error()
    assert lib.tdkv_diff_compare(null, 1, null, null, null, null, 1, 8, 1, 8, 0, 0, null) == 1
    assert lib.tdkv_diff_compare(null, 1, null, null, null, null, 1, 8, 1, 8, 8, 7, null) == 2
    assert lib.tdkv_rows(null, 1, 8, null, 1, 1, 8, 8, 0, 0, 0, 0, null) == 1
    assert lib.tdkv_gemm(null, 8, null, 8, null, 8, 4, 4, 4, 0, 0, null) == 1
    assert lib.tdkv_select_important(null, null, null, null, 1, 100000, null, null, null,
                                     null) == 2
    assert lib.tdkv_rope_table(null, 4, null, 4, 0, null, null) == 1
    # zero-size work is a successful no-op
    assert lib.tdkv_collect(null, null, 0, null, 0, 8, null, null, null, 0, null, null, 0,
                            2, 2, 8, 0, 0, null) == 0
    assert lib.tdkv_rows(null, 0, 8, null, 1, 1, 8, 8, 0, 0, 0, 0, null) == 0


def test_collect_sources_rejects_bad_arguments_without_a_gpu():
    """tdkv_collect_sources (the peer-read K1) validates its source table
    before any CUDA call."""
    import ctypes
    from paper_2604_03143_b200 import _lib
    lib = _lib.load()
    null = ctypes.c_void_p(0)
    fake = ctypes.c_void_p(0x100000)              # never dereferenced: validation fails first
    tbl = (ctypes.c_void_p * 2)(fake.value, fake.value)
    tail = [null, 1, 8, null, null, null, 0, null, null, 0, 2, 2, 8, 1, 0, null]
    assert lib.tdkv_collect_sources(tbl, tbl, 0, null, 0, *tail) == 1
    assert b"sources" in lib.tdkv_last_error()
    assert lib.tdkv_collect_sources(tbl, tbl, 17, fake, 0, *tail) == 1
    assert lib.tdkv_collect_sources(tbl, tbl, 2, null, 0, *tail) == 1      # no unit map
    tail_v = tail[:8] + [fake] + tail[9:]         # a V destination for the K+V form
    odd = (ctypes.c_void_p * 2)(fake.value, fake.value + 8)
    assert lib.tdkv_collect_sources(odd, odd, 2, fake, 0, *tail_v) == 1
    assert b"aligned" in lib.tdkv_last_error()
    holes = (ctypes.c_void_p * 2)(fake.value, None)
    assert lib.tdkv_collect_sources(holes, tbl, 2, fake, 0, *tail_v) == 1
    assert b"null" in lib.tdkv_last_error()
    # K+V sources with a K-only destination (and the converse) are rejected
    assert lib.tdkv_collect_sources(tbl, None, 2, fake, 0, *tail_v) == 1
    assert lib.tdkv_collect_sources(tbl, tbl, 2, fake, 0, *tail) == 1


def test_missing_library_fails_loudly():
    """No CPU fallback: with the library absent the entry points raise
    TdkvUnavailable instead of computing anything on the host."""
    import subprocess
    import sys
    code = (
        "import paper_2604_03143_b200 as p\n"
        "for fn in (p.launch_count, lambda: p.SegmentIndex(4)):\n"
        "    try:\n"
        "        fn()\n"
        "    except p.TdkvUnavailable:\n"
        "        continue\n"
        "    raise SystemExit('entry point ran without libtdkv.so')\n"
        "print('ok')\n")
    env = dict(os.environ, TDKV_LIBRARY=os.path.join(ROOT, "no-such-dir", "libtdkv.so"))
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True,
                         text=True, timeout=300)
    assert out.returncode == 0 and out.stdout.strip() == "ok", out.stdout + out.stderr


def test_integration_binding_matches_library_signatures():
    """The ctypes stub INTEGRATION.md shows a maintainer declares the same
    argument types as the repo's own binding (and so as include/tdkv.h)."""
    import ctypes
    from paper_2604_03143_b200 import _lib
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    names = {"_P": ctypes.c_void_p, "_I32": ctypes.c_int32, "_I64": ctypes.c_int64,
             "ctypes.c_float": ctypes.c_float, "ctypes.c_uint32": ctypes.c_uint32}
    found = re.findall(r"_lib\.(tdkv_\w+)\.argtypes = \[([^\]]*)\]", text, re.S)
    assert len(found) >= 15
    for fn, body in found:
        args = [names[a.strip()] for a in re.sub(r"#[^\n]*", "", body).split(",") if a.strip()]
        assert args == _lib._SIGS[fn][1], fn


def test_binding_signatures_match_header_prototypes():
    """Every prototype in include/tdkv.h and its ctypes declaration agree
    argument by argument (pointer / int32 / int64 / float), so a stale
    binding cannot shift arguments silently."""
    import ctypes
    from paper_2604_03143_b200 import _lib
    text = open(os.path.join(ROOT, "include", "tdkv.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    text = re.sub(r"//[^\n]*", "", text)

    def ctype(decl):
        decl = decl.strip()
        if "*" in decl:
            return ctypes.c_void_p
        base = decl.replace("const ", "").split()[0]
        return {"int32_t": ctypes.c_int32, "int64_t": ctypes.c_int64, "float": ctypes.c_float,
                "uint32_t": ctypes.c_uint32, "tdkv_pinned_fn": ctypes.c_void_p}[base]

    seen = set()
    for fn, body in re.findall(r"(?<!\*)\b(tdkv_\w+)\s*\(([^;{]*?)\)\s*;", text, re.S):
        body = body.strip()
        args = [] if body in ("", "void") else [ctype(a) for a in body.split(",")]
        assert args == _lib._SIGS[fn][1], fn
        seen.add(fn)
    assert seen == set(_lib.EXPORTS)

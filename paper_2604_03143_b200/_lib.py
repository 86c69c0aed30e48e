"""ctypes binding of libtdkv.so (the C-ABI declared in include/tdkv.h).

The shared library is built in-tree by ``build_library()`` (nvcc, sm_100a)
and loaded from this package directory.  There is no fallback: if the
library is missing every entry point raises ``TdkvUnavailable``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from typing import Optional

import numpy as np

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG_DIR)
LIB_PATH = os.path.join(PKG_DIR, "libtdkv.so")
CSRC = os.path.join(PKG_DIR, "csrc")
INCLUDE = os.path.join(ROOT, "include")

TDKV_F32 = 0
TDKV_BF16 = 1
NO_VIOLATION = 0x7F7F7F7F
ROWS_CONTIGUOUS = 1
ROWS_JOB_MINOR = 2
ROUND_FUSE_TABLE = 1
ROUND_NEOX = 2
ROUND_ONE_ITEM = 4

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
]


class TdkvUnavailable(RuntimeError):
    """libtdkv.so is not built or cannot be loaded (no CPU fallback exists)."""


class TdkvError(RuntimeError):
    """A tdkv C-ABI call returned a non-zero status."""


# ---------------------------------------------------------------------------
# build


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def build_library(force: bool = False, verbose: bool = False) -> str:
    """Compile csrc/*.cu into libtdkv.so for sm_100a (cross-compiles without a GPU)."""
    srcs = sources()
    deps = srcs + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cuh")]
    deps.append(os.path.join(INCLUDE, "tdkv.h"))
    if not force and os.path.exists(LIB_PATH):
        built = os.path.getmtime(LIB_PATH)
        if all(os.path.getmtime(d) <= built for d in deps):
            return LIB_PATH
    nvcc = os.environ.get("NVCC", "nvcc")
    tmp = LIB_PATH + ".tmp"
    cmd = [nvcc, *NVCC_FLAGS, "-I", INCLUDE, *srcs, "-o", tmp]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


# ---------------------------------------------------------------------------
# descriptor layouts (must match include/tdkv.h)

COLLECT_JOB = np.dtype([("dst_off", "<i8"), ("seg_row0", "<i4"), ("tbl_row", "<i4"),
                        ("tbl_stride", "<i4"), ("pad", "<i4")])
COLLECT_UNIT = np.dtype([("row0", "<i4"), ("nrows", "<i4"), ("job_begin", "<i4"),
                         ("job_end", "<i4")])
DIFF_PAIR = np.dtype([("master_k", "<u8"), ("master_v", "<u8"), ("mirror_k", "<u8"),
                      ("mirror_v", "<u8")])
DIFF_OUT = np.dtype([("payload_k", "<u8"), ("payload_v", "<u8"), ("indices", "<u8"),
                     ("blkmap", "<u8"), ("cap", "<i4"), ("pad", "<i4")])
ROWS_JOB = np.dtype([("src_k", "<u8"), ("src_v", "<u8"), ("src_layer_stride", "<i8"),
                     ("src_rows", "<u8"), ("pay_k", "<u8"), ("pay_v", "<u8"),
                     ("map_k", "<u8"), ("map_v", "<u8"), ("dst_k", "<u8"), ("dst_v", "<u8"),
                     ("dst_layer_stride", "<i8"), ("dst_rows", "<u8"), ("num_tokens", "<i4"),
                     ("tbl_row", "<i4"), ("tbl_stride", "<i4"), ("rotate", "<i4")])
WIRE_SEG = np.dtype([("offset", "<u8"), ("nbytes", "<u8"), ("ptr", "<u8"), ("kind", "<i4"),
                     ("pad", "<i4")])
ATTN_MEMBER = np.dtype([("ctx_k", "<u8"), ("ctx_v", "<u8"), ("fresh_of", "<u8"),
                        ("fix_idx", "<u8"), ("ctx_layer_stride", "<i8"), ("row0", "<i4"),
                        ("n_rows", "<i4"), ("num_tokens", "<i4"), ("tile0", "<i4")])
COLLECT_OVERLAY = np.dtype([("pay_k", "<u8"), ("pay_v", "<u8"), ("map_k", "<u8"),
                            ("map_v", "<u8")])
WIRE_RAW, WIRE_BF16_TO_F32, WIRE_F32_TO_BF16 = 0, 1, 2
assert WIRE_SEG.itemsize == 32 and ATTN_MEMBER.itemsize == 56
assert COLLECT_JOB.itemsize == 24 and COLLECT_UNIT.itemsize == 16
assert COLLECT_OVERLAY.itemsize == 32
assert DIFF_PAIR.itemsize == 32 and DIFF_OUT.itemsize == 40 and ROWS_JOB.itemsize == 112

EXPORTS = (
    "tdkv_version", "tdkv_last_error", "tdkv_launch_count", "tdkv_host_is_pinned",
    "tdkv_copy_h2d", "tdkv_rope_table",
    "tdkv_collect", "tdkv_collect_round", "tdkv_collect_sources", "tdkv_restore_family", "tdkv_diff_compare", "tdkv_diff_compact", "tdkv_diff_encode", "tdkv_rows",
    "tdkv_keydiff", "tdkv_select_important", "tdkv_gemm", "tdkv_tf32_split", "tdkv_gemm_tf32x3",
    "tdkv_qkv_rope", "tdkv_attention",
    "tdkv_attention_many",
    "tdkv_fill_rows", "tdkv_alloc_create", "tdkv_alloc_destroy", "tdkv_alloc_free_count",
    "tdkv_alloc_take", "tdkv_alloc_release", "tdkv_wire_pack", "tdkv_wire_unpack",
    "tdkv_segidx_create", "tdkv_segidx_destroy", "tdkv_segidx_count", "tdkv_segidx_total",
    "tdkv_segidx_insert", "tdkv_segidx_lookup", "tdkv_segidx_remove", "tdkv_segidx_evict",
    "tdkv_segidx_entries", "tdkv_prepare_batch", "tdkv_plan_offsets",
)

_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_SIGS = {
    "tdkv_version": (_I32, []),
    "tdkv_last_error": (ctypes.c_char_p, []),
    "tdkv_launch_count": (_I64, []),
    "tdkv_host_is_pinned": (_I32, [_P]),
    "tdkv_copy_h2d": (_I32, [_P, _P, _I64, _P]),
    "tdkv_rope_table": (_I32, [_P, _I64, _P, _I32, _I32, _P, _P]),
    "tdkv_collect": (_I32, [_P, _P, _I64, _P, _I32, _I32, _P, _P, _P, _I32, _P, _P, _I64,
                            _I32, _I32, _I32, _I32, _I32, _P]),
    "tdkv_collect_round": (_I32, [_P, _I64, _P, _P, _P, _P, _I64, _P, _I32, _I32, _P, _P, _P,
                                  _P, _I64, _I32, _I32, _I32, _I32, _I32, _I32, _P]),
    "tdkv_collect_sources": (_I32, [_P, _P, _I32, _P, _I64, _P, _I32, _I32, _P, _P, _P, _I32,
                                    _P, _P, _I64, _I32, _I32, _I32, _I32, _I32, _P]),
    "tdkv_restore_family": (_I32, [_P, _P, _I32, _I64, _P, _I32, _I32, _P, _I32, _P, _P,
                                   _I32, _I32, _P, _I32, _P, _P, _I64, _I32, _I32, _I32, _I32,
                                   _I32, _P]),
    "tdkv_diff_compare": (_I32, [_P, _I32, _P, _P, _P, _P, _I32, _I32, _I32, _I32, _I32,
                                 _I32, _P]),
    "tdkv_diff_compact": (_I32, [_P, _P, _I32, _P, _P, _I32, _I32, _I32, _I32, _I32, _I32,
                                 _P]),
    "tdkv_rows": (_I32, [_P, _I32, _I32, _P, _I32, _I32, _I32, _I32, _I32, _I32, _I32, _I32,
                         _P]),
    "tdkv_diff_encode": (_I32, [_P, _P, _I32, _P, _P, _P, _P, _P, _P, _I32, _I32, _I32, _I32,
                                _I32, _I32, _P]),
    "tdkv_fill_rows": (_I32, [_P, _I64, _I32, _P, _I64, _I32, _I32, ctypes.c_uint32, _P]),
    "tdkv_keydiff": (_I32, [_P, _P, _P, _I64, _I32, _I32, _P, _P]),
    "tdkv_select_important": (_I32, [_P, _P, _P, _P, _I32, _I32, _P, _P, _P, _P]),
    "tdkv_gemm": (_I32, [_P, _I32, _P, _I32, _P, _I32, _I32, _I32, _I32, _I32, _I32, _P]),
    "tdkv_tf32_split": (_I32, [_P, _I64, _P, _P, _P]),
    "tdkv_gemm_tf32x3": (_I32, [_P, _P, _I32, _P, _P, _I32, _P, _I32, _I32, _I32, _I32, _I32, _P]),
    "tdkv_qkv_rope": (_I32, [_P, _P, _I32, _I32, _I32, _P, _P, _P, _P]),
    "tdkv_alloc_create": (_P, [_I64, _I32]),
    "tdkv_alloc_destroy": (None, [_P]),
    "tdkv_alloc_free_count": (_I64, [_P]),
    "tdkv_alloc_take": (_I32, [_P, _I64, _P]),
    "tdkv_alloc_release": (_I32, [_P, _P, _I64]),
    "tdkv_wire_pack": (_I32, [_P, _I32, _I64, _P, _P]),
    "tdkv_segidx_create": (_P, [_I64]),
    "tdkv_segidx_destroy": (None, [_P]),
    "tdkv_segidx_count": (_I64, [_P]),
    "tdkv_segidx_total": (_I64, [_P]),
    "tdkv_segidx_insert": (_I32, [_P, _P, _I64, _I64, _P, _P, _P, _I32, _P]),
    "tdkv_segidx_lookup": (_I32, [_P, _P, _I32, _I32, _P]),
    "tdkv_segidx_remove": (_I32, [_P, _I64, _I64]),
    "tdkv_segidx_evict": (_I32, [_P, _I64, _P, _P, _P, _I32, _P]),
    "tdkv_segidx_entries": (_I32, [_P, _P, _I64, _P]),
    "tdkv_wire_unpack": (_I32, [_P, _I32, _I64, _P, _P]),
    "tdkv_plan_offsets": (_I32, [_I32, _P, _P, _I32, _P, _P, _P, _I32, _I32, _I64, _P, _P, _P,
                                 _I64, _P]),
    "tdkv_prepare_batch": (_I32, [_P, _I32, _P, _P, _I32, _P, _P, _P, _P, _I64, _P, _I64, _P,
                                  _P, _P, _P, _P, _P, _P, _P, _P, _P, _I32]),
    "tdkv_attention_many": (_I32, [_P, _P, _P, _P, _I32, _I32, _I32, _I32, _I32, _I32, _I32,
                                   _I32, ctypes.c_float, _P, _P]),
    "tdkv_attention": (_I32, [_P, _P, _P, _P, _P, _P, _P, _I32, _I32, _I32, _I32,
                              ctypes.c_float, _P, _P]),
}

_lib: Optional[ctypes.CDLL] = None
_lock = threading.Lock()


def load(path: Optional[str] = None) -> ctypes.CDLL:
    """Load libtdkv.so (once; ``TDKV_LIBRARY`` overrides the in-tree path for
    A/B builds).  Raises TdkvUnavailable when it is missing."""
    global _lib
    if _lib is not None:                 # every launch passes here: no env lookup
        return _lib
    path = path or os.environ.get("TDKV_LIBRARY") or LIB_PATH
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise TdkvUnavailable(
                f"{path} is not built; run __graft_entry__.build() (nvcc sm_100a). "
                "There is no CPU fallback.")
        lib = ctypes.CDLL(path)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def call(name: str, *args) -> None:
    """Invoke a tdkv entry point; raise TdkvError with the library's message."""
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != 0:
        raise_last(name, rc)


def raise_last(name: str, rc: int = -1) -> None:
    """Raise TdkvError with the library's last message for a failed ``name``."""
    msg = load().tdkv_last_error().decode(errors="replace")
    raise TdkvError(f"{name} failed ({rc}): {msg}")


PINNED_FN = ctypes.CFUNCTYPE(ctypes.c_int32, ctypes.c_void_p, ctypes.c_int64)


_graph_launches = [0]


def note_launches(n: int) -> None:
    """Count kernels launched by a CUDA graph replay (their launches bypass
    the library's own counter)."""
    _graph_launches[0] += int(n)


def launch_count() -> int:
    """tdkv kernels launched by this process: the library's counter plus the
    kernels of replayed graphs."""
    return int(load().tdkv_launch_count()) + _graph_launches[0]


def version() -> int:
    return int(load().tdkv_version())

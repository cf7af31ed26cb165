"""ctypes binding of ``libfiltra_b200.so`` (the C-ABI in ``include/filtra_b200.h``).

This is the only path to compute in the package: there is no CPU or PyTorch
fallback. ``lib()`` raises ``NativeUnavailable`` when the library was not built or
no sm_100 device is present, so a missing extension fails loudly.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from . import errors

_LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libfiltra_b200.so"
_lib = None

c_i8p = ctypes.POINTER(ctypes.c_int8)
c_u64p = ctypes.POINTER(ctypes.c_uint64)
c_i64p = ctypes.POINTER(ctypes.c_int64)
c_i32p = ctypes.POINTER(ctypes.c_int32)
c_vp = ctypes.c_void_p

FB_OK = 0
FB_ERR_INVALID = 1
FB_ERR_DIM_MISMATCH = 2
FB_ERR_LENGTH_MISMATCH = 3
FB_ERR_DEGENERATE = 4
FB_ERR_CUDA = 5
FB_ERR_UNSUPPORTED = 6
FB_ERR_NO_DEVICE = 7
FB_ERR_PARSE = 8

FB_PLAN_FORCE_FALLBACK = 1
FB_PLAN_SIMT = 2
FB_PLAN_NO_SAMPLE = 4

FB_MAX_K_HASHES = 32
FB_MAX_STACK = 64
FB_MAX_LEAVES = 16384

# every symbol include/filtra_b200.h declares (checked by tests/test_native_cpu.py)
EXPORTED = (
    "fb_abi_version", "fb_last_error", "fb_device_ok", "fb_hash_leaves", "fb_bloom_build",
    "fb_filter_eval", "fb_quantize", "fb_quantize_f64", "fb_row_sums", "fb_topk_plan_create",
    "fb_topk_plan_destroy", "fb_topk_plan_stats", "fb_topk_execute", "fb_merge_topk",
    "fb_dequant_scores", "fb_int8_dot_rows", "fb_dot_rows_f64", "fb_launch_count",
    "fb_topk_set_timing", "fb_topk_last_timing", "fb_topk_scan_path", "fb_debug_tc_scores",
    "fb_task_dots_f64", "fb_kmeans_min_sqdist", "fb_pairwise_sum_scratch",
    "fb_pairwise_sum_f64", "fb_kmeans_draw", "fb_row_sqnorm_f64", "fb_kmeans_assign",
    "fb_kmeans_means", "fb_ivf_topk", "fb_merge_union", "fb_final_topk", "fb_value_model", "fb_vocab_create", "fb_vocab_free",
    "fb_pack_text", "fb_pack_postfix", "fb_pack_meta", "fb_pack_array", "fb_pack_free",
)


ABI_VERSION = 5  # include/filtra_b200.h FB_ABI_VERSION


class FbIndex(ctypes.Structure):
    _fields_ = [
        ("items", c_vp), ("planes", c_vp), ("valid", c_vp), ("id_rank", c_vp),
        ("item_ids", c_vp), ("row_sum", c_vp),
        ("n_slots", ctypes.c_int64), ("n_words", ctypes.c_int64),
        ("dim", ctypes.c_int32), ("dim_pad", ctypes.c_int32),
        ("m_bits", ctypes.c_int32), ("k_hashes", ctypes.c_int32),
        ("slot_of_rank", c_vp), ("id_of_rank", c_vp),
        ("id_dense", ctypes.c_int32), ("id_base", ctypes.c_uint64),
    ]


class FbFilterProg(ctypes.Structure):
    _fields_ = [
        ("n_queries", ctypes.c_int32), ("n_leaves", ctypes.c_int32),
        ("k_max", ctypes.c_int32), ("max_stack", ctypes.c_int32),
        ("leaf_pos", c_vp), ("op_offset", c_vp), ("ops", c_vp),
        ("n_planes", ctypes.c_int32), ("rmax_stack", ctypes.c_int32),
        ("n_rops", ctypes.c_int32), ("reserved", ctypes.c_int32),
        ("plane_list", c_vp), ("leaf_slot", c_vp), ("rop_offset", c_vp), ("rops", c_vp),
        ("n_cols", ctypes.c_int32), ("cnf_words", ctypes.c_int32),
        ("cnf_gmax", ctypes.c_int32), ("cnf_windowed", ctypes.c_int32),
        ("col_leaf", c_vp), ("qmask", c_vp), ("qgroups", c_vp),
    ]


class FbStats(ctypes.Structure):
    _fields_ = [
        ("slots_scanned", ctypes.c_int64), ("tiles", ctypes.c_int64),
        ("max_tile_rows", ctypes.c_int64), ("slots_evaluated", ctypes.c_int64),
        ("fallback_queries", ctypes.c_int64),
    ]


class NativeUnavailable(RuntimeError):
    """The sm_100a library is missing or no B200 is visible: the product has no fallback."""


def library_path() -> Path:
    return _LIB_PATH


def load_library() -> ctypes.CDLL:
    """Load the shared library without requiring a GPU (symbol checks on CPU)."""
    global _lib
    if _lib is not None:
        return _lib
    path = _LIB_PATH
    variant = os.environ.get("FB_LIB_VARIANT", "")  # A/B builds of the same sources (tools/)
    if variant:
        path = _LIB_PATH.with_name(f"libfiltra_b200_{variant}.so")
    if not path.exists():
        raise NativeUnavailable(
            f"{path} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(str(path))
    _declare(lib)
    if lib.fb_abi_version() != ABI_VERSION:
        raise NativeUnavailable(f"{path} has ABI {lib.fb_abi_version()}, expected "
                                f"{ABI_VERSION}: rebuild the library")
    _lib = lib
    return lib


def _declare(lib) -> None:
    i32, i64, dbl = ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    sig = {
        "fb_abi_version": ([], i32),
        "fb_last_error": ([], ctypes.c_char_p),
        "fb_device_ok": ([], i32),
        "fb_hash_leaves": ([c_vp, c_vp, i64, i32, i32, c_vp, c_vp], i32),
        "fb_bloom_build": ([c_vp, c_vp, c_vp, i64, i64, i32, i32, c_vp, c_vp], i32),
        "fb_filter_eval": ([ctypes.POINTER(FbIndex), ctypes.POINTER(FbFilterProg), i64, i64, i32,
                            c_vp, c_vp], i32),
        "fb_quantize": ([c_vp, i64, i32, dbl, dbl, c_vp, i32, c_vp], i32),
        "fb_quantize_f64": ([c_vp, i64, i32, dbl, dbl, c_vp, i32, c_vp], i32),
        "fb_row_sums": ([c_vp, i64, i32, i32, c_vp, c_vp], i32),
        "fb_topk_plan_create": ([ctypes.POINTER(FbIndex), i32, i32, c_vp, i32, i32,
                                 ctypes.POINTER(c_vp)], i32),
        "fb_topk_plan_destroy": ([c_vp], i32),
        "fb_topk_plan_stats": ([c_vp, ctypes.POINTER(FbStats)], i32),
        "fb_topk_execute": ([c_vp, c_vp, ctypes.POINTER(FbFilterProg), c_vp, c_vp, c_vp, c_vp,
                             c_vp, c_vp, dbl, dbl, c_vp], i32),
        "fb_merge_topk": ([c_vp, c_vp, c_vp, c_vp, i32, i32, i32, i32, c_vp, c_vp, c_vp, c_vp,
                           c_vp], i32),
        "fb_dequant_scores": ([c_vp, c_vp, c_vp, i32, i32, c_vp, i32, dbl, dbl, c_vp, c_vp], i32),
        "fb_int8_dot_rows": ([c_vp, i64, i32, i32, c_vp, c_vp, c_vp], i32),
        "fb_dot_rows_f64": ([c_vp, i64, i32, c_vp, c_vp, c_vp], i32),
        "fb_task_dots_f64": ([c_vp, i64, i32, c_vp, c_vp, i64, c_vp, i32, i32, c_vp, c_vp], i32),
        "fb_kmeans_min_sqdist": ([c_vp, i64, i32, i64, c_vp, i32, c_vp], i32),
        "fb_pairwise_sum_scratch": ([i64], i64),
        "fb_pairwise_sum_f64": ([c_vp, i64, c_vp, c_vp, i64, c_vp], i32),
        "fb_kmeans_draw": ([c_vp, c_vp, i64, c_vp, dbl, c_vp, c_vp, c_vp, c_vp], i32),
        "fb_row_sqnorm_f64": ([c_vp, i64, i32, c_vp, c_vp], i32),
        "fb_kmeans_assign": ([c_vp, i64, i32, c_vp, i32, c_vp, c_vp, c_vp, c_vp, c_vp], i32),
        "fb_kmeans_means": ([c_vp, i32, c_vp, c_vp, c_vp, i32, c_vp, c_vp], i32),
        "fb_ivf_topk": ([ctypes.POINTER(FbIndex), c_vp, i32, ctypes.POINTER(FbFilterProg), c_vp, i32,
                         i32, i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, dbl, dbl, c_vp],
                        i32),
        "fb_value_model": ([c_vp, i32, c_vp, c_vp, i32, i32, i64, c_vp, c_vp, c_vp, c_vp], i32),
        "fb_final_topk": ([c_vp, i64, c_vp, i32, i32, c_vp, c_vp, c_vp], i32),
        "fb_merge_union": ([c_vp, c_vp, i32, i32, i32, i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp],
                           i32),
        "fb_launch_count": ([], ctypes.c_uint64),
        "fb_vocab_create": ([i32, c_vp, c_vp, i32, c_vp, c_vp, c_vp], i32),
        "fb_vocab_free": ([c_vp], None),
        "fb_pack_text": ([i32, c_vp, c_vp, i32, i32, c_vp, c_vp], i32),
        "fb_pack_postfix": ([i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, i32, i32, c_vp], i32),
        "fb_pack_meta": ([c_vp, c_vp], i32),
        "fb_pack_array": ([c_vp, i32, c_vp, c_vp], i32),
        "fb_pack_free": ([c_vp], None),
        "fb_topk_scan_path": ([c_vp], i32),
        "fb_debug_tc_scores": ([ctypes.POINTER(FbIndex), c_vp, i32, c_vp, c_vp], i32),
        "fb_topk_set_timing": ([c_vp, i32], i32),
        "fb_topk_last_timing": ([c_vp, ctypes.POINTER(ctypes.c_float),
                                 ctypes.POINTER(ctypes.c_float)], i32),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res


def lib() -> ctypes.CDLL:
    """The library, verified usable on the current CUDA device (raises otherwise)."""
    l = load_library()
    if not getattr(l, "_device_checked", False):
        import torch
        if not torch.cuda.is_available():
            raise NativeUnavailable("no CUDA device visible; the filtered top-k path needs a B200")
        torch.cuda.init()
        if l.fb_device_ok() != 1:
            raise NativeUnavailable(l.fb_last_error().decode())
        l._device_checked = True
    return l


def check(rc: int) -> None:
    """Map a C-ABI status onto the reference exception types."""
    if rc == FB_OK:
        return
    msg = load_library().fb_last_error().decode()
    if rc == FB_ERR_INVALID:
        raise ValueError(msg)
    if rc == FB_ERR_DIM_MISMATCH:
        raise errors.FiltraError(msg)
    if rc == FB_ERR_LENGTH_MISMATCH:
        raise errors.FiltraError(msg)
    if rc == FB_ERR_DEGENERATE:
        raise errors.DegenerateRange(msg)
    if rc == FB_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    if rc == FB_ERR_PARSE:
        raise ValueError(msg)
    raise RuntimeError(f"filtra_b200 error {rc}: {msg}")


def ptr(t) -> int:
    """Raw data pointer of a torch tensor or numpy array (None -> NULL)."""
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        return t.data_ptr()
    return t.ctypes.data


def stream_ptr(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def env_flag(name: str) -> bool:
    return os.environ.get(name, "") not in ("", "0")

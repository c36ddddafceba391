"""Loader and ctypes signatures of the C-ABI library ``_lib/libam_b200.so``.

The library is built in-tree by ``paper_2106_10031_b200.build`` (nvcc, sm_100a).
There is no fallback: if the library or a CUDA device is missing, every entry
point raises ``NativeUnavailable`` (the product path must never silently run
anything else).
"""

from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# AM_LIB_PATH: load an alternative in-tree build (tuning variants, tools/variants.sh)
LIB_PATH = os.environ.get("AM_LIB_PATH") or os.path.join(HERE, "_lib", "libam_b200.so")

STEP_FIELDS = 12
SUB_FIELDS = 6

AM_OK = 0
_ERRORS = {-1: "bad argument", -2: "CUDA error", -3: "capacity", -4: "no CUDA device", -5: "overflow"}


class NativeUnavailable(RuntimeError):
    """The CUDA extension is not built or no B200 is visible."""


class NativeError(RuntimeError):
    pass


class NetDesc(ctypes.Structure):
    _fields_ = [
        ("h_params", ctypes.c_void_p), ("n_params", ctypes.c_int64),
        ("h_steps", ctypes.c_void_p), ("n_steps", ctypes.c_int32),
        ("h_subs", ctypes.c_void_p), ("n_subs", ctypes.c_int32),
        ("n_bits", ctypes.c_int32), ("ensemble", ctypes.c_int32),
    ]


class MarchParams(ctypes.Structure):
    _fields_ = [
        ("bbox_lo", ctypes.c_double * 3), ("bbox_hi", ctypes.c_double * 3),
        ("tol_cell", ctypes.c_double), ("tol_weld", ctypes.c_double),
        ("tol_onplane", ctypes.c_double), ("probe_delta", ctypes.c_double),
        ("max_cells", ctypes.c_int64), ("batch_cells", ctypes.c_int64),
        ("mem_budget", ctypes.c_int64), ("rank", ctypes.c_int32), ("world", ctypes.c_int32),
        ("n_shapes", ctypes.c_int32), ("precision", ctypes.c_int32),
    ]


# name -> (restype, argtypes); every function of include/am_b200.h
P, I64, I32, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double
SIGNATURES = {
    "am_last_error": (ctypes.c_char_p, []),
    "am_device_info": (ctypes.c_int, [ctypes.c_int, P, P, P]),
    "am_engine_create": (ctypes.c_int, [P, P, P, ctypes.c_int, P]),
    "am_engine_destroy": (ctypes.c_int, [P]),
    "am_engine_key_words": (ctypes.c_int, [P]),
    "am_engine_reset": (ctypes.c_int, [P]),
    "am_forward": (ctypes.c_int, [P, P, I64, P, P]),
    "am_affine_maps": (ctypes.c_int, [P, P, I64, P, P, P]),
    "am_seed": (ctypes.c_int, [P, P, I64]),
    "am_dichotomy": (ctypes.c_int, [P, P, P, I64, D, D, ctypes.c_int, P]),
    "am_push_candidates": (ctypes.c_int, [P, P, I64]),
    "am_wave": (ctypes.c_int, [P, P]),
    "am_run": (ctypes.c_int, [P, P]),
    "am_outbox_counts": (ctypes.c_int, [P, P]),
    "am_outbox_take": (ctypes.c_int, [P, P, P]),
    "am_queue_size": (ctypes.c_int, [P, P]),
    "am_result_counts": (ctypes.c_int, [P, P]),
    "am_result_copy": (ctypes.c_int, [P, P, P, P, P, P]),
    "am_result_copy_device": (ctypes.c_int, [P, P, P, P, P, P]),
    "am_stats": (ctypes.c_int, [P, P]),
    "am_set_timing": (ctypes.c_int, [P, ctypes.c_int]),
    "am_bench_fp64_peak": (ctypes.c_int, [ctypes.c_int, P]),
    "am_debug_counters": (ctypes.c_int, [P, P]),
    "am_engine_load_params": (ctypes.c_int, [P, P, ctypes.c_int64]),
    "am_engine_set_shape_params": (ctypes.c_int, [P, P, ctypes.c_int64, P]),
    "am_engine_set_shape": (ctypes.c_int, [P, ctypes.c_int32]),
    "am_forward_shapes": (ctypes.c_int, [P, P, P, ctypes.c_int64, P, P]),
    "am_seed_shapes": (ctypes.c_int, [P, P, P, ctypes.c_int64]),
    "am_dichotomy_shapes": (ctypes.c_int, [P, P, P, P, ctypes.c_int64, ctypes.c_double, ctypes.c_double,
                                           ctypes.c_int, P]),
    "am_trace": (ctypes.c_int, [P, P, ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_int, ctypes.c_double,
                                ctypes.c_double, P, P, P]),
    "am_kernel_times": (ctypes.c_int, [P, P]),
    "am_shard_rows": (ctypes.c_int, [P, ctypes.c_int64]),
    "am_shard_iterate": (ctypes.c_int, [P, ctypes.c_int, ctypes.c_int64, P]),
    "am_shard_pack": (ctypes.c_int, [P, P, ctypes.c_int64]),
    "am_shard_absorb": (ctypes.c_int, [P, P, ctypes.c_int64]),
    "am_shard_stats": (ctypes.c_int, [P, P]),
    "am_unique_planes": (ctypes.c_int, [P, ctypes.c_int64, ctypes.c_double, P, ctypes.c_int64, P, P]),
    "am_weld": (ctypes.c_int, [P, ctypes.c_int64, P, P, ctypes.c_int64, ctypes.c_double, P, P, P, P, P, P, P]),
}

_lib = None


def load(require: bool = True):
    """Load the library (no device needed to load; calls need a GPU)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        if require:
            raise NativeUnavailable(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
        return None
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int, what: str):
    if rc != AM_OK:
        msg = _lib.am_last_error().decode(errors="replace") if _lib is not None else ""
        kind = _ERRORS.get(rc, f"error {rc}")
        if rc == -4:
            raise NativeUnavailable(f"{what}: {kind}: {msg}")
        raise NativeError(f"{what}: {kind}: {msg}")

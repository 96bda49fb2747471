"""ctypes binding of libdmqr_b200.so (include/dmqr_b200.h).

This is the binding INTEGRATION.md shows a reference maintainer adding.  The
library is required: there is no CPU fallback, and importing the product API
on a machine without the built .so or without a CUDA device fails loudly.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libdmqr_b200.so"
if os.environ.get("DMQR_LIB_PATH"):  # A/B builds (tools/); the product loads the in-tree library
    LIB_PATH = Path(os.environ["DMQR_LIB_PATH"]).resolve()

EXPORTS = (
    "dmqr_workspace_bytes",
    "dmqr_qrdm_f64",
    "dmqr_qrdm_stream_f64",
    "dmqr_qrp_f64",
    "dmqr_qrp_stream_f64",
    "dmqr_qrdm_batched_f64",
    "dmqr_batched_workspace_bytes",
    "dmqr_batched_group",
    "dmqr_form_q_f64",
    "dmqr_form_q_workspace_bytes",
    "dmqr_check_finite_f64",
    "dmqr_jacobi_svd_batched_f64",
    "dmqr_strerror",
    "dmqr_version",
    "dmqr_debug_ctl",
    "dmqr_stats_enable",
    "dmqr_stats_get",
    "dmqr_debug_panel_clocks",
    "dmqr_debug_timeline",
    "dmqr_release_resources",
    "dmqr_debug_small_clocks",
)

DMQR_OK, DMQR_EINVAL, DMQR_ENONFINITE, DMQR_EZEROCOL, DMQR_ECUDA, DMQR_ECAP = 0, -1, -2, -3, -4, -5


class Params(C.Structure):
    _fields_ = [
        ("tau", C.c_double),
        ("delta", C.c_double),
        ("epsilon", C.c_double),
        ("k_dm", C.c_int32),
        ("use_delta_max", C.c_int32),
        ("stop_rule", C.c_int32),
        ("break_check", C.c_int32),
        ("trace_norms", C.c_int32),
        ("max_steps", C.c_int32),
    ]


class Step(C.Structure):
    _fields_ = [
        ("n_s", C.c_int64),
        ("k_selected", C.c_int64),
        ("k_accepted", C.c_int64),
        ("k_max", C.c_int64),
        ("broke_early", C.c_int32),
        ("fell_back_to_scalar", C.c_int32),
        ("eps_s", C.c_double),
        ("gamma", C.c_double),
    ]


class Info(C.Structure):
    _fields_ = [
        ("rank", C.c_int64),
        ("n_factored", C.c_int64),
        ("n_steps", C.c_int64),
        ("n_swaps", C.c_int64),
        ("stopped_early", C.c_int32),
        ("status", C.c_int32),
        ("a_max0", C.c_double),
    ]


class Stats(C.Structure):
    _fields_ = [
        ("kernel_launches", C.c_int64),
        ("calls", C.c_int64),
        ("timed_steps", C.c_int64),
        ("ms_select", C.c_double),
        ("ms_panel", C.c_double),
        ("ms_trailing", C.c_double),
        ("ms_norms", C.c_double),
        ("ms_pivot", C.c_double),
    ]


STEP_BYTES = C.sizeof(Step)  # 56
INFO_BYTES = C.sizeof(Info)

_lib = None


def load() -> C.CDLL:
    """Load the library (no compute); raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise RuntimeError(
            f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`"
        )
    lib = C.CDLL(str(LIB_PATH))
    P, I64, I32, D, SZ, VP = C.c_void_p, C.c_int64, C.c_int32, C.c_double, C.c_size_t, C.c_void_p
    lib.dmqr_workspace_bytes.argtypes = [I64, I64, C.POINTER(Params)]
    lib.dmqr_workspace_bytes.restype = SZ
    lib.dmqr_qrdm_f64.argtypes = [P, I64, I64, I64, C.POINTER(Params), P, P, P, I64, P, I64, P, P, SZ,
                                  C.POINTER(Info), VP]
    lib.dmqr_qrdm_f64.restype = C.c_int
    lib.dmqr_qrdm_stream_f64.argtypes = [P, I64, I64, I64, C.POINTER(Params), P, P, P, I64, P, I64, P, P, SZ,
                                         C.POINTER(Info), P, I64, VP]
    lib.dmqr_qrdm_stream_f64.restype = C.c_int
    lib.dmqr_qrp_f64.argtypes = lib.dmqr_qrdm_f64.argtypes
    lib.dmqr_qrp_f64.restype = C.c_int
    lib.dmqr_qrp_stream_f64.argtypes = lib.dmqr_qrdm_stream_f64.argtypes
    lib.dmqr_qrp_stream_f64.restype = C.c_int
    lib.dmqr_qrdm_batched_f64.argtypes = [P, I64, I64, I64, I64, I64, C.POINTER(Params), P, P, P, I64, P, I64,
                                          P, I32, P, SZ, VP]
    lib.dmqr_qrdm_batched_f64.restype = C.c_int
    lib.dmqr_batched_workspace_bytes.argtypes = [I64, I64, C.POINTER(Params), I32]
    lib.dmqr_batched_workspace_bytes.restype = SZ
    lib.dmqr_batched_group.argtypes = [I64, I64]
    lib.dmqr_batched_group.restype = I32
    lib.dmqr_form_q_f64.argtypes = [P, I64, I64, I64, P, I64, P, I64, I64, P, SZ, VP]
    lib.dmqr_form_q_f64.restype = C.c_int
    lib.dmqr_form_q_workspace_bytes.argtypes = [I64, I64]
    lib.dmqr_form_q_workspace_bytes.restype = SZ
    lib.dmqr_jacobi_svd_batched_f64.argtypes = [P, I64, I64, I64, I64, I64, D, I32, P, P, P, VP]
    lib.dmqr_jacobi_svd_batched_f64.restype = C.c_int
    lib.dmqr_check_finite_f64.argtypes = [P, I64, I64, I64, P, VP]
    lib.dmqr_check_finite_f64.restype = C.c_int
    lib.dmqr_strerror.argtypes = [C.c_int]
    lib.dmqr_strerror.restype = C.c_char_p
    lib.dmqr_debug_ctl.argtypes = [P, P, VP]
    lib.dmqr_debug_ctl.restype = C.c_int
    lib.dmqr_stats_enable.argtypes = [C.c_int32]
    lib.dmqr_stats_enable.restype = None
    lib.dmqr_stats_get.argtypes = [C.POINTER(Stats), C.c_int32]
    lib.dmqr_stats_get.restype = None
    lib.dmqr_debug_panel_clocks.argtypes = [P, I64, I64, P]
    lib.dmqr_debug_panel_clocks.restype = C.c_int
    lib.dmqr_debug_timeline.argtypes = [P, I64, I64, P]
    lib.dmqr_debug_timeline.restype = C.c_int
    lib.dmqr_debug_small_clocks.argtypes = [P]
    lib.dmqr_debug_small_clocks.restype = C.c_int
    lib.dmqr_release_resources.argtypes = []
    lib.dmqr_release_resources.restype = None
    lib.dmqr_version.argtypes = []
    lib.dmqr_version.restype = C.c_char_p
    _lib = lib
    return lib


def stats(reset: bool = False) -> dict:
    st = Stats()
    load().dmqr_stats_get(C.byref(st), int(reset))
    return {k: getattr(st, k) for k, _ in Stats._fields_}


def strerror(code: int) -> str:
    return load().dmqr_strerror(code).decode()

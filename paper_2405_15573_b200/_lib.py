"""ctypes binding of the C ABI declared in include/uhmv.h (libuhmv.so, sm_100a).

The product path has no CPU fallback: if the shared library is missing or cannot be
loaded, every entry point raises.  Build it with ``python -c "import __graft_entry__ as g;
g.build()"`` (nvcc -gencode arch=compute_100a,code=sm_100a).
"""

from __future__ import annotations

import ctypes
import os

__all__ = ["lib", "UhmvProgram", "UhmvDesc", "UhmvPeerRank", "check", "LIB_PATH", "MAX_PHASES"]

LIB_PATH = os.environ.get("UHMV_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "_build", "libuhmv.so")
MAX_PHASES = 8
ABI_VERSION = 13
MODE_PHASED, MODE_FUSED, MODE_BULK = 0, 1, 2


class UhmvProgram(ctypes.Structure):
    _fields_ = [
        ("n_ops", ctypes.c_int32),
        ("ops", ctypes.c_void_p),
        ("segs", ctypes.c_void_p),
        ("runs", ctypes.c_void_p),
        ("waits", ctypes.c_void_p),
        ("sigs", ctypes.c_void_p),
        ("fused_order", ctypes.c_void_p),
        ("pieces", ctypes.c_void_p),
        ("n_phases", ctypes.c_int32),
        ("phase_lo", ctypes.c_int32 * MAX_PHASES),
        ("phase_hi", ctypes.c_int32 * MAX_PHASES),
        ("in_max", ctypes.c_int32),
        ("out_max", ctypes.c_int32),
        ("n_counters", ctypes.c_int32),
        ("xin_max", ctypes.c_int32),
        ("zero_output", ctypes.c_int32),
        ("stage_elems", ctypes.c_int32),
        ("mr_segs", ctypes.c_void_p),
        ("mr_ranges", ctypes.c_void_p),
        ("n_tmaps", ctypes.c_int32),
        ("tmap_lds", ctypes.c_void_p),
        ("tmaps", ctypes.c_void_p),
        ("flags", ctypes.c_int32),
    ]


PROG_SYM = 1  # uhmv_program.flags: symmetric single-triangle program (bulk engine only)
PROG_WORDER = 4  # uhmv_program.flags: ordered output (NEAR stores, FAR waits and adds; no memset, no atomics)
PROG_XWIN = 2  # uhmv_program.flags: windowed-input ops (H-format FAR; bulk engine only)


class UhmvDesc(ctypes.Structure):
    _fields_ = [
        ("abi_version", ctypes.c_int32),
        ("device", ctypes.c_int32),
        ("n_rows", ctypes.c_int64),
        ("n_cols", ctypes.c_int64),
        ("arena", ctypes.c_void_p),
        ("arena_len", ctypes.c_int64),
        ("work", ctypes.c_void_p),
        ("work_len", ctypes.c_int64),
        ("counters", ctypes.c_void_p),
        ("ticket", ctypes.c_void_p),
        ("exit_count", ctypes.c_void_p),
        ("x_scratch", ctypes.c_void_p),
        ("w_scratch", ctypes.c_void_p),
        ("fwd", UhmvProgram),
        ("adj", UhmvProgram),
    ]


class UhmvPeerRank(ctypes.Structure):
    _fields_ = [
        ("work", ctypes.c_void_p),
        ("work_len", ctypes.c_int64),
        ("counters", ctypes.c_void_p),
        ("done", ctypes.c_void_p),
    ]


_lib = None

EXPORTS = (
    "uhmv_abi_version",
    "uhmv_plan_create",
    "uhmv_execute",
    "uhmv_execute_phases",
    "uhmv_matvec_host",
    "uhmv_execute_mrhs",
    "uhmv_matmat_host",
    "uhmv_execute_peer",
    "uhmv_peer_set_diag",
    "uhmv_plan_set_io",
    "uhmv_plan_set_host_path",
    "uhmv_plan_last_host_path",
    "uhmv_host_pinned",
    "uhmv_plan_info",
    "uhmv_plan_set_profile",
    "uhmv_plan_set_trace",
    "uhmv_dmma_peak",
    "uhmv_plan_destroy",
    "uhmv_last_error",
)


def lib():
    """Load libuhmv.so once; raise (never fall back) when it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"uniform-H CUDA library not built: {LIB_PATH} is missing "
            "(run __graft_entry__.build()); there is no CPU fallback"
        )
    L = ctypes.CDLL(LIB_PATH)
    missing = [name for name in EXPORTS if not hasattr(L, name)]
    if missing:  # a stale build: ensure_built() rebuilds on RuntimeError
        raise RuntimeError(f"libuhmv.so lacks {missing}; rebuild")
    vp, i32 = ctypes.c_void_p, ctypes.c_int
    L.uhmv_abi_version.restype = i32
    L.uhmv_plan_create.argtypes = [ctypes.POINTER(UhmvDesc), ctypes.POINTER(vp)]
    L.uhmv_plan_create.restype = i32
    L.uhmv_execute.argtypes = [vp, vp, vp, i32, i32, vp]
    L.uhmv_execute.restype = i32
    L.uhmv_execute_phases.argtypes = [vp, vp, vp, i32, i32, i32, vp]
    L.uhmv_execute_phases.restype = i32
    L.uhmv_matvec_host.argtypes = [vp, vp, vp, i32, i32, vp]
    L.uhmv_execute_mrhs.argtypes = [vp, vp, vp, vp, i32, i32, vp]
    L.uhmv_execute_mrhs.restype = i32
    L.uhmv_matmat_host.argtypes = [vp, vp, vp, i32, vp, vp, vp, i32, i32, vp]
    L.uhmv_matmat_host.restype = i32
    L.uhmv_execute_peer.argtypes = [vp, i32, i32, i32, ctypes.POINTER(UhmvPeerRank), vp, vp, i32, ctypes.c_uint32, vp]
    L.uhmv_execute_peer.restype = i32
    L.uhmv_peer_set_diag.argtypes = [vp, i32]
    L.uhmv_peer_set_diag.restype = i32
    L.uhmv_plan_set_io.argtypes = [vp, ctypes.POINTER(UhmvProgram), ctypes.POINTER(UhmvProgram), vp]
    L.uhmv_plan_set_io.restype = i32
    L.uhmv_matvec_host.restype = i32
    L.uhmv_plan_set_host_path.argtypes = [vp, i32, i32]
    L.uhmv_plan_set_host_path.restype = i32
    L.uhmv_plan_last_host_path.argtypes = [vp, i32]
    L.uhmv_plan_last_host_path.restype = i32
    L.uhmv_host_pinned.argtypes = [vp]
    L.uhmv_host_pinned.restype = i32
    pi = ctypes.POINTER(i32)
    L.uhmv_plan_info.argtypes = [vp, i32, i32, pi, pi, pi, pi]
    L.uhmv_plan_info.restype = i32
    L.uhmv_dmma_peak.argtypes = [i32, ctypes.POINTER(ctypes.c_double)]
    L.uhmv_dmma_peak.restype = i32
    L.uhmv_plan_set_profile.argtypes = [vp, vp]
    L.uhmv_plan_set_profile.restype = i32
    L.uhmv_plan_set_trace.argtypes = [vp, vp]
    L.uhmv_plan_set_trace.restype = i32
    L.uhmv_plan_destroy.argtypes = [vp]
    L.uhmv_plan_destroy.restype = i32
    L.uhmv_last_error.restype = ctypes.c_char_p
    if L.uhmv_abi_version() != ABI_VERSION:
        raise RuntimeError("libuhmv.so ABI version mismatch; rebuild")
    _lib = L
    return L


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = lib().uhmv_last_error().decode(errors="replace")
        raise RuntimeError(f"{what} failed ({rc}): {msg}")

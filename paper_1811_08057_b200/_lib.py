"""ctypes binding of libmcnd_b200.so (include/mcnd_b200.h).

There is no CPU fallback: if the library is missing or no CUDA device is
usable, every entry point raises.  The reference (`mcnd`) has no FFI; this is
the binding its Python callers get.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .build import LIB

MCND_OK = 0
MCND_EINVAL = 1
MCND_ECUDA = 2
MCND_ENCCL = 3
MCND_EDEVICE = 4
MCND_EPIVOT = 5
MCND_EPIVOT_SHORT = 6
FLAG_FAST = 1
FLAG_GROUPS = 2


class McndLogDet(ctypes.Structure):
    _fields_ = [("sign", ctypes.c_int32), ("singular", ctypes.c_int32), ("log_abs", ctypes.c_double),
                ("singular_step", ctypes.c_int64), ("invalid_step", ctypes.c_int64),
                ("invalid_row", ctypes.c_int64), ("device_ms", ctypes.c_double), ("steps", ctypes.c_int64),
                ("launches", ctypes.c_int64), ("torn_reads", ctypes.c_int64)]


class McndCommStats(ctypes.Structure):
    _fields_ = [("broadcasts", ctypes.c_int64), ("broadcast_bytes", ctypes.c_int64),
                ("pivot_search_msgs", ctypes.c_int64), ("scalar_updates", ctypes.c_int64),
                ("aborted_step", ctypes.c_int64), ("scatter_seconds", ctypes.c_double),
                ("comm_seconds", ctypes.c_double)]


# host-transport callbacks of the native multi-GPU driver (mcnd_mg_attach_host)
HOST_BCAST = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32)
HOST_ALLGATHER = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64)

_lock = threading.Lock()
LAST_LAUNCHES = 0  # GPU kernels launched by the most recent single-matrix call (bench accounting)
LAST_TORN_READS = 0  # panel records the most recent blocked call saw half-written (re-polled)
_lib = None

EXPORTS = (
    "mcnd_logdet_condensation_dev", "mcnd_logdet_condensation",
    "mcnd_mc_parallel_dev", "mcnd_mc_parallel",
    "mcnd_logdet_batched_dev", "mcnd_logdet_batched", "mcnd_fold_mc_parallel",
    "mcnd_dist_ipc_handle_bytes", "mcnd_dist_create", "mcnd_dist_connect", "mcnd_dist_mc_parallel",
    "mcnd_dist_destroy",
    "mcnd_last_error", "mcnd_version", "mcnd_k1_grid", "mcnd_release_workspace",
    "mcnd_logdet_blocked_dev", "mcnd_logdet_blocked", "mcnd_blocked_panel",
    "mcnd_mg_create", "mcnd_mg_load", "mcnd_mg_pair", "mcnd_mg_trailing", "mcnd_mg_export", "mcnd_mg_tail",
    "mcnd_mg_records", "mcnd_mg_gather_bytes", "mcnd_mg_ld", "mcnd_mg_destroy",
    "mcnd_nccl_id_bytes", "mcnd_nccl_unique_id", "mcnd_mg_attach", "mcnd_mg_logdet", "mcnd_mg_schedule",
    "mcnd_logdet_lu_dev", "mcnd_logdet_lu", "mcnd_mg_attach_host",
)


def load(path: str | None = None):
    """Load (never build) the shared library and declare its signatures."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = path or LIB
        if not os.path.exists(path):
            raise RuntimeError(
                f"libmcnd_b200.so not found at {path}: run __graft_entry__.build() "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(path)
        P, i64, i32, u32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint32
        LD = ctypes.POINTER(McndLogDet)
        CS = ctypes.POINTER(McndCommStats)
        for name in ("mcnd_logdet_condensation_dev", "mcnd_logdet_condensation"):
            f = getattr(lib, name)
            f.argtypes = [P, i64, i64, P, i64, u32, P, LD, P, P]
            f.restype = ctypes.c_int
        for name in ("mcnd_mc_parallel_dev", "mcnd_mc_parallel"):
            f = getattr(lib, name)
            f.argtypes = [P, i64, i64, i32, u32, P, LD, CS, P, P, P]
            f.restype = ctypes.c_int
        lib.mcnd_logdet_batched_dev.argtypes = [P, i64, i64, i64, u32, P, P, P, P, P]
        lib.mcnd_logdet_batched_dev.restype = ctypes.c_int
        lib.mcnd_logdet_batched.argtypes = [P, i64, i64, i64, u32, P, P, P]
        lib.mcnd_logdet_batched.restype = ctypes.c_int
        lib.mcnd_fold_mc_parallel.argtypes = [i64, i32, P, P, i64, P, P, LD, CS, P, P]
        lib.mcnd_fold_mc_parallel.restype = ctypes.c_int
        lib.mcnd_dist_ipc_handle_bytes.argtypes = []
        lib.mcnd_dist_ipc_handle_bytes.restype = ctypes.c_int32
        lib.mcnd_dist_create.argtypes = [i32, i32, i64, ctypes.POINTER(ctypes.c_void_p), P]
        lib.mcnd_dist_create.restype = ctypes.c_int
        lib.mcnd_dist_connect.argtypes = [P, P]
        lib.mcnd_dist_connect.restype = ctypes.c_int
        lib.mcnd_dist_mc_parallel.argtypes = [P, P, i64, i64, u32, P, P, P, P, P, P, P]
        lib.mcnd_dist_mc_parallel.restype = ctypes.c_int
        lib.mcnd_dist_destroy.argtypes = [P]
        lib.mcnd_dist_destroy.restype = None
        for name in ("mcnd_logdet_blocked_dev", "mcnd_logdet_blocked"):
            f = getattr(lib, name)
            f.argtypes = [P, i64, i64, u32, P, LD, P, P]
            f.restype = ctypes.c_int
        lib.mcnd_blocked_panel.restype = ctypes.c_int32
        for name in ("mcnd_logdet_lu_dev", "mcnd_logdet_lu"):
            f = getattr(lib, name)
            f.argtypes = [P, i64, i64, P, u32, P, LD, P, P]
            f.restype = ctypes.c_int
        VP = ctypes.POINTER(ctypes.c_void_p)
        sigs = {
            "mcnd_mg_create": [i64, i64, VP],
            "mcnd_mg_load": [P, P, i64, P],
            "mcnd_mg_pair": [P, i64, i64, i64, P, i64, P, P, P],
            "mcnd_mg_trailing": [P, i64, i64, i64, P, i64, P, P, i32, i32, P],
            "mcnd_mg_export": [P, i64, i64, i64, P, i64, P, P],
            "mcnd_mg_tail": [P, P, i64, P, i64, P, P, P],
            "mcnd_mg_records": [P, P, P, P],
            "mcnd_mg_destroy": [P],
        }
        for name, args in sigs.items():
            f = getattr(lib, name)
            f.argtypes = args
            f.restype = ctypes.c_int
        lib.mcnd_nccl_id_bytes.argtypes = []
        lib.mcnd_nccl_id_bytes.restype = ctypes.c_int32
        lib.mcnd_nccl_unique_id.argtypes = [P]
        lib.mcnd_nccl_unique_id.restype = ctypes.c_int
        lib.mcnd_mg_attach.argtypes = [P, i32, i32, P, i32]
        lib.mcnd_mg_attach.restype = ctypes.c_int
        lib.mcnd_mg_attach_host.argtypes = [P, i32, i32, HOST_BCAST, HOST_ALLGATHER]
        lib.mcnd_mg_attach_host.restype = ctypes.c_int
        lib.mcnd_mg_logdet.argtypes = [P, P, i64, i64, P, LD]
        lib.mcnd_mg_logdet.restype = ctypes.c_int
        lib.mcnd_mg_schedule.argtypes = [i64, i32, i64, P, i64]
        lib.mcnd_mg_schedule.restype = ctypes.c_int64
        lib.mcnd_mg_gather_bytes.argtypes = []
        lib.mcnd_mg_gather_bytes.restype = ctypes.c_int64
        lib.mcnd_mg_ld.argtypes = [P]
        lib.mcnd_mg_ld.restype = ctypes.c_int64
        lib.mcnd_last_error.argtypes = []
        lib.mcnd_last_error.restype = ctypes.c_char_p
        lib.mcnd_version.restype = ctypes.c_int32
        lib.mcnd_k1_grid.restype = ctypes.c_int32
        lib.mcnd_release_workspace.restype = None
        _lib = lib
        return lib


def last_error() -> str:
    return load().mcnd_last_error().decode(errors="replace")


def check(rc: int) -> None:
    if rc == MCND_OK:
        return
    msg = last_error()
    if rc in (MCND_EINVAL, MCND_EPIVOT):
        raise ValueError(msg)
    if rc == MCND_EPIVOT_SHORT:
        raise IndexError(msg)
    raise RuntimeError(f"mcnd_b200 error {rc}: {msg}")

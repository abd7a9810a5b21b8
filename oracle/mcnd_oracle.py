"""ORACLE -- test infrastructure only (tests/, __graft_entry__.smoke(), bench.py's
CPU-baseline leg).  Never imported by the product package.

ctypes front end of oracle/mcnd_oracle.c, the plain-C restatement of the
reference CPU path (mcnd/condense.py:82-160, mcnd/runtime.py:123-229,
mcnd/gauss.py:16-68).  Parity of this restatement with the reference itself
is pinned by tests/test_oracle_golden.py against tests/golden/cases/*.json,
which tests/golden/make_golden.py produced by running the reference.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from typing import NamedTuple, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "liboracle.so")

_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def _load():
    global _lib
    if _lib is not None:
        return _lib
    src = os.path.join(HERE, "mcnd_oracle.c")
    if not os.path.exists(LIB_PATH) or os.path.getmtime(src) > os.path.getmtime(LIB_PATH):
        build()
    lib = ctypes.CDLL(LIB_PATH)
    P = ctypes.c_void_p
    i64, i32 = ctypes.c_int64, ctypes.c_int
    lib.oracle_logdet_condensation.argtypes = [P, i64, P, i32, P, P, P, P, P, P]
    lib.oracle_logdet_lu.argtypes = [P, i64, P, P, P]
    lib.oracle_mc_parallel.argtypes = [P, i64, i64, i32, P, P, P, P, P, P, P, P, P, P, i64]
    lib.oracle_logdet_batched.argtypes = [P, i64, i64, i32, P, P]
    lib.oracle_condense_steps.argtypes = [P, i64, P, i32, P, P, P, P, P, P, i64]
    lib.oracle_condense_steps.restype = ctypes.c_int
    for f in (lib.oracle_logdet_condensation, lib.oracle_logdet_lu, lib.oracle_mc_parallel,
              lib.oracle_logdet_batched):
        f.restype = ctypes.c_int
    _lib = lib
    return lib


def _ptr(x):
    return ctypes.c_void_p(x.ctypes.data) if x is not None else None


class OracleResult(NamedTuple):
    sign: int
    log_abs: float
    pivots: np.ndarray       # per-step pivot values (n entries, last = final 1x1)
    cols: np.ndarray         # per-step pivot columns
    singular_step: int


def logdet_condensation(a, pivot_sequence: Optional[Sequence[int]] = None, threads: int = 0) -> OracleResult:
    lib = _load()
    a = np.ascontiguousarray(a, dtype=np.float64)
    n = a.shape[0]
    seq = None
    if pivot_sequence is not None:
        seq = np.ascontiguousarray(np.asarray(pivot_sequence, dtype=np.int64)[: n - 1])
        if seq.shape[0] < n - 1:
            raise IndexError("pivot_sequence shorter than n-1")
    sign = ctypes.c_int32()
    la = ctypes.c_double()
    piv = np.zeros(n, dtype=np.float64)
    cols = np.zeros(n, dtype=np.int32)
    ss = ctypes.c_int64()
    bad = ctypes.c_int64()
    rc = lib.oracle_logdet_condensation(_ptr(a), n, _ptr(seq), threads, ctypes.byref(sign),
                                        ctypes.byref(la), _ptr(piv), _ptr(cols), ctypes.byref(ss),
                                        ctypes.byref(bad))
    if rc == 2:
        raise ValueError(f"row {int(seq[bad.value])} is not active")
    if rc:
        raise MemoryError("oracle allocation failed")
    return OracleResult(int(sign.value), float(la.value), piv, cols, int(ss.value))


def condense_prefix(a, steps: int, threads: int = 0):
    """Run only the first `steps` condensation steps (bounded CPU-baseline sample)."""
    lib = _load()
    a = np.ascontiguousarray(a, dtype=np.float64)
    sign = ctypes.c_int32()
    la = ctypes.c_double()
    ss = ctypes.c_int64()
    bad = ctypes.c_int64()
    lib.oracle_condense_steps(_ptr(a), a.shape[0], None, threads, ctypes.byref(sign), ctypes.byref(la),
                              None, None, ctypes.byref(ss), ctypes.byref(bad), int(steps))
    return int(sign.value), float(la.value)


def logdet_lu(a, row_witness=None):
    lib = _load()
    a = np.ascontiguousarray(a, dtype=np.float64)
    w = None if row_witness is None else np.ascontiguousarray(row_witness, dtype=np.float64)
    sign = ctypes.c_int32()
    la = ctypes.c_double()
    lib.oracle_logdet_lu(_ptr(a), a.shape[0], _ptr(w), ctypes.byref(sign), ctypes.byref(la))
    return int(sign.value), float(la.value)


class OracleParallel(NamedTuple):
    sign: int
    log_abs: float
    broadcasts: int
    broadcast_bytes: int
    scalar_updates: int
    aborted_step: int
    payload_entries: list
    row_updates: list
    owners: np.ndarray
    pivots: np.ndarray
    cols: np.ndarray
    rem: np.ndarray          # p x p remainder (row w = worker w's last live row)
    rem_wit: np.ndarray      # its witnesses


def mc_parallel(a, p: int, threads: int = 0, max_steps: int | None = None) -> OracleParallel:
    """runtime.py:123-229; max_steps bounds the number of broadcast steps (a prefix of the
    workload for the CPU-baseline timing; the result is then the partial accumulators)."""
    lib = _load()
    a = np.ascontiguousarray(a, dtype=np.float64)
    n = a.shape[0]
    if p < 1 or p > n:
        raise ValueError(f"invalid plan: need 1 <= p <= n, got p={p}, n={n}")
    sign = ctypes.c_int32()
    la = ctypes.c_double()
    stats = np.zeros(4, dtype=np.int64)
    payload = np.zeros(max(n - p, 1), dtype=np.int64)
    rows = np.zeros(p, dtype=np.int64)
    owners = np.full(max(n - p + 1, 1), -1, dtype=np.int64)
    piv = np.zeros(max(n - p + 1, 1), dtype=np.float64)
    cols = np.zeros(max(n - p + 1, 1), dtype=np.int32)
    rem = np.zeros((p, p), dtype=np.float64)
    rem_wit = np.zeros(p, dtype=np.float64)
    lib.oracle_mc_parallel(_ptr(a), n, p, threads, ctypes.byref(sign), ctypes.byref(la), _ptr(stats),
                           _ptr(payload), _ptr(rows), _ptr(owners), _ptr(piv), _ptr(cols), _ptr(rem),
                           _ptr(rem_wit), ctypes.c_int64(n if max_steps is None else int(max_steps)))
    aborted = int(stats[3])
    n_bcast_payload = (aborted if aborted >= 0 else n - p)
    return OracleParallel(int(sign.value), float(la.value), int(stats[0]), int(stats[1]),
                          int(stats[2]), aborted, [int(x) for x in payload[:n_bcast_payload]],
                          [int(x) for x in rows], owners, piv, cols, rem, rem_wit)


def logdet_batched(a3, threads: int = 0):
    lib = _load()
    a3 = np.ascontiguousarray(a3, dtype=np.float64)
    b, n, _ = a3.shape
    signs = np.zeros(b, dtype=np.int32)
    logs = np.zeros(b, dtype=np.float64)
    lib.oracle_logdet_batched(_ptr(a3), b, n, threads if threads > 0 else (os.cpu_count() or 1),
                              _ptr(signs), _ptr(logs))
    return signs, logs


def tolerance(n: int, ref_log: float) -> float:
    """north_star tolerance: |d log| <= max(1e-8*N, 1e-10*|log|)."""
    if math.isinf(ref_log):
        return 0.0
    return max(1e-8 * n, 1e-10 * abs(ref_log))

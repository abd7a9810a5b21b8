"""Drop-in for mcnd.gauss / the GE half of mcnd.runtime: Gaussian elimination with row
pivoting on the GPU -- the paper's comparison baseline (SURVEY.md §8(f)
rank 3).

* ``logdet_lu(a, row_witness=None) -> LogDet`` (gauss.py:34-68): column k's pivot is the
  max-|a[r, k]| unprocessed row (ties -> lowest row), rows never move, the pivot
  permutation's parity goes into the sign; singular = an exactly zero pivot, or
  |pivot| <= 1e-12 * row_witness[row] when a witness is given.
* ``ge_parallel(a, p) -> RunResult`` (runtime.py:232-321): rows dealt cyclically (row i on
  worker i mod p), a global pivot search per column (2(p-1) messages when p > 1), the pivot
  row broadcast (n-k-1 entries + 1 word), per-worker log sums reduced in rank order.

Both run csrc/k1_condense.cu in GE mode on A^T (mcnd_logdet_lu*): pivots, log|det| and sign
are bitwise the reference's.  ge_parallel's arithmetic is serial GE's (the global pivot and
the updates are the same), so one elimination on the device gives every worker's pivots;
its log|det| sums them per owner like runtime.py:296, and the accounting is the reference's
_Fabric law (runtime.py:82-104) replayed from the pivot rows.
"""

from __future__ import annotations

import ctypes
import time

import numpy as np

from . import _lib
from .condense import SINGULAR, LogDet, _is_torch_cuda, _torch_device_args
from .matrix import square_for_device
from .runtime import CommStats, RunResult


def _ge(a, row_witness=None, fast: bool = False):
    """(LogDet, device_ms, pivot values, pivot rows, steps published)."""
    lib = _lib.load()
    out = _lib.McndLogDet()
    flags = _lib.FLAG_FAST if fast else 0
    if _is_torch_cuda(a):
        import torch

        keep, ptr, n, ld, stream = _torch_device_args(a)
        w = None
        if row_witness is not None:
            w = torch.as_tensor(np.ascontiguousarray(row_witness, dtype=np.float64)).to(keep.device)
        piv = np.zeros(n, dtype=np.float64)
        rows = np.full(n, -1, dtype=np.int32)
        rc = lib.mcnd_logdet_lu_dev(ptr, n, ld, None if w is None else w.data_ptr(), flags, stream,
                                    ctypes.byref(out), piv.ctypes.data, rows.ctypes.data)
        del keep, w
    else:
        a = square_for_device(a)
        n = a.shape[0]
        w = None if row_witness is None else np.ascontiguousarray(row_witness, dtype=np.float64)
        if w is not None and w.shape != (n,):
            raise ValueError(f"row_witness must have {n} entries, got shape {w.shape}")
        piv = np.zeros(n, dtype=np.float64)
        rows = np.full(n, -1, dtype=np.int32)
        rc = lib.mcnd_logdet_lu(a.ctypes.data, n, n, None if w is None else w.ctypes.data, flags, None,
                                ctypes.byref(out), piv.ctypes.data, rows.ctypes.data)
    _lib.check(rc)
    _lib.LAST_LAUNCHES = int(out.launches)
    res = SINGULAR if out.singular else LogDet(int(out.sign), float(out.log_abs))
    k = int(out.singular_step) + 1 if out.singular else n
    return res, float(out.device_ms), piv[:k], rows[:k]


def logdet_lu(a, row_witness=None, *, fast: bool = False, return_pivots: bool = False):
    """gauss.py:34-68 on the GPU (see the module docstring)."""
    res, ms, piv, rows = _ge(a, row_witness, fast)
    if return_pivots:
        return res, piv, rows, ms
    return res


def ge_parallel(a, p: int, *, fast: bool = False) -> RunResult:
    """runtime.py:232-321: cyclic-distributed Gaussian elimination with partial pivoting."""
    import math

    shape = tuple(getattr(a, "shape", ()))
    if len(shape) == 2 and not (1 <= p <= shape[0]):
        raise ValueError(f"invalid worker count: need 1 <= p <= n, got p={p}")
    t0 = time.perf_counter()
    res, ms, piv, rows = _ge(a, None, fast)
    n = shape[0] if len(shape) == 2 else len(rows)
    stats = CommStats(compute_seconds=ms / 1e3)
    remaining = [len(range(w, n, p)) for w in range(p)]  # unprocessed rows per worker
    local_logs = [0.0] * p
    row_updates = [0] * p
    payload = []
    scalar_updates = 0
    singular = res.sign == 0
    for k in range(len(rows)):
        if p > 1:
            stats.pivot_search_msgs += 2 * (p - 1)  # candidates in, the winner back (runtime.py:92-104)
        if singular and k == len(rows) - 1:
            break  # the zero pivot: searched, never broadcast (runtime.py:274-276)
        owner = int(rows[k]) % p
        remaining[owner] -= 1
        local_logs[owner] += math.log(abs(float(piv[k])))
        if k == n - 1:
            break
        stats.broadcasts += 1
        stats.broadcast_bytes += 8 * (n - k - 1) + 8  # the pivot row + 1 word (runtime.py:285)
        payload.append(n - k - 1)
        for w in range(p):
            if remaining[w]:
                row_updates[w] += remaining[w]
                scalar_updates += remaining[w] * (n - k - 1)
    if not singular:
        total = 0.0
        for v in local_logs:  # _Fabric.reduce_sum: rank order (runtime.py:114-120)
            total += v
        res = LogDet(res.sign, total)
    return RunResult(logdet=res, stats=stats, n_workers=p, total_seconds=time.perf_counter() - t0,
                     broadcast_payload_entries=payload, row_updates=row_updates, scalar_updates=scalar_updates)

"""Drop-in for mcnd.condense: serial condensation log-determinant on a B200.

Same names, argument meaning, return type and error behaviour as
/root/reference/pkg/src/mcnd/condense.py:24-160:

* ``logdet_condensation(a, pivot_sequence=None) -> LogDet``
  (condense.py:134-160).  Default pivot order is top-to-bottom; a caller
  sequence of original row ids is honoured (condense.py:147-152) and an
  inactive/out-of-range row raises ``ValueError`` (condense.py:85-86), a
  short sequence ``IndexError`` -- but, as in the reference, only if the
  matrix did not turn out singular first.
* singular matrices return ``SINGULAR == LogDet(0, -inf)``, never raise.
* the input is never modified.

The whole O(N^3) loop runs in one persistent sm_100a kernel
(csrc/k1_condense.cu); the host only validates, builds the pivot schedule
and folds the returned N pivots into (sign, log|det|) in reference order, so
the default (parity) mode is bitwise equal to the reference.  ``fast=True``
switches the rank-1 update to FMA (one rounding; differs from numpy in the
last bits, well inside the north_star tolerance).

Accepted inputs: anything ``np.ascontiguousarray(.., float64)`` accepts
(host path: the H2D copy is part of the call), or a float64 CUDA torch tensor
with unit column stride (device path: used in place, no copy).
"""

from __future__ import annotations

import ctypes
import math
from typing import NamedTuple, Optional, Sequence

import numpy as np

from . import _lib
from .matrix import square_for_device

SINGULAR_RTOL = 1e-12  # condense.py:29


class SingularRowError(ArithmeticError):
    """condense.py:32-33 (kept for API parity; the GPU path reports singular
    matrices as SINGULAR, as logdet_condensation does)."""


class LogDet(NamedTuple):
    """Determinant as (sign, ln|det|); sign 0 means singular, log_abs -inf."""

    sign: int
    log_abs: float


SINGULAR = LogDet(0, -math.inf)


def _is_torch_cuda(a) -> bool:
    return type(a).__module__.startswith("torch") and getattr(a, "is_cuda", False)


def _torch_device_args(a):
    """Validate a CUDA torch tensor like require_square and return (ptr, n, ld, stream)."""
    import torch

    if a.dim() != 2:
        raise ValueError(f"matrix must be 2-D, got {a.dim()}-D")
    if a.shape[0] == 0 or a.shape[1] == 0:
        raise ValueError("matrix dimensions must be positive")
    if a.dtype != torch.float64:
        a = a.to(torch.float64)
    if a.stride(1) != 1 or a.stride(0) < a.shape[1]:
        a = a.contiguous()
    if a.shape[0] != a.shape[1]:
        if not bool(torch.isfinite(a).all()):
            raise ValueError("matrix entries must be finite (no NaN/Inf)")
        raise ValueError(f"matrix must be square, got {tuple(a.shape)}")
    # finiteness (matrix.py:39-40) is checked on the device, fused into the copy
    torch.cuda.set_device(a.device)
    stream = torch.cuda.current_stream(a.device).cuda_stream
    return a, a.data_ptr(), a.shape[0], a.stride(0), stream


def _seq_array(pivot_sequence, n):
    if pivot_sequence is None:
        return None, 0
    seq = np.ascontiguousarray([int(x) for x in list(pivot_sequence)[: max(n - 1, 0)]], dtype=np.int64)
    return seq, seq.shape[0]


def logdet_condensation(a, pivot_sequence: Optional[Sequence[int]] = None, *, fast: bool = False,
                        return_pivots: bool = False):
    """Full log-determinant by repeated condensation on the GPU (condense.py:134)."""
    lib = _lib.load()
    out = _lib.McndLogDet()
    flags = _lib.FLAG_FAST if fast else 0
    if _is_torch_cuda(a):
        keep, ptr, n, ld, stream = _torch_device_args(a)
        seq, slen = _seq_array(pivot_sequence, n)
        piv = np.zeros(n, dtype=np.float64)
        cols = np.zeros(n, dtype=np.int32)
        rc = lib.mcnd_logdet_condensation_dev(
            ptr, n, ld, None if seq is None else seq.ctypes.data, slen, flags, stream,
            ctypes.byref(out), piv.ctypes.data, cols.ctypes.data)
        del keep
    else:
        a = square_for_device(a)
        n = a.shape[0]
        seq, slen = _seq_array(pivot_sequence, n)
        piv = np.zeros(n, dtype=np.float64)
        cols = np.zeros(n, dtype=np.int32)
        rc = lib.mcnd_logdet_condensation(
            a.ctypes.data, n, n, None if seq is None else seq.ctypes.data, slen, flags, None,
            ctypes.byref(out), piv.ctypes.data, cols.ctypes.data)
    _lib.check(rc)
    _lib.LAST_LAUNCHES = int(out.launches)
    res = SINGULAR if out.singular else LogDet(int(out.sign), float(out.log_abs))
    if return_pivots:
        steps = int(out.steps)
        k = steps if out.singular else n
        return res, piv[: k + (1 if out.singular else 0)], cols[: k + (1 if out.singular else 0)], float(out.device_ms)
    return res



def _perm_parity(perm) -> int:
    """Parity of a permutation (cycle decomposition, as gauss.py:16-31)."""
    seen = np.zeros(len(perm), dtype=bool)
    par = 1
    for s in range(len(perm)):
        if seen[s]:
            continue
        ln, j = 0, s
        while not seen[j]:
            seen[j] = True
            j = int(perm[j])
            ln += 1
        if ln % 2 == 0:
            par = -par
    return par


def logdet_blocked(a, pivot_sequence: Optional[Sequence[int]] = None, *, fast: bool = False,
                   return_pivots: bool = False):
    """Blocked rank-64 condensation (K2, csrc/k2_blocked.cu): panels of 64 pivot
    rows chosen by the reference's rule, trailing update on FP64 tensor cores.
    Same result type and pivot rule as logdet_condensation; rounding differs from
    the reference, so parity is by tolerance.  Input handling as
    logdet_condensation.

    ``pivot_sequence`` (condense.py:147-152): the rows are taken in that order.  The
    blocked kernels always run top to bottom, so the rows are gathered into that order on
    the device first (the condensation steps only see which row is the pivot, never where
    it sits) and the sign picks up the permutation's parity: det(A) = sgn(P) det(PA).  A
    sequence that names an inactive row, or is too short, goes to logdet_condensation,
    which raises exactly when the reference would (or returns SINGULAR first)."""
    if pivot_sequence is not None:
        n = int(a.shape[0]) if len(getattr(a, "shape", ())) == 2 else None
        seq = [int(x) for x in list(pivot_sequence)[: max((n or 1) - 1, 0)]]
        ok = n is not None and len(seq) >= n - 1 and all(0 <= r < n for r in seq) and len(set(seq)) == len(seq)
        if not ok:
            return logdet_condensation(a, pivot_sequence, fast=fast, return_pivots=return_pivots)
        rest = sorted(set(range(n)) - set(seq))
        perm = np.array(seq + rest, dtype=np.int64)
        if _is_torch_cuda(a):
            import torch

            pa = a.index_select(0, torch.as_tensor(perm, device=a.device))
        else:
            pa = np.ascontiguousarray(np.asarray(a, dtype=np.float64)[perm])
        out = logdet_blocked(pa, fast=fast, return_pivots=return_pivots)
        res = out[0] if return_pivots else out
        if res.sign != 0:
            res = LogDet(res.sign * _perm_parity(perm), res.log_abs)
        return (res,) + tuple(out[1:]) if return_pivots else res
    lib = _lib.load()
    out = _lib.McndLogDet()
    flags = _lib.FLAG_FAST if fast else 0
    if _is_torch_cuda(a):
        keep, ptr, n, ld, stream = _torch_device_args(a)
        piv = np.zeros(n, dtype=np.float64)
        cols = np.zeros(n, dtype=np.int32)
        rc = lib.mcnd_logdet_blocked_dev(ptr, n, ld, flags, stream, ctypes.byref(out), piv.ctypes.data,
                                         cols.ctypes.data)
        del keep
    else:
        a = square_for_device(a)
        n = a.shape[0]
        piv = np.zeros(n, dtype=np.float64)
        cols = np.zeros(n, dtype=np.int32)
        rc = lib.mcnd_logdet_blocked(a.ctypes.data, n, n, flags, None, ctypes.byref(out), piv.ctypes.data,
                                     cols.ctypes.data)
    _lib.check(rc)
    _lib.LAST_LAUNCHES = int(out.launches)
    _lib.LAST_TORN_READS = int(out.torn_reads)
    res = SINGULAR if out.singular else LogDet(int(out.sign), float(out.log_abs))
    if return_pivots:
        k = int(out.steps) + (0 if out.singular else 1)
        return res, piv[:k], cols[:k], float(out.device_ms)
    return res

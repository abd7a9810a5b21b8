"""Drop-in for mcnd.runtime's condensation half: block-row parallel condensation.

Mirrors /root/reference/pkg/src/mcnd/runtime.py:25-66 and :123-229:

* ``plan_blocks(n, p) -> WorkerPlan`` (runtime.py:33-44), same ValueError;
* ``CommStats`` / ``RunResult`` with the same fields (runtime.py:47-66);
* ``mc_parallel(a, p) -> RunResult`` (runtime.py:123): p contiguous row
  blocks, round-robin owners taking their topmost live row, one pivot-row
  "broadcast" per step (N - p of them, zero pivot-search messages), the p x p
  remainder finished by row-pivoted elimination.  The result is bitwise the
  reference's (same pivots, same arithmetic, same log summation order:
  per-worker step-ordered sums, rank-ordered reduce, + the LU tail).

On one GPU the p "workers" are a pivot schedule for the persistent kernel
(the broadcast is the in-kernel pivot-row publication; accounting follows the
reference's _Fabric byte law, runtime.py:82-90).  ``n_workers=`` is accepted
as an alias of ``p`` (README.md:65 uses it).  Across GPUs see
``paper_1811_08057_b200.dist``.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .condense import SINGULAR, LogDet, _is_torch_cuda, _torch_device_args
from .matrix import square_for_device


@dataclass(frozen=True)
class WorkerPlan:
    """Contiguous block row assignment: per-worker (start, length)."""

    n_workers: int
    assignments: tuple[tuple[int, int], ...]


def plan_blocks(n: int, p: int) -> WorkerPlan:
    """runtime.py:33-44: the first n % p workers get one extra row."""
    if p < 1 or p > n:
        raise ValueError(f"invalid plan: need 1 <= p <= n, got p={p}, n={n}")
    base, extra = divmod(n, p)
    out, start = [], 0
    for w in range(p):
        ln = base + (1 if w < extra else 0)
        out.append((start, ln))
        start += ln
    return WorkerPlan(p, tuple(out))


@dataclass
class CommStats:
    broadcasts: int = 0
    broadcast_bytes: int = 0
    pivot_search_msgs: int = 0
    scatter_seconds: float = 0.0
    comm_seconds: float = 0.0
    compute_seconds: float = 0.0


@dataclass
class RunResult:
    logdet: LogDet
    stats: CommStats
    n_workers: int
    total_seconds: float = 0.0
    broadcast_payload_entries: list[int] = field(default_factory=list)
    row_updates: list[int] = field(default_factory=list)
    scalar_updates: int = 0


def mc_parallel(a, p: int | None = None, *, n_workers: int | None = None, fast: bool = False,
                groups: bool = False) -> RunResult:
    """Block-distributed parallel matrix condensation (runtime.py:123-229) on the GPU.

    ``groups=True`` runs the p workers as p CTA groups with private workspaces
    that exchange pivot rows through the multi-GPU push protocol (p <= 8);
    results are identical either way."""
    if p is None:
        p = n_workers
    if p is None:
        raise TypeError("mc_parallel() missing required argument: 'p'")
    p = int(p)
    lib = _lib.load()
    out = _lib.McndLogDet()
    st = _lib.McndCommStats()
    flags = (_lib.FLAG_FAST if fast else 0) | (_lib.FLAG_GROUPS if groups else 0)
    t0 = time.perf_counter()
    if _is_torch_cuda(a):
        keep, ptr, n, ld, stream = _torch_device_args(a)
        fn, args = lib.mcnd_mc_parallel_dev, (ptr, n, ld)
    else:
        a = square_for_device(a)
        n = a.shape[0]
        keep, stream = a, None
        fn, args = lib.mcnd_mc_parallel, (a.ctypes.data, n, n)
    if p < 1 or p > n:
        raise ValueError(f"invalid plan: need 1 <= p <= n, got p={p}, n={n}")
    payload = np.zeros(max(n - p, 1), dtype=np.int64)
    rows = np.zeros(p, dtype=np.int64)
    rc = fn(*args, p, flags, stream, ctypes.byref(out), ctypes.byref(st), payload.ctypes.data,
            rows.ctypes.data, None)
    del keep
    _lib.check(rc)
    total = time.perf_counter() - t0
    n_payload = int(out.steps)
    # scatter: the rows distributed into the workers' workspaces (+ the H2D copy for a host
    # matrix); comm: the pivot-row broadcasts (in-kernel publication time, summed over steps)
    stats = CommStats(broadcasts=int(st.broadcasts), broadcast_bytes=int(st.broadcast_bytes),
                      pivot_search_msgs=int(st.pivot_search_msgs), scatter_seconds=float(st.scatter_seconds),
                      comm_seconds=float(st.comm_seconds),
                      compute_seconds=max(0.0, float(out.device_ms) / 1e3 - float(st.comm_seconds)))
    ld_res = SINGULAR if out.singular else LogDet(int(out.sign), float(out.log_abs))
    return RunResult(logdet=ld_res, stats=stats, n_workers=p, total_seconds=total,
                     broadcast_payload_entries=[int(x) for x in payload[:n_payload]],
                     row_updates=[int(x) for x in rows], scalar_updates=int(st.scalar_updates))

"""The reference's plugin seam: ALGORITHMS + run_algorithm (mcnd/bench.py:25, :50-65).

``run_algorithm(name, a, p) -> RunResult`` dispatches by string exactly like
the reference so its bench/CLI layers can call the GPU path by name.  Only
the condensation algorithms are on the GPU path; the Gaussian-elimination
names (ge-serial, ge-parallel) are the paper's comparison baseline and are
out of scope here -- asking for them raises ValueError with
a pointer back to the reference package.
"""

from __future__ import annotations

import time

from .condense import logdet_blocked, logdet_condensation
from .runtime import CommStats, RunResult, mc_parallel

ALGORITHMS = ("mc-serial", "mc-parallel", "mc-blocked")
REFERENCE_ONLY = ("ge-serial", "ge-parallel")


def run_algorithm(algorithm: str, a, p: int, *, fast: bool = False) -> RunResult:
    """bench.py:50-65: serial variants report empty comm stats."""
    if algorithm == "mc-parallel":
        return mc_parallel(a, p, fast=fast)
    if algorithm == "mc-serial":
        t0 = time.perf_counter()
        ld = logdet_condensation(a, fast=fast)
        return RunResult(logdet=ld, stats=CommStats(), n_workers=1, total_seconds=time.perf_counter() - t0)
    if algorithm == "mc-blocked":
        t0 = time.perf_counter()
        ld = logdet_blocked(a, fast=fast)
        return RunResult(logdet=ld, stats=CommStats(), n_workers=1, total_seconds=time.perf_counter() - t0)
    if algorithm in REFERENCE_ONLY:
        raise ValueError(f"algorithm {algorithm!r} is not on the GPU condensation path; use mcnd for it")
    raise ValueError(f"unknown algorithm {algorithm!r}")

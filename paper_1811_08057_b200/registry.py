"""The reference's plugin seam: ALGORITHMS + run_algorithm (mcnd/bench.py:25, :50-65).

``run_algorithm(name, a, p) -> RunResult`` dispatches by string exactly like
the reference so its bench/CLI layers can call the GPU path by name: the
condensation algorithms (mc-serial, mc-parallel, + mc-blocked) and the paper's
Gaussian-elimination baseline (ge-serial = gauss.py:34-68 logdet_lu, ge-parallel =
runtime.py:232-321), all on the GPU.
"""

from __future__ import annotations

import csv
import math
import time
from dataclasses import dataclass

from .condense import logdet_blocked, logdet_condensation
from .gauss import ge_parallel, logdet_lu
from .runtime import CommStats, RunResult, mc_parallel

ALGORITHMS = ("mc-serial", "mc-parallel", "ge-serial", "ge-parallel", "mc-blocked")


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
    if algorithm == "ge-parallel":
        return ge_parallel(a, p, fast=fast)
    if algorithm == "ge-serial":
        t0 = time.perf_counter()
        ld = logdet_lu(a, fast=fast)
        return RunResult(logdet=ld, stats=CommStats(), n_workers=1, total_seconds=time.perf_counter() - t0)
    raise ValueError(f"unknown algorithm {algorithm!r}")


# ---- benchmark records in the reference's CSV format ----
# mcnd/bench.py:26-43: BenchRecord / CSV_HEADER; a GPU sweep written with
# write_records() is read back by mcnd.bench.read_records, so the reference's
# format_report (speedup T_s / T_p, bench.py:178-195) covers GPU runs unchanged.
CSV_HEADER = ["algorithm", "n", "p", "run", "total_s", "scatter_s", "comm_s", "sign", "logabs"]
GPU_ALGORITHMS = {"mc-gpu": "mc-serial", "mc-gpu-parallel": "mc-parallel", "mc-gpu-blocked": "mc-blocked",
                  "ge-gpu": "ge-serial", "ge-gpu-parallel": "ge-parallel", "ge-cusolver": "ge-cusolver"}


def _ge_cusolver(d):
    """The paper's Gaussian-elimination comparison point on the GPU (SURVEY.md §8(f)
    rank 3): cuSOLVER LU via torch.linalg.slogdet -- a library baseline, not this
    package's path."""
    import torch

    from .condense import SINGULAR, LogDet

    sign, la = torch.linalg.slogdet(d)
    sg = int(sign.item())
    return SINGULAR if sg == 0 else LogDet(sg, float(la.item()))


@dataclass(frozen=True)
class BenchRecord:
    algorithm: str
    n: int
    p: int
    run_index: int
    total_seconds: float
    scatter_seconds: float
    comm_seconds: float
    sign: int
    log_abs: float


def run_bench(sizes, workers, repeats: int = 5, kind: str = "uniform-random", seed: int = 0,
              algorithms=tuple(GPU_ALGORITHMS)) -> list:
    """The reference's sweep protocol (bench.py:68-108) on the GPU path: one record
    per (algorithm, n, p, run).  The matrix is made resident on the device once per
    (n, p) (its copy time = scatter_s, excluded from total_s as in the reference,
    bench.py:3-4); total_s = wall time of the (synchronous) call: device work + host
    fold; comm_s = 0 (the exchange is fused into the kernels).  Serial algorithms run only
    at p = 1."""
    import torch

    from .matrix import MatrixSpec, generate

    if repeats < 1:
        raise ValueError("repeats must be >= 1")
    records = []
    for n in sizes:
        a = generate(MatrixSpec(size=n, kind=kind, seed=seed))
        for p in workers:
            if p > n:
                continue
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            d = torch.from_numpy(a).cuda()
            e1.record()
            e1.synchronize()
            scatter = e0.elapsed_time(e1) / 1e3
            for run in range(repeats):
                for alg in algorithms:
                    base = GPU_ALGORITHMS[alg]
                    if base not in ("mc-parallel", "ge-parallel") and p != 1:
                        continue
                    torch.cuda.synchronize()
                    t0 = time.perf_counter()
                    if base == "ge-cusolver":
                        ld = _ge_cusolver(d)
                    else:
                        ld = run_algorithm(base, d, p).logdet
                    total = time.perf_counter() - t0
                    records.append(BenchRecord(alg, n, p, run, total, scatter, 0.0, ld.sign, ld.log_abs))
    return records


def write_records(records, path) -> None:
    """CSV exactly as mcnd.bench.write_records (bench.py:111-128)."""
    with open(path, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(CSV_HEADER)
        for r in records:
            w.writerow([r.algorithm, r.n, r.p, r.run_index, repr(r.total_seconds), repr(r.scatter_seconds),
                        repr(r.comm_seconds), r.sign, repr(r.log_abs)])


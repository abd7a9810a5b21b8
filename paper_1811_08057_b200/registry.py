"""The reference's plugin seam: ALGORITHMS + run_algorithm (mcnd/bench.py:25, :50-65).

``run_algorithm(name, a, p) -> RunResult`` dispatches by string exactly like
the reference so its bench/CLI layers can call the GPU path by name.  Only
the condensation algorithms are on the GPU path; the Gaussian-elimination
names (ge-serial, ge-parallel) are the paper's comparison baseline and are
out of scope here -- asking for them raises ValueError with
a pointer back to the reference package.
"""

from __future__ import annotations

import csv
import math
import time
from dataclasses import dataclass

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


# ---- benchmark records in the reference's CSV format ----
# mcnd/bench.py:26-43: BenchRecord / CSV_HEADER; a GPU sweep written with
# write_records() is read back by mcnd.bench.read_records, so the reference's
# format_report (speedup T_s / T_p, bench.py:178-195) covers GPU runs unchanged.
CSV_HEADER = ["algorithm", "n", "p", "run", "total_s", "scatter_s", "comm_s", "sign", "logabs"]
GPU_ALGORITHMS = {"mc-gpu": "mc-serial", "mc-gpu-parallel": "mc-parallel", "mc-gpu-blocked": "mc-blocked",
                  "ge-gpu": "ge-cusolver"}


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
                    if base != "mc-parallel" and p != 1:
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


# ---- the reference's report over benchmark CSVs (bench.py:130-258), restated so the
# CLI's `report` works on GPU sweeps without the reference installed ----
class ReportError(ValueError):
    """Malformed benchmark CSV (bench.py:ReportError)."""


def read_records(path) -> list:
    """bench.py:130-160: header must match CSV_HEADER; per-line field count and types."""
    records = []
    with open(path, newline="") as f:
        reader = csv.reader(f)
        try:
            header = next(reader)
        except StopIteration:
            raise ReportError("empty CSV") from None
        if header != CSV_HEADER:
            raise ReportError(f"line 1: bad header {header!r}")
        for line_no, row in enumerate(reader, 2):
            if not row:
                continue
            if len(row) != len(CSV_HEADER):
                raise ReportError(f"line {line_no}: expected {len(CSV_HEADER)} fields, got {len(row)}")
            try:
                records.append(BenchRecord(row[0], int(row[1]), int(row[2]), int(row[3]), float(row[4]),
                                           float(row[5]), float(row[6]), int(row[7]), float(row[8])))
            except ValueError as exc:
                raise ReportError(f"line {line_no}: {exc}") from exc
    return records


def _mean(values) -> float:
    values = list(values)
    return sum(values) / len(values)


def mean_totals(records) -> dict:
    """bench.py:168-173: mean total seconds per (algorithm, n, p)."""
    groups = {}
    for r in records:
        groups.setdefault((r.algorithm, r.n, r.p), []).append(r.total_seconds)
    return {k: _mean(v) for k, v in groups.items()}


def serial_reference_times(records) -> dict:
    """bench.py:176-183: per size, the fastest single-worker mean across algorithms (T_s)."""
    out = {}
    for (_alg, n, p), t in mean_totals(records).items():
        if p == 1 and (n not in out or t < out[n]):
            out[n] = t
    return out


def speedup_table(records) -> dict:
    """bench.py:186-193: T_s / T_p per (algorithm, n, p)."""
    t_serial = serial_reference_times(records)
    return {(alg, n, p): t_serial[n] / t for (alg, n, p), t in mean_totals(records).items()
            if n in t_serial and t > 0}


def average_speedups(records) -> dict:
    """bench.py:196-203: mean of the per-size speedups per (algorithm, p)."""
    groups = {}
    for (alg, _n, p), s in speedup_table(records).items():
        groups.setdefault((alg, p), []).append(s)
    return {k: _mean(v) for k, v in groups.items()}


def comm_summary(records) -> dict:
    """bench.py:206-218: mean (scatter_s, comm_s) per (algorithm, p)."""
    groups = {}
    for r in records:
        groups.setdefault((r.algorithm, r.p), []).append((r.scatter_seconds, r.comm_seconds))
    return {k: (_mean(s for s, _ in v), _mean(c for _, c in v)) for k, v in groups.items()}


def format_report(records) -> str:
    """bench.py:221-258: the same deterministic text report."""
    if not records:
        raise ReportError("no records to report")
    table, t_serial, means = speedup_table(records), serial_reference_times(records), mean_totals(records)
    lines = ["== Speedup per size (T_s / T_p; T_s = fastest 1-worker mean) ==",
             f"{'algorithm':<12} {'n':>6} {'p':>4} {'mean_total_s':>14} {'speedup':>10}"]
    for (alg, n, p) in sorted(means, key=lambda k: (k[1], k[0], k[2])):
        lines.append(f"{alg:<12} {n:>6} {p:>4} {means[(alg, n, p)]:>14.6f} {table.get((alg, n, p), math.nan):>10.4f}")
    lines += ["", "== Average speedup across sizes ==", f"{'algorithm':<12} {'p':>4} {'avg_speedup':>12}"]
    avgs = average_speedups(records)
    for (alg, p) in sorted(avgs):
        lines.append(f"{alg:<12} {p:>4} {avgs[(alg, p)]:>12.4f}")
    lines += ["", "== Scatter / communication averages ==", f"{'algorithm':<12} {'p':>4} {'avg_scatter_s':>14} {'avg_comm_s':>12}"]
    comms = comm_summary(records)
    for (alg, p) in sorted(comms):
        sc, cm = comms[(alg, p)]
        lines.append(f"{alg:<12} {p:>4} {sc:>14.6f} {cm:>12.6f}")
    lines += ["", "reference serial times: " + ", ".join(f"n={n}: {t_serial[n]:.6f}s" for n in sorted(t_serial))]
    return "\n".join(lines) + "\n"

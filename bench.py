#!/usr/bin/env python
"""Benchmark: time-to-logdet / effective GFLOP/s of matrix condensation on B200.

Default workload (BASELINE.json metric): C3, one dense N=8000 FP64 matrix with
iid U[-1,1] entries (numpy PCG64 seed 3), log-determinant by condensation.
A "step" is one full log-determinant of that matrix.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3|c1|c2|c4|c5]
                    [--method unblocked|blocked] [--fast] [--impl mc|reference]

value      effective GFLOP/s = (2 N^3 / 3) / (device time per step), input resident
           in HBM, CUDA events on the launching stream (max over ranks).
e2e        same metric through the public API with the matrix in pinned HOST
           memory: H2D copy, condensation, D2H of the pivots, host sign/log.
roofline   HBM-bound: algorithmic bytes B(N) = 8 sum_{m=2}^{N} [(m-1)m + m + (m-1)^2]
           per logdet / kernel time, against MEASURED_PEAKS.json hbm_gbs.
cpu_baseline  the oracle (plain-C port of the reference algorithm, OpenMP over
           rows, all host threads) on a bounded prefix of the same workload,
           extrapolated by sum m^2 (work per step ~ m^2).
--impl reference  the same CPU port as the whole measurement (rank 0 only).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

PAPER_TABLE3_N8000 = {1: 170.80, 2: 94.06, 4: 46.85, 8: 33.73}  # PAPER.md:193, seconds


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--method", default=None, choices=["unblocked", "blocked"],
                    help="condensation variant (default: unblocked for n < 2048 (c1, c2), blocked otherwise (c3, c5))")
    ap.add_argument("--fast", action="store_true", help="FMA update (default: reference-exact arithmetic)")
    ap.add_argument("--impl", default="mc", choices=["mc", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--force-dist", action="store_true",
                    help="use the multi-GPU block-row driver even with one rank (test hook)")
    ap.add_argument("--no-c5", action="store_true", help="skip the C5 sub-record of the default (C3) line")
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU check of the multi-rank launcher and schedule (gloo, no GPU work)")
    return ap.parse_args()


def algorithmic_bytes(n: int) -> float:
    m = np.arange(2, n + 1, dtype=np.float64)
    return float(8.0 * np.sum((m - 1) * m + m + (m - 1) ** 2))


def flops(n: int) -> float:
    return 2.0 * n ** 3 / 3.0


def workload(cfg: str):
    from paper_1811_08057_b200 import matrix as M

    if cfg == "c1":
        return "C1 dense N(0,1) N=1000 seed 1", M.config_dense_normal(1000, 1), 1000
    if cfg == "c2":
        return "C2 SPD X X^T/2N + 1e-3 I, N=4000 seed 2", M.config_spd(4000, 2), 4000
    if cfg == "c3":
        return "C3 dense U[-1,1] N=8000 seed 3", M.config_uniform(8000, 3), 8000
    if cfg == "c4":
        return "C4 batched 4096 x SPD 64x64 seed 4", M.config_batched_spd(4096, 64, 4), 64
    if cfg == "c5":
        return ("C5 SPD X X^T/N + 1e-2 I, N=32768 (X from a seeded CUDA generator, seed 5)",
                M.config_spd_device(32768, 5), 32768)
    raise ValueError(cfg)


def fp64_peak(local: int) -> dict:
    """The FP64 roofline denominator, measured in this run: cuBLAS DGEMM (torch.matmul,
    float64, 8192^3; FP64 tensor cores, DMMA), best of 5 with CUDA events, SM clocks
    sampled meanwhile.  (MEASURED_PEAKS.json has no FP64 entry; a DMMA register-only
    microbenchmark gives 37.0 TFLOP/s, profiles/r1_dmma_peak.txt.)"""
    import torch

    n = 8192
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.rand((n, n), dtype=torch.float64, device="cuda", generator=g)
    y = torch.rand((n, n), dtype=torch.float64, device="cuda", generator=g)
    for _ in range(2):
        torch.matmul(x, y)
    torch.cuda.synchronize()
    best = float("inf")
    with ClockSampler(local) as clk:
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch.matmul(x, y)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
    del x, y
    return {"tflops": 2.0 * n ** 3 / (best * 1e-3) / 1e12, "ms": best,
            "how": "cuBLAS DGEMM (torch.matmul float64) 8192^3, best of 5, measured in this run",
            "clocks": clk.summary()}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region: NVML polled
    every 2 ms from a thread (short regions such as C4's still get samples); falls
    back to `nvidia-smi -lms 100` without NVML."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []
        self.samples = []  # (sm_mhz, max_mhz, reasons)
        self._stop = threading.Event()
        self._nvml = None

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            self._nvml = pynvml
            self._t = threading.Thread(target=self._poll_nvml, daemon=True)
            self._t.start()
            t0 = time.perf_counter()
            while not self.samples and time.perf_counter() - t0 < 0.2:  # poller running
                time.sleep(0.0005)
            return self
        except Exception:
            self._nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:
            self.proc = None
        return self

    def _poll_nvml(self):
        nv = self._nvml
        bits = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}
        mx = nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM)
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h) if hasattr(
                    nv, "nvmlDeviceGetCurrentClocksEventReasons") else nv.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
                self.samples.append((float(sm), float(mx), {k for k, b in bits.items() if rs & b}))
            except Exception:
                pass
            self._stop.wait(0.002)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self._nvml is not None:  # one last sample right at the end of the region
            time.sleep(0.003)
        self._stop.set()
        if self._nvml is not None:
            self._t.join(timeout=1)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        for (c, m, r) in self.samples:
            sm.append(c)
            mx = max(mx, m)
            reasons |= r
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = max(mx, float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(self.NAMES, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvml" if self.samples else "nvidia-smi"}


def prefix_work_fraction(n: int, steps: int) -> float:
    """Share of the condensation work (sum over steps of (m-1)^2, m = active width) done
    by the first `steps` steps: the extrapolation factor of a bounded CPU sample."""
    m = np.arange(n, 1, -1, dtype=np.float64)
    return float(np.sum((m[:steps] - 1) ** 2) / np.sum((m - 1) ** 2))


class CpuSample:
    """The reference's CPU path (oracle: plain-C port of condense.py:134-160 /
    runtime.py:123-229, OpenMP over rows, all host threads) on a bounded prefix of the
    workload: the first S condensation steps (S calibrated once so that one sample takes
    about `budget_s`), serial top-to-bottom order at one GPU and the p-worker block-row
    schedule (mc_parallel(a, p)) at p GPUs."""

    def __init__(self, a: np.ndarray, budget_s: float, p: int = 1):
        from oracle import mcnd_oracle as O

        self.O, self.a, self.p = O, a, p
        self.n = a.shape[0]
        self.threads = os.cpu_count() or 1
        self.total = self.n - p  # broadcast steps of the full run
        self._run(min(self.total, 8))  # load the library, spin up the thread pool
        steps = min(self.total, 16)
        for _ in range(4):  # grow the prefix until one sample takes about budget_s
            t = self._run(steps)
            if t >= 0.6 * budget_s or steps == self.total:
                break
            steps = int(min(self.total, max(steps + 1, steps * 0.9 * budget_s / max(t, 1e-3))))
        self.steps = steps
        self.frac = prefix_work_fraction(self.n, steps)

    def _run(self, steps: int) -> float:
        t0 = time.perf_counter()
        if self.p == 1:
            self.O.condense_prefix(self.a, steps, self.threads)
        else:
            self.O.mc_parallel(self.a, self.p, self.threads, max_steps=steps)
        return time.perf_counter() - t0

    def time_one(self) -> float:
        return self._run(self.steps)

    def describe(self, t: float) -> dict:
        """cpu_baseline object for one measured sample time t (seconds)."""
        call = "logdet_condensation" if self.p == 1 else f"mc_parallel(a, {self.p})"
        return {"value": flops(self.n) * self.frac / t / 1e9, "unit": "GFLOP/s", "cores": self.threads,
                "kind": "port",
                "sample": (f"reference {call} (oracle C port, {self.threads} threads): first {self.steps} of "
                           f"{self.total} condensation steps of the same matrix, {100 * self.frac:.1f}% of the "
                           f"work, {t:.2f} s measured; value = that work / that time"),
                "sample_seconds": t,
                "time_to_logdet_s_extrapolated": t / self.frac}


def cpu_baseline(a: np.ndarray, budget_s: float, p: int = 1):
    s = CpuSample(a, budget_s, p)
    return s.describe(s.time_one())


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def default_method(args, n: int) -> str:
    return args.method or ("unblocked" if n < 2048 else "blocked")


def bench_config(args, name: str, n: int, world: int, batch: int | None = None) -> dict:
    """The workload `config` both arms print (the driver compares them)."""
    if batch is not None:
        return {"workload": name, "batch": batch, "n": n, "l2": "L2 flushed between iterations",
                "parallelism": "1 GPU" if world == 1 else f"batch sharded x{world} GPUs"}
    method = default_method(args, n)
    if world == 1:
        par = "1 GPU"
    elif method == "blocked":
        par = (f"block rows x{world} GPUs: panel pairs from the rank with the most live rows, "
               "W broadcast (NCCL), local rank-128 updates")
    else:
        par = f"block-row x{world} GPUs, pivot rows pushed over NVLink"
    return {"workload": name, "n": n, "method": method, "mode": "fast-fma" if args.fast else "reference-exact",
            "l2": ("input larger than L2 (%.0f MB vs 126 MB); workspace re-read from the caller's matrix each step"
                   % (8 * n * n / 1e6)) if 8 * n * n > 126e6 else "input fits L2 (%.0f MB)" % (8 * n * n / 1e6),
            "parallelism": par}


def run_reference(args):
    """--impl reference: the reference's CPU path (oracle port, all host threads) on this
    arm's workload, rank 0 only; every timed step is one bounded sample (the first S
    condensation steps, S calibrated during the warm-up), so steps x ms_per_step is the
    time actually measured."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    p = max(world, args.gpus)
    name, a, n = workload(args.config)
    if not isinstance(a, np.ndarray):  # C5 is generated on the GPU; the CPU port gets a host copy
        a = a.cpu().numpy()
    threads = os.cpu_count() or 1
    if a.ndim == 3:
        from oracle import mcnd_oracle as O

        for _ in range(args.warmup):
            O.logdet_batched(a[:256], threads)
        times = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            O.logdet_batched(a, threads)
            times.append(time.perf_counter() - t0)
        t = statistics.mean(times)
        val = a.shape[0] * flops(n) / t / 1e9
        cb = {"value": val, "unit": "GFLOP/s", "cores": threads, "kind": "port",
              "sample": f"full batch of {a.shape[0]} matrices per step (oracle C port, {threads} threads)"}
        cfg = bench_config(args, name, n, p, batch=a.shape[0])
    else:
        total_budget = 150.0  # seconds of CPU work for the whole --steps/--warmup run
        budget = max(1.0, min(args.cpu_seconds, total_budget / max(args.steps + 1, 1)))
        smp = CpuSample(a, budget, p)  # its calibration samples are the warm-up
        times = [smp.time_one() for _ in range(args.steps)]
        t = statistics.mean(times)
        cb = smp.describe(t)
        val = cb["value"]
        cfg = bench_config(args, name, n, p)
    line = {"impl": "reference", "metric": metric_name(args.config), "value": val, "unit": "GFLOP/s",
            "n_gpus": p, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (numpy PCG64)", "config": cfg, "cpu_baseline": cb,
            "e2e": {"value": val, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def metric_name(cfg):
    if cfg == "c5":
        return "effective GFLOP/s (2N^3/3) of the blocked condensation log-determinant, N=32768 FP64 (time-to-logdet in ms_per_step)"
    if cfg == "c4":
        return "effective GFLOP/s (2n^3/3 per matrix), batched 4096 x 64x64 SPD FP64 logdet"
    return "effective GFLOP/s (2N^3/3) of the condensation log-determinant, FP64 (time-to-logdet in ms_per_step)"


def traffic_from_profiles(cfg):
    path = os.path.join(ROOT, "profiles", f"ncu_{cfg}_traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get("traffic_bytes_per_launch")
    except Exception:
        return None


def run_single(args):
    import torch

    import paper_1811_08057_b200 as mc

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    name, a, n = workload(args.config)
    if a.ndim == 3:
        return run_batched(args, name, a, n)
    # default: the blocked rank-64 variant where the unblocked rank-1 chain is HBM-bound
    # (north_star (2)); C1 stays unblocked (L2/latency-bound, 8 MB).  The other variant
    # is measured too and reported under "alt" (unblocked = bitwise-reference arithmetic).
    method = default_method(args, n)
    fn = mc.logdet_blocked if method == "blocked" else mc.logdet_condensation
    if isinstance(a, np.ndarray):
        d = torch.from_numpy(a).cuda()
    else:
        d, a = a, None
    try:
        h = torch.empty(tuple(d.shape), dtype=torch.float64, pin_memory=True)
        h.copy_(d)
        hv = h.numpy()
    except Exception:  # not enough pinned host memory: e2e from pageable memory
        hv = d.cpu().numpy()
    if a is None and not args.no_cpu_baseline:
        a = hv
    stream = torch.cuda.current_stream()

    for _ in range(args.warmup):
        res = fn(d, fast=args.fast)
    torch.cuda.synchronize()
    kernel_ms = []
    launches = 0
    torn = 0
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            res, piv, cols, kms = fn(d, fast=args.fast, return_pivots=True)
            kernel_ms.append(kms)
            launches += mc._lib.LAST_LAUNCHES  # counted by the library per call
            torn += mc._lib.LAST_TORN_READS if method == "blocked" else 0
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / args.steps

    # e2e: public API on a pinned HOST matrix (H2D + condensation + D2H + host fold)
    fn(hv, fast=args.fast)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        res_e2e = fn(hv, fast=args.fast)
    e1.record(stream)
    torch.cuda.synchronize()
    ms_e2e = e0.elapsed_time(e1) / args.steps
    assert res_e2e == res, (res_e2e, res)

    kms = statistics.mean(kernel_ms)
    hbm, peak_kind = peaks()
    fp64 = fp64_peak(local)
    if method == "blocked":
        achieved = flops(n) / (kms * 1e-3) / 1e12  # the pivot chain, not DMMA, bounds small N
        roof = {"bound": "tensor", "achieved": achieved, "peak": fp64["tflops"],
                "peak_kind": fp64["how"], "unit": "TFLOP/s",
                "frac": achieved / fp64["tflops"], "traffic": traffic_from_profiles(args.config + "_blocked"),
                "algorithmic_flops_per_launch": flops(n), "peak_clocks": fp64["clocks"]}
        chain = panel_chain(mc, d, args.fast)
        if chain:
            roof["panel_chain"] = chain
    else:
        B = algorithmic_bytes(n)
        achieved = B / (kms * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "peak_kind": peak_kind, "unit": "GB/s",
                "frac": achieved / hbm, "traffic": traffic_from_profiles(args.config),
                "algorithmic_bytes_per_launch": B}
    parity = check_parity(args.config, res, args.fast or method == "blocked")
    line = {
        "metric": metric_name(args.config),
        "value": flops(n) / (ms * 1e-3) / 1e9,
        "unit": "GFLOP/s",
        "n_gpus": 1,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "time_to_logdet_s": ms / 1e3,
        "kernel_ms": kms,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": (PAPER_TABLE3_N8000[1] / (ms / 1e3)) if args.config == "c3" else None,
        "vs_baseline_note": "paper Table 3 (PAPER.md:193): N=8000, 1 CPU processor, 170.80 s" if args.config == "c3" else None,
        "dtype": "f64",
        "data": "synthetic (seeded, BASELINE recipe)",
        "config": bench_config(args, name, n, 1),
        "result": {"sign": res.sign, "log_abs": res.log_abs, "parity": parity,
                   "panel_torn_reads": torn if method == "blocked" else None},
        "roofline": roof,
        "e2e": {"value": flops(n) / (ms_e2e * 1e-3) / 1e9, "unit": "GFLOP/s", "ms_per_step": ms_e2e,
                "h2d_bytes_per_step": 8 * n * n, "d2h_bytes_per_step": 12 * n + 16},
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    bad = [parity] if parity.startswith("MISMATCH") else []
    if args.method is None and args.config in ("c2", "c3"):
        other = mc.logdet_condensation if method == "blocked" else mc.logdet_blocked
        other(d, fast=args.fast)
        oms = []
        for _ in range(max(2, min(args.steps, 4))):
            r2, _, _, k2 = other(d, fast=args.fast, return_pivots=True)
            oms.append(k2)
        okms = statistics.mean(oms)
        omethod = "unblocked" if method == "blocked" else "blocked"
        opar = check_parity(args.config, r2, args.fast or omethod == "blocked")
        bad += [opar] if opar.startswith("MISMATCH") else []
        alt = {"method": omethod, "kernel_ms": okms, "value": flops(n) / (okms * 1e-3) / 1e9, "unit": "GFLOP/s",
               "result": {"sign": r2.sign, "log_abs": r2.log_abs, "parity": opar}}
        if omethod == "unblocked":
            B = algorithmic_bytes(n)
            alt["roofline"] = {"bound": "hbm", "achieved": B / (okms * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
                               "frac": B / (okms * 1e-3) / 1e9 / hbm, "traffic": traffic_from_profiles(args.config)}
        line["alt"] = alt
    if args.config == "c3" and not args.no_c5:
        del d
        torch.cuda.empty_cache()
        c5 = c5_record(args, mc, fp64, local)
        line["c5"] = c5
        if c5["parity"].startswith("MISMATCH"):
            bad.append("C5 " + c5["parity"])
    if not args.no_cpu_baseline and a is not None:
        line["cpu_baseline"] = cpu_baseline(a, args.cpu_seconds)
    print(json.dumps(line), flush=True)
    if bad:
        print("bench.py: PARITY FAILURE: " + "; ".join(bad), file=sys.stderr, flush=True)
        return 3
    return 0


def c5_record(args, mc, fp64, local: int) -> dict:
    """C5 (N=32768 SPD, 8.6 GB, blocked b=64 on the FP64 tensor cores) as a sub-record of
    the default line: device time per logdet against the in-run DGEMM peak, cuSOLVER LU
    (torch.linalg.slogdet, getrf) on the same matrix as the library reference point and
    the value oracle (the reference CPU path is infeasible at this size)."""
    import torch

    from paper_1811_08057_b200 import matrix as M

    n = 32768
    a = M.config_spd_device(n, 5)
    stream = torch.cuda.current_stream()
    mc.logdet_blocked(a)
    torch.cuda.synchronize()
    times, kms, launches = [], [], 0
    with ClockSampler(local) as clk:
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            res, _, _, k = mc.logdet_blocked(a, return_pivots=True)
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
            kms.append(k)
            launches += mc._lib.LAST_LAUNCHES
    torn = mc._lib.LAST_TORN_READS
    cus = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        s_ref, l_ref = torch.linalg.slogdet(a)
        e1.record(stream)
        torch.cuda.synchronize()
        cus.append(e0.elapsed_time(e1))
    s_ref, l_ref = int(s_ref.item()), float(l_ref.item())
    tol = max(1e-8 * n, 1e-10 * abs(l_ref))
    d = abs(res.log_abs - l_ref)
    parity = (f"within tolerance of cuSOLVER LU slogdet (|d|={d:.3e} <= {tol:.2e})"
              if res.sign == s_ref and d <= tol else
              f"MISMATCH vs cuSOLVER LU slogdet ({res.sign},{res.log_abs}) != ({s_ref},{l_ref})")
    ms = statistics.mean(times)
    ach = flops(n) / (ms * 1e-3) / 1e12
    del a
    torch.cuda.empty_cache()
    return {"workload": "C5 SPD X X^T/N + 1e-2 I, N=32768 (X from a seeded CUDA generator, seed 5)",
            "method": "blocked", "ms_per_step": ms, "kernel_ms": statistics.mean(kms), "steps": len(times),
            "value": flops(n) / (ms * 1e-3) / 1e9, "unit": "GFLOP/s",
            "roofline": {"bound": "tensor", "achieved": ach, "peak": fp64["tflops"], "peak_kind": fp64["how"],
                         "unit": "TFLOP/s", "frac": ach / fp64["tflops"],
                         "traffic": traffic_from_profiles("c5_blocked")},
            "result": {"sign": res.sign, "log_abs": res.log_abs, "panel_torn_reads": torn},
            "parity": parity,
            "cusolver_getrf_ms": statistics.mean(cus), "speedup_vs_cusolver": statistics.mean(cus) / ms,
            "gpu_launches": launches, "clocks": clk.summary()}


def panel_chain(mc, d, fast):
    """In-kernel time of the panel kernels of one blocked call (device globaltimer
    spans logged by the panel kernel's CTA 0): the latency-bound pivot chain that
    bounds the blocked path at moderate N, as a share of the call."""
    import ctypes

    lib = mc._lib.load()
    if not hasattr(lib, "mcnd_debug_kp_spans"):
        return None
    buf = np.zeros((4096, 2), dtype=np.uint64)
    lib.mcnd_debug_kp_spans(ctypes.c_void_p(buf.ctypes.data), 4096)  # reset
    r = mc.logdet_blocked(d, fast=fast, return_pivots=True)
    k = lib.mcnd_debug_kp_spans(ctypes.c_void_p(buf.ctypes.data), 4096)
    if k <= 0:
        return None
    sp = buf[:k].astype(np.int64)
    kp_ms = float((sp[:, 1] - sp[:, 0]).sum()) / 1e6
    return {"panels": int(k), "panel_kernel_ms": kp_ms, "call_ms": r[3], "share": kp_ms / r[3],
            "pivots": int(k) * 64, "us_per_pivot": 1e3 * kp_ms / (int(k) * 64)}


def check_parity(cfg, res, fast):
    """Compare with the reference's golden (when committed) -- reported, not asserted."""
    names = {"c1": "c1_normal_1000_s1", "c3": "c3_uniform_8000_s3"}
    nm = names.get(cfg)
    if not nm:
        return "see tests/test_gpu_parity.py"
    path = os.path.join(ROOT, "tests", "golden", "cases", nm + ".json")
    if not os.path.exists(path):
        return "golden missing"
    with open(path) as f:
        c = json.load(f)
    exp_s, exp_l = c["expect"]["sign"], float.fromhex(c["expect"]["log_abs"])
    if res.sign == exp_s and res.log_abs == exp_l:
        return "bitwise equal to reference mcnd.logdet_condensation"
    if res.sign == exp_s and abs(res.log_abs - exp_l) <= max(1e-8 * 8000, 1e-10 * abs(exp_l)):
        return f"within tolerance (|d|={abs(res.log_abs - exp_l):.3e})"
    return f"MISMATCH vs reference ({res.sign},{res.log_abs}) != ({exp_s},{exp_l})"


def run_batched(args, name, a, n):
    import torch

    import paper_1811_08057_b200 as mc

    d = torch.from_numpy(a).cuda()
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        mc.logdet_batched(d, fast=args.fast)
    torch.cuda.synchronize()
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
    times = []
    with ClockSampler(int(os.environ.get("LOCAL_RANK", "0"))) as clk:
        for _ in range(args.steps):
            flush.fill_(1.0)  # L2 flush between iterations (input is 134 MB, L2 126 MB)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            s, l = mc.logdet_batched(d, fast=args.fast)
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
    ms = statistics.mean(times)
    h = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
    h.numpy()[...] = a
    mc.logdet_batched(h.numpy(), fast=args.fast)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        mc.logdet_batched(h.numpy(), fast=args.fast)
    ms_e2e = (time.perf_counter() - t0) * 1e3 / args.steps
    hbm, peak_kind = peaks()
    B = a.nbytes + a.shape[0] * 12
    fl = a.shape[0] * flops(n)
    line = {"metric": metric_name("c4"), "value": fl / (ms * 1e-3) / 1e9, "unit": "GFLOP/s", "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (numpy PCG64 seed 4)",
            "config": bench_config(args, name, n, 1, batch=a.shape[0]),
            "roofline": {"bound": "hbm", "achieved": B / (ms * 1e-3) / 1e9, "peak": hbm, "peak_kind": peak_kind,
                         "unit": "GB/s", "frac": B / (ms * 1e-3) / 1e9 / hbm, "traffic": traffic_from_profiles("c4")},
            "e2e": {"value": fl / (ms_e2e * 1e-3) / 1e9, "unit": "GFLOP/s", "ms_per_step": ms_e2e,
                    "h2d_bytes_per_step": a.nbytes, "d2h_bytes_per_step": a.shape[0] * 12},
            "gpu_launches": args.steps, "clocks": clk.summary()}
    if not args.no_cpu_baseline:
        from oracle import mcnd_oracle as O

        threads = os.cpu_count() or 1
        sub = a[:1024]
        t0 = time.perf_counter()
        O.logdet_batched(sub, threads)
        t = time.perf_counter() - t0
        line["cpu_baseline"] = {"value": sub.shape[0] * flops(n) / t / 1e9, "unit": "GFLOP/s", "cores": threads,
                                "kind": "port", "sample": "first 1024 of 4096 matrices"}
    print(json.dumps(line), flush=True)
    return 0


def spawn(args) -> int:
    """`bench.py --gpus N` outside torchrun: launch N ranks (one process per GPU) through
    torch.distributed.run on 127.0.0.1 and return their exit status; rank 0 prints the line."""
    import socket

    if not args.dry_run:
        import torch

        have = torch.cuda.device_count()
        if have < args.gpus:
            print(f"bench.py: --gpus {args.gpus} but only {have} CUDA device(s) visible", file=sys.stderr)
            return 2
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def dry_run(args) -> int:
    """CPU check of the multi-rank plumbing (gloo): every rank derives its block rows and
    the blocked pair schedule, the ranks agree on them, rank 0 prints the line it would
    print (no GPU work, value null)."""
    import torch
    import torch.distributed as dist

    from paper_1811_08057_b200 import dist as D
    from paper_1811_08057_b200.runtime import plan_blocks

    rank, world, _ = dist_env()
    dist.init_process_group("gloo")
    n = {"c1": 1000, "c2": 4000, "c3": 8000, "c5": 32768}.get(args.config, 8000)
    start, rows = plan_blocks(n, world).assignments[rank]
    sched = D.blocked_schedule(n, world)
    mine = torch.tensor([rows, len(sched[0])], dtype=torch.int64)
    allv = [torch.zeros_like(mine) for _ in range(world)]
    dist.all_gather(allv, mine)
    ok = sum(int(v[0]) for v in allv) == n and len({int(v[1]) for v in allv}) == 1
    if rank == 0:
        print(json.dumps({"metric": metric_name(args.config), "value": None, "unit": "GFLOP/s", "n_gpus": world,
                          "steps": 0, "warmup": 0, "dry_run": True, "schedule_consistent": ok,
                          "config": {"workload": args.config, "n": n, "ranks_rows": [int(v[0]) for v in allv]}}),
              flush=True)
    dist.destroy_process_group()
    return 0 if ok else 1


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":  # CPU only: rank 0 runs it (torchrun or not), p = the GPU count
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn(args)
    if args.gpus > 1 and world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        return 2
    if args.dry_run:
        return dry_run(args)
    if world > 1 or args.force_dist:
        from paper_1811_08057_b200 import dist

        return dist.bench_main(args)
    return run_single(args)


if __name__ == "__main__":
    sys.exit(main())

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


FP64_PEAK_TFLOPS = 35.47  # cuBLAS DGEMM 8192^3 measured on this pool (profiles/r1_fp64_peak.json);
#                           DMMA-only register microbenchmark: 37.0 (profiles/r1_dmma_peak.txt)


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


def cpu_baseline(a: np.ndarray, budget_s: float):
    """Oracle (C port, OpenMP) on a bounded prefix of the condensation, extrapolated by sum m^2."""
    from oracle import mcnd_oracle as O

    n = a.shape[0]
    threads = os.cpu_count() or 1
    O.condense_prefix(a[:64, :64], 8, threads)  # load + spin up the thread pool
    steps = min(n - 1, 16)
    for _ in range(3):  # grow the prefix until it takes about budget_s
        t0 = time.perf_counter()
        O.condense_prefix(a, steps, threads)
        t = time.perf_counter() - t0
        if t >= 0.5 * budget_s or steps == n - 1:
            break
        steps = int(min(n - 1, max(steps + 1, steps * 0.9 * budget_s / max(t, 1e-3))))
    m = np.arange(n, 1, -1, dtype=np.float64)  # active size at each step
    w_all = float(np.sum((m - 1) ** 2))
    w_pre = float(np.sum((m[:steps] - 1) ** 2))
    t_full = t * w_all / w_pre
    return {"value": flops(n) / t_full / 1e9, "unit": "GFLOP/s", "cores": threads, "kind": "port",
            "sample": f"first {steps} of {n - 1} condensation steps of the same matrix "
                      f"({t:.1f} s, {100 * w_pre / w_all:.1f}% of the work), extrapolated by sum m^2",
            "time_to_logdet_s_extrapolated": t_full}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    name, a, n = workload(args.config)
    if not isinstance(a, np.ndarray):  # C5 is generated on the GPU; the CPU port gets a host copy
        a = a.cpu().numpy()
    if a.ndim == 3:
        from oracle import mcnd_oracle as O

        threads = os.cpu_count() or 1
        times = []
        for _ in range(args.warmup):
            O.logdet_batched(a[:256], threads)
        for _ in range(args.steps):
            t0 = time.perf_counter()
            O.logdet_batched(a, threads)
            times.append(time.perf_counter() - t0)
        t = statistics.mean(times)
        val = a.shape[0] * flops(n) / t / 1e9
        cb = {"value": val, "unit": "GFLOP/s", "cores": threads, "kind": "port", "sample": "full batch"}
    else:
        budget = max(2.0, min(args.cpu_seconds, 150.0 / max(args.steps + args.warmup, 1)))
        for _ in range(args.warmup):
            cpu_baseline(a, budget / 4)
        vals = [cpu_baseline(a, budget) for _ in range(args.steps)]
        val = statistics.mean(v["value"] for v in vals)
        cb = dict(vals[-1])
        cb["value"] = val
        t = flops(n) / (val * 1e9)
    line = {"impl": "reference", "metric": metric_name(args.config), "value": val, "unit": "GFLOP/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (numpy PCG64)", "config": {"workload": name, "n": n},
            "cpu_baseline": cb,
            "e2e": {"value": val, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


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
    method = args.method or ("unblocked" if n < 2048 else "blocked")
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
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            res, piv, cols, kms = fn(d, fast=args.fast, return_pivots=True)
            kernel_ms.append(kms)
            launches += mc._lib.LAST_LAUNCHES  # counted by the library per call
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
    assert res_e2e == res

    kms = statistics.mean(kernel_ms)
    hbm, peak_kind = peaks()
    if method == "blocked":
        achieved = flops(n) / (kms * 1e-3) / 1e12  # the pivot chain, not DMMA, bounds small N
        roof = {"bound": "tensor", "achieved": achieved, "peak": FP64_PEAK_TFLOPS,
                "peak_kind": "measured here (cuBLAS DGEMM, FP64 DMMA)", "unit": "TFLOP/s",
                "frac": achieved / FP64_PEAK_TFLOPS, "traffic": traffic_from_profiles(args.config + "_blocked"),
                "algorithmic_flops_per_launch": flops(n)}
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
        "config": {"workload": name, "n": n, "method": method,
                   "mode": "fast-fma" if args.fast else "reference-exact",
                   "l2": "input larger than L2 (%.0f MB vs 126 MB); workspace re-read from the caller's matrix each step" % (8 * n * n / 1e6),
                   "parallelism": "1 GPU"},
        "result": {"sign": res.sign, "log_abs": res.log_abs, "parity": parity},
        "roofline": roof,
        "e2e": {"value": flops(n) / (ms_e2e * 1e-3) / 1e9, "unit": "GFLOP/s", "ms_per_step": ms_e2e,
                "h2d_bytes_per_step": 8 * n * n, "d2h_bytes_per_step": 12 * n + 16},
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    if args.method is None and args.config in ("c2", "c3"):
        other = mc.logdet_condensation if method == "blocked" else mc.logdet_blocked
        other(d, fast=args.fast)
        oms = []
        for _ in range(max(2, min(args.steps, 4))):
            r2, _, _, k2 = other(d, fast=args.fast, return_pivots=True)
            oms.append(k2)
        okms = statistics.mean(oms)
        omethod = "unblocked" if method == "blocked" else "blocked"
        alt = {"method": omethod, "kernel_ms": okms, "value": flops(n) / (okms * 1e-3) / 1e9, "unit": "GFLOP/s",
               "result": {"sign": r2.sign, "log_abs": r2.log_abs,
                          "parity": check_parity(args.config, r2, args.fast or omethod == "blocked")}}
        if omethod == "unblocked":
            B = algorithmic_bytes(n)
            alt["roofline"] = {"bound": "hbm", "achieved": B / (okms * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
                               "frac": B / (okms * 1e-3) / 1e9 / hbm, "traffic": traffic_from_profiles(args.config)}
        line["alt"] = alt
    if not args.no_cpu_baseline and a is not None:
        line["cpu_baseline"] = cpu_baseline(a, args.cpu_seconds)
    print(json.dumps(line), flush=True)


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
            "config": {"workload": name, "batch": a.shape[0], "n": n, "l2": "L2 flushed between iterations"},
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


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    rank, world, local = dist_env()
    if world > 1 or args.force_dist:
        from paper_1811_08057_b200 import dist

        return dist.bench_main(args)
    return run_single(args)


if __name__ == "__main__":
    main()

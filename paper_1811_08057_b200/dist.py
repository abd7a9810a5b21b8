"""Multi-GPU block-row condensation: one process per GPU (D1).

Replaces the reference's in-process fabric (mcnd/runtime.py:69-120) with real
transport.  Rank w holds rows plan_blocks(n, world)[w] (runtime.py:33-44) in a
full n x ld workspace; the pivot owner of each step (round-robin over ranks
with > 1 live row, its topmost live row -- runtime.py:153-165, which for
divisible n is exactly "the rank holding the most live rows") publishes the
scaled pivot row by storing it straight into the matching row slot of every
peer's workspace over NVLink (CUDA IPC mappings), followed by a system-scope
release flag.  Every rank's persistent kernel (csrc/k1_condense.cu) waits only
for that flag, so the "broadcast" of runtime.py:185 is fused into the kernel
that computes it -- no NCCL call and no host round trip per step.

After n - p steps every rank holds one live row; the p rows (first p
columns) and their witnesses are all-gathered and folded exactly like
runtime.py:206-229 (mcnd_fold_mc_parallel), so the result is bitwise the
reference's mc_parallel(a, world).

The host-side gather/fold (``fold_gathered``) is transport-agnostic and is
covered by world_size-2 gloo tests on CPU (tests/test_dist_host.py).
"""

from __future__ import annotations

import ctypes
import os
import time

import numpy as np

from . import _lib
from .condense import SINGULAR, LogDet
from .runtime import CommStats, RunResult, plan_blocks


def fold_gathered(n: int, p: int, piv_vals, piv_cols, singular_at: int, rem_rows, rem_wits) -> RunResult:
    """runtime.py:206-229 on gathered data: rem_rows[w] = worker w's last live row
    (first p columns), rem_wits[w] its witness; pivots as published."""
    lib = _lib.load()
    out = _lib.McndLogDet()
    st = _lib.McndCommStats()
    pv = np.ascontiguousarray(piv_vals, dtype=np.float64)
    pc = np.ascontiguousarray(piv_cols, dtype=np.int32)
    rem = np.ascontiguousarray(np.asarray(rem_rows, dtype=np.float64).reshape(p, p))
    wit = np.ascontiguousarray(rem_wits, dtype=np.float64).reshape(p)
    payload = np.zeros(max(n - p, 1), dtype=np.int64)
    rows = np.zeros(p, dtype=np.int64)
    rc = lib.mcnd_fold_mc_parallel(n, p, pv.ctypes.data, pc.ctypes.data, int(singular_at), rem.ctypes.data,
                                   wit.ctypes.data, ctypes.byref(out), ctypes.byref(st), payload.ctypes.data,
                                   rows.ctypes.data)
    _lib.check(rc)
    stats = CommStats(broadcasts=int(st.broadcasts), broadcast_bytes=int(st.broadcast_bytes),
                      pivot_search_msgs=0)
    res = SINGULAR if out.singular else LogDet(int(out.sign), float(out.log_abs))
    return RunResult(logdet=res, stats=stats, n_workers=p,
                     broadcast_payload_entries=[int(x) for x in payload[: int(out.steps)]],
                     row_updates=[int(x) for x in rows], scalar_updates=int(st.scalar_updates))


class BlockRowGroup:
    """Collective handle over the ranks of a torch.distributed process group
    (one GPU per rank, current device already set).  n is fixed per handle."""

    def __init__(self, n: int, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.n = int(n)
        self.plan = plan_blocks(self.n, self.world)
        lib = _lib.load()
        self.lib = lib
        hb = lib.mcnd_dist_ipc_handle_bytes()
        buf = ctypes.create_string_buffer(hb)
        h = ctypes.c_void_p()
        _lib.check(lib.mcnd_dist_create(self.rank, self.world, self.n, ctypes.byref(h), buf))
        self.handle = h
        objs = [None] * self.world
        dist.all_gather_object(objs, bytes(buf.raw), group=group)
        allb = ctypes.create_string_buffer(b"".join(objs), hb * self.world)
        _lib.check(lib.mcnd_dist_connect(self.handle, allb))
        dist.barrier(group=group)
        self.last_device_ms = 0.0

    def local_rows(self):
        s, ln = self.plan.assignments[self.rank]
        return s, ln

    def mc_parallel(self, rows, *, fast: bool = False) -> RunResult:
        """rows: this rank's block (plan_blocks rows x n), float64 CUDA tensor."""
        import torch

        n, p = self.n, self.world
        s, ln = self.local_rows()
        if tuple(rows.shape) != (ln, n):
            raise ValueError(f"rank {self.rank} expects its block of shape {(ln, n)}, got {tuple(rows.shape)}")
        if rows.dtype != torch.float64 or rows.stride(1) != 1:
            rows = rows.to(torch.float64).contiguous()
        t0 = time.perf_counter()
        stream = torch.cuda.current_stream().cuda_stream
        piv = np.zeros(max(n - p, 1), dtype=np.float64)
        cols = np.zeros(max(n - p, 1), dtype=np.int32)
        sing = ctypes.c_int64(-1)
        rem = np.zeros(p, dtype=np.float64)
        wit = np.zeros(1, dtype=np.float64)
        dms = ctypes.c_double(0.0)
        # every rank's kernel waits on its peers: launch them together
        self.dist.barrier(group=self.group)
        rc = self.lib.mcnd_dist_mc_parallel(self.handle, rows.data_ptr(), n, rows.stride(0),
                                            _lib.FLAG_FAST if fast else 0, stream, piv.ctypes.data,
                                            cols.ctypes.data, ctypes.byref(sing), rem.ctypes.data,
                                            wit.ctypes.data, ctypes.byref(dms))
        _lib.check(rc)
        self.last_device_ms = float(dms.value)
        gathered = [None] * p
        self.dist.all_gather_object(gathered, (rem.tolist(), float(wit[0])), group=self.group)
        res = fold_gathered(n, p, piv, cols, int(sing.value), [g[0] for g in gathered], [g[1] for g in gathered])
        res.total_seconds = time.perf_counter() - t0
        res.stats.compute_seconds = self.last_device_ms / 1e3
        return res

    def close(self):
        if self.handle:
            self.lib.mcnd_dist_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


def bench_main(args):
    """bench.py --gpus N under torchrun: C3 on N GPUs (strong scaling)."""
    import json
    import statistics

    import torch
    import torch.distributed as dist

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", rank))
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29511")
    os.environ.setdefault("RANK", str(rank))
    os.environ.setdefault("WORLD_SIZE", str(world))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import bench as B

    name, a, n = B.workload(args.config)
    if a.ndim != 2:
        raise SystemExit("multi-GPU bench needs a single-matrix config")
    grp = BlockRowGroup(n)
    s, ln = grp.local_rows()
    block = np.ascontiguousarray(a[s:s + ln])
    d = torch.from_numpy(block).cuda()
    h = torch.empty(block.shape, dtype=torch.float64, pin_memory=True)
    h.numpy()[...] = block
    for _ in range(args.warmup):
        res = grp.mc_parallel(d, fast=args.fast)
    torch.cuda.synchronize()
    dist.barrier()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    kms = []
    with B.ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            res = grp.mc_parallel(d, fast=args.fast)
            kms.append(grp.last_device_ms)
        e1.record(stream)
        torch.cuda.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1) / args.steps], device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    km = torch.tensor([statistics.mean(kms)], device="cuda")
    dist.all_reduce(km, op=dist.ReduceOp.MAX)
    # e2e: block rows from pinned host memory each step, result back to the host
    dist.barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for _ in range(args.steps):
        dd = h.cuda(non_blocking=True)
        res_e = grp.mc_parallel(dd, fast=args.fast)
    f1.record(stream)
    torch.cuda.synchronize()
    ms_e = torch.tensor([f0.elapsed_time(f1) / args.steps], device="cuda")
    dist.all_reduce(ms_e, op=dist.ReduceOp.MAX)
    assert res_e.logdet == res.logdet
    grp.close()
    if rank == 0:
        t = float(ms.item())
        hbm, peak_kind = B.peaks()
        Bb = B.algorithmic_bytes(n)
        achieved = Bb / (float(km.item()) * 1e-3) / 1e9
        line = {
            "metric": B.metric_name(args.config), "value": B.flops(n) / (t * 1e-3) / 1e9, "unit": "GFLOP/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t,
            "time_to_logdet_s": t / 1e3, "kernel_ms": float(km.item()), "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": (B.PAPER_TABLE3_N8000.get(world) / (t / 1e3)) if (args.config == "c3" and world in B.PAPER_TABLE3_N8000) else None,
            "dtype": "f64", "data": "synthetic (numpy PCG64 seed, BASELINE recipe)",
            "config": {"workload": name, "n": n, "parallelism": f"block-row x{world} GPUs, pivot rows pushed over NVLink",
                       "mode": "fast-fma" if args.fast else "reference-exact",
                       "l2": "input larger than L2 per rank" if 8 * n * n / world > 126e6 else "per-rank block fits L2"},
            "result": {"sign": res.logdet.sign, "log_abs": res.logdet.log_abs,
                       "broadcasts": res.stats.broadcasts},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm * world, "peak_kind": peak_kind + f" x{world}",
                         "unit": "GB/s", "frac": achieved / (hbm * world), "traffic": None},
            "e2e": {"value": B.flops(n) / (float(ms_e.item()) * 1e-3) / 1e9, "unit": "GFLOP/s",
                    "ms_per_step": float(ms_e.item()), "h2d_bytes_per_step": int(block.nbytes) * world,
                    "d2h_bytes_per_step": (12 * n + 8 * world) * world},
            "gpu_launches": args.steps * world,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()

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


_PIVREC = np.dtype([("v", "<f8"), ("l", "<i4"), ("flag", "<u4")])


def blocked_schedule(n: int, world: int, tail: int = 64, b: int = 64):
    """Host schedule of the multi-GPU blocked condensation (deterministic, identical
    on every rank).  Rows: contiguous blocks (plan_blocks, runtime.py:33-44).  Each
    panel pair (2b rows) comes from the rank holding the most live rows, ties ->
    lowest rank (north_star (3)), as that rank's topmost 2b live rows; the pivot
    position k_pos = live rows of the ranks before it (runtime.py:158-160).  Returns
    (pairs, tops, lives, t_tail): pairs = [(owner, local_row0, t, m, k_pos)]."""
    plan = plan_blocks(n, world)
    live = [ln for (_, ln) in plan.assignments]
    top = [0] * world
    pairs = []
    t = 0
    while True:
        m = n - t
        o = max(range(world), key=lambda r: (live[r], -r))
        if live[o] < 2 * b or m - 2 * b < max(tail, 2):
            break
        pairs.append((o, top[o], t, m, sum(live[:o])))
        live[o] -= 2 * b
        top[o] += 2 * b
        t += 2 * b
    return pairs, top, live, t


def blocked_pivot_sequence(n: int, world: int, tail: int = 64):
    """Original row ids in the order the blocked multi-GPU schedule eliminates them
    (for the oracle: logdet_condensation(a, pivot_sequence=...))."""
    plan = plan_blocks(n, world)
    pairs, top, live, _ = blocked_schedule(n, world, tail)
    seq = []
    for (o, lr0, _, _, _) in pairs:
        s0 = plan.assignments[o][0]
        seq.extend(range(s0 + lr0, s0 + lr0 + 128))
    for r in range(world):  # tail: the remaining rows top to bottom in global order
        s0 = plan.assignments[r][0]
        seq.extend(range(s0 + top[r], s0 + top[r] + live[r]))
    return seq[: n - 1]


class BlockedGroup:
    """Multi-GPU BLOCKED condensation over the ranks of a torch.distributed group
    (one GPU per rank, current device set).  Per panel pair: the owner factors its
    2x64 rows (mcnd_mg_pair), W / Wp / the gather descriptor are broadcast, every
    rank applies the rank-128 update to its own live rows (mcnd_mg_trailing); the
    last rows are all-gathered and finished by K1 on every rank (mcnd_mg_tail).
    Kernels = the single-GPU K2 kernels ("one broadcast per panel
    of W").  Same result type as logdet_condensation; parity by tolerance."""

    def __init__(self, n: int, group=None, tail: int | None = None, native: bool | None = None):
        import torch
        import torch.distributed as dist

        self.torch, self.dist, self.group = torch, dist, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.nccl = dist.get_backend(group) == "nccl"
        self.n = int(n)
        self.plan = plan_blocks(self.n, self.world)
        self.row0, self.rows = self.plan.assignments[self.rank]
        self.tail = int(os.environ.get("MCND_K2_TAIL", 64) if tail is None else tail)
        self.pairs, self.tops, self.lives, self.t_tail = blocked_schedule(self.n, self.world, self.tail)
        lib = _lib.load()
        self.lib = lib
        h = ctypes.c_void_p()
        _lib.check(lib.mcnd_mg_create(self.n, self.rows, ctypes.byref(h)))
        self.h = h
        dev = torch.device("cuda", torch.cuda.current_device())
        wmax = 128 * (self.n - 64 + 1)
        self.W = [torch.empty(wmax, dtype=torch.float64, device=dev) for _ in range(2)]
        self.Wp = [torch.empty(64 * 64, dtype=torch.float64, device=dev) for _ in range(2)]
        gb = int(lib.mcnd_mg_gather_bytes())
        self.gp = [torch.zeros(gb, dtype=torch.uint8, device=dev) for _ in range(2)]
        # MCND_MG_FORCE_COMM=1: run the broadcast/comm-stream path even with one rank (test hook)
        self.force_comm = os.environ.get("MCND_MG_FORCE_COMM", "0") == "1"
        self.comm = torch.cuda.Stream() if (self.nccl and (self.world > 1 or self.force_comm)) else None
        # the panel chain on a high-priority stream, overlapped trailing updates on a low one
        self.crit = torch.cuda.Stream(priority=-1)
        self.side = self.crit if os.environ.get("MCND_MG_SERIAL", "0") == "1" else torch.cuda.Stream(priority=0)
        self.last_device_ms = 0.0
        self.last_launches = 0
        # the native driver (mcnd_mg_logdet: the per-pair loop in C++, NCCL on the library's own
        # communicator) whenever the group is NCCL or a single rank; the Python loop below stays
        # for gloo groups (host-staged broadcasts: the CPU / shared-GPU tests)
        self.native = (self.nccl or self.world == 1) if native is None else bool(native)
        if self.native and not self.nccl and self.world > 1:
            # gloo group (tests: ranks sharing one GPU): the native driver with host collectives
            import torch as _t

            def _bcast(ptr, nbytes, root):
                try:
                    t = _t.frombuffer((ctypes.c_ubyte * nbytes).from_address(ptr), dtype=_t.uint8)
                    dist.broadcast(t, root, group=self.group)
                    return 0
                except Exception:  # pragma: no cover
                    return 1

            def _allgather(send, recv, nbytes):
                try:
                    s = _t.frombuffer((ctypes.c_ubyte * nbytes).from_address(send), dtype=_t.uint8)
                    r = _t.frombuffer((ctypes.c_ubyte * (nbytes * self.world)).from_address(recv), dtype=_t.uint8)
                    dist.all_gather(list(r.view(self.world, nbytes).unbind(0)), s, group=self.group)
                    return 0
                except Exception:  # pragma: no cover
                    return 1

            self._cbs = (_lib.HOST_BCAST(_bcast), _lib.HOST_ALLGATHER(_allgather))  # kept alive
            _lib.check(lib.mcnd_mg_attach_host(h, self.world, self.rank, *self._cbs))
        elif self.native:
            idb = int(lib.mcnd_nccl_id_bytes())
            uid = bytes(idb)
            need = self.world > 1 or self.force_comm
            if need and self.rank == 0:
                buf = ctypes.create_string_buffer(idb)
                _lib.check(lib.mcnd_nccl_unique_id(buf))
                uid = buf.raw
            if need and self.world > 1:
                box = [uid]
                dist.broadcast_object_list(box, src=0, group=self.group)
                uid = box[0]
            _lib.check(lib.mcnd_mg_attach(h, self.world, self.rank, uid if need else None, 1 if need else 0))

    def _bcast(self, t, src):
        if self.world == 1:
            return
        if self.nccl:
            self.dist.broadcast(t, src, group=self.group)
        else:  # gloo (tests): host staging
            c = t.cpu()
            self.dist.broadcast(c, src, group=self.group)
            t.copy_(c)

    def _all_gather(self, t):
        """all_gather of equal-shape device tensors -> list (rank order)."""
        if self.world == 1:
            return [t]
        if self.nccl:
            out = [self.torch.empty_like(t) for _ in range(self.world)]
            self.dist.all_gather(out, t, group=self.group)
            return out
        out = [self.torch.empty_like(t, device="cpu") for _ in range(self.world)]
        self.dist.all_gather(out, t.cpu(), group=self.group)
        return [o.to(t.device) for o in out]

    def logdet(self, rows) -> LogDet:
        """rows: this rank's block (plan_blocks rows x n), float64 CUDA tensor."""
        import math

        torch, lib, h = self.torch, self.lib, self.h
        n, rank = self.n, self.rank
        if tuple(rows.shape) != (self.rows, n):
            raise ValueError(f"rank {rank} expects its block of shape {(self.rows, n)}, got {tuple(rows.shape)}")
        if rows.dtype != torch.float64 or rows.stride(1) != 1:
            rows = rows.to(torch.float64).contiguous()
        if self.native:
            out = _lib.McndLogDet()
            _lib.check(lib.mcnd_mg_logdet(h, rows.data_ptr(), rows.stride(0), self.tail,
                                          torch.cuda.current_stream().cuda_stream, ctypes.byref(out)))
            self.last_device_ms = float(out.device_ms)
            self.last_launches = int(out.launches)
            return SINGULAR if out.singular else LogDet(int(out.sign), float(out.log_abs))
        cur = torch.cuda.current_stream()
        crit, side = self.crit, self.side
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(cur)
        crit.wait_stream(cur)
        side.wait_stream(cur)
        hc, hs = crit.cuda_stream, side.cuda_stream
        _lib.check(lib.mcnd_mg_load(h, rows.data_ptr(), rows.stride(0), hc))
        nl = 1  # kernels launched on this rank
        plan = self.plan
        live = [ln for (_, ln) in plan.assignments]
        top = [0] * self.world
        pairs = self.pairs
        comm = self.comm
        ev_pair = [torch.cuda.Event(), torch.cuda.Event()]
        ev_bc = [torch.cuda.Event(), torch.cuda.Event()]
        ev_trc = [torch.cuda.Event(), torch.cuda.Event()]  # crit / side users of W[q & 1] done
        ev_trs = [torch.cuda.Event(), torch.cuda.Event()]
        ev_side = torch.cuda.Event()
        ev_crit = torch.cuda.Event()  # the next owner's critical rows updated (releases the side update)
        side_pending = False

        def ldw_of(m):
            return (m - 64 + 1) // 2 * 2

        def launch_pair(q):
            o, lr0, t, m, _ = pairs[q]
            W, Wp, gp = self.W[q & 1], self.Wp[q & 1], self.gp[q & 1]
            _lib.check(lib.mcnd_mg_pair(h, lr0, t, m, W.data_ptr(), ldw_of(m), Wp.data_ptr(), gp.data_ptr(), hc))
            ev_pair[q & 1].record(crit)

        def trailing(r0, nrows, m, W, ldw, Wp, gp, q, on_side):
            _lib.check(lib.mcnd_mg_trailing(h, r0, nrows, m, W.data_ptr(), ldw, Wp.data_ptr(), gp.data_ptr(),
                                            -1 if on_side else 0, q & 1, hs if on_side else hc))

        if pairs and pairs[0][0] == rank:
            launch_pair(0)
            nl += 2
        for q, (o, lr0, t, m, _) in enumerate(pairs):
            W, Wp, gp = self.W[q & 1], self.Wp[q & 1], self.gp[q & 1]
            ldw = ldw_of(m)
            if comm is not None:
                # broadcast on its own stream: it waits only for the pair (owner) and for the
                # buffer's previous users (pair q-2's updates on this rank)
                if rank == o:
                    comm.wait_event(ev_pair[q & 1])
                if q >= 2:
                    comm.wait_event(ev_trc[q & 1])
                    comm.wait_event(ev_trs[q & 1])
                with torch.cuda.stream(comm):
                    self.dist.broadcast(W[: 128 * ldw], o, group=self.group)
                    self.dist.broadcast(Wp, o, group=self.group)
                    self.dist.broadcast(gp, o, group=self.group)
                ev_bc[q & 1].record(comm)
                crit.wait_event(ev_bc[q & 1])
                side.wait_event(ev_bc[q & 1])
            elif self.world == 1:
                side.wait_event(ev_pair[q & 1])  # the side update reads the pair's W, Wp, descriptor
            else:  # gloo (tests): synchronous host-staged broadcasts
                crit.synchronize()
                side.synchronize()
                self._bcast(W[: 128 * ldw], o)
                self._bcast(Wp, o)
                self._bcast(gp, o)
                crit.wait_stream(cur)  # the host-staged copies landed on the caller's stream
                side.wait_stream(cur)
            live[o] -= 128
            top[o] += 128
            # look-ahead: the next owner updates the 128 rows it contributes next on the
            # high-priority stream, factors them at once (its broadcast can start), and
            # updates the rest on the low-priority stream meanwhile (single-GPU schedule)
            nxt = pairs[q + 1][0] if q + 1 < len(pairs) else -1
            r0, rows_r = top[rank], live[rank]
            if side_pending:  # rows about to be touched on crit were last updated on side
                crit.wait_event(ev_side)
                side_pending = False
            if nxt == rank and rows_r > 128:
                trailing(r0, 128, m, W, ldw, Wp, gp, q, False)
                ev_crit.record(crit)
                launch_pair(q + 1)
                # the side update is released only after the critical rows' update (its CTAs
                # would otherwise take the SMs the critical kernels need; single-GPU schedule)
                side.wait_event(ev_crit)
                trailing(r0 + 128, rows_r - 128, m, W, ldw, Wp, gp, q, True)
                ev_side.record(side)
                side_pending = True
                nl += 2 + 4
            else:
                if rows_r > 0:
                    trailing(r0, rows_r, m, W, ldw, Wp, gp, q, False)
                    nl += 2
                if nxt == rank:
                    launch_pair(q + 1)
                    nl += 2
            ev_trc[q & 1].record(crit)
            ev_trs[q & 1].record(side)
        crit.wait_stream(side)
        cur.wait_stream(crit)
        stream = cur.cuda_stream
        # tail: every rank's remaining rows (first mt columns), gathered in rank order
        mt = n - self.t_tail
        ldr = (mt + 1) // 2 * 2
        rmax = max(live)
        dev = rows.device
        buf = torch.zeros((max(rmax, 1), ldr), dtype=torch.float64, device=dev)
        wbuf = torch.zeros(max(rmax, 1), dtype=torch.float64, device=dev)
        if live[rank] > 0:
            _lib.check(lib.mcnd_mg_export(h, top[rank], live[rank], mt, buf.data_ptr(), ldr, wbuf.data_ptr(), stream))
        bufs = self._all_gather(buf)
        wbufs = self._all_gather(wbuf)
        tail_rows = torch.cat([bufs[r][: live[r]] for r in range(self.world)]).contiguous()
        tail_wit = torch.cat([wbufs[r][: live[r]] for r in range(self.world)]).contiguous()
        trec = np.zeros(mt, dtype=_PIVREC)
        terr = np.zeros(4, dtype=np.uint32)
        stream = torch.cuda.current_stream().cuda_stream
        _lib.check(lib.mcnd_mg_tail(h, tail_rows.data_ptr(), ldr, tail_wit.data_ptr(), mt, stream, trec.ctypes.data,
                                    terr.ctypes.data))
        self.last_launches = nl + 1
        rec = np.zeros(n, dtype=_PIVREC)
        err = np.zeros(4, dtype=np.uint32)
        _lib.check(lib.mcnd_mg_records(h, rec.ctypes.data, err.ctypes.data, stream))
        e1.record()
        e1.synchronize()
        self.last_device_ms = e0.elapsed_time(e1)
        if self.world > 1:
            gathered = [None] * self.world
            self.dist.all_gather_object(gathered, (rec.tobytes(), err.tolist()), group=self.group)
        else:
            gathered = [(rec.tobytes(), err.tolist())]
        recs = [np.frombuffer(g[0], dtype=_PIVREC) for g in gathered]
        errs = [g[1] for g in gathered]
        if any(e[2] for e in errs) or terr[2]:
            raise ValueError("matrix entries must be finite (no NaN/Inf)")
        if any(e[0] for e in errs) or terr[0]:
            raise RuntimeError(f"mcnd_b200 multi-GPU blocked: device timeout (errors {errs}, tail {terr.tolist()})")
        # fold: the reference's sign / log bookkeeping (condense.py:124-128, 159-160) in step order
        sign, log_acc = 1, 0.0
        for (o, lr0, t, m, kpos) in self.pairs:
            ro, ep = recs[o], errs[o][3]
            for s_ in range(128):
                v, l, fl = float(ro["v"][t + s_]), int(ro["l"][t + s_]), int(ro["flag"][t + s_])
                if fl != ep or l < 0:
                    return SINGULAR
                ms = m - s_
                sign *= (1 if v > 0 else -1) * (-1 if l != ms - 1 else 1) * (-1 if (kpos + ms - 1) & 1 else 1)
                log_acc += math.log(abs(v))
        ep0 = errs[rank][3]
        for j in range(mt):
            v, l, fl = float(trec["v"][j]), int(trec["l"][j]), int(trec["flag"][j])
            if fl != ep0 or l < 0:
                return SINGULAR
            mj = mt - j
            if j < mt - 1:
                sign *= (1 if v > 0 else -1) * (-1 if l != mj - 1 else 1) * (-1 if (mj - 1) & 1 else 1)
            else:
                sign *= 1 if v > 0 else -1
            log_acc += math.log(abs(v))
        return LogDet(sign, log_acc)

    def close(self):
        if self.h:
            self.lib.mcnd_mg_destroy(self.h)
            self.h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


def bench_main(args):
    """bench.py --gpus N under torchrun: one matrix, block rows over N GPUs (strong
    scaling).  Default method as on one GPU: blocked for N >= 2048 (BlockedGroup:
    panel pairs from the rank with the most live rows, W broadcast, local rank-128
    updates), unblocked below (BlockRowGroup: pivot rows pushed over NVLink)."""
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
    if a.ndim == 3:
        return _bench_batched(args, B, name, a, n, rank, world, local)
    method = args.method or ("unblocked" if n < 2048 else "blocked")
    if method == "blocked":
        grp = BlockedGroup(n)
        s, ln = grp.row0, grp.rows
        run = lambda d: grp.logdet(d)
    else:
        grp = BlockRowGroup(n)
        s, ln = grp.local_rows()
        run = lambda d: grp.mc_parallel(d, fast=args.fast).logdet
    if isinstance(a, np.ndarray):
        block = np.ascontiguousarray(a[s:s + ln])
        d = torch.from_numpy(block).cuda()
    else:  # device-generated workload (C5)
        d = a[s:s + ln].contiguous()
        block = None
    h = torch.empty(tuple(d.shape), dtype=torch.float64, pin_memory=True)
    h.copy_(d)
    nbytes = h.numel() * 8
    for _ in range(args.warmup):
        res = run(d)
    torch.cuda.synchronize()
    dist.barrier()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    kms = []
    launches0 = 0
    with B.ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            res = run(d)
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
        res_e = run(dd)
    f1.record(stream)
    torch.cuda.synchronize()
    ms_e = torch.tensor([f0.elapsed_time(f1) / args.steps], device="cuda")
    dist.all_reduce(ms_e, op=dist.ReduceOp.MAX)
    assert res_e == res
    lt = torch.tensor([getattr(grp, "last_launches", 1) * args.steps], device="cuda")
    dist.all_reduce(lt)  # every rank's kernels
    launches = int(lt.item())
    grp.close()
    peak = B.fp64_peak(local) if (rank == 0 and method == "blocked") else None
    if rank == 0:
        t = float(ms.item())
        hbm, peak_kind = B.peaks()
        if method == "blocked":
            achieved = B.flops(n) / (float(km.item()) * 1e-3) / 1e12
            pk = peak["tflops"]
            roof = {"bound": "tensor", "achieved": achieved, "peak": pk * world,
                    "peak_kind": peak["how"] + f" (rank 0) x{world}", "unit": "TFLOP/s",
                    "frac": achieved / (pk * world), "traffic": None}
        else:
            Bb = B.algorithmic_bytes(n)
            achieved = Bb / (float(km.item()) * 1e-3) / 1e9
            roof = {"bound": "hbm", "achieved": achieved, "peak": hbm * world, "peak_kind": peak_kind + f" x{world}",
                    "unit": "GB/s", "frac": achieved / (hbm * world), "traffic": None}
        line = {
            "metric": B.metric_name(args.config), "value": B.flops(n) / (t * 1e-3) / 1e9, "unit": "GFLOP/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t,
            "time_to_logdet_s": t / 1e3, "kernel_ms": float(km.item()), "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": (B.PAPER_TABLE3_N8000.get(world) / (t / 1e3)) if (args.config == "c3" and world in B.PAPER_TABLE3_N8000) else None,
            "dtype": "f64", "data": "synthetic (numpy PCG64 seed, BASELINE recipe)",
            "config": B.bench_config(args, name, n, world),
            "result": {"sign": res.sign, "log_abs": res.log_abs},
            "roofline": roof,
            "e2e": {"value": B.flops(n) / (float(ms_e.item()) * 1e-3) / 1e9, "unit": "GFLOP/s",
                    "ms_per_step": float(ms_e.item()), "h2d_bytes_per_step": int(nbytes) * world,
                    "d2h_bytes_per_step": 16 * n * world},
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def _bench_batched(args, B, name, a, n, rank, world, local):
    """C4 over N GPUs: the batch is sharded (contiguous slices), no exchange
    (replicas of K3); total batch fixed (strong scaling)."""
    import json
    import statistics

    import torch
    import torch.distributed as dist

    from .batched import logdet_batched

    plan = plan_blocks(a.shape[0], world)
    s, ln = plan.assignments[rank]
    d = torch.from_numpy(np.ascontiguousarray(a[s:s + ln])).cuda()
    for _ in range(args.warmup):
        logdet_batched(d, fast=args.fast)
    torch.cuda.synchronize()
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
    stream = torch.cuda.current_stream()
    times = []
    with B.ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.fill_(1.0)
            dist.barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            sg, lg = logdet_batched(d, fast=args.fast)
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
    ms = torch.tensor([statistics.mean(times)], device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    h = torch.empty(d.shape, dtype=torch.float64, pin_memory=True)
    h.copy_(d)
    logdet_batched(h.numpy(), fast=args.fast)
    dist.barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for _ in range(args.steps):
        logdet_batched(h.numpy(), fast=args.fast)
    f1.record(stream)
    torch.cuda.synchronize()
    ms_e = torch.tensor([f0.elapsed_time(f1) / args.steps], device="cuda")
    dist.all_reduce(ms_e, op=dist.ReduceOp.MAX)
    if rank == 0:
        t = float(ms.item())
        hbm, peak_kind = B.peaks()
        byt = a.nbytes + a.shape[0] * 12
        fl = a.shape[0] * B.flops(n)
        line = {"metric": B.metric_name("c4"), "value": fl / (t * 1e-3) / 1e9, "unit": "GFLOP/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": t, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (numpy PCG64 seed 4)",
                "config": B.bench_config(args, name, n, world, batch=a.shape[0]),
                "roofline": {"bound": "hbm", "achieved": byt / (t * 1e-3) / 1e9, "peak": hbm * world,
                             "peak_kind": peak_kind + f" x{world}", "unit": "GB/s",
                             "frac": byt / (t * 1e-3) / 1e9 / (hbm * world), "traffic": None},
                "e2e": {"value": fl / (float(ms_e.item()) * 1e-3) / 1e9, "unit": "GFLOP/s",
                        "ms_per_step": float(ms_e.item()), "h2d_bytes_per_step": a.nbytes,
                        "d2h_bytes_per_step": a.shape[0] * 12},
                "gpu_launches": args.steps * world, "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()

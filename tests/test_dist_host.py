"""Multi-process (gloo, world_size 2 and 3) CPU tests of the block-row driver's
host side: plan, schedule, the all-gather of the remaining rows and the fold
into (sign, log|det|) + accounting (runtime.py:206-229).

Each rank plays one worker.  The per-step pivots and the remaining rows come
from the oracle (what every rank's GPU kernel would hand back); the ranks
exchange their remaining row through torch.distributed (gloo) exactly as
dist.BlockRowGroup does and fold with the C-ABI's host-only
mcnd_fold_mc_parallel.  The result must equal the reference's mc_parallel
bitwise, on every rank.
"""

import os
import socket

import numpy as np
import pytest

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n, seed, kind, q):
    import sys

    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import mcnd_oracle as O
        from paper_1811_08057_b200 import dist as D
        from paper_1811_08057_b200 import matrix as M
        from paper_1811_08057_b200.runtime import plan_blocks

        if kind == "planted":
            a = M.generate(M.MatrixSpec(n, "singular-planted", seed))
        else:
            a = np.random.default_rng(seed).uniform(-1, 1, (n, n))
        ref = O.mc_parallel(a, world)
        s, ln = plan_blocks(n, world).assignments[rank]
        # what this rank's kernel returns: all pivots + its own remaining row/witness
        singular_at = ref.aborted_step
        k = (singular_at + 1) if singular_at >= 0 else n - world
        my_row = ref.rem[rank].tolist()
        my_wit = float(ref.rem_wit[rank])
        gathered = [None] * world
        dist.all_gather_object(gathered, (my_row, my_wit))
        res = D.fold_gathered(n, world, ref.pivots[:k], ref.cols[:k], singular_at,
                              [g[0] for g in gathered], [g[1] for g in gathered])
        ok = (res.logdet.sign == ref.sign and (res.logdet.log_abs == ref.log_abs
              or (np.isinf(ref.log_abs) and np.isinf(res.logdet.log_abs)))
              and res.stats.broadcasts == ref.broadcasts and res.stats.broadcast_bytes == ref.broadcast_bytes
              and res.row_updates == ref.row_updates and res.scalar_updates == ref.scalar_updates
              and res.broadcast_payload_entries == ref.payload_entries)
        q.put((rank, ok, (res.logdet, (ref.sign, ref.log_abs)), (s, ln)))
    except Exception as e:  # pragma: no cover - surfaced by the assert below
        q.put((rank, False, repr(e), None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,seed,kind", [(2, 64, 1, "uniform"), (2, 101, 2, "uniform"),
                                               (3, 50, 3, "uniform"), (2, 16, 16, "planted"),
                                               (3, 17, 5, "uniform")])
def test_gloo_gather_and_fold_matches_reference(world, n, seed, kind):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, seed, kind, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, detail, _ in sorted(results, key=lambda x: x[0]):
        assert ok, f"rank {rank}: {detail}"
    # the block plan each rank used tiles [0, n)
    spans = sorted(r[3] for r in results)
    assert spans[0][0] == 0 and sum(ln for _, ln in spans) == n


def test_round_robin_owner_equals_most_live_rows_when_divisible():
    """north_star owner rule ("rank with the most live rows, ties -> lowest")
    coincides with the reference's round-robin (runtime.py:153-156) for p | n."""
    from paper_1811_08057_b200.runtime import plan_blocks

    for n, p in ((1000, 1), (4000, 2), (8000, 2), (8000, 4), (8000, 8), (64, 8), (96, 3)):
        lens = [ln for _, ln in plan_blocks(n, p).assignments]
        consumed = [0] * p
        rr = []
        while any(lens[w] - consumed[w] > 1 for w in range(p)):
            for w in range(p):
                if lens[w] - consumed[w] <= 1:
                    continue
                rr.append(w)
                consumed[w] += 1
        consumed = [0] * p
        most = []
        for _ in range(n - p):
            live = [lens[w] - consumed[w] for w in range(p)]
            w = max(range(p), key=lambda u: (live[u], -u))
            most.append(w)
            consumed[w] += 1
        assert rr == most, (n, p)


# ---- multi-GPU blocked schedule (host logic of dist.BlockedGroup) ----
@pytest.mark.parametrize("n,world,tail", [(8000, 8, 256), (8000, 2, 256), (4000, 2, 256), (1000, 3, 100),
                                          (700, 2, 2), (32768, 8, 256)])
def test_blocked_schedule_invariants(n, world, tail):
    from paper_1811_08057_b200.dist import blocked_schedule, blocked_pivot_sequence
    from paper_1811_08057_b200.runtime import plan_blocks

    plan = plan_blocks(n, world)
    pairs, top, live, t_tail = blocked_schedule(n, world, tail)
    lv = [ln for (_, ln) in plan.assignments]
    tp = [0] * world
    t = 0
    for (o, lr0, tt, m, kpos) in pairs:
        assert tt == t and m == n - t
        assert lv[o] == max(lv) and all(lv[r] < lv[o] for r in range(o))  # most live rows, ties -> lowest
        assert lr0 == tp[o] and lv[o] >= 128
        assert kpos == sum(lv[:o])
        lv[o] -= 128
        tp[o] += 128
        t += 128
    assert (tp, lv, t) == (top, live, t_tail)
    assert sum(live) == n - t_tail and n - t_tail >= 2
    seq = blocked_pivot_sequence(n, world, tail)
    assert len(seq) == n - 1 and len(set(seq)) == n - 1 and all(0 <= r < n for r in seq)


def test_blocked_pivot_sequence_oracle_consistent():
    """The schedule's pivot order is a valid reference pivot_sequence (condense.py:147-152):
    the oracle accepts it and lands within tolerance of the top-to-bottom result."""
    from oracle import mcnd_oracle as O
    from paper_1811_08057_b200.dist import blocked_pivot_sequence

    a = np.random.default_rng(5).uniform(-1, 1, (600, 600))
    ref = O.logdet_condensation(a)
    for world in (1, 2, 3):
        seq = np.array(blocked_pivot_sequence(600, world, 2), dtype=np.int64)
        got = O.logdet_condensation(a, pivot_sequence=seq)
        assert got.sign == ref.sign
        assert abs(got.log_abs - ref.log_abs) <= max(1e-8 * 600, 1e-10 * abs(ref.log_abs))


def test_native_schedule_matches_python():
    """The C++ pair schedule of the native driver (mcnd_mg_schedule) is dist.blocked_schedule."""
    import ctypes

    from paper_1811_08057_b200 import _lib
    from paper_1811_08057_b200 import dist as D

    lib = _lib.load()
    for n, world, tail in [(300, 1, 2), (1000, 2, 64), (4000, 2, 64), (8000, 8, 64), (8001, 3, 100),
                           (10007, 5, 256), (32768, 8, 64), (129, 2, 2), (1100, 4, 256)]:
        pairs, _, _, _ = D.blocked_schedule(n, world, tail)
        buf = np.zeros((max(len(pairs), 1), 5), dtype=np.int64)
        k = lib.mcnd_mg_schedule(n, world, tail, buf.ctypes.data, buf.shape[0])
        assert k == len(pairs)
        assert [tuple(int(x) for x in r) for r in buf[:k]] == [tuple(p) for p in pairs]

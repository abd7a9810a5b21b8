"""Multi-GPU BLOCKED condensation (dist.BlockedGroup, csrc mcnd_mg_*): the per-rank
engine and the host schedule, checked against the oracle run with the SAME pivot
order (logdet_condensation(a, pivot_sequence=...), condense.py:147-152).

World size 1 runs in-process; world size 2 runs two processes that share cuda:0
over gloo: their kernels never wait on one another (every exchange is a host-side
collective), so this is a faithful test of the protocol on one GPU."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def tol(n, la):
    return max(1e-8 * n, 1e-10 * abs(la))


@pytest.fixture(scope="module")
def mc():
    import torch

    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    import paper_1811_08057_b200 as mc

    return mc


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, seed, tail, out_path):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1811_08057_b200 import dist as D

    a = np.random.default_rng(seed).uniform(-1, 1, (n, n))
    g = D.BlockedGroup(n, tail=tail)  # the Python loop (host-staged broadcasts)
    s, ln = g.plan.assignments[rank]
    res = g.logdet(torch.from_numpy(np.ascontiguousarray(a[s:s + ln])).cuda())
    res2 = g.logdet(torch.from_numpy(np.ascontiguousarray(a[s:s + ln])).cuda())  # reuse of the handle
    g.close()
    # the native per-rank driver (mcnd_mg_logdet) with its collectives over gloo: the same
    # kernels in the same order on every rank -> the same result to the last bit
    gn = D.BlockedGroup(n, tail=tail, native=True)
    res3 = gn.logdet(torch.from_numpy(np.ascontiguousarray(a[s:s + ln])).cuda())
    gn.close()
    if rank == 0:
        np.save(out_path, np.array([res.sign, res.log_abs, res2.sign, res2.log_abs, res3.sign, res3.log_abs]))
    dist.barrier()
    dist.destroy_process_group()


def _oracle(a, world, tail):
    from oracle import mcnd_oracle as O
    from paper_1811_08057_b200 import dist as D

    seq = D.blocked_pivot_sequence(a.shape[0], world, tail)
    return O.logdet_condensation(a, pivot_sequence=np.array(seq, dtype=np.int64))


@pytest.mark.parametrize("n,tail", [(300, 2), (700, 100), (1100, 256)])
def test_mg_world1_vs_oracle(mc, n, tail):
    import torch
    import torch.distributed as dist
    from paper_1811_08057_b200 import dist as D

    port = _port()
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        a = np.random.default_rng(n).uniform(-1, 1, (n, n))
        g = D.BlockedGroup(n, tail=tail)
        got = g.logdet(torch.from_numpy(a).cuda())
        g.close()
    finally:
        dist.destroy_process_group()
    ref = _oracle(a, 1, tail)
    assert got.sign == ref.sign
    assert abs(got.log_abs - ref.log_abs) <= tol(n, ref.log_abs)


@pytest.mark.parametrize("n,tail,world", [(700, 2, 2), (1500, 256, 2), (2000, 64, 3)])
def test_mg_world2_gloo_vs_oracle(mc, tmp_path, n, tail, world):
    import torch.multiprocessing as tmp

    out = str(tmp_path / "res.npy")
    tmp.start_processes(_worker, args=(world, _port(), n, 7, tail, out), nprocs=world, join=True, start_method="spawn")
    r = np.load(out)
    a = np.random.default_rng(7).uniform(-1, 1, (n, n))
    ref = _oracle(a, world, tail)
    assert int(r[0]) == ref.sign and int(r[2]) == ref.sign
    assert abs(r[1] - ref.log_abs) <= tol(n, ref.log_abs)
    assert r[1] == r[3]  # deterministic across calls
    assert int(r[4]) == ref.sign and r[5] == r[1]  # native driver == Python loop, bitwise


def test_mg_singular_and_nonfinite(mc):
    import torch
    import torch.distributed as dist
    from paper_1811_08057_b200 import dist as D
    from paper_1811_08057_b200 import matrix as M

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{_port()}", rank=0, world_size=1)
    try:
        z = M.generate(M.MatrixSpec(400, "singular-planted", 3))
        g = D.BlockedGroup(400, tail=2)
        assert g.logdet(torch.from_numpy(z).cuda()) == mc.SINGULAR
        bad = np.eye(400)
        bad[7, 3] = np.nan
        with pytest.raises(ValueError, match="finite"):
            g.logdet(torch.from_numpy(bad).cuda())
        g.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [700, 1500, 4000])
def test_mg_native_driver_matches_python_loop(mc, n, monkeypatch):
    """mcnd_mg_logdet (the per-pair loop in C++) runs exactly the kernels of the Python loop in
    the same order: the same result to the last bit, without NCCL (one rank) and with the
    broadcasts issued through a one-rank NCCL communicator (MCND_MG_FORCE_COMM=1)."""
    import torch
    import torch.distributed as dist
    from paper_1811_08057_b200 import dist as D

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{_port()}", rank=0, world_size=1)
    try:
        a = torch.from_numpy(np.random.default_rng(n + 1).uniform(-1, 1, (n, n))).cuda()
        loop = D.BlockedGroup(n, native=False)
        ref = loop.logdet(a)
        loop.close()
        nat = D.BlockedGroup(n, native=True)
        got = [nat.logdet(a), nat.logdet(a)]
        assert nat.last_launches > 2 and nat.last_device_ms > 0
        nat.close()
        monkeypatch.setenv("MCND_MG_FORCE_COMM", "1")
        nc = D.BlockedGroup(n, native=True)
        got.append(nc.logdet(a))
        nc.close()
    finally:
        dist.destroy_process_group()
    assert all(g == ref for g in got), (got, ref)
    single = mc.logdet_blocked(a)
    assert single.sign == ref.sign and abs(single.log_abs - ref.log_abs) <= tol(n, ref.log_abs)

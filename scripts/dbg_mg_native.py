"""Debug: world-N gloo ranks on one GPU, the Python loop vs the native driver, repeated."""
import os, sys, socket
import numpy as np
import torch
import torch.multiprocessing as tmp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def worker(rank, world, port, n, tail, serial):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    if serial:
        os.environ["MCND_MG_SERIAL"] = "1"
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1811_08057_b200 import dist as D
    a = np.random.default_rng(7).uniform(-1, 1, (n, n))
    out = []
    for native in (False, True, True, False, True):
        g = D.BlockedGroup(n, tail=tail, native=native)
        s, ln = g.plan.assignments[rank]
        r = g.logdet(torch.from_numpy(np.ascontiguousarray(a[s:s + ln])).cuda())
        g.close()
        out.append((native, r.log_abs.hex()))
    if rank == 0:
        print(n, tail, world, "serial" if serial else "", out, flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    for n, tail, world in ((1500, 256, 2), (2000, 64, 3), (700, 2, 2)):
        for serial in (False,):
            s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
            tmp.start_processes(worker, args=(world, port, n, tail, serial), nprocs=world, join=True, start_method="spawn")

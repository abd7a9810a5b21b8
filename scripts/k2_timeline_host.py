"""Critical-stream timeline of one blocked call on a PINNED HOST matrix (streamed input):
run with MCND_DEBUG_TIMELINE=2; prints the device time of each step of the last call."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1811_08057_b200 as mc
from paper_1811_08057_b200 import matrix as M
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8000
host = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
host.copy_(torch.from_numpy(M.config_uniform(n, 3)))
for it in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = mc.logdet_blocked(host.numpy())
    torch.cuda.synchronize()
    print(f"call {it}: {1e3 * (time.perf_counter() - t0):.2f} ms wall", r, flush=True)

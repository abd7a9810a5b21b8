"""Time cuSOLVER LU (torch.linalg.slogdet, FP64) at the C3 / C2 / C5 sizes: the library
reference point for the blocked condensation (not our path)."""
import json, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1811_08057_b200 import matrix as M
out = {}
for name, n in [("c3", 8000), ("c2", 4000), ("n16384", 16384)]:
    a = torch.from_numpy(M.config_uniform(n, 3)).cuda()
    for _ in range(3):
        torch.linalg.slogdet(a)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(5):
        e0.record(); torch.linalg.slogdet(a); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    out[name] = {"n": n, "ms": sorted(ts)[len(ts) // 2], "gflops": 2 * n**3 / 3 / (sorted(ts)[len(ts) // 2] * 1e-3) / 1e9}
    del a
print(json.dumps(out))

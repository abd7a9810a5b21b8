"""Time the blocked K2 path at C3 (N=8000) and C5 (N=32768) on one GPU."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1811_08057_b200 as mc
from paper_1811_08057_b200 import matrix as M
out = {}
a = torch.from_numpy(M.config_uniform(8000, 3)).cuda()
for _ in range(2): r = mc.logdet_blocked(a, return_pivots=True)
ts = [mc.logdet_blocked(a, return_pivots=True)[3] for _ in range(3)]
out["c3_blocked"] = {"ms": ts, "res": list(r[0])}
out["c3_unblocked"] = {"res": list(mc.logdet_condensation(a))}
del a
for n in [int(x) for x in (sys.argv[1:] or ["16384", "32768"])]:
    a = M.config_spd_device(n, 5)
    torch.cuda.synchronize()
    t0 = time.time(); s, l = torch.linalg.slogdet(a); torch.cuda.synchronize(); tsl = time.time() - t0
    r = mc.logdet_blocked(a, return_pivots=True)
    r2 = mc.logdet_blocked(a, return_pivots=True)
    out[f"spd{n}"] = {"ms": [r[3], r2[3]], "res": list(r2[0]), "slogdet": [int(s.item()), float(l)], "slogdet_s": tsl,
                      "gflops": 2 * n**3 / 3 / (r2[3] * 1e-3) / 1e9}
    del a
    torch.cuda.empty_cache()
print(json.dumps(out))

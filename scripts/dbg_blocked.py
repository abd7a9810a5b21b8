"""Debug: repeated blocked C3 runs with the overlap knob (prints per-call status)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1811_08057_b200 as mc
from paper_1811_08057_b200 import matrix as M
a = torch.from_numpy(M.config_uniform(int(sys.argv[1]) if len(sys.argv) > 1 else 8000, 3)).cuda()
for ov in sys.argv[2:] or ["0", "1"]:
    os.environ["MCND_K2_OVERLAP"] = ov
    for i in range(4):
        t0 = time.time()
        try:
            r = mc.logdet_blocked(a, return_pivots=True)
            print(ov, i, r[0], r[3], flush=True)
        except Exception as e:
            print(ov, i, "ERR", e, time.time() - t0, flush=True)

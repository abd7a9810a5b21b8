"""One blocked logdet call at C3 (N=8000) or C5 (N=32768) after one warm-up call:
run under ncu (--launch-skip past the warm-up) for the per-call DRAM traffic."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1811_08057_b200 as mc
from paper_1811_08057_b200 import matrix as M
cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
a = torch.from_numpy(M.config_uniform(8000, 3)).cuda() if cfg == "c3" else M.config_spd_device(32768, 5)
torch.cuda.synchronize()
print("marker: start", flush=True)
r = mc.logdet_blocked(a, return_pivots=True)
print(cfg, r[0], r[3], flush=True)

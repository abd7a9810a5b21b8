"""One warm + one profiled condensation of a BASELINE config (for ncu -k regex:k1_condense)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1811_08057_b200 as mc
from paper_1811_08057_b200 import matrix as M
cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
if cfg == "c4":
    d = torch.from_numpy(M.config_batched_spd(4096, 64, 4)).cuda()
    for _ in range(2): print(mc.logdet_batched(d)[1][:2])
else:
    a = {"c1": lambda: M.config_dense_normal(1000, 1), "c2": lambda: M.config_spd(4000, 2),
         "c3": lambda: M.config_uniform(8000, 3)}[cfg]()
    d = torch.from_numpy(a).cuda()
    for _ in range(2): print(mc.logdet_condensation(d))
torch.cuda.synchronize()

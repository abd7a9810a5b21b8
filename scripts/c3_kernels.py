"""One blocked C3 logdet (for a per-kernel launch list under ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1811_08057_b200 as mc
from paper_1811_08057_b200 import matrix as M
a = torch.from_numpy(M.config_uniform(8000, 3)).cuda()
print(mc.logdet_blocked(a, return_pivots=True)[3])

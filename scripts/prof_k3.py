import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1811_08057_b200 as mc
from paper_1811_08057_b200 import matrix as M
d = torch.from_numpy(M.config_batched_spd(4096, 64, 4)).cuda()
for _ in range(3): s, l = mc.logdet_batched(d)
torch.cuda.synchronize(); print(l[:3])

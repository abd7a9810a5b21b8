"""Blocked K2 on an SPD matrix of size N (argv[1]), run twice (warm + profiled)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1811_08057_b200 as mc
from paper_1811_08057_b200 import matrix as M
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
a = M.config_spd_device(n, 5)
for _ in range(2):
    print(mc.logdet_blocked(a, return_pivots=True)[3])
torch.cuda.synchronize()

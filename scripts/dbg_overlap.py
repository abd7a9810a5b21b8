"""Debug: compare blocked pivots with and without the look-ahead overlap."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1811_08057_b200 as mc
from paper_1811_08057_b200 import matrix as M
for n in [int(x) for x in sys.argv[1:]] or [2000, 4000, 8000]:
    a = torch.from_numpy(M.config_uniform(n, 3)).cuda()
    os.environ["MCND_K2_OVERLAP"] = "0"
    r0 = mc.logdet_blocked(a, return_pivots=True)
    os.environ["MCND_K2_OVERLAP"] = "1"
    for rep in range(2):
        r1 = mc.logdet_blocked(a, return_pivots=True)
        d = np.nonzero((r0[1] != r1[1]) | (r0[2] != r1[2]))[0]
        print(n, rep, r0[0], r1[0], "first diff", d[:5], len(d), flush=True)

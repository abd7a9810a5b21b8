"""A/B an env knob on the blocked path: pivots (bitwise?) and device time."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1811_08057_b200 as mc
from paper_1811_08057_b200 import matrix as M
knob = sys.argv[1]
vals = sys.argv[2].split(",")
for n in [int(x) for x in sys.argv[3:]] or [8000]:
    a = torch.from_numpy(M.config_uniform(n, 3)).cuda() if n <= 16384 else M.config_spd_device(n, 5)
    res = {}
    for v in vals:
        os.environ[knob] = v
        r = [mc.logdet_blocked(a, return_pivots=True) for _ in range(3)]
        res[v] = r[-1]
        print(n, f"{knob}={v}", [round(x[3], 2) for x in r], r[-1][0], flush=True)
    d = np.nonzero((res[vals[0]][1] != res[vals[1]][1]) | (res[vals[0]][2] != res[vals[1]][2]))[0]
    print("  pivot diffs:", len(d), "first", d[:3])

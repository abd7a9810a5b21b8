"""Panel-kernel timeline of one blocked call: KP spans (device globaltimer) vs the
whole call -> how much of the critical path is panel factorisation vs gaps."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1811_08057_b200 as mc
from paper_1811_08057_b200 import _lib, matrix as M
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8000
a = torch.from_numpy(M.config_uniform(n, 3)).cuda() if n <= 16384 else M.config_spd_device(n, 5)
lib = _lib.load()
buf = np.zeros((4096, 2), dtype=np.uint64)
for it in range(3):
    lib.mcnd_debug_kp_spans(ctypes.c_void_p(buf.ctypes.data), 4096)
    r = mc.logdet_blocked(a, return_pivots=True)
    k = lib.mcnd_debug_kp_spans(ctypes.c_void_p(buf.ctypes.data), 4096)
    sp = buf[:k].astype(np.int64)
    dur = (sp[:, 1] - sp[:, 0]) / 1e3
    gaps = (sp[1:, 0] - sp[:-1, 1]) / 1e3
    total = (sp[-1, 1] - sp[0, 0]) / 1e3
    print(f"call {it}: device {r[3]:.2f} ms, {k} panels, first->last panel {total/1e3:.2f} ms, "
          f"panel time {dur.sum()/1e3:.2f} ms (mean {dur.mean():.1f} us), gaps {gaps.sum()/1e3:.2f} ms "
          f"(mean {gaps.mean():.1f} us; odd {gaps[0::2].mean():.1f} even {gaps[1::2].mean():.1f})")
    if it == 2:
        for j in [0, 1, 2, 3, k // 2, k // 2 + 1, k - 2, k - 1]:
            print(f"  panel {j}: {dur[j]:.1f} us, gap after {gaps[j] if j < k - 1 else 0:.1f} us")

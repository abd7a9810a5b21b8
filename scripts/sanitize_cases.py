"""Small invocations of every kernel family for compute-sanitizer (memcheck / racecheck /
synccheck): K1 (serial, mc_parallel with CTA groups = the multi-GPU push protocol), the
blocked path (KP panel kernel incl. the fused first-panel update and pair prep, gather +
L correction, both DMMA GEMMs, K1 tail), K3 batched.  Host numpy inputs only (no torch
CUDA context), results checked against the oracle so a sanitizer-perturbed schedule that
computes garbage also fails.

    compute-sanitizer --tool memcheck python scripts/sanitize_cases.py
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_1811_08057_b200 as mc  # noqa: E402
from oracle import mcnd_oracle as O  # noqa: E402


def tol(n, la):
    return max(1e-8 * n, 1e-10 * abs(la))


def main():
    which = sys.argv[1:] or ["k1", "groups", "blocked", "batched"]
    if "k1" in which:
        a = np.random.default_rng(1).uniform(-1, 1, (300, 300))
        r = O.logdet_condensation(a)
        assert mc.logdet_condensation(a) == (r.sign, r.log_abs)
        print("k1 ok", flush=True)
    if "groups" in which:
        a = np.random.default_rng(2).uniform(-1, 1, (200, 200))
        r = O.mc_parallel(a, 4)
        g = mc.mc_parallel(a, 4, groups=True)
        assert (g.logdet.sign, g.logdet.log_abs) == (r.sign, r.log_abs)
        print("groups ok", flush=True)
    if "blocked" in which:
        # n = 700: 5 pairs of panels (KP with r1 prologue + pair prep), critical and side
        # GEMMs, gather + L correction, the single-panel path and the K1 tail
        a = np.random.default_rng(3).uniform(-1, 1, (700, 700))
        r = O.logdet_condensation(a)
        got = mc.logdet_blocked(a)
        assert got.sign == r.sign and abs(got.log_abs - r.log_abs) <= tol(700, r.log_abs), (got, r)
        print("blocked ok", flush=True)
    if "batched" in which:
        b = np.random.default_rng(4).uniform(-1, 1, (8, 64, 64))
        s, l = mc.logdet_batched(b)
        rs, rl = O.logdet_batched(b)
        assert np.array_equal(s, rs) and np.all(np.abs(l - rl) <= 1e-8 * 64)
        print("batched ok", flush=True)


if __name__ == "__main__":
    main()

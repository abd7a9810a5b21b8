import glob
import hashlib
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden", "cases")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long-running (large N)")


def load_cases():
    out = []
    for f in sorted(glob.glob(os.path.join(GOLDEN_DIR, "*.json"))):
        with open(f) as fh:
            out.append(json.load(fh))
    return out


def digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()[:32]


def case_input(case) -> np.ndarray:
    """Rebuild the exact input the reference saw (explicit KAT matrix or recipe)."""
    from paper_1811_08057_b200 import matrix as M

    if "matrix" in case:
        return np.array([[float.fromhex(v) for v in row] for row in case["matrix"]], dtype=np.float64)
    r = case["recipe"]
    kind, n, seed = r["kind"], r["n"], r["seed"]
    if kind == "normal":
        return M.config_dense_normal(n, seed)
    if kind == "uniform":
        return M.config_uniform(n, seed)
    return M.generate(M.MatrixSpec(n, kind, seed))


def expect(case):
    return case["expect"]["sign"], float.fromhex(case["expect"]["log_abs"])


@pytest.fixture(scope="session")
def golden_cases():
    cases = load_cases()
    assert cases, "no golden fixtures under tests/golden/cases"
    return cases


def cuda_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False

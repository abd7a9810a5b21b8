"""CPU-only checks: the C-ABI library loads and exports every declared symbol,
and the host-side mirror of the reference interface validates like mcnd does
(errors raised before any device work)."""

import ctypes
import math
import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "mcnd_b200.h")


def declared_symbols():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(mcnd_[a-z0-9_]+)\s*\(", txt)))


def test_library_builds_and_exports_every_header_symbol():
    from paper_1811_08057_b200 import _lib
    from paper_1811_08057_b200.build import build

    path = build()
    lib = ctypes.CDLL(path)
    syms = declared_symbols()
    assert len(syms) >= 10
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in include/mcnd_b200.h but not exported"
    assert set(_lib.EXPORTS) <= set(syms)


def test_library_is_sm100a():
    import subprocess

    from paper_1811_08057_b200.build import build

    path = build()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", path], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_version_and_error_string():
    from paper_1811_08057_b200 import _lib

    lib = _lib.load()
    assert lib.mcnd_version() >= 100
    assert isinstance(_lib.last_error(), str)


def test_invalid_shapes_raise_value_error_before_device_work():
    """matrix.py:32-48 messages (no GPU needed: validation precedes the call)."""
    from paper_1811_08057_b200 import logdet_condensation, mc_parallel

    with pytest.raises(ValueError, match="square"):
        logdet_condensation(np.zeros((2, 3)))
    with pytest.raises(ValueError, match="2-D"):
        logdet_condensation(np.zeros(3))
    with pytest.raises(ValueError, match="positive"):
        logdet_condensation(np.zeros((0, 0)))
    with pytest.raises(ValueError, match="finite"):  # non-square AND non-finite: finiteness first
        logdet_condensation(np.array([[1.0, np.nan, 2.0], [0.0, 1.0, 3.0]]))
    with pytest.raises(ValueError, match="invalid plan"):
        mc_parallel(np.eye(4), 5)
    with pytest.raises(ValueError, match="invalid plan"):
        mc_parallel(np.eye(4), 0)


def test_abi_rejects_bad_arguments_without_gpu():
    from paper_1811_08057_b200 import _lib

    lib = _lib.load()
    out = _lib.McndLogDet()
    rc = lib.mcnd_logdet_condensation_dev(None, 4, 4, None, 0, 0, None, ctypes.byref(out), None, None)
    assert rc == _lib.MCND_EINVAL
    rc = lib.mcnd_logdet_batched_dev(None, 1, 200, 40000, 0, None, None, None, None, None)
    assert rc == _lib.MCND_EINVAL
    assert "n <= 128" in _lib.last_error()


def test_plan_blocks_mirror():
    """runtime.py:33-44 / test_runtime.py:14-45."""
    from paper_1811_08057_b200 import plan_blocks

    assert plan_blocks(16, 4).assignments == ((0, 4), (4, 4), (8, 4), (12, 4))
    assert [ln for _, ln in plan_blocks(10, 4).assignments] == [3, 3, 2, 2]
    assert [ln for _, ln in plan_blocks(5, 5).assignments] == [1] * 5
    for n in (7, 12, 31):
        for p in range(1, n + 1):
            pos = 0
            for s, ln in plan_blocks(n, p).assignments:
                assert s == pos
                pos += ln
            assert pos == n
    for bad in ((4, 0), (4, 5)):
        with pytest.raises(ValueError):
            plan_blocks(*bad)


def test_registry_seam():
    from paper_1811_08057_b200 import ALGORITHMS, run_algorithm

    assert set(ALGORITHMS) >= {"mc-serial", "mc-parallel", "ge-serial", "ge-parallel"}  # bench.py:25
    with pytest.raises(ValueError):
        run_algorithm("nope", np.eye(2), 1)


def test_logdet_namedtuple_parity():
    from paper_1811_08057_b200 import SINGULAR, LogDet

    assert SINGULAR == LogDet(0, -math.inf)
    assert LogDet(1, 0.0) == (1, 0.0)


def test_generators_reproduce_reference_recipes():
    """matrix.py:69-106 restatement, pinned by digests recorded from the reference."""
    from conftest import case_input, digest, load_cases

    checked = 0
    for c in load_cases():
        if "recipe" in c and not c.get("blas") and c["n"] <= 1000:
            assert digest(case_input(c)) == c["input_digest"], c["name"]
            checked += 1
    assert checked > 20

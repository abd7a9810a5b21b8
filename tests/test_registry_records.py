"""GPU benchmark records in the reference's CSV format (registry.py; mcnd/bench.py:26-43, 111-128)."""

import csv
import math
import os

import pytest

from paper_1811_08057_b200 import registry as R

REF_SRC = "/root/reference/pkg/src"


def _records():
    return [R.BenchRecord("mc-gpu", 64, 1, 0, 0.001, 0.0002, 0.0, -1, 12.5),
            R.BenchRecord("mc-gpu-parallel", 64, 2, 0, 0.0008, 0.0002, 0.0, -1, 12.5),
            R.BenchRecord("mc-gpu-blocked", 64, 1, 0, 0.0009, 0.0002, 0.0, 1, -math.inf)]


def test_csv_layout(tmp_path):
    p = tmp_path / "r.csv"
    R.write_records(_records(), p)
    rows = list(csv.reader(open(p)))
    assert rows[0] == ["algorithm", "n", "p", "run", "total_s", "scatter_s", "comm_s", "sign", "logabs"]
    assert rows[1] == ["mc-gpu", "64", "1", "0", "0.001", "0.0002", "0.0", "-1", "12.5"]
    assert rows[3][-1] == "-inf"


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference not mounted")
def test_reference_report_reads_gpu_records(tmp_path):
    """The reference's own reader and report accept the file (CPU, reference imported read-only)."""
    import sys

    sys.path.insert(0, REF_SRC)
    try:
        from mcnd import bench as ref_bench
    finally:
        sys.path.remove(REF_SRC)
    p = tmp_path / "r.csv"
    R.write_records(_records(), p)
    recs = ref_bench.read_records(p)
    rep = ref_bench.format_report(recs)
    assert "mc-gpu-parallel" in rep and "speedup" in rep.lower()


@pytest.mark.gpu
def test_run_bench_gpu():
    recs = R.run_bench([64, 200], [1, 2], repeats=2)
    algs = {r.algorithm for r in recs}
    assert algs == {"mc-gpu", "mc-gpu-parallel", "mc-gpu-blocked", "ge-gpu", "ge-gpu-parallel", "ge-cusolver"}
    assert all(r.total_seconds > 0 and r.scatter_seconds > 0 for r in recs)
    assert not any(r.algorithm not in ("mc-gpu-parallel", "ge-gpu-parallel") and r.p != 1 for r in recs)
    serial = {(r.n, r.run_index): (r.sign, r.log_abs) for r in recs if r.algorithm == "mc-gpu"}
    for r in recs:
        s, l = serial[(r.n, r.run_index)]
        assert r.sign == s and abs(r.log_abs - l) <= max(1e-8 * r.n, 1e-10 * abs(l))

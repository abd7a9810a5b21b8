"""CLI parity with the reference's front end (cli.py; mcnd/cli.py:55-191, SURVEY.md §8(f)
rank 4): subcommands, exit codes (0 / 1 usage / 2 I/O), messages, the logdet output line,
CSV matrix I/O (matrix.py:154-180) and the sweep CSV (the reference's own report reads it:
tests/test_registry_records.py).  CPU tests cover the parser and I/O paths; the GPU tests
run logdet and a tiny sweep on the device."""

import os
import re
import sys

import numpy as np
import pytest

from paper_1811_08057_b200 import cli
from paper_1811_08057_b200 import io as mio
from paper_1811_08057_b200 import registry as R
from paper_1811_08057_b200.matrix import MatrixSpec, generate

REF_SRC = "/root/reference/pkg/src"


def run(argv, capsys):
    rc = cli.main(argv)
    out = capsys.readouterr()
    return rc, out.out, out.err


def test_gen_round_trip(tmp_path, capsys):
    p = tmp_path / "m.mcnd"
    rc, _, _ = run(["gen", "--size", "7", "--kind", "diag", "--seed", "3", "--out", str(p)], capsys)
    assert rc == 0
    a = mio.read_matrix(p)
    assert np.array_equal(a, generate(MatrixSpec(7, "diagonally-dominant", 3)))


@pytest.mark.parametrize("argv", [["gen", "--size", "0", "--out", "x.mcnd"], ["gen", "--size", "3", "--kind", "nope", "--out", "x"],
                                  ["bogus"], [], ["logdet"], ["bench", "--sizes", "1,x", "--out", "o.csv"]])
def test_usage_errors_exit_1(argv, capsys, tmp_path, monkeypatch):
    monkeypatch.chdir(tmp_path)
    rc, _, err = run(argv, capsys)
    assert rc == 1 and err


def test_logdet_io_errors_exit_2(tmp_path, capsys):
    rc, _, err = run(["logdet", str(tmp_path / "missing.mcnd")], capsys)
    assert rc == 2 and err.startswith("cannot read ")
    bad = tmp_path / "bad.mcnd"
    bad.write_bytes(b"XXXX" + b"\0" * 30)
    rc, _, err = run(["logdet", str(bad)], capsys)
    assert rc == 2 and "bad matrix file" in err and "bad magic" in err
    rag = tmp_path / "rag.csv"
    rag.write_text("1,2\n3\n")
    rc, _, err = run(["logdet", str(rag)], capsys)
    assert rc == 2 and "ragged row width" in err


def test_logdet_workers_and_reference_only_algorithms(tmp_path, capsys):
    p = tmp_path / "m.mcnd"
    mio.write_matrix(np.eye(3), p)
    rc, _, err = run(["logdet", str(p), "--workers", "0"], capsys)
    assert rc == 1 and "workers must be >= 1" in err
    rc, _, err = run(["logdet", str(p), "--algorithm", "ge-bogus"], capsys)
    assert rc == 1 and "invalid choice" in err


def test_csv_matrix_round_trip_and_errors(tmp_path):
    a = np.random.default_rng(5).normal(size=(4, 4))
    p = tmp_path / "a.csv"
    mio.write_matrix_csv(a, p)
    assert np.array_equal(mio.read_matrix_csv(p), a)  # repr() floats: bit-exact
    (tmp_path / "e.csv").write_text("\n\n")
    with pytest.raises(mio.FormatError, match="empty CSV matrix"):
        mio.read_matrix_csv(tmp_path / "e.csv")
    (tmp_path / "t.csv").write_text("1,2\n3,abc\n")
    with pytest.raises(mio.FormatError, match="line 2"):
        mio.read_matrix_csv(tmp_path / "t.csv")


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference not mounted")
def test_csv_reader_matches_reference(tmp_path):
    sys.path.insert(0, REF_SRC)
    try:
        from mcnd import matrix as ref_matrix
    finally:
        sys.path.remove(REF_SRC)
    a = np.random.default_rng(9).uniform(-1, 1, (6, 6))
    p = tmp_path / "a.csv"
    ref_matrix.write_matrix_csv(a, p)
    assert np.array_equal(mio.read_matrix_csv(p), ref_matrix.read_matrix_csv(p))


@pytest.mark.gpu
def test_logdet_cli_on_gpu(tmp_path, capsys):
    from oracle import mcnd_oracle as O

    a = generate(MatrixSpec(40, "uniform-random", 2))
    p = tmp_path / "m.mcnd"
    mio.write_matrix(a, p)
    ref = O.logdet_condensation(a)
    for alg, workers in [("mc-serial", 1), ("mc-parallel", 4), ("mc-blocked", 1), ("ge-serial", 1), ("ge-parallel", 3)]:
        rc, out, _ = run(["logdet", str(p), "--algorithm", alg, "--workers", str(workers)], capsys)
        assert rc == 0, out
        m = re.match(r"status=ok sign=([+-]1) logabs=(\S+) algorithm=(\S+) workers=(\d+) broadcasts=(\d+) "
                     r"broadcast_bytes=(\d+) pivot_search_msgs=(\d+) scatter_s=\S+ comm_s=\S+ total_s=\S+$", out.strip())
        assert m, out
        assert int(m.group(1)) == ref.sign and abs(float(m.group(2)) - ref.log_abs) <= 1e-8 * 40
        if alg == "mc-parallel":
            assert int(m.group(5)) == 40 - 4  # broadcasts = N - p (test_acceptance.py:107)
    sing = tmp_path / "s.csv"
    mio.write_matrix_csv(generate(MatrixSpec(9, "singular-planted", 1)), sing)
    rc, out, _ = run(["logdet", str(sing)], capsys)
    assert rc == 0 and out.startswith("status=singular sign=0 logabs=-inf")


@pytest.mark.gpu
def test_bench_cli_on_gpu(tmp_path, capsys):
    import csv

    p = tmp_path / "b.csv"
    rc, out, _ = run(["bench", "--sizes", "32,48", "--workers", "1,2", "--repeats", "2", "--out", str(p)], capsys)
    assert rc == 0 and out.startswith("wrote ")
    with open(p) as f:
        rows = list(csv.reader(f))
    assert rows[0] == R.CSV_HEADER
    assert {r[0] for r in rows[1:]} >= {"mc-gpu", "mc-gpu-parallel", "mc-gpu-blocked"}

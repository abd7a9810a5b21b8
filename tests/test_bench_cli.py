"""bench.py's driver contract on CPU: the --gpus N launcher (torchrun, gloo dry run) and
the reference arm's record (timed samples, same config as the repo arm)."""

import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args, timeout=300):
    t0 = time.perf_counter()
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    wall = time.perf_counter() - t0
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    return r.returncode, lines, wall, r.stderr


def test_gpus_n_spawns_ranks_dry_run():
    """`bench.py --gpus 2` outside torchrun launches 2 ranks; rank 0 prints one line with n_gpus=2."""
    rc, lines, _, err = _run("--gpus", "2", "--dry-run", "--config", "c3")
    assert rc == 0, err
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["schedule_consistent"] and d["config"]["ranks_rows"] == [4000, 4000]


def test_reference_arm_record_is_what_was_timed():
    sys.path.insert(0, ROOT)
    import argparse

    import bench

    rc, lines, wall, err = _run("--impl", "reference", "--gpus", "2", "--steps", "3", "--warmup", "1",
                                "--config", "c1", "--cpu-seconds", "1")
    assert rc == 0, err
    d = json.loads(lines[-1])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["steps"] == 3
    # the timed steps fit in the process's own wall clock
    assert d["steps"] * d["ms_per_step"] / 1e3 < wall
    assert "mc_parallel(a, 2)" in d["cpu_baseline"]["sample"]
    assert d["e2e"]["value"] == d["value"]
    # the repo arm prints the same config dict for the same arguments
    ns = argparse.Namespace(method=None, fast=False)
    assert d["config"] == bench.bench_config(ns, d["config"]["workload"], 1000, 2)

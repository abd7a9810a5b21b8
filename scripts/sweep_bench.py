"""Tuning sweep: run bench.py (C3, no C5 / CPU legs) under a list of environment settings and
print one line per setting (ms per step, parity).  Usage:
    python scripts/sweep_bench.py 'VAR=a,VAR2=b' 'VAR=c' ...   (empty string = defaults)"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for spec in sys.argv[1:]:
    env = dict(os.environ)
    for kv in filter(None, spec.split(",")):
        k, v = kv.split("=")
        env[k] = v
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "6", "--warmup", "3", "--no-c5",
                        "--no-cpu-baseline"], env=env, capture_output=True, text=True, cwd=ROOT)
    try:
        d = json.loads(r.stdout.strip().splitlines()[-1])
        print(f"{spec or 'default':40s} {d['ms_per_step']:.3f} ms  {d['result']['parity']}", flush=True)
    except Exception:
        print(f"{spec:40s} ERR {r.stderr[-400:]}", flush=True)

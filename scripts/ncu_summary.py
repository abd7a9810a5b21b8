"""Summarise an ncu report (--set full) or a launch-list CSV into profiles/.

usage: python scripts/ncu_summary.py report.ncu-rep out_prefix [config]
       python scripts/ncu_summary.py launches.csv out_prefix --launches
"""
import csv, io, json, subprocess, sys
from collections import defaultdict

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__bytes.sum.per_second",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard", "lts__t_bytes.sum", "l1tex__t_bytes.sum"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
         "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "nsecond": 1e-9}


def rep(path, prefix, cfg):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = {"value": vals[i], "unit": units[i]}
        out.append(d)
    lines = []
    for d in out:
        lines.append(f"kernel: {d['kernel'][:120]}")
        for k in KEYS:
            if k in d:
                lines.append(f"  {k:70s} {d[k]['value']:>20s} {d[k]['unit']}")
    open(prefix + ".txt", "w").write("\n".join(lines) + "\n")
    d = out[0]
    def val(k):
        v = float(d[k]["value"].replace(",", ""))
        return v * SCALE.get(d[k]["unit"], 1.0)
    traffic = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
    summ = {"config": cfg, "kernel": d["kernel"], "traffic_bytes_per_launch": traffic,
            "duration_s": val("gpu__time_duration.sum"), "source": path}
    json.dump(summ, open(prefix + ".json", "w"), indent=1)
    print("\n".join(lines))


def launches(path, prefix):
    txt = open(path).read()
    body = "\n".join(l for l in txt.splitlines() if not l.startswith("=="))
    rows = list(csv.DictReader(io.StringIO(body)))
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", "")) * SCALE.get(r["Metric Unit"], 1.0)
        k = r["Kernel Name"][:100]
        agg[k][0] += 1
        agg[k][1] += v
    tot = sum(v[1] for v in agg.values())
    lines = [f"{'kernel':100s} {'launches':>8s} {'total_ms':>10s} {'share':>7s}"]
    for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"{k:100s} {c:8d} {t*1e3:10.3f} {100*t/tot:6.2f}%")
    open(prefix + ".txt", "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    if "--launches" in sys.argv:
        launches(sys.argv[1], sys.argv[2])
    else:
        rep(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")

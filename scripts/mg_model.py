"""Critical-path model of the multi-GPU paths at 1/2/4/8 B200s, from single-GPU
measurements (profiles/r2_bench_default.json, r2_k2_timeline_c3.txt, r2_kp_bench_*.txt) and the
NVLink 5 peer bandwidth.  Prints the predicted time per logdet and the parallel efficiency
t1 / (p tp).  Not a measurement: this pool has one GPU per box.

    python scripts/mg_model.py
"""

HBM = 5.95e12         # B/s, what K1 sustains (0.91 of the 6.54 TB/s copy peak; C3 unblocked 461 ms)
NVL = 770e9           # B/s, NVLink 5 peer bandwidth per direction (bulk, NCCL broadcast)
NVL_LAT = 10e-6       # s, per NCCL broadcast (launch + protocol latency)
PUSH_SM = 120e9       # B/s, remote stores from ONE SM (the unblocked pivot-row push)
DGEMM = 25.6e12       # flop/s, the trailing GEMM as it runs beside the panels (C5 0.918 s)
PIVOT = 3.3e-6        # s per pivot, column-distributed panel kernel (active widths above 6400)
PIVOT_KC = 1.97e-6    # s per pivot, cluster panel kernel at m = 4000 (pair 252 us; 2.3 at m = 6400), 1.6 at m <= 1000
KC_MAXM = 6400        # active widths the cluster panel kernel takes
PAIR_EXTRA = 40e-6    # s, per pair on the critical stream besides the panels (prologue, W, pair prep)
CRIT_GAP = 80e-6      # s, per pair: join, gather + L correction, the next 128 rows' update, launch gaps (r2_k2_timeline_c3.txt)
K1_STEP = 4.5e-6      # s, unblocked per-step chain (publish -> flag -> stage), C1 3.8 us + NVLink flag


def blocked(n, p, t1_meas=None):
    """Per pair: the owner factors 2 x 64 pivots (serial), W (128 x m) is broadcast, every rank
    updates its rows (the GEMM splits p ways and overlaps the next pairs' panels)."""
    t_chain = t_bcast = t_gemm = 0.0
    b = 64
    for k in range(0, n - 128, 2 * b):
        m = n - k
        piv = PIVOT if m > KC_MAXM else (1.6e-6 + (PIVOT_KC - 1.6e-6) * max(0.0, (m - 1000) / 3000.0))
        t_chain += 2 * b * piv + (PAIR_EXTRA if m > KC_MAXM else 0.0) + CRIT_GAP
        if p > 1:
            t_bcast += NVL_LAT + 128 * m * 8 / NVL
        t_gemm += 2.0 * (m - 2 * b) * (m - 2 * b) * 2 * b / DGEMM
    # the trailing update overlaps the panel chain (look-ahead); the broadcast sits on the
    # critical path once per pair (the next owner's critical rows need this pair's W)
    return max(t_chain + t_bcast, t_gemm / p + t_bcast) + 0.25e-3


def unblocked(n, p):
    """Per step: every rank updates its N/p live rows at HBM speed; the owner's scaled pivot row
    goes to p-1 peers from one SM; the next step waits for max(update, chain + push)."""
    t = 0.0
    for m in range(n, 1, -1):
        upd = 16.0 * (m - 1) * m / p / HBM
        push = (p - 1) * 8.0 * m / PUSH_SM if p > 1 else 0.0
        t += max(upd, K1_STEP + push)
    return t


def main():
    rows = [("C3 N=8000 blocked (default)", lambda p: blocked(8000, p)),
            ("C3 N=8000 unblocked (per-step push)", lambda p: unblocked(8000, p)),
            ("C5 N=32768 blocked", lambda p: blocked(32768, p))]
    print(f"{'workload':40s} " + " ".join(f"{'p=' + str(p):>16s}" for p in (1, 2, 4, 8)))
    for name, f in rows:
        t1 = f(1)
        cells = []
        for p in (1, 2, 4, 8):
            tp = f(p)
            cells.append(f"{tp * 1e3:8.1f} ms {t1 / (p * tp) * 100:4.0f}%")
        print(f"{name:40s} " + " ".join(f"{c:>16s}" for c in cells))


if __name__ == "__main__":
    main()

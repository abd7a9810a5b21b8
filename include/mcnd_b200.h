/*
 * mcnd_b200 -- C ABI of the B200-native matrix-condensation log-determinant.
 *
 * Drop-in boundary for the reference package `mcnd` (pure Python/numpy; it
 * has no FFI of its own).  Each entry point replaces one reference call; the
 * Python mirror (paper_1811_08057_b200/condense.py, runtime.py) binds them via
 * ctypes exactly as INTEGRATION.md shows.  Plain pointers and sizes only.
 *
 * Conventions
 *   - matrices are row-major float64 with a leading dimension (elements);
 *   - `*_dev` entry points take DEVICE pointers and a cudaStream_t (as void*);
 *     the others take HOST pointers and perform the host<->device copies
 *     inside the call (pinned memory makes them asynchronous DMA);
 *   - return 0 on success, otherwise an MCND_E* code; mcnd_last_error()
 *     gives a thread-local message.  A singular matrix is a VALUE
 *     (sign 0, log_abs -inf), never an error, as in condense.py:153-158;
 *   - the caller's matrix is never modified (condense.py:72, runtime.py:139).
 */
#ifndef MCND_B200_H
#define MCND_B200_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MCND_OK 0
#define MCND_EINVAL 1        /* bad shape / argument  -> Python ValueError       */
#define MCND_ECUDA 2         /* CUDA runtime failure  -> RuntimeError            */
#define MCND_ENCCL 3         /* NCCL failure          -> RuntimeError            */
#define MCND_EDEVICE 4       /* device-side timeout / protocol error             */
#define MCND_EPIVOT 5        /* pivot_sequence names an inactive row (ValueError) */
#define MCND_EPIVOT_SHORT 6  /* pivot_sequence shorter than n-1 (IndexError)      */

/* flags */
#define MCND_FLAG_FAST 1u     /* fused multiply-add update (default: reference-exact
                                 multiply-then-subtract, bitwise equal to numpy)   */
#define MCND_FLAG_GROUPS 2u   /* mc_parallel only: run the p workers as p CTA groups with
                                 separate workspaces on one GPU, exchanging pivot rows
                                 through the same push protocol the multi-GPU driver uses
                                 over NVLink (p <= 8)                               */

/* Result of one log-determinant (mirrors mcnd.LogDet, condense.py:36-43). */
typedef struct mcnd_logdet {
    int32_t sign;            /* +1 / -1, 0 = singular                            */
    int32_t singular;        /* 1 if singular                                    */
    double log_abs;          /* ln|det|, -inf if singular                        */
    int64_t singular_step;   /* step whose pivot failed the witness test, or -1 */
    int64_t invalid_step;    /* first invalid pivot_sequence step, or -1        */
    int64_t invalid_row;     /* the offending row id (MCND_EPIVOT)              */
    double device_ms;        /* device time of the condensation (CUDA events)   */
    int64_t steps;           /* condensation steps executed                      */
    int64_t launches;        /* GPU kernels this call launched (0 if not counted) */
    int64_t torn_reads;      /* blocked: panel records observed half-written (one 8-byte word
                                of the new store, one stale) and re-polled; informational */
} mcnd_logdet;

/* Communication accounting of the block-row driver (runtime.py:47-66). */
typedef struct mcnd_comm_stats {
    int64_t broadcasts;
    int64_t broadcast_bytes;
    int64_t pivot_search_msgs;
    int64_t scalar_updates;
    int64_t aborted_step;    /* -1 if no abort */
    double scatter_seconds;  /* rows distributed to the workers (+ the H2D copy for host input) */
    double comm_seconds;     /* time in the pivot-row broadcasts (device, summed over steps)  */
} mcnd_comm_stats;

/* ---- serial condensation: replaces mcnd.logdet_condensation (condense.py:134) ----
 * pivot_sequence: optional HOST array of >= n-1 original row ids (condense.py:147-152),
 *                 NULL = top-to-bottom.  pivots_out / cols_out: optional HOST arrays
 *                 of n entries receiving each step's pivot value / column (the
 *                 last entry is the final 1x1). */
int mcnd_logdet_condensation_dev(const double* d_a, int64_t n, int64_t lda,
                                 const int64_t* pivot_sequence, int64_t pivot_sequence_len,
                                 uint32_t flags, void* stream, mcnd_logdet* out,
                                 double* pivots_out, int32_t* cols_out);
int mcnd_logdet_condensation(const double* h_a, int64_t n, int64_t lda,
                             const int64_t* pivot_sequence, int64_t pivot_sequence_len,
                             uint32_t flags, void* stream, mcnd_logdet* out,
                             double* pivots_out, int32_t* cols_out);

/* ---- block-row parallel condensation: replaces mcnd.mc_parallel(a, p) (runtime.py:123) ----
 * One GPU runs the exact p-worker schedule (round-robin owners, topmost live row,
 * runtime.py:153-204) and the p x p LU tail (runtime.py:206-219).
 * payload_entries: optional HOST array of n-p entries; row_updates: optional HOST
 * array of p entries; owners_out: optional HOST array (n-p) of the owner per step. */
int mcnd_mc_parallel_dev(const double* d_a, int64_t n, int64_t lda, int32_t p, uint32_t flags,
                         void* stream, mcnd_logdet* out, mcnd_comm_stats* stats,
                         int64_t* payload_entries, int64_t* row_updates, int32_t* owners_out);
int mcnd_mc_parallel(const double* h_a, int64_t n, int64_t lda, int32_t p, uint32_t flags,
                     void* stream, mcnd_logdet* out, mcnd_comm_stats* stats,
                     int64_t* payload_entries, int64_t* row_updates, int32_t* owners_out);

/* ---- blocked rank-b condensation (b = mcnd_blocked_panel() = 64): panels of b pivot
 * rows factorised with the unblocked rule, then one rank-b trailing update on FP64
 * tensor cores (DMMA).  Same pivot rule and result type as logdet_condensation
 * (top-to-bottom order); rounding differs from the reference (tolerance parity).
 * No reference counterpart (PAPER.md:89 leaves it to future work). */
int mcnd_logdet_blocked_dev(const double* d_a, int64_t n, int64_t lda, uint32_t flags, void* stream,
                            mcnd_logdet* out, double* pivots_out, int32_t* cols_out);
/* Host input: a pinned (page-locked) h_a is copied in row chunks that overlap the first
 * panel pairs (bitwise the result of the _dev call); a pageable h_a is copied whole first. */
int mcnd_logdet_blocked(const double* h_a, int64_t n, int64_t lda, uint32_t flags, void* stream,
                        mcnd_logdet* out, double* pivots_out, int32_t* cols_out);
int32_t mcnd_blocked_panel(void);

/* ---- Gaussian elimination with row pivoting: replaces mcnd.logdet_lu (gauss.py:34-68), the
 * paper's comparison baseline.  Bitwise the reference's pivots and log|det| (K1 run on A^T).
 * row_witness: optional n per-row bounds (DEVICE for _dev, HOST otherwise; NULL = only an exactly
 * zero pivot is singular).  pivots_out / rows_out: optional HOST arrays of n entries: each
 * step's pivot value and ORIGINAL pivot row (ge_parallel's owners and accounting, runtime.py:232). */
int mcnd_logdet_lu_dev(const double* d_a, int64_t n, int64_t lda, const double* d_row_witness, uint32_t flags,
                       void* stream, mcnd_logdet* out, double* pivots_out, int32_t* rows_out);
int mcnd_logdet_lu(const double* h_a, int64_t n, int64_t lda, const double* h_row_witness, uint32_t flags,
                   void* stream, mcnd_logdet* out, double* pivots_out, int32_t* rows_out);

/* Fold per-step pivots and the p x p remainder of the block-row driver into the
 * reference's result and accounting (runtime.py:185-229): sign parity, per-worker
 * log sums reduced in rank order, row-pivoted LU tail (gauss.py:34-68).
 * piv_vals/piv_cols: n-p (or singular_at+1) entries; rem: p x p row-major (row w =
 * worker w's last live row); rem_wit: p witnesses; singular_at: -1 or the pivot that
 * failed the witness test. */
int mcnd_fold_mc_parallel(int64_t n, int32_t p, const double* piv_vals, const int32_t* piv_cols,
                          int64_t singular_at, const double* rem, const double* rem_wit, mcnd_logdet* out,
                          mcnd_comm_stats* stats, int64_t* payload_entries, int64_t* row_updates);

/* ---- multi-GPU block-row driver, one process per GPU (replaces the in-process
 * _Fabric of runtime.py:69-120 with stores into peer memory over NVLink) ----
 * 1. mcnd_dist_create on every rank (current device = the rank's GPU) -> handle and an
 *    opaque IPC handle of mcnd_dist_ipc_handle_bytes() bytes;
 * 2. all-gather the IPC handles (any host transport), mcnd_dist_connect(all handles);
 * 3. mcnd_dist_mc_parallel with this rank's block rows (plan_blocks(n, world), DEVICE
 *    pointer, row stride lda): returns every pivot (all ranks receive all of them),
 *    this rank's remaining row (first `world` columns) and its witness;
 * 4. all-gather the remaining rows; mcnd_fold_mc_parallel gives the result.
 * n must equal n_max.  world <= 8. */
int32_t mcnd_dist_ipc_handle_bytes(void);
int mcnd_dist_create(int32_t rank, int32_t world, int64_t n_max, void** handle, void* ipc_out);
int mcnd_dist_connect(void* handle, const void* ipc_all);
int mcnd_dist_mc_parallel(void* handle, const double* d_rows, int64_t n, int64_t lda, uint32_t flags,
                          void* stream, double* piv_vals, int32_t* piv_cols, int64_t* singular_at,
                          double* rem_row, double* rem_wit, double* device_ms);
void mcnd_dist_destroy(void* handle);

/* ---- multi-GPU BLOCKED condensation, one process per GPU: the per-rank engine.
 * Replaces mc_parallel's block-row worker loop (runtime.py:153-204) for the blocked
 * variant ("K2: one broadcast per panel of W").  Rank r holds a
 * contiguous block of rows (plan_blocks, runtime.py:33-44) x all n columns.  The host
 * schedule (paper_1811_08057_b200/dist.py BlockedGroup) gives each panel pair to the
 * rank with the most live rows (its topmost 128 live rows, north_star (3)); that rank
 * runs mcnd_mg_pair, the host broadcasts W / Wp / the gather descriptor (NCCL), and
 * every rank runs mcnd_mg_trailing on its own live rows.  The last rows are exported
 * (mcnd_mg_export), gathered to one rank and finished by mcnd_mg_tail (K1).
 * Records are 16 bytes {double v; int32 l; uint32 flag}; flag == the epoch returned
 * in err[3] by mcnd_mg_records.  All device pointers; asynchronous unless stated. */
int mcnd_mg_create(int64_t n, int64_t local_rows, void** handle);
int mcnd_mg_load(void* handle, const double* d_rows, int64_t lds, void* stream);
int mcnd_mg_pair(void* handle, int64_t lr0, int64_t t, int64_t m, double* d_W, int64_t ldw, double* d_Wp,
                 void* d_gather, void* stream);
int mcnd_mg_trailing(void* handle, int64_t lr0, int64_t rows, int64_t m, const double* d_W, int64_t ldw,
                     const double* d_Wp, const void* d_gather, int32_t sm_budget, int32_t par, void* stream);
int mcnd_mg_export(void* handle, int64_t lr0, int64_t rows, int64_t mt, double* d_out, int64_t ldo, double* d_wit,
                   void* stream);
/* synchronous: h_recs receives mt records, h_err {error, step, nonfinite} */
int mcnd_mg_tail(void* handle, double* d_rows, int64_t ldr, const double* d_wit, int64_t mt, void* stream,
                 void* h_recs, uint32_t* h_err);
/* synchronous: n records (global step index) + {error, step, nonfinite, epoch} */
int mcnd_mg_records(void* handle, void* h_recs, uint32_t* h_err, void* stream);
int64_t mcnd_mg_gather_bytes(void);   /* size of the gather descriptor to broadcast */
/* Native driver: the whole per-rank schedule above in one call (dist.BlockedGroup's loop in
 * C++), W / Wp / descriptor broadcast and the tail / records all-gathered with NCCL on the
 * library's own communicator (libnccl.so.2 resolved at run time).  Set up once per handle:
 * rank 0 fills an id (mcnd_nccl_id_bytes() bytes) with mcnd_nccl_unique_id, the ranks share it
 * over any host transport, every rank calls mcnd_mg_attach (world 1 needs no id and no NCCL;
 * force_comm = 1 runs the broadcasts even then).  mcnd_mg_logdet takes this rank's block rows
 * (plan_blocks(n, world), DEVICE pointer, row stride lds; `tail` rows finished by K1, 0 = 64) and
 * returns the whole matrix's result
 * on every rank (synchronous; device_ms = this rank's time from entry to the folded records).
 * Replaces mc_parallel's worker loop (runtime.py:153-204) for the blocked variant. */
int32_t mcnd_nccl_id_bytes(void);
int mcnd_nccl_unique_id(void* id_out);
int mcnd_mg_attach(void* handle, int32_t world, int32_t rank, const void* nccl_id, int32_t force_comm);
int mcnd_mg_logdet(void* handle, const double* d_rows, int64_t lds, int64_t tail, void* stream, mcnd_logdet* out);
/* Test transport: the same driver with its collectives done by host callbacks on pinned
 * buffers (bcast(buf, bytes, root); allgather(send, recv = world x bytes, bytes)), e.g. over
 * gloo for ranks that share one GPU.  Callbacks return 0 on success. */
int mcnd_mg_attach_host(void* handle, int32_t world, int32_t rank, int (*bcast)(void*, int64_t, int32_t),
                        int (*allgather)(const void*, void*, int64_t));
/* Host only: the pair schedule (5 int64 per pair: owner, local row, first pivot, active width,
 * k_pos) of n rows over world ranks with a `tail`-row K1 finish; returns the pair count. */
int64_t mcnd_mg_schedule(int64_t n, int32_t world, int64_t tail, int64_t* pairs_out, int64_t max_pairs);
int64_t mcnd_mg_ld(void* handle);      /* workspace row stride (W buffers use it)    */
int mcnd_mg_destroy(void* handle);

/* ---- batched: two warps per small matrix (no reference counterpart; oracle = a loop
 * of logdet_condensation).  d_sign/d_log_abs: DEVICE outputs (batch entries);
 * d_pivots: optional DEVICE batch x n pivot values (for bitwise checks); d_nonfinite:
 * optional DEVICE flag set nonzero when any entry is NaN/Inf (the host entry point
 * turns it into MCND_EINVAL, like matrix.py:39-40). n <= 128.  Asynchronous. */
int mcnd_logdet_batched_dev(const double* d_a, int64_t batch, int64_t n, int64_t stride,
                            uint32_t flags, void* stream, int32_t* d_sign, double* d_log_abs,
                            double* d_pivots, uint32_t* d_nonfinite);
/* host in / host out */
int mcnd_logdet_batched(const double* h_a, int64_t batch, int64_t n, int64_t stride,
                        uint32_t flags, void* stream, int32_t* h_sign, double* h_log_abs);

/* ---- introspection ---- */
const char* mcnd_last_error(void);
int32_t mcnd_version(void);
/* Number of CTAs the persistent condensation kernel runs with on the current device. */
int32_t mcnd_k1_grid(void);
/* Free the library's cached device workspace and pinned staging buffers. */
void mcnd_release_workspace(void);

#ifdef __cplusplus
}
#endif
#endif /* MCND_B200_H */

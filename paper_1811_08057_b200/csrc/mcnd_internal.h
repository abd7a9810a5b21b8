// Internal interfaces shared by the kernels (.cu) and the host runtime.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace mcnd {

constexpr double kSingularRtol = 1e-12;  // condense.py:29
constexpr int kK1Threads = 1024;         // one CTA per SM, 32 warps
constexpr int kK1MaxRowsPerCta = 512;    // per-CTA row table lives in shared memory
constexpr int kK1MaxChunk = 16384;       // pivot-row chunk staged in smem (doubles)
constexpr int kMaxGroups = 8;            // block-row workers (ranks) one launch can address
constexpr int32_t kNever = 0x7fffffff;   // pivot index of a row that is never a pivot

// One published pivot.  Written once per call by the owner CTA into EVERY
// group's record array (local or peer memory); `flag` is release-stored last
// with the call's epoch, so no per-call reset is needed.
struct PivRec {
    double v;       // pivot value
    int32_t l;      // pivot column (-1: failed the witness test -> singular)
    uint32_t flag;  // == epoch once v/l and the scaled pivot row are visible
};

struct K1Err {
    unsigned error;     // nonzero: device-side timeout
    unsigned err_step;
    unsigned nonfinite; // nonzero: the input held NaN/Inf (-> ValueError)
    unsigned torn;      // panel records read torn (one word stale) and re-polled
    unsigned dbg[8];    // diagnostics of the first timeout (panel kernel)
    unsigned long long scatter_ns;  // K1: rows distributed into the workspaces (slowest CTA's prologue)
    unsigned long long comm_ns;     // K1: time in pivot-row publications (the broadcasts of runtime.py:185)
};

// Persistent, barrier-free condensation kernel parameters (k1_condense.cu).
//
// "Groups" are the block-row workers of mc_parallel (runtime.py:123): group g
// owns a contiguous block of rows and keeps a full n x ld workspace in which
// the rows it does not own serve as mailboxes for the scaled pivot rows.  One
// launch runs `n_local_groups` groups starting at global id `group0`:
//   single GPU  : 1 group, no peers;
//   multi GPU   : 1 group per rank, ws[]/rec[] of other ranks are peer
//                 (CUDA IPC, NVLink) mappings, sys-scope flags;
//   emulation   : all P groups on one GPU (tests the same push protocol).
struct K1Params {
    const double* src[kMaxGroups];   // input rows of each local group
    int64_t src_row0[kMaxGroups];    // global row id of src[g]'s first row
    int64_t lds;
    double* ws[kMaxGroups];          // workspace of every group (n rows x ld)
    PivRec* rec[kMaxGroups];         // pivot records of every group
    double* row_wit[kMaxGroups];     // per-row witnesses at exit (local groups; global row index)
    int64_t ld;
    int32_t n;                       // rows of the workspace (global row ids < n)
    int32_t ncol0;                   // active width at step 0 (n for a whole logdet)
    int32_t n_steps;                 // S condensation steps
    int32_t in_place;                // 1: rows already in ws (panel mode): no copy, witness
                                     //    starts from wit_in[r] (blocked K2)
    const double* wit_in;            // carried-in witnesses (in_place mode)
    const unsigned* abort_flag;      // nullable: nonzero -> exit immediately
    int32_t n_groups;                // P
    int32_t group0;
    int32_t n_local_groups;
    int32_t ctas_per_group;
    int32_t sys_scope;               // 1: peers live on other GPUs
    uint32_t epoch;
    const int32_t* seq;              // global pivot schedule (pivot row of pivot t)
    const int32_t* row_pstep;        // pivot index of each row (kNever: never a pivot)
    int32_t pstep_offset;            // subtracted from row_pstep (panel launches of K2)
    const int32_t* cta_row_ptr;      // [n_local_groups * ctas_per_group + 1]
    const int32_t* cta_rows;         // rows dealt to each CTA, ascending pivot index
    K1Err* err;
    int32_t chunk;                   // staged pivot-row chunk (even, <= kK1MaxChunk)
    unsigned long long timeout_ns;
    // Gaussian-elimination mode (logdet_lu, gauss.py:34-68, run on A^T: the pivot row of A^T
    // is the elimination column of A, its argmax the row pivot): ge_ids[c] = original row id
    // of A at column position c (kept current across the column exchanges by the publishers),
    // ties -> lowest ORIGINAL id, singular iff the pivot is exactly 0 or
    // |v| <= 1e-12 * ge_rowwit[id] (optional caller witness).  nullptr: condensation.
    int32_t* ge_ids;
    const double* ge_rowwit;
};

cudaError_t k1_launch(const K1Params& p, bool fast, cudaStream_t s);
// out = a^T (n x n; row strides lda, ldo)
cudaError_t transpose_launch(const double* a, int64_t n, int64_t lda, double* out, int64_t ldo, cudaStream_t s);
size_t k1_smem_bytes(int chunk);

// ---- K2: blocked rank-b condensation (k2_blocked.cu) ----
constexpr int kK2B = 64;  // panel height b (rank of the trailing update)
constexpr long kK2GroupAbove = 12000;  // pairs grouped into rank-256 updates above this active width
// Gather descriptor of a trailing update: the K multiplier columns P (positions
// in the layout the trailing rows are in) and the final columns whose source
// column moved (composition of the column exchanges of condense.py:104-107).
struct K2Gather {
    int32_t P[2 * kK2B];
    int32_t l[kK2B];           // pivot positions of the producing panel (layout of each step)
    int32_t n_moved;
    int32_t moved_c[2 * kK2B];
    int32_t moved_src[2 * kK2B];
};
// Column-distributed panel factorisation (k2_panel.cu).  Every exchanged
// value travels in a 16-byte record of two tagged 8-byte words
// {tag:16 | aux:16 | half of the value} written with ONE 16-byte store, so readers
// poll the records themselves (no fences, no counters) and detect a torn read
// deterministically (a tag mismatch in either word).
struct KPParams {
    double* ws;
    int64_t ld;
    int32_t row0;             // first panel row
    int32_t m;                // active width at panel start
    int32_t G;                // CTAs (column chunks)
    int32_t cw;               // chunk width (columns per CTA)
    const double* wit;        // running witnesses, global row index
    PivRec* rec;              // this panel's 64 pivot records
    uint32_t epoch;
    uint32_t tag0;            // record tag of step s is tag0 + s (the global step + 1 < 65535; slots cleared per call)
    double* W;                // out: T^{-1} U, 64 x (m - 64), row stride ldw
    int64_t ldw;
    K2Gather* pan;            // out: panel-start pivot columns (P[0..63]), moved columns
    unsigned* abort;
    ulonglong2* cand;         // [64][G]   {candidate value, pos, tag}
    ulonglong2* wrec;         // [64][G]   {running max of the pivot row, tag}
    ulonglong2* colbuf;       // [64][G][64] {candidate column values, tag}
    ulonglong2* lastbuf;      // [64][64]  {last active column values, tag}
    K1Err* err;
    unsigned long long timeout_ns;
    // second panel of a pair: CTA 0 also runs the pair prep (k2_pair_prep.cuh) at the end
    const K2Gather* pp_g0;    // the pair's first descriptor (nullptr: no pair prep)
    double* pp_W;             // W of the pair (rows 0..63 = W_k), row stride pp_ldw
    int64_t pp_ldw;
    double* pp_Wp;
    K2Gather* pp_gpair;
    int32_t pp_m;             // active width at the first panel of the pair
    // second panel of a pair: the first panel's update of these 64 rows is applied in
    // the prologue (gather of -A[rows, P0], moved columns, rank-64 FMA update) instead
    // of by separate gather + GEMM launches
    const K2Gather* r1_g0;    // the first panel's descriptor (nullptr: rows already updated)
    const double* r1_W;       // its W (64 rows, row stride r1_ldw)
    int64_t r1_ldw;
    // pair prep spread over every CTA of the second panel (Wp rows and W's moved columns
    // in slices, the composite descriptor in CTA 0) around one grid barrier on this
    // counter (zeroed per call, one per pair); nullptr: CTA 0 does all of it
    unsigned* pp_bar;
    // second half of a two-panel launch: the grid barrier between the panels (zeroed per call)
    unsigned* half_bar;
};
constexpr int kKPMaxG = 160;
// lastbuf allocation: the LAST records [64][64], then the pair-prep barrier counters
constexpr int kPPBars = 1024;  // pairs per call (n <= 131072)
constexpr size_t kLastBufBytes = (size_t)64 * 64 * 16 + (size_t)2 * kPPBars * sizeof(unsigned);  // + pp / half barriers
// ~176 columns per panel CTA (C3 sweep with the 4-warp GEMM: 128: 31.26, 160: 31.19, 176: 31.03,
// 184: 31.54, 192: 31.50, 224: 31.74 ms): the pivot latency is flat up to ~200 columns and fewer
// panel CTAs leave more SMs to the overlapped trailing GEMM
constexpr int kKPCols = 176;
// while the trailing GEMM bounds the pair (m above ~6000 at the panel's ~3.2 us per pivot), wider
// chunks: fewer panel CTAs, more SMs for the overlapped GEMM (C3 sweep: 176 everywhere 30.77 ms;
// 208 / 240 / 272 / 320 above 6000: 30.59 / 30.36 / 30.54 / 30.45; 240 above 4500 / 6500 / 7200:
// 30.60 / 30.54 / 30.67)
constexpr int kKPColsWide = 240;
constexpr int kKPWideAbove = 6000;
// far above (C5, m up to 32768): 300 columns -- 110 CTAs instead of 136 at m = 32768, the rest of
// the SMs for the GEMM (C5 sweep: 240 / 280 / 300 / 320 / 368 above 12000: 0.915 / - / 0.904 / 0.923
// / 0.921 s; 300 above 9000 / 16000: 0.905 / 0.904 s)
constexpr int kKPColsXL = 300;
constexpr int kKPXLAbove = 12000;
__host__ __device__ constexpr int kp_cols_for(long long m) {
    return m > kKPXLAbove ? kKPColsXL : m > kKPWideAbove ? kKPColsWide : kKPCols;
}
// columns per panel CTA: 64 x 368 doubles = 184 KB of dynamic shared memory, + the kernel's 42 KB
// static, inside the 227 KB a CTA may have (n up to 368 x 148 = 54464 on one B200)
constexpr int kKPMaxCw = 368;
// 16-bit record tags: step t's tag t + 1, unique within a call (n <= kKPMaxCw * kKPMaxG)
static_assert((long long)kKPMaxCw * kKPMaxG + 64 < 0xffff, "panel record tags are 16-bit");
inline uint32_t kp_tag0(int64_t t) { return (uint32_t)t + 1u; }
// second != nullptr: one launch runs p then *second (the pair's second panel, same G / cw)
cudaError_t kp_launch(const KPParams& p, cudaStream_t s, const KPParams* second = nullptr);
size_t kp_smem_bytes(int cw);
// Cluster-resident panel kernel (k2_cpanel.cu): the 64 x m panel in the shared memory of ONE
// thread-block cluster (G = cluster size <= 16 CTAs, cw columns each), pivots exchanged over
// distributed shared memory in micro-panels of 8 rows.  Same parameters and outputs as kp_launch
// (cand / wrec / lastbuf unused, colbuf is a small scratch).
constexpr int kKCMaxC = 16;
constexpr int kKCMaxCw = 400;  // 64 x 400 doubles = 200 KB dynamic + 24 KB static shared memory
// cluster size for active width m and its chunk width; 0: m is outside the cluster kernel's range
// on the current device (kc_max_cluster: the largest cluster it can co-schedule, probed once)
int kc_plan(int64_t m, int* cw_out);
int kc_max_cluster();
cudaError_t kc_launch(const KPParams& p, cudaStream_t s, const KPParams* second = nullptr);
size_t kc_smem_bytes(int cw);
int kc_debug_spans(unsigned long long* out, int max_spans);
// debug: (entry, exit) globaltimer of the panel launches since the last call; returns the count
int kp_debug_spans(unsigned long long* out, int max_spans);

// All launches are asynchronous on `s`; `abort` (device) short-circuits every
// kernel once a panel pivot failed the witness test.
// Per trailing row: L[r, 0:K] = -A[r, P[0:K]] (negated), then A[r, c] = A[r, src] for the moved columns.
cudaError_t k2_gather_fix(double* ws, int64_t ld, int32_t rbase, int32_t nrows, int32_t K, const K2Gather* gp,
                          double* L, const unsigned* abort, cudaStream_t s);
// Pair gather (K = 128) fused with the L correction NL[:, 64:128] += NL[:, 0:64] * Wp.
cudaError_t k2_gather_lcorr(double* ws, int64_t ld, int32_t rbase, int32_t nrows, const K2Gather* gp, double* L,
                            const double* Wp, const unsigned* abort, cudaStream_t s, int64_t ldl = 128);
// a group of two pairs (a, b): Wx = lcorr_b(-W_a[:, P_b]) (128 x 128), then b's column moves
// applied to W_a in place (k2_blocked.cu)
cudaError_t k2_group_prep(double* Wa, int64_t ldw, const K2Gather* gb, const double* Wpb, double* Wx,
                          const unsigned* abort, cudaStream_t s);

// C[M x N2] (rows rbase.. of ws) += NL[M x K] W[K x N2], K in {64, 128}; NL (= -L, as written by
// k2_gather_fix) row stride ldl;
// row_wit (nullable) receives the running max |C| per row.
// sm_budget > 0: at most that many SMs, one "fat" CTA each (the rest stay free).
cudaError_t k2_gemm(double* ws, int64_t ld, int32_t rbase, int32_t M, int32_t N2, int32_t K, const double* L,
                    int64_t ldl, const double* W, int64_t ldw, double* row_wit, const unsigned* abort, cudaStream_t s,
                    int sm_budget = 0, const double* W1 = nullptr);

// The blocked path's tail (k3_batched.cu): rows row0 .. row0+n-1 x n columns of the workspace (n <= 128)
// condensed to the end by one pair of warps, K1's in-place arithmetic; records rec[0 .. n-1].
cudaError_t k3_tail_launch(const double* ws, int64_t ldw, int32_t row0, int32_t n, bool fast, const double* wit_in,
                           PivRec* rec, uint32_t epoch, const unsigned* abort, cudaStream_t s);
// nonfinite (nullable, device): set to nonzero if any input entry is NaN/Inf.
cudaError_t k3_launch(const double* a, int64_t batch, int64_t n, int64_t stride, bool fast,
                      int32_t* sign, double* log_abs, double* pivots, unsigned* nonfinite, cudaStream_t s);

}  // namespace mcnd

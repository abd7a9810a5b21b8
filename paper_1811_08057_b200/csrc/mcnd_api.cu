// Host runtime + C ABI (include/mcnd_b200.h).
//
// Everything the reference does on the host around the hot loop lives here,
// in native code: argument validation (matrix.py:32-48, condense.py:85-86,
// runtime.py:35-36), the pivot schedule (condense.py:147-152 top-to-bottom or
// a caller sequence; runtime.py:153-156 round-robin block owners), the exact
// sign bookkeeping (condense.py:125-128, runtime.py:179-182), the sequential
// log sum (condense.py:124; runtime.py:114-120 rank-ordered reduce), the p x p
// elimination tail of the block-row driver (runtime.py:206-219 ->
// gauss.py:34-68), the communication accounting (runtime.py:47-66, 82-90) and
// the multi-GPU plumbing (CUDA IPC mappings of every rank's workspace).
// The GPU does all O(N^3) work; the host touches O(N) numbers.
//
// Compiled with -ffp-contract=off: the tail LU must round exactly like numpy.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>  // types only: libnccl.so.2 is resolved at run time (mg_nccl)
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <map>
#include <mutex>
#include <string>
#include <vector>
#include "../../include/mcnd_b200.h"
#include "mcnd_internal.h"

namespace mcnd {
namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CUDA_TRY(expr)                                                                      \
    do {                                                                                    \
        cudaError_t _e = (expr);                                                            \
        if (_e != cudaSuccess)                                                              \
            return fail(MCND_ECUDA, "%s failed: %s", #expr, cudaGetErrorString(_e));        \
    } while (0)

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

long env_long(const char* name, long dflt) {
    const char* v = std::getenv(name);
    if (!v || !*v) return dflt;
    return std::strtol(v, nullptr, 10);
}

// One panel (second == nullptr) or both panels of a pair in one launch: the cluster-resident
// kernel (k2_cpanel.cu) while the panel fits one thread-block cluster (active width <= 16 x 400
// columns), the column-distributed kernel (k2_panel.cu) above.  Test hooks: MCND_KC=0 keeps the
// column-distributed kernel everywhere, MCND_KC_MAXM lowers the cluster kernel's range, MCND_KC_C
// caps the cluster size.
cudaError_t panel_launch(KPParams q0, cudaStream_t st, KPParams* q1) {
    int cw = 0;
    int C = (env_long("MCND_KC", 1) != 0 && q0.m <= env_long("MCND_KC_MAXM", 1L << 30)) ? kc_plan(q0.m, &cw) : 0;
    if (C > 0) {
        const long fc = env_long("MCND_KC_C", 0);  // test hook: a smaller cluster (wider chunks, more columns per thread)
        if (fc > 0 && fc < C && (q0.m + fc - 1) / fc <= kKCMaxCw - 31) {
            C = (int)fc;
            cw = (int)(((q0.m + fc - 1) / fc + 31) / 32 * 32);
        }
        KPParams c0 = q0, c1 = q1 ? *q1 : q0;
        c0.G = C; c0.cw = cw;
        c1.G = C; c1.cw = cw;
        const cudaError_t e = kc_launch(c0, st, q1 ? &c1 : nullptr);
        // a cluster the device cannot place after all (the probe of kc_max_cluster is an estimate):
        // nothing was launched, the column-distributed kernel takes the panel
        if (e != cudaErrorLaunchOutOfResources && e != cudaErrorInvalidConfiguration && e != cudaErrorInvalidClusterSize)
            return e;
        (void)cudaGetLastError();
    }
    if (q0.cw > kKPMaxCw) return cudaErrorInvalidValue;
    return kp_launch(q0, st, q1);
}

// ---- cached device/pinned buffers (one set per device; calls are serialised) ----
struct Buffers {
    int device = -1;
    void* dws = nullptr;   size_t dws_bytes = 0;    // condensation workspace(s) + records + metadata
    void* din = nullptr;   size_t din_bytes = 0;    // H2D staging for host-input calls
    void* hpin = nullptr;  size_t hpin_bytes = 0;   // pinned metadata / result staging
    void* dge = nullptr;   size_t dge_bytes = 0;    // GE: transposed matrix, row ids, witness
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    cudaStream_t side = nullptr;                 // K2: trailing updates overlapped with the next panels (lowest priority)
    cudaStream_t crit = nullptr;                 // K2: the panel chain (highest priority)
    cudaEvent_t ev_a = nullptr, ev_b = nullptr, ev_c = nullptr;  // K2: stream joins
    cudaEvent_t ev_in = nullptr, ev_out = nullptr;
    cudaEvent_t ev_h0 = nullptr, ev_h1 = nullptr;  // timed: host-input staging (mc_parallel's scatter)
    cudaStream_t cpy = nullptr;                  // K2 host input: row chunks copied while the first pairs run
    std::mutex mu;                               // calls on this device are serialised; other devices run concurrently
    static constexpr int kMaxChunks = 32;
    cudaEvent_t ev_arr[kMaxChunks] = {};
    int sms = 0;
    uint32_t epoch = 0;
};
std::mutex g_mu;             // guards g_bufs (the list, not the buffers)
std::deque<Buffers> g_bufs;  // one per device; deque: element addresses are stable

int init_buffers(Buffers& b, int dev) {
    b.device = dev;
    cudaDeviceGetAttribute(&b.sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaEventCreate(&b.ev0) != cudaSuccess || cudaEventCreate(&b.ev1) != cudaSuccess ||
        cudaEventCreate(&b.ev_h0) != cudaSuccess || cudaEventCreate(&b.ev_h1) != cudaSuccess)
        return fail(MCND_ECUDA, "cudaEventCreate failed");
    int prio_lo = 0, prio_hi = 0;
    cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
    if (cudaEventCreateWithFlags(&b.ev_a, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&b.ev_b, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&b.ev_c, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&b.ev_in, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&b.ev_out, cudaEventDisableTiming) != cudaSuccess ||
        cudaStreamCreateWithPriority(&b.side, cudaStreamNonBlocking, prio_lo) != cudaSuccess ||
        cudaStreamCreateWithPriority(&b.crit, cudaStreamNonBlocking, prio_hi) != cudaSuccess ||
        cudaStreamCreateWithFlags(&b.cpy, cudaStreamNonBlocking) != cudaSuccess)
        return fail(MCND_ECUDA, "cudaEventCreate/cudaStreamCreate failed");
    for (auto& ev : b.ev_arr)
        if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) return fail(MCND_ECUDA, "cudaEventCreate failed");
    return MCND_OK;
}

Buffers* buffers_for_current(int* code) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) { *code = fail(MCND_ECUDA, "cudaGetDevice: %s", cudaGetErrorString(e)); return nullptr; }
    std::lock_guard<std::mutex> lk(g_mu);
    for (auto& b : g_bufs) if (b.device == dev) return &b;
    g_bufs.emplace_back();
    if ((*code = init_buffers(g_bufs.back(), dev)) != MCND_OK) {
        g_bufs.pop_back();
        return nullptr;
    }
    return &g_bufs.back();
}

int ensure_dev(void** p, size_t* have, size_t need) {
    if (*have >= need) return MCND_OK;
    if (*p) cudaFree(*p);
    *p = nullptr;
    *have = 0;
    cudaError_t e = cudaMalloc(p, need);
    if (e != cudaSuccess) return fail(MCND_ECUDA, "cudaMalloc(%zu): %s", need, cudaGetErrorString(e));
    *have = need;
    return MCND_OK;
}

int ensure_pinned(void** p, size_t* have, size_t need) {
    if (*have >= need) return MCND_OK;
    if (*p) cudaFreeHost(*p);
    *p = nullptr;
    *have = 0;
    cudaError_t e = cudaMallocHost(p, need);
    if (e != cudaSuccess) return fail(MCND_ECUDA, "cudaMallocHost(%zu): %s", need, cudaGetErrorString(e));
    *have = need;
    return MCND_OK;
}

// ---- schedules ----
struct Blocks {  // plan_blocks (runtime.py:33-44)
    std::vector<int64_t> start, len;
    int32_t group_of(int64_t r) const {
        for (size_t w = 0; w < start.size(); ++w) if (r < start[w] + len[w]) return (int32_t)w;
        return (int32_t)start.size() - 1;
    }
};

Blocks plan_blocks(int64_t n, int32_t p) {
    Blocks b;
    const int64_t base = n / p, extra = n % p;
    int64_t s0 = 0;
    for (int32_t w = 0; w < p; ++w) {
        b.start.push_back(s0);
        b.len.push_back(base + (w < extra ? 1 : 0));
        s0 += b.len.back();
    }
    return b;
}

// Round-robin owner schedule of mc_parallel (runtime.py:153-156): each pass
// visits workers in rank order, skipping those with <= 1 live row; the owner's
// pivot row is its topmost live row.  n - p steps.
void round_robin(const Blocks& b, std::vector<int32_t>* seq, std::vector<int32_t>* owner) {
    const int32_t p = (int32_t)b.start.size();
    std::vector<int64_t> consumed((size_t)p, 0);
    for (;;) {
        bool any = false;
        for (int32_t w = 0; w < p; ++w) any |= (b.len[(size_t)w] - consumed[(size_t)w] > 1);
        if (!any) break;
        for (int32_t w = 0; w < p; ++w) {
            if (b.len[(size_t)w] - consumed[(size_t)w] <= 1) continue;
            seq->push_back((int32_t)(b.start[(size_t)w] + consumed[(size_t)w]));
            owner->push_back(w);
            consumed[(size_t)w] += 1;
        }
    }
}

// ---- K1 plan and run ----
struct K1Run {
    int64_t n = 0;
    int64_t steps = 0;              // S
    std::vector<int32_t> seq;       // S (+1 when a final 1x1 pivot is published)
    std::vector<double> piv_val;    // outputs, seq.size()
    std::vector<int32_t> piv_col;
    int64_t singular_at = -1;       // pivot index with failed witness test
    double device_ms = 0.0;
    double scatter_s = 0.0, comm_s = 0.0;  // in-kernel distribution / pivot-row publication time
};

// Per-group workspace layout: [matrix n x ld][records npv][row_wit n]
struct GroupLayout {
    int64_t ld = 0;
    size_t o_rec = 0, o_wit = 0, bytes = 0;
};

GroupLayout group_layout(int64_t n, int64_t npv) {
    GroupLayout L;
    L.ld = (int64_t)align_up((size_t)n, 16);
    size_t off = align_up((size_t)n * L.ld * sizeof(double), 256);
    L.o_rec = off;
    off = align_up(off + (size_t)npv * sizeof(PivRec), 256);
    L.o_wit = off;
    off = align_up(off + (size_t)n * sizeof(double), 256);
    L.bytes = off;
    return L;
}

// Rows of each local group dealt cyclically over its CTAs, ascending pivot index.
void deal_rows(int64_t n, const std::vector<int32_t>& seq, const std::vector<int32_t>& row_group,
               int32_t group0, int32_t n_local, int32_t cpg, std::vector<int32_t>* pstep,
               std::vector<int32_t>* row_ptr, std::vector<int32_t>* rows) {
    pstep->assign((size_t)n, kNever);
    for (size_t t = 0; t < seq.size(); ++t) (*pstep)[(size_t)seq[t]] = (int32_t)t;
    std::vector<int32_t> order;
    order.reserve((size_t)n);
    for (int32_t r : seq) order.push_back(r);
    for (int64_t r = 0; r < n; ++r) if ((*pstep)[(size_t)r] == kNever) order.push_back((int32_t)r);
    std::vector<std::vector<int32_t>> per_cta((size_t)n_local * cpg);
    std::vector<int64_t> dealt((size_t)n_local, 0);
    for (int32_t r : order) {
        const int32_t g = row_group[(size_t)r] - group0;
        if (g < 0 || g >= n_local) continue;
        per_cta[(size_t)g * cpg + (size_t)(dealt[(size_t)g]++ % cpg)].push_back(r);
    }
    row_ptr->assign(per_cta.size() + 1, 0);
    rows->clear();
    for (size_t c = 0; c < per_cta.size(); ++c) {
        (*row_ptr)[c + 1] = (*row_ptr)[c] + (int32_t)per_cta[c].size();
        rows->insert(rows->end(), per_cta[c].begin(), per_cta[c].end());
    }
}

// Launch description shared by the single-process and multi-process paths.
struct K1Launch {
    int64_t n = 0, lda = 0;
    int32_t n_groups = 1, group0 = 0, n_local = 1, cpg = 1;
    bool sys = false;
    uint32_t epoch = 1;
    double* ws[kMaxGroups] = {};
    PivRec* rec[kMaxGroups] = {};
    double* wit[kMaxGroups] = {};         // local groups
    const double* src[kMaxGroups] = {};   // local groups
    int64_t src_row0[kMaxGroups] = {};
    std::vector<int32_t> row_group;       // group of every row
    void* d_meta = nullptr;               // device metadata area
    size_t meta_bytes = 0;
    unsigned long long timeout_ns = 20ull * 1000000000ull;
    bool reset_records = true;
    int32_t* ge_ids = nullptr;            // GE mode (K1Params::ge_ids)
    const double* ge_rowwit = nullptr;
};

size_t meta_bytes_for(int64_t n, int64_t npv, int64_t ctas) {
    return align_up((size_t)(npv + n + ctas + 1 + n) * sizeof(int32_t), 256) + align_up(sizeof(K1Err), 256);
}

// Uploads the schedule, launches K1, downloads the pivot records of the first
// local group.  Leaves the stream synchronised.
int k1_execute(Buffers& B, K1Launch& L, bool fast, cudaStream_t st, K1Run& run) {
    const int64_t n = L.n;
    const int64_t npiv = (int64_t)run.seq.size();
    const int64_t npv = std::max<int64_t>(npiv, 1);
    const int64_t ctas = (int64_t)L.n_local * L.cpg;

    std::vector<int32_t> pstep, row_ptr, rows;
    deal_rows(n, run.seq, L.row_group, L.group0, L.n_local, L.cpg, &pstep, &row_ptr, &rows);
    for (int64_t c = 0; c < ctas; ++c)
        if (row_ptr[(size_t)c + 1] - row_ptr[(size_t)c] > kK1MaxRowsPerCta)
            return fail(MCND_EINVAL, "n=%lld needs more than %d rows per CTA on this device", (long long)n,
                        kK1MaxRowsPerCta);

    const size_t n_int = (size_t)(npv + n + ctas + 1 + n);
    const size_t rec_bytes = (size_t)npv * sizeof(PivRec);
    if (meta_bytes_for(n, npv, ctas) > L.meta_bytes) return fail(MCND_EINVAL, "metadata area too small");
    int rc = ensure_pinned(&B.hpin, &B.hpin_bytes, std::max(n_int * sizeof(int32_t), rec_bytes + 256) + 256);
    if (rc) return rc;
    int32_t* hi = (int32_t*)B.hpin;
    std::memset(hi, 0, (size_t)npv * sizeof(int32_t));
    std::memcpy(hi, run.seq.data(), (size_t)npiv * sizeof(int32_t));
    std::memcpy(hi + npv, pstep.data(), (size_t)n * sizeof(int32_t));
    std::memcpy(hi + npv + n, row_ptr.data(), (size_t)(ctas + 1) * sizeof(int32_t));
    std::memcpy(hi + npv + n + ctas + 1, rows.data(), (size_t)n * sizeof(int32_t));
    char* meta = (char*)L.d_meta;
    const size_t o_err = align_up(n_int * sizeof(int32_t), 256);
    CUDA_TRY(cudaMemcpyAsync(meta, hi, n_int * sizeof(int32_t), cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemsetAsync(meta + o_err, 0, sizeof(K1Err), st));
    if (L.reset_records)
        for (int32_t g = 0; g < L.n_local; ++g)
            CUDA_TRY(cudaMemsetAsync(L.rec[L.group0 + g], 0, rec_bytes, st));

    K1Params p{};
    for (int g = 0; g < kMaxGroups; ++g) {
        p.src[g] = L.src[g];
        p.src_row0[g] = L.src_row0[g];
        p.ws[g] = L.ws[g];
        p.rec[g] = L.rec[g];
        p.row_wit[g] = L.wit[g];
    }
    p.lds = L.lda;
    p.ld = (int64_t)align_up((size_t)n, 16);
    p.n = (int32_t)n;
    p.n_steps = (int32_t)run.steps;
    p.n_groups = L.n_groups;
    p.group0 = L.group0;
    p.n_local_groups = L.n_local;
    p.ctas_per_group = L.cpg;
    p.sys_scope = L.sys ? 1 : 0;
    p.epoch = L.epoch;
    int32_t* di = (int32_t*)meta;
    p.seq = di;
    p.row_pstep = di + npv;
    p.cta_row_ptr = di + npv + n;
    p.cta_rows = di + npv + n + ctas + 1;
    p.err = (K1Err*)(meta + o_err);
    p.chunk = (int32_t)std::min<int64_t>((int64_t)align_up((size_t)n, 2), kK1MaxChunk);
    const long ck = env_long("MCND_K1_CHUNK", 0);  // test knob: force multi-chunk staging
    if (ck >= 2 && ck <= kK1MaxChunk) p.chunk = (int32_t)std::min<int64_t>(p.chunk, ck & ~1L);
    p.timeout_ns = L.timeout_ns;
    p.ncol0 = (int32_t)n;
    p.in_place = 0;
    p.wit_in = nullptr;
    p.abort_flag = nullptr;
    p.pstep_offset = 0;
    p.ge_ids = L.ge_ids;
    p.ge_rowwit = L.ge_rowwit;

    CUDA_TRY(cudaEventRecord(B.ev0, st));
    cudaError_t e = k1_launch(p, fast, st);
    if (e != cudaSuccess) return fail(MCND_ECUDA, "condensation kernel launch: %s", cudaGetErrorString(e));
    CUDA_TRY(cudaEventRecord(B.ev1, st));

    char* hp = (char*)B.hpin;
    PivRec* h_rec = (PivRec*)hp;
    K1Err* h_err = (K1Err*)(hp + align_up(rec_bytes, 64));
    CUDA_TRY(cudaMemcpyAsync(h_rec, L.rec[L.group0], rec_bytes, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(h_err, meta + o_err, sizeof(K1Err), cudaMemcpyDeviceToHost, st));
    e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return fail(MCND_ECUDA, "condensation kernel: %s", cudaGetErrorString(e));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, B.ev0, B.ev1);
    run.device_ms = ms;
    run.scatter_s = (double)h_err->scatter_ns * 1e-9;
    run.comm_s = (double)h_err->comm_ns * 1e-9;
    if (h_err->nonfinite) return fail(MCND_EINVAL, "matrix entries must be finite (no NaN/Inf)");
    if (h_err->error) return fail(MCND_EDEVICE, "device timeout waiting for pivot %u", h_err->err_step);
    run.piv_val.resize((size_t)npiv);
    run.piv_col.resize((size_t)npiv);
    run.singular_at = -1;
    int64_t published = 0;
    for (int64_t t = 0; t < npiv; ++t) {
        if (h_rec[t].flag != L.epoch) break;
        run.piv_val[(size_t)t] = h_rec[t].v;
        run.piv_col[(size_t)t] = h_rec[t].l;
        ++published;
        if (h_rec[t].l < 0) { run.singular_at = t; break; }
    }
    if (run.singular_at < 0 && published != npiv)
        return fail(MCND_EDEVICE, "protocol error: %lld of %lld pivots published", (long long)published,
                    (long long)npiv);
    return MCND_OK;
}

// Single-process run: P groups (1 = plain single GPU; p > 1 = the p workers as
// CTA groups with separate workspaces, exercising the multi-GPU push protocol).
int k1_run_local(Buffers& B, const double* d_a, int64_t n, int64_t lda, bool fast, cudaStream_t st,
                 K1Run& run, const Blocks* groups, const std::vector<int32_t>* keep_rows, int64_t keep_cols,
                 std::vector<double>* keep_out, std::vector<double>* keep_wit, int32_t* ge_ids = nullptr,
                 const double* ge_rowwit = nullptr) {
    const int32_t P = groups ? (int32_t)groups->start.size() : 1;
    if (P > kMaxGroups) return fail(MCND_EINVAL, "at most %d CTA groups", kMaxGroups);
    const int64_t npv = std::max<int64_t>((int64_t)run.seq.size(), 1);
    const GroupLayout GL = group_layout(n, npv);
    int64_t cpg = P == 1 ? std::min<int64_t>(B.sms, n) : std::max<int64_t>(B.sms / P, 1);
    const long eg = env_long("MCND_K1_GRID", 0);  // test knob: fewer CTAs, more rows per CTA
    if (eg > 0) cpg = std::max<int64_t>(1, std::min<int64_t>(cpg, eg));
    const size_t mb = meta_bytes_for(n, npv, P * cpg);
    int rc = ensure_dev(&B.dws, &B.dws_bytes, (size_t)P * GL.bytes + mb);
    if (rc) return rc;
    char* base = (char*)B.dws;
    K1Launch L;
    L.n = n;
    L.lda = lda;
    L.n_groups = P;
    L.group0 = 0;
    L.n_local = P;
    L.cpg = (int32_t)cpg;
    L.sys = false;
    L.epoch = ++B.epoch;
    for (int32_t g = 0; g < P; ++g) {
        char* gb = base + (size_t)g * GL.bytes;
        L.ws[g] = (double*)gb;
        L.rec[g] = (PivRec*)(gb + GL.o_rec);
        L.wit[g] = (double*)(gb + GL.o_wit);
        L.src[g] = d_a;
        L.src_row0[g] = 0;
    }
    L.row_group.assign((size_t)n, 0);
    if (groups)
        for (int64_t r = 0; r < n; ++r) L.row_group[(size_t)r] = groups->group_of(r);
    L.d_meta = base + (size_t)P * GL.bytes;
    L.meta_bytes = mb;
    L.ge_ids = ge_ids;
    L.ge_rowwit = ge_rowwit;
    rc = k1_execute(B, L, fast, st, run);
    if (rc) return rc;
    if (keep_rows && keep_out) {
        keep_out->assign(keep_rows->size() * (size_t)keep_cols, 0.0);
        keep_wit->assign(keep_rows->size(), 0.0);
        for (size_t i = 0; i < keep_rows->size(); ++i) {
            const int32_t r = (*keep_rows)[i], g = L.row_group[(size_t)r];
            CUDA_TRY(cudaMemcpy(keep_out->data() + i * keep_cols, L.ws[g] + (int64_t)r * GL.ld,
                                (size_t)keep_cols * sizeof(double), cudaMemcpyDeviceToHost));
            CUDA_TRY(cudaMemcpy(keep_wit->data() + i, L.wit[g] + r, sizeof(double), cudaMemcpyDeviceToHost));
        }
    }
    return MCND_OK;
}

// Fenwick tree over row ids: k_pos = number of live rows before the pivot row
// (the pivot's position in active_rows, condense.py:113).
struct Fenwick {
    std::vector<int32_t> t;
    explicit Fenwick(int64_t n) : t((size_t)n + 1, 0) {
        for (int64_t i = 1; i <= n; ++i) {
            t[(size_t)i] += 1;
            int64_t j = i + (i & -i);
            if (j <= n) t[(size_t)j] += t[(size_t)i];
        }
    }
    int64_t prefix(int64_t i) const {  // live rows with id < i
        int64_t s = 0;
        for (; i > 0; i -= i & -i) s += t[(size_t)i];
        return s;
    }
    void remove(int64_t i) {
        for (++i; i < (int64_t)t.size(); i += i & -i) t[(size_t)i] -= 1;
    }
};

// gauss.py:16-31
int permutation_parity(const std::vector<int64_t>& perm) {
    std::vector<char> seen(perm.size(), 0);
    int parity = 1;
    for (size_t s = 0; s < perm.size(); ++s) {
        if (seen[s]) continue;
        size_t len = 0, j = s;
        while (!seen[j]) { seen[j] = 1; j = (size_t)perm[j]; ++len; }
        if (len % 2 == 0) parity = -parity;
    }
    return parity;
}

// gauss.py:34-68, row-pivoted elimination on the tiny p x p remainder.
void logdet_lu_host(std::vector<double> a, int64_t n, const std::vector<double>& wit, int32_t* sign,
                    double* log_abs) {
    std::vector<int64_t> unproc((size_t)n), perm;
    for (int64_t i = 0; i < n; ++i) unproc[(size_t)i] = i;
    double log_acc = 0.0;
    int signs = 1;
    for (int64_t k = 0; k < n; ++k) {
        size_t bi = 0;
        double bv = std::fabs(a[(size_t)(unproc[0] * n + k)]);
        for (size_t i = 1; i < unproc.size(); ++i) {
            const double v = std::fabs(a[(size_t)(unproc[i] * n + k)]);
            if (v > bv) { bv = v; bi = i; }
        }
        const int64_t pr = unproc[bi];
        const double piv = a[(size_t)(pr * n + k)];
        if (piv == 0.0 || std::fabs(piv) <= kSingularRtol * wit[(size_t)pr]) {
            *sign = 0;
            *log_abs = -INFINITY;
            return;
        }
        perm.push_back(pr);
        unproc.erase(unproc.begin() + (long)bi);
        log_acc += std::log(std::fabs(piv));
        signs *= piv > 0 ? 1 : -1;
        for (int64_t r : unproc) {
            const double f = a[(size_t)(r * n + k)] / piv;
            for (int64_t c = k + 1; c < n; ++c) {
                const double prod = f * a[(size_t)(pr * n + c)];
                a[(size_t)(r * n + c)] = a[(size_t)(r * n + c)] - prod;
            }
        }
    }
    *sign = signs * permutation_parity(perm);
    *log_abs = log_acc;
}

void clear_out(mcnd_logdet* out) {
    std::memset(out, 0, sizeof(*out));
    out->singular_step = -1;
    out->invalid_step = -1;
    out->invalid_row = -1;
}

int check_shape(const void* a, int64_t n, int64_t lda) {
    if (!a) return fail(MCND_EINVAL, "null matrix pointer");
    if (n < 1) return fail(MCND_EINVAL, "matrix dimensions must be positive");
    if (lda < n) return fail(MCND_EINVAL, "lda (%lld) < n (%lld)", (long long)lda, (long long)n);
    return MCND_OK;
}

int serial_dev(const double* d_a, int64_t n, int64_t lda, const int64_t* seq_in, int64_t seq_len,
               uint32_t flags, cudaStream_t st, mcnd_logdet* out, double* pivots_out, int32_t* cols_out) {
    clear_out(out);
    int rc = check_shape(d_a, n, lda);
    if (rc) return rc;
    int code = MCND_OK;
    Buffers* B = buffers_for_current(&code);
    if (!B) return code;

    // pivot schedule (condense.py:147-152); validation mirrors select_pivot's
    // "row is not active" (condense.py:85-86) and the IndexError of a short
    // sequence, which the reference only raises when it reaches that step.
    K1Run run;
    run.n = n;
    int64_t bad = -1, bad_row = -1;
    int bad_code = MCND_OK;
    if (seq_in == nullptr) {
        run.seq.resize((size_t)n);
        for (int64_t i = 0; i < n; ++i) run.seq[(size_t)i] = (int32_t)i;
        run.steps = n - 1;
    } else {
        std::vector<char> used((size_t)n, 0);
        for (int64_t t = 0; t < n - 1; ++t) {
            if (t >= seq_len) { bad = t; bad_code = MCND_EPIVOT_SHORT; break; }
            const int64_t r = seq_in[t];
            if (r < 0 || r >= n || used[(size_t)r]) { bad = t; bad_row = r; bad_code = MCND_EPIVOT; break; }
            used[(size_t)r] = 1;
            run.seq.push_back((int32_t)r);
        }
        if (bad < 0) {
            for (int64_t r = 0; r < n; ++r) if (!used[(size_t)r]) { run.seq.push_back((int32_t)r); break; }
            run.steps = n - 1;
        } else {
            run.steps = bad;  // run the valid prefix; the error surfaces unless it went singular first
        }
    }
    rc = k1_run_local(*B, d_a, n, lda, (flags & MCND_FLAG_FAST) != 0, st, run, nullptr, nullptr, 0, nullptr,
                      nullptr);
    if (rc) return rc;
    out->device_ms = run.device_ms;
    out->launches = 1;
    if (pivots_out) for (size_t t = 0; t < run.piv_val.size(); ++t) pivots_out[t] = run.piv_val[t];
    if (cols_out) for (size_t t = 0; t < run.piv_col.size(); ++t) cols_out[t] = run.piv_col[t];
    if (run.singular_at >= 0) {
        out->sign = 0;
        out->singular = 1;
        out->log_abs = -INFINITY;
        out->singular_step = run.singular_at;
        out->steps = run.singular_at;
        return MCND_OK;
    }
    if (bad >= 0) {
        out->invalid_step = bad;
        out->invalid_row = bad_row;
        out->steps = bad;
        if (bad_code == MCND_EPIVOT) return fail(MCND_EPIVOT, "row %lld is not active", (long long)bad_row);
        return fail(MCND_EPIVOT_SHORT, "pivot_sequence index %lld out of range", (long long)bad);
    }
    // sign and log in reference order (condense.py:124-128, 159-160)
    Fenwick live(n);
    double log_acc = 0.0;
    int sign_acc = 1;
    for (int64_t t = 0; t < n - 1; ++t) {
        const int64_t m = n - t;
        const int64_t r = run.seq[(size_t)t];
        const double v = run.piv_val[(size_t)t];
        const int64_t k_pos = seq_in ? live.prefix(r) : 0;
        if (seq_in) live.remove(r);
        log_acc += std::log(std::fabs(v));
        const int swap_parity = (run.piv_col[(size_t)t] != m - 1) ? -1 : 1;
        const int parity = ((k_pos + m - 1) % 2) ? -1 : 1;
        sign_acc *= (v > 0 ? 1 : -1) * swap_parity * parity;
    }
    const double vf = run.piv_val[(size_t)(n - 1)];
    out->sign = sign_acc * (vf > 0 ? 1 : -1);
    out->log_abs = log_acc + std::log(std::fabs(vf));
    out->steps = n - 1;
    return MCND_OK;
}

// ---- Gaussian elimination with row pivoting: logdet_lu (gauss.py:34-68) on the GPU ----
// K1 in GE mode on A^T.  Column k of A is row k of A^T; gauss.py's pivot (max |a[r, k]| over
// the unprocessed rows r, ties -> lowest r) is K1's argmax over that row with ties broken by
// the original row id; its update a[r, j] -= (a[r, k] / piv) * a[p, j] is, transposed, K1's
// b[j, c] -= b[j, l] * (b[k, c] / v) with the same three roundings (the product commutes).  So
// the pivots are bitwise gauss.py's and so is log|det| (summed in pivot order); the sign is
// prod sgn(piv) x parity(pivot rows) (gauss.py:16-31, 64-68).  Singular: an exactly zero
// pivot, or |piv| <= 1e-12 x row_witness[pivot row] when the caller passes one (gauss.py:55-58).
int ge_dev(const double* d_a, int64_t n, int64_t lda, const double* d_rowwit, uint32_t flags, cudaStream_t st,
           mcnd_logdet* out, double* pivots_out, int32_t* rows_out, const double* h_rowwit = nullptr) {
    clear_out(out);
    int rc = check_shape(d_a, n, lda);
    if (rc) return rc;
    int code = MCND_OK;
    Buffers* B = buffers_for_current(&code);
    if (!B) return code;
    // transposed matrix + row ids (+ the witness), in the library's GE scratch area
    const size_t o_t = 0, o_ids = align_up((size_t)n * n * sizeof(double), 256);
    const size_t o_w = o_ids + align_up((size_t)n * sizeof(int32_t), 256);
    rc = ensure_dev(&B->dge, &B->dge_bytes, o_w + (size_t)n * sizeof(double));
    if (rc) return rc;
    char* base = (char*)B->dge;
    double* at = (double*)(base + o_t);
    int32_t* ids = (int32_t*)(base + o_ids);
    if (h_rowwit) {
        d_rowwit = (const double*)(base + o_w);
        CUDA_TRY(cudaMemcpyAsync((void*)d_rowwit, h_rowwit, (size_t)n * sizeof(double), cudaMemcpyHostToDevice, st));
    }
    cudaError_t e = transpose_launch(d_a, n, lda, at, n, st);
    if (e != cudaSuccess) return fail(MCND_ECUDA, "transpose: %s", cudaGetErrorString(e));
    std::vector<int32_t> iota((size_t)n);
    for (int64_t i = 0; i < n; ++i) iota[(size_t)i] = (int32_t)i;
    CUDA_TRY(cudaMemcpyAsync(ids, iota.data(), (size_t)n * sizeof(int32_t), cudaMemcpyHostToDevice, st));
    K1Run run;
    run.n = n;
    run.seq = iota;
    run.steps = n - 1;
    rc = k1_run_local(*B, at, n, n, (flags & MCND_FLAG_FAST) != 0, st, run, nullptr, nullptr, 0, nullptr, nullptr,
                      ids, d_rowwit);
    if (rc) return rc;
    out->device_ms = run.device_ms;
    out->launches = 2;
    // replay the column exchanges: position l at step t holds original row ids[l]
    std::vector<int64_t> perm;
    perm.reserve((size_t)n);
    std::vector<int32_t> cur = iota;
    const int64_t np = run.singular_at >= 0 ? run.singular_at + 1 : n;
    for (int64_t t = 0; t < np; ++t) {
        const int64_t m = n - t;
        const int32_t lr = run.piv_col[(size_t)t];
        const int32_t l = lr >= 0 ? lr : -lr - 2;  // a singular record keeps its position as -(l + 2)
        const int32_t id = cur[(size_t)l];
        if (pivots_out) pivots_out[t] = run.piv_val[(size_t)t];
        if (rows_out) rows_out[t] = id;
        if (lr >= 0) { perm.push_back(id); if (l != m - 1) cur[(size_t)l] = cur[(size_t)(m - 1)]; }
    }
    if (run.singular_at >= 0) {
        out->sign = 0; out->singular = 1; out->log_abs = -INFINITY;
        out->singular_step = run.singular_at; out->steps = run.singular_at;
        return MCND_OK;
    }
    double log_acc = 0.0;
    int signs = 1;
    for (int64_t t = 0; t < n; ++t) {
        const double v = run.piv_val[(size_t)t];
        log_acc += std::log(std::fabs(v));
        signs *= v > 0 ? 1 : -1;
    }
    out->sign = signs * permutation_parity(perm);
    out->log_abs = log_acc;
    out->steps = n;
    return MCND_OK;
}

// Folds the mc_parallel pivots + p x p remainder into the reference's result
// and accounting (runtime.py:185-229).  Shared by the single-process and the
// multi-GPU drivers.  singular_at: first pivot that failed the witness test, or -1.
int fold_parallel(int64_t n, int32_t p, const double* piv_vals, const int32_t* piv_cols, int64_t singular_at,
                  const double* rem, const double* rem_wit, mcnd_logdet* out, mcnd_comm_stats* stats,
                  int64_t* payload_out, int64_t* row_updates_out) {
    const Blocks b = plan_blocks(n, p);
    std::vector<int32_t> seq, owner;
    round_robin(b, &seq, &owner);
    const int64_t S = (int64_t)seq.size();
    const int64_t done = singular_at >= 0 ? singular_at : S;
    std::vector<int64_t> cons((size_t)p, 0), row_upd((size_t)p, 0);
    int64_t bbytes = 0, scalar = 0;
    std::vector<double> local_logs((size_t)p, 0.0);
    Fenwick live(n);
    int sign = 1;
    for (int64_t t = 0; t < done; ++t) {
        const int32_t w = owner[(size_t)t];
        const int64_t m = n - t, last = m - 1;
        const double v = piv_vals[t];
        const int64_t r = seq[(size_t)t];
        local_logs[(size_t)w] += std::log(std::fabs(v));
        cons[(size_t)w] += 1;
        const int64_t k_pos = live.prefix(r);
        live.remove(r);
        const int swap_parity = (piv_cols[t] != last) ? -1 : 1;
        const int parity = ((k_pos + m - 1) % 2) ? -1 : 1;
        sign *= (v > 0 ? 1 : -1) * swap_parity * parity;
        bbytes += 8 * last + 8;
        if (payload_out) payload_out[t] = last;
        for (int32_t u = 0; u < p; ++u) {
            const int64_t lv = b.len[(size_t)u] - cons[(size_t)u];
            row_upd[(size_t)u] += lv;
            scalar += lv * last;
        }
    }
    if (row_updates_out) for (int32_t u = 0; u < p; ++u) row_updates_out[u] = row_upd[(size_t)u];
    if (stats) {
        stats->broadcasts = done + (singular_at >= 0 ? 1 : 0);
        stats->broadcast_bytes = bbytes + (singular_at >= 0 ? 1 : 0);
        stats->pivot_search_msgs = 0;
        stats->scalar_updates = scalar;
        stats->aborted_step = singular_at;
    }
    out->steps = done;
    if (singular_at >= 0) {
        out->sign = 0;
        out->singular = 1;
        out->log_abs = -INFINITY;
        out->singular_step = singular_at;
        return MCND_OK;
    }
    // gather -> reduce_sum -> LU tail (runtime.py:209-219)
    std::vector<double> remv(rem, rem + (size_t)p * p), fw(rem_wit, rem_wit + p);
    double total = 0.0;
    for (int32_t w = 0; w < p; ++w) total += local_logs[(size_t)w];
    int32_t rs = 0;
    double rl = 0.0;
    logdet_lu_host(remv, p, fw, &rs, &rl);
    if (rs == 0) {
        out->sign = 0;
        out->singular = 1;
        out->log_abs = -INFINITY;
        out->singular_step = S;
        return MCND_OK;
    }
    out->sign = sign * rs;
    out->log_abs = total + rl;
    return MCND_OK;
}

int parallel_dev(const double* d_a, int64_t n, int64_t lda, int32_t p, uint32_t flags, cudaStream_t st,
                 mcnd_logdet* out, mcnd_comm_stats* stats, int64_t* payload_out, int64_t* row_updates_out,
                 int32_t* owners_out) {
    clear_out(out);
    if (stats) std::memset(stats, 0, sizeof(*stats));
    int rc = check_shape(d_a, n, lda);
    if (rc) return rc;
    if (p < 1 || p > n) return fail(MCND_EINVAL, "invalid plan: need 1 <= p <= n, got p=%d, n=%lld", p, (long long)n);
    const bool groups = (flags & MCND_FLAG_GROUPS) != 0;
    if (groups && p > kMaxGroups) return fail(MCND_EINVAL, "MCND_FLAG_GROUPS supports p <= %d", kMaxGroups);
    int code = MCND_OK;
    Buffers* B = buffers_for_current(&code);
    if (!B) return code;

    const Blocks blk = plan_blocks(n, p);
    K1Run run;
    run.n = n;
    std::vector<int32_t> owner;
    round_robin(blk, &run.seq, &owner);
    run.steps = (int64_t)run.seq.size();  // n - p
    std::vector<int32_t> rem_rows((size_t)p);
    for (int32_t w = 0; w < p; ++w) rem_rows[(size_t)w] = (int32_t)(blk.start[(size_t)w] + blk.len[(size_t)w] - 1);
    std::vector<double> rem, rem_wit;
    rc = k1_run_local(*B, d_a, n, lda, (flags & MCND_FLAG_FAST) != 0, st, run, groups ? &blk : nullptr, &rem_rows,
                      p, &rem, &rem_wit);
    if (rc) return rc;
    out->device_ms = run.device_ms;
    out->launches = 1;
    if (owners_out) for (size_t t = 0; t < owner.size(); ++t) owners_out[t] = owner[t];
    rc = fold_parallel(n, p, run.piv_val.data(), run.piv_col.data(), run.singular_at, rem.data(), rem_wit.data(),
                       out, stats, payload_out, row_updates_out);
    if (stats) {
        stats->scatter_seconds = run.scatter_s;
        stats->comm_seconds = run.comm_s;
    }
    return rc;
}

// Host-input staging: copy an n x n (lda) host matrix into a cached device buffer.
int stage_input(Buffers& B, const double* h_a, int64_t rows, int64_t n, int64_t lda, cudaStream_t st,
                const double** d_out) {
    const size_t need = (size_t)rows * n * sizeof(double);
    int rc = ensure_dev(&B.din, &B.din_bytes, need);
    if (rc) return rc;
    CUDA_TRY(cudaMemcpy2DAsync(B.din, (size_t)n * sizeof(double), h_a, (size_t)lda * sizeof(double),
                               (size_t)n * sizeof(double), (size_t)rows, cudaMemcpyHostToDevice, st));
    *d_out = (const double*)B.din;
    return MCND_OK;
}

// ---- blocked rank-b condensation (K2) ----
// Panels of b = 64 pivot rows while at least `m_tail` columns remain after the
// panel, then the unblocked K1 finishes the last m_tail..m_tail+b-1 rows.  All
// launches are asynchronous; a failed witness test raises a device abort flag
// that turns every later launch into a no-op; one D2H at the end.
int blocked_dev(const double* d_a, int64_t n, int64_t lda, uint32_t flags, cudaStream_t st_caller, mcnd_logdet* out,
                double* pivots_out, int32_t* cols_out, const double* h_src = nullptr) {
    clear_out(out);
    int rc = check_shape(h_src ? h_src : d_a, n, lda);
    if (rc) return rc;
    int code = MCND_OK;
    Buffers* B = buffers_for_current(&code);
    if (!B) return code;
    // The panel chain runs on a highest-priority stream, the overlapped trailing
    // updates on a lowest-priority one: SMs freed by the trailing GEMM's CTAs go to
    // the next panel first.  Joined with the caller's stream at entry and exit; the
    // copy stream of the previous call is drained first (it may still hold reads of
    // its caller's buffer and writes into din).
    cudaStream_t st = B->crit;
    CUDA_TRY(cudaEventRecord(B->ev_in, st_caller));
    CUDA_TRY(cudaStreamWaitEvent(st, B->ev_in, 0));
    // any early return after this point drains the library's streams first: the next call
    // reuses din and the workspace, and a streamed copy may still read the caller's buffer
    struct Drain {
        Buffers* B;
        bool armed = true;
        ~Drain() {
            if (!armed) return;
            cudaStreamSynchronize(B->cpy);
            cudaStreamSynchronize(B->side);
            cudaStreamSynchronize(B->crit);
            cudaGetLastError();
        }
    } drain{B};
    const bool fast = (flags & MCND_FLAG_FAST) != 0;
    const int64_t b = kK2B;
    int64_t m_tail = env_long("MCND_K2_TAIL", 64);  // test hook: rows finished by the unblocked K1 tail
    if (m_tail < 2) m_tail = 2;
    const int64_t n_panels = (n - m_tail >= b) ? (n - m_tail) / b : 0;
    const int64_t kb_end = n_panels * b;
    const int64_t mt = n - kb_end;
    const int64_t ld = (int64_t)align_up((size_t)n, 16);
    const int64_t G0 = std::min<int64_t>(B->sms, n);
    const int64_t Gt = std::min<int64_t>(B->sms, mt);
    if ((n + G0 - 1) / G0 > kK1MaxRowsPerCta) return fail(MCND_EINVAL, "n=%lld too large for one GPU", (long long)n);
    if (n > (int64_t)kKPMaxCw * std::min<int64_t>(B->sms, kKPMaxG))  // panel chunks must fit shared memory
        return fail(MCND_EINVAL, "n=%lld too large for the one-GPU blocked path (at most %d panel columns per SM); "
                    "use logdet_condensation (unblocked)", (long long)n, kKPMaxCw);

    // Streamed host input (a pinned host matrix, the pair schedule with look-ahead): the rows
    // arrive in chunks on a copy stream while the first pairs run.  A pair's side update
    // covers only the chunks expected to have landed by then (a static plan from the copy
    // rate and the pair times; a late chunk only makes the side stream wait for its event);
    // a chunk first covered at pair q is caught up on the side stream first: its K1 init,
    // then the updates of pairs 0..q-1 in order, each with that pair's own L/W/descriptor
    // slot (kept alive: the slot ring grows to the last catch-up).  Every row sees the same
    // kernels in the same order as with the matrix resident, so the result is bitwise the same.
    int n_chunks = 1;
    std::vector<int64_t> cr{0, n};  // chunk row boundaries
    std::vector<int> cov_of;        // per pair: last chunk covered by its side update
    // groups of two pairs: the rows past the second pair's next pair take both pairs' update as
    // ONE rank-256 GEMM (k2_group_prep, k2_gemm K = 256), only while the trailing GEMM bounds
    // the pairs by far -- a group halves the time the side stream has for a pair's bulk rows:
    // C5 0.895 -> 0.853 s with groups above 12000 (8000 / 16000 / 20000: 0.851 / 0.853 / 0.858),
    // C3 30.5 -> 31.4 ms with groups everywhere.  Test hook MCND_K2_GROUP_ABOVE: the active width
    // above which a pair may start a group (0: always).
    const int64_t group_above = env_long("MCND_K2_GROUP_ABOVE", kK2GroupAbove);
    const bool groups = n - 4 * b > group_above;
    // pair slots (L, W, Wp, descriptor): a side update may read slot q while pairs q+1, q+2
    // factor (depth-2 look-ahead); a group's update reads the slots of both its pairs while
    // the next two factor
    int ring = groups ? 4 : 3;
    const bool overlap = env_long("MCND_K2_OVERLAP", 1) != 0;  // test hook: 0 = serial schedule (same arithmetic)
    if (h_src && overlap && n_panels >= 8) {
        cudaPointerAttributes pa{};
        const bool pinned = cudaPointerGetAttributes(&pa, h_src) == cudaSuccess && pa.type == cudaMemoryTypeHost;
        cudaGetLastError();
        // chunk 0 (>= 512 rows) holds the rows pairs 0 and 1 update on the critical stream and in
        // their part A; later parts A touch rows covered two pairs earlier
        const int64_t min_rows = 1024;  // C3 sweep (end to end): 512: 35.2, 768: 34.9, 1024: 34.6, 1536: 34.9 ms
        const int64_t rows_c = (int64_t)align_up((size_t)std::max<int64_t>(min_rows, (n + Buffers::kMaxChunks - 1) / Buffers::kMaxChunks), 128);
        if (pinned && rows_c < n) {
            n_chunks = (int)((n + rows_c - 1) / rows_c);
            cr.assign(1, 0);
            for (int c = 0; c < n_chunks; ++c) cr.push_back(std::min<int64_t>(n, cr.back() + rows_c));
            std::vector<double> arr(n_chunks);  // expected landing times at 60 GB/s (C3 sweep 40: 36.7, 50: 35.9, 56: 35.3, 70: 35.2, 200: 37.1 ms e2e)
            const double gbs = 60e9;
            double t = 0.0;
            for (int c = 0; c < n_chunks; ++c) { t += (double)(cr[c + 1] - cr[c]) * (double)n * 8.0 / gbs; arr[c] = t; }
            auto chunk_of = [&](int64_t row) { return (int)std::min<int64_t>(n_chunks - 1, row / rows_c); };
            double tq = arr[0];
            int cov = 0, q_last = 0;
            for (int64_t k = 0, q = 0; k + 1 < n_panels; k += 2, ++q) {
                const int64_t kb = k * b, m = n - kb, nr = m - 2 * b;
                const double t_pan = 2.0 * 64 * 3.4e-6;
                int c = std::max(cov, chunk_of(std::min<int64_t>(n, kb + 10 * b) - 1));  // through pair q+4's rows
                while (c + 1 < n_chunks && arr[c + 1] <= tq + t_pan) ++c;
                if (k + 3 >= n_panels) c = n_chunks - 1;  // the next unit is not a pair: everything
                if (c > cov || q == 0) q_last = (int)q;
                cov = c;
                cov_of.push_back(c);
                tq += std::max(t_pan, 2.0 * (double)nr * (double)(m - 2 * b) * 128.0 / 26e12) + 60e-6;
            }
            if (cov != n_chunks - 1) { n_chunks = 1; cr.assign({0, n}); cov_of.clear(); }
            else ring = std::max(ring, q_last + 3);
        }
    }
    const bool streamed = n_chunks > 1;
    const int64_t lda_h = lda;
    if (h_src) {  // host input: staged in din (whole, or chunk by chunk when streamed)
        rc = ensure_dev(&B->din, &B->din_bytes, (size_t)n * n * sizeof(double));
        if (rc) return rc;
        if (!streamed)
            CUDA_TRY(cudaMemcpy2DAsync(B->din, (size_t)n * sizeof(double), h_src, (size_t)lda * sizeof(double),
                                       (size_t)n * sizeof(double), (size_t)n, cudaMemcpyHostToDevice, st));
        d_a = (const double*)B->din;
        lda = n;
    }

    // device layout
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off = align_up(off + bytes, 256); return o; };
    const size_t o_ws = take((size_t)n * ld * sizeof(double));
    const size_t o_wit = take((size_t)n * sizeof(double));
    const size_t o_rec = take((size_t)n * sizeof(PivRec));
    // L, W, Wp and the pair's gather descriptor in a ring of kRing pair slots: the side update
    // of pair q may still read its slot while pairs q+1 and q+2 factor (depth-2 look-ahead)
    const int kRing = ring;
    const size_t o_L = take((size_t)kRing * std::max<int64_t>(n, 1) * 2 * b * sizeof(double));
    const size_t o_W = take((size_t)kRing * 2 * b * ld * sizeof(double));
    const size_t o_pan = take((2 + kRing) * sizeof(K2Gather));           // gp0, gp1, gpair ring
    const size_t o_Wp = take((size_t)kRing * b * b * sizeof(double));
    // groups: [NL_a | NL_b] of every row (absolute row index, side stream only) and each group's Wx
    const int64_t n_groups = groups ? n_panels / 4 + 1 : 0;
    const size_t o_Lc = take(groups ? (size_t)n * 4 * b * sizeof(double) : 0);
    const size_t o_Wx = take((size_t)n_groups * 2 * b * 2 * b * sizeof(double));
    const size_t o_cand = take((size_t)64 * kKPMaxG * sizeof(ulonglong2));
    const size_t o_wrec = take((size_t)64 * kKPMaxG * sizeof(ulonglong2));
    const size_t o_colb = take((size_t)64 * kKPMaxG * 64 * sizeof(ulonglong2));
    const size_t o_lastb = take(kLastBufBytes);
    const size_t o_ctl = take(sizeof(K1Err) + 16);
    // int metadata: iota[n] | never[n] | panel_ptr[b+1] | init_ptr[G0+1] init_rows[n] | tail_ptr[Gt+1] tail_rows[mt]
    //               | per-chunk init_ptr[n_chunks][G0+1] (streamed input; rows dealt inside init_rows)
    const size_t n_int = (size_t)(n + n + (b + 1) + (G0 + 1) + n + (Gt + 1) + mt + (streamed ? n_chunks * (G0 + 1) : 0));
    const size_t o_int = take(n_int * sizeof(int32_t));
    rc = ensure_dev(&B->dws, &B->dws_bytes, off);
    if (rc) return rc;
    rc = ensure_pinned(&B->hpin, &B->hpin_bytes, std::max(n_int * sizeof(int32_t), (size_t)n * sizeof(PivRec) + 256) + 256);
    if (rc) return rc;
    char* base = (char*)B->dws;
    int32_t* hi = (int32_t*)B->hpin;
    int32_t* h_iota = hi;
    int32_t* h_never = h_iota + n;
    int32_t* h_pptr = h_never + n;
    int32_t* h_iptr = h_pptr + (b + 1);
    int32_t* h_irows = h_iptr + (G0 + 1);
    int32_t* h_tptr = h_irows + n;
    int32_t* h_trows = h_tptr + (Gt + 1);
    for (int64_t i = 0; i < n; ++i) { h_iota[i] = (int32_t)i; h_never[i] = kNever; }
    for (int64_t i = 0; i <= b; ++i) h_pptr[i] = (int32_t)i;
    auto deal = [](int64_t first, int64_t count, int64_t G, int32_t* ptr, int32_t* rows) {
        ptr[0] = 0;
        for (int64_t c = 0; c < G; ++c) ptr[c + 1] = ptr[c] + (int32_t)((count - c + G - 1) / G);
        std::vector<int32_t> fill(ptr, ptr + G);
        for (int64_t i = 0; i < count; ++i) rows[fill[(size_t)(i % G)]++] = (int32_t)(first + i);
    };
    int32_t* h_cptr = h_trows + mt;
    if (streamed) {
        for (int c = 0; c < n_chunks; ++c) {
            int32_t* ptr = h_cptr + (size_t)c * (G0 + 1);
            deal(cr[c], cr[c + 1] - cr[c], G0, ptr, h_irows + cr[c]);
            for (int64_t g = 0; g <= G0; ++g) ptr[g] += (int32_t)cr[c];
        }
    } else {
        deal(0, n, G0, h_iptr, h_irows);
    }
    deal(kb_end, mt, Gt, h_tptr, h_trows);
    CUDA_TRY(cudaMemcpyAsync(base + o_int, hi, n_int * sizeof(int32_t), cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemsetAsync(base + o_rec, 0, (size_t)n * sizeof(PivRec), st));
    CUDA_TRY(cudaMemsetAsync(base + o_ctl, 0, sizeof(K1Err) + 16, st));
    // the panel kernels' record slots: cleared per call, so a record's tag only has to
    // be unique within the call (its global step + 1)
    CUDA_TRY(cudaMemsetAsync(base + o_cand, 0, o_lastb + kLastBufBytes - o_cand, st));
    const int32_t* d_int = (const int32_t*)(base + o_int);
    const int32_t* d_iota = d_int;
    const int32_t* d_never = d_iota + n;
    const int32_t* d_pptr = d_never + n;
    const int32_t* d_iptr = d_pptr + (b + 1);
    const int32_t* d_irows = d_iptr + (G0 + 1);
    const int32_t* d_tptr = d_irows + n;
    const int32_t* d_trows = d_tptr + (Gt + 1);
    const int32_t* d_cptr = d_trows + mt;
    double* ws = (double*)(base + o_ws);
    double* wit = (double*)(base + o_wit);
    PivRec* recs = (PivRec*)(base + o_rec);
    double* Lb = (double*)(base + o_L);
    double* Wb = (double*)(base + o_W);
    K2Gather* gp0 = (K2Gather*)(base + o_pan);
    K2Gather* gp1 = gp0 + 1;
    K2Gather* const gpair2 = gp0 + 2;  // ring, like L and W
    double* const Wp2 = (double*)(base + o_Wp);
    double* const Lc = (double*)(base + o_Lc);
    double* const Wx2 = (double*)(base + o_Wx);
    K1Err* err = (K1Err*)(base + o_ctl);
    unsigned* abort = (unsigned*)(base + o_ctl + sizeof(K1Err));
    const uint32_t epoch = ++B->epoch;

    K1Params p{};
    p.src[0] = d_a;
    p.src_row0[0] = 0;
    p.lds = lda;
    p.ws[0] = ws;
    p.row_wit[0] = wit;
    p.ld = ld;
    p.n = (int32_t)n;
    p.n_groups = 1;
    p.group0 = 0;
    p.n_local_groups = 1;
    p.sys_scope = 0;
    p.epoch = epoch;
    p.err = err;
    p.chunk = (int32_t)std::min<int64_t>((int64_t)align_up((size_t)n, 2), kK1MaxChunk);
    p.timeout_ns = 20ull * 1000000000ull;
    p.abort_flag = abort;

    if (streamed) {  // the row chunks, in order, on the copy stream
        CUDA_TRY(cudaEventRecord(B->ev_in, st_caller));
        CUDA_TRY(cudaStreamWaitEvent(B->cpy, B->ev_in, 0));
        for (int c = 0; c < n_chunks; ++c) {
            CUDA_TRY(cudaMemcpy2DAsync((double*)B->din + cr[c] * n, (size_t)n * sizeof(double), h_src + cr[c] * lda_h,
                                       (size_t)lda_h * sizeof(double), (size_t)n * sizeof(double), (size_t)(cr[c + 1] - cr[c]),
                                       cudaMemcpyHostToDevice, B->cpy));
            CUDA_TRY(cudaEventRecord(B->ev_arr[c], B->cpy));
        }
    }
    CUDA_TRY(cudaEventRecord(B->ev0, st));
    // 1. copy + initial witness + finiteness (no pivots); streamed: chunk 0 now, the others at their catch-up
    p.ncol0 = (int32_t)n; p.n_steps = 0; p.in_place = 0; p.wit_in = nullptr;
    p.seq = d_iota; p.row_pstep = d_never; p.pstep_offset = 0;
    p.cta_row_ptr = d_iptr; p.cta_rows = d_irows; p.ctas_per_group = (int32_t)G0; p.rec[0] = recs;
    auto init_chunk = [&](int c, cudaStream_t ss) -> cudaError_t {
        K1Params pc = p;
        pc.cta_row_ptr = d_cptr + (size_t)c * (G0 + 1);
        cudaError_t ee = cudaStreamWaitEvent(ss, B->ev_arr[c], 0);
        return ee == cudaSuccess ? k1_launch(pc, fast, ss) : ee;
    };
    cudaError_t e = streamed ? init_chunk(0, st) : k1_launch(p, fast, st);
    if (e != cudaSuccess) return fail(MCND_ECUDA, "K2 init launch: %s", cudaGetErrorString(e));
    // 2. panels: column-distributed panel factorisation, gather, DMMA trailing update
    KPParams kp{};
    kp.ws = ws;
    kp.ld = ld;
    kp.wit = wit;
    kp.epoch = epoch;
    kp.ldw = ld;
    kp.abort = abort;
    kp.cand = (ulonglong2*)(base + o_cand);
    kp.wrec = (ulonglong2*)(base + o_wrec);
    kp.colbuf = (ulonglong2*)(base + o_colb);
    kp.lastbuf = (ulonglong2*)(base + o_lastb);
    kp.err = err;
    kp.timeout_ns = 20ull * 1000000000ull;
    auto split = [&](int64_t m, int64_t G, int64_t* cw_out) {
        int64_t cw = 0;
        for (;; --G) {
            cw = (int64_t)align_up((size_t)((m + G - 1) / G), 2);
            if (G == 1 || m - (G - 1) * cw >= b) break;
        }
        *cw_out = cw;
        return G;
    };
    // panel chunk width: kp_cols_for(m) (mcnd_internal.h: the sweeps behind 176 / 240 columns)
    const int64_t kp_maxg = std::min<int64_t>(B->sms, env_long("MCND_KP_MAXG", kKPMaxG));  // test hook: wide chunks
    auto kp_ctas = [&](int64_t m) {  // ~kp_cols_for(m) columns per CTA, at most 256 unless the SM count caps G
        const int64_t cols = kp_cols_for(m);
        const int64_t cap = std::max<int64_t>(256, cols);
        return std::min<int64_t>({kp_maxg, (int64_t)kKPMaxG, std::max<int64_t>((m + cap - 1) / cap, m / cols)});
    };
    // the parameters of the panel at kb; its column chunks split the active width `m_split`
    // (the pair's first panel's: the second panel runs on the same CTAs and chunks)
    auto kp_at = [&](int64_t kb, K2Gather* gp, double* Wout, int64_t m_split) -> KPParams {
        KPParams q = kp;
        int64_t cw = 0;
        const int64_t G = split(m_split, kp_ctas(m_split), &cw);
        q.row0 = (int32_t)kb;
        q.m = (int32_t)(n - kb);
        q.G = (int32_t)G;
        q.cw = (int32_t)cw;
        q.rec = recs + kb;
        q.pan = gp;
        q.W = Wout;
        q.tag0 = kp_tag0(kb);  // slots cleared per call
        return q;
    };
    auto run_kp = [&](int64_t kb, K2Gather* gp, double* Wout) -> cudaError_t {
        return panel_launch(kp_at(kb, gp, Wout, n - kb), st, nullptr);
    };
    // Panels go in pairs: panel k, then its update of panel k+1's 64 rows, panel
    // k+1, and ONE rank-128 trailing update (half the C traffic of two rank-64
    // updates).  L of the pair = [A[R, P_k], A'[R, P_{k+1}]] where the second
    // half is corrected for panel k by a 64-wide DMMA update: L1 -= L0 * W_k[:, P_{k+1}].
    //
    // Look-ahead: the trailing update is split.  The rows the NEXT pair factors are
    // updated first on the critical (highest-priority) stream; the rest goes to the
    // lowest-priority side stream (part A: the rows of the pair after next, part B: the
    // remainder), running while the next panels are factored.  The next pair's critical
    // update waits for part A only.  L, W, Wp and the pair descriptor live in a ring of
    // pair slots so the side GEMM can read pair q's while pairs q+1, q+2 write theirs.
    bool side_pending = false, sideA_pending = false;
    cudaStream_t side = B->side;
    auto join_side = [&]() -> cudaError_t {  // all side work
        sideA_pending = false;
        if (!side_pending) return cudaSuccess;
        side_pending = false;
        return cudaStreamWaitEvent(st, B->ev_b, 0);
    };
    auto join_rows = [&]() -> cudaError_t {  // the side work the next critical update depends on
        if (sideA_pending) {
            sideA_pending = false;
            return cudaStreamWaitEvent(st, B->ev_c, 0);
        }
        return join_side();
    };
    int64_t k = 0;
    int par = 0;  // ring slot
    int64_t n_launch = 1;  // kernels launched by this call (K1 init so far)
    // a finished unit a late chunk of streamed input catches up on: one pair (par2 < 0) or a
    // group of two (slots par, par2; kb, m of its first pair; its Wx)
    struct PairSlot { int64_t kb, m; int par, par2; const double* wx; };
    std::vector<PairSlot> done_pairs;
    // a group's update of absolute rows [r0, r0 + rows): the two gathers (each with its pair's
    // column moves and L correction) into Lc, NL_b += NL_a Wx, then the rank-256 update
    auto group_update = [&](const PairSlot& G, int64_t r0, int64_t rows, cudaStream_t ss, int sm_budget) -> cudaError_t {
        if (rows <= 0) return cudaSuccess;
        double* const Lr = Lc + r0 * 4 * b;
        cudaError_t ee = k2_gather_lcorr(ws, ld, (int32_t)r0, (int32_t)rows, gpair2 + G.par, Lr, Wp2 + (size_t)G.par * b * b,
                                         abort, ss, 4 * b);
        if (ee == cudaSuccess)
            ee = k2_gather_lcorr(ws, ld, (int32_t)r0, (int32_t)rows, gpair2 + G.par2, Lr + 2 * b,
                                 Wp2 + (size_t)G.par2 * b * b, abort, ss, 4 * b);
        if (ee == cudaSuccess)
            ee = k2_gemm(Lr + 2 * b, 4 * b, 0, (int32_t)rows, (int32_t)(2 * b), 128, Lr, 4 * b, G.wx, 2 * b, nullptr, abort, ss,
                         sm_budget);
        if (ee == cudaSuccess)
            ee = k2_gemm(ws, ld, (int32_t)r0, (int32_t)rows, (int32_t)(G.m - 4 * b), 256, Lr, 4 * b,
                         Wb + (size_t)G.par * 2 * b * ld, ld, wit, abort, ss, sm_budget, Wb + (size_t)G.par2 * 2 * b * ld);
        n_launch += 4;
        return ee;
    };
    bool grp_open = false;  // the previous pair started a group
    PairSlot grp{};
    int cov_prev = 0;
    // debug timeline (MCND_DEBUG_TIMELINE=1): an event after every critical-stream step,
    // per-label device time printed to stderr at the end of the call
    const long dbg_tl = env_long("MCND_DEBUG_TIMELINE", 0);  // 2: every step
    std::vector<std::pair<const char*, cudaEvent_t>> tl;
    auto mark = [&](const char* label) {
        if (!dbg_tl) return;
        cudaEvent_t ev;
        cudaEventCreate(&ev);
        cudaEventRecord(ev, st);
        tl.emplace_back(label, ev);
    };
    mark("init");
    while (k < n_panels) {
        const int64_t kb = k * b, m = n - kb;
        double* const Wq = Wb + (size_t)par * 2 * b * ld;
        double* const Lq = Lb + (size_t)par * std::max<int64_t>(n, 1) * 2 * b;
        double* const Wp = Wp2 + (size_t)par * b * b;
        K2Gather* const gpair = gpair2 + par;
        int cov_q = n_chunks - 1;
        if (streamed && k + 1 < n_panels) {
            const size_t q = (size_t)(k / 2);
            cov_q = q < cov_of.size() ? cov_of[q] : n_chunks - 1;
        }
        // chunks first covered at this pair: K1 init, then pairs 0..q-1 in order, on the side
        // stream (after pair q-1's side work, so every slot they read is final; after this
        // pair's part A, which only touches rows covered two pairs ago)
        auto catch_up = [&]() -> cudaError_t {
            cudaError_t ee = cudaSuccess;
            for (int c = cov_prev + 1; c <= cov_q && ee == cudaSuccess; ++c) {
                ee = init_chunk(c, side);
                ++n_launch;
                for (const PairSlot& ps : done_pairs) {
                    if (ee != cudaSuccess) break;
                    if (ps.par2 >= 0) {
                        ee = group_update(ps, cr[c], cr[c + 1] - cr[c], side, -1);
                        continue;
                    }
                    const int64_t r0 = cr[c] - (ps.kb + 2 * b);  // rows relative to that pair's trailing block
                    double* const Lp = Lb + (size_t)ps.par * std::max<int64_t>(n, 1) * 2 * b + r0 * 2 * b;
                    ee = k2_gather_lcorr(ws, ld, (int32_t)cr[c], (int32_t)(cr[c + 1] - cr[c]), gpair2 + ps.par, Lp,
                                         Wp2 + (size_t)ps.par * b * b, abort, side);
                    if (ee == cudaSuccess)
                        ee = k2_gemm(ws, ld, (int32_t)cr[c], (int32_t)(cr[c + 1] - cr[c]), (int32_t)(ps.m - 2 * b), 128, Lp,
                                     2 * b, Wb + (size_t)ps.par * 2 * b * ld, ld, wit, abort, side, -1);
                    n_launch += 2;
                }
            }
            cov_prev = std::max(cov_prev, cov_q);
            return ee;
        };
        const int64_t cov_end = cr[cov_q + 1];  // rows past it are not resident yet
        if (k + 1 < n_panels) {
            // both panels of the pair in ONE launch on the same CTAs: the second applies the
            // first's update to its own rows in its prologue and runs the pair prep (spread over
            // its CTAs around one grid barrier)
            {
                const KPParams q0 = kp_at(kb, gp0, Wq, m);
                KPParams q1 = kp_at(kb + b, gp1, Wq + b * ld, m);
                unsigned* const bars = reinterpret_cast<unsigned*>(kp.lastbuf + 64 * 64);
                q1.r1_g0 = gp0; q1.r1_W = Wq; q1.r1_ldw = ld;
                q1.pp_g0 = gp0; q1.pp_W = Wq; q1.pp_ldw = ld; q1.pp_Wp = Wp; q1.pp_gpair = gpair; q1.pp_m = (int32_t)m;
                q1.pp_bar = bars + kb / (2 * b);
                q1.half_bar = bars + kPPBars + kb / (2 * b);
                e = panel_launch(q0, st, &q1);  // (checks the chunk width)
            }
            mark("kp_pair");
            if (e == cudaSuccess) e = join_rows();  // the critical rows final for the previous pair
            mark("join");
            const int32_t nr = (int32_t)(n - kb - 2 * b);
            // rows the next unit factors (a pair: 128, a last single panel: 64, or the tail: all)
            // and, when the next unit is a pair, the rows of the unit after it
            const int64_t k2 = k + 2, k4 = k + 4;
            const int64_t unit1 = (k2 + 1 < n_panels) ? 2 * b : (k2 < n_panels ? b : nr);
            const int64_t unit2 = (k2 + 1 < n_panels) ? ((k4 + 1 < n_panels) ? 2 * b : (k4 < n_panels ? b : nr - unit1)) : 0;
            // groups: this pair (a) starts one when the next unit is a pair (b) and rows are left
            // past b's next unit; those rows take a and b together at b (group_update)
            const bool g_end = grp_open;
            const bool g_start = groups && !g_end && m > group_above && k + 3 < n_panels && unit1 + unit2 < nr;
            // rows this pair updates on its own; the rest is deferred (g_start) or the group's (g_end)
            const int64_t own = g_start ? unit1 + unit2 : (g_end ? unit1 : nr);
            // (serial schedule, MCND_K2_OVERLAP=0: everything on the critical stream, same arithmetic)
            const int64_t ahead = overlap ? unit1 : own;
            // gather + L correction + trailing update of `rows` rows starting at row offset r0
            // (relative to the pair's trailing block) on stream `ss`
            auto trailing = [&](int64_t r0, int64_t rows, cudaStream_t ss, int sm_budget) -> cudaError_t {
                if (rows <= 0) return cudaSuccess;
                double* const Lr = Lq + r0 * 2 * b;
                // gather + NL[:, 64:128] += NL[:, 0:64] * (-Wp) in one pass, then the DMMA update
                cudaError_t ee = k2_gather_lcorr(ws, ld, (int32_t)(kb + 2 * b + r0), (int32_t)rows, gpair, Lr, Wp, abort, ss);
                if (ss == st) mark("gather_lcorr");
                if (ee == cudaSuccess)
                    ee = k2_gemm(ws, ld, (int32_t)(kb + 2 * b + r0), (int32_t)rows, (int32_t)(m - 2 * b), 128, Lr, 2 * b,
                                 Wq, ld, wit, abort, ss, sm_budget);
                if (ss == st) mark("trailing");
                n_launch += 2;
                return ee;
            };
            PairSlot gq{};
            if (g_end) {
                gq = grp;
                gq.par2 = par;
            }
            // the group's preparation (Wx from W_a, then b's column moves into W_a): after every
            // per-pair use of W_a (the critical rows of a and its part A precede it in stream order)
            auto group_prep = [&](cudaStream_t ss) -> cudaError_t {
                n_launch += 2;
                return k2_group_prep(Wb + (size_t)gq.par * 2 * b * ld, ld, gpair, Wp, const_cast<double*>(gq.wx), abort, ss);
            };
            const int64_t r_end = std::min<int64_t>(nr, cov_end - (kb + 2 * b));  // resident rows
            if (streamed && cov_q > cov_prev && ahead >= nr) {
                // no side work: new rows caught up first
                if (e == cudaSuccess) e = cudaEventRecord(B->ev_a, st);
                if (e == cudaSuccess) e = cudaStreamWaitEvent(side, B->ev_a, 0);
                if (e == cudaSuccess) e = catch_up();
                if (e == cudaSuccess) e = cudaEventRecord(B->ev_b, side);
                side_pending = (e == cudaSuccess);
                if (e == cudaSuccess) e = join_side();
            }
            // the critical rows first (serial: every row this pair updates on its own)
            if (e == cudaSuccess) e = trailing(0, ahead, st, 0);
            if (!overlap) {
                if (g_end && e == cudaSuccess) e = group_prep(st);
                if (g_end && e == cudaSuccess) e = group_update(gq, kb + 2 * b + own, nr - own, st, 0);
            } else if (ahead < nr) {
                // side stream: W, Wp and the gather descriptor are final once the pair prep is done;
                // started only after the critical rows' update, so the side kernels do not take the
                // SMs the critical ones need
                if (e == cudaSuccess) e = cudaEventRecord(B->ev_a, st);
                if (e == cudaSuccess) e = cudaStreamWaitEvent(side, B->ev_a, 0);
                if (g_end && e == cudaSuccess) e = group_prep(side);
                // part A: the rows of the unit after next, when the next unit is a pair; the next
                // pair waits for it alone.  Part B: the rest (deferred when this pair starts a group)
                const int64_t a_rows = unit2 < nr - unit1 ? unit2 : 0;
                if (a_rows > 0) {
                    // (defensive: part A's rows not resident yet -> catch up first)
                    if (e == cudaSuccess && streamed && kb + 2 * b + unit1 + a_rows > cr[cov_prev + 1]) e = catch_up();
                    if (e == cudaSuccess)
                        e = g_end ? group_update(gq, kb + 2 * b + unit1, a_rows, side, -1) : trailing(unit1, a_rows, side, -1);
                    if (e == cudaSuccess) e = cudaEventRecord(B->ev_c, side);
                    sideA_pending = (e == cudaSuccess);
                }
                if (e == cudaSuccess && streamed) e = catch_up();
                if (!g_start) {
                    const int64_t r_b = unit1 + a_rows;
                    if (e == cudaSuccess)
                        e = g_end ? group_update(gq, kb + 2 * b + r_b, r_end - r_b, side, -1) : trailing(r_b, r_end - r_b, side, -1);
                }
                if (e == cudaSuccess) e = cudaEventRecord(B->ev_b, side);
                side_pending = (e == cudaSuccess);
            }
            ++n_launch;  // the panel pair
            if (g_start) {
                grp = PairSlot{kb, m, par, -1, Wx2 + (size_t)(k / 4) * 4 * b * b};
                grp_open = true;
            } else {
                grp_open = false;
                if (streamed) done_pairs.push_back(g_end ? gq : PairSlot{kb, m, par, -1, nullptr});
            }
            k += 2;
            par = (par + 1) % kRing;
        } else {
            e = run_kp(kb, gp0, Wq);
            if (e == cudaSuccess) e = join_side();
            if (e == cudaSuccess)
                e = k2_gather_fix(ws, ld, (int32_t)(kb + b), (int32_t)(n - kb - b), 64, gp0, Lq, abort, st);
            if (e == cudaSuccess)
                e = k2_gemm(ws, ld, (int32_t)(kb + b), (int32_t)(n - kb - b), (int32_t)(m - b), 64, Lq, 64, Wq, ld, wit,
                            abort, st);
            n_launch += 3;
            k += 1;
            par = (par + 1) % kRing;
        }
        if (e != cudaSuccess) {
            join_side();
            return fail(MCND_ECUDA, "K2 panel kernels: %s", cudaGetErrorString(e));
        }
    }
    e = join_side();
    if (e != cudaSuccess) return fail(MCND_ECUDA, "K2 stream join: %s", cudaGetErrorString(e));
    mark("final_join");
    // 3. unblocked tail (publishes the final 1x1)
    p.in_place = 1; p.wit_in = wit; p.row_pstep = d_iota;
    p.ncol0 = (int32_t)mt; p.n_steps = (int32_t)(mt - 1); p.seq = d_iota + kb_end; p.pstep_offset = (int32_t)kb_end;
    p.cta_row_ptr = d_tptr; p.cta_rows = d_trows; p.ctas_per_group = (int32_t)Gt; p.rec[0] = recs + kb_end;
    // (after panels, a tail of at most 128 rows goes to one pair of warps -- the same arithmetic,
    //  bitwise, without K1's per-step publication between 148 CTAs: 20 us instead of 240 us at
    //  64 rows; MCND_K2_SMALL_TAIL=0: K1)
    if (n_panels > 0 && mt >= 2 && mt <= 128 && env_long("MCND_K2_SMALL_TAIL", 1) != 0)
        e = k3_tail_launch(ws, ld, (int32_t)kb_end, (int32_t)mt, fast, wit, recs + kb_end, epoch, abort, st);
    else
        e = k1_launch(p, fast, st);
    if (e != cudaSuccess) return fail(MCND_ECUDA, "K2 tail launch: %s", cudaGetErrorString(e));
    CUDA_TRY(cudaEventRecord(B->ev1, st));
    out->launches = n_launch + 1;
    if (dbg_tl) {
        mark("tail");
        cudaStreamSynchronize(st);
        std::map<std::string, std::pair<double, int>> acc;
        for (size_t i = 1; i < tl.size(); ++i) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, tl[i - 1].second, tl[i].second);
            auto& a = acc[tl[i].first];
            a.first += ms;
            a.second += 1;
            if (dbg_tl > 1) std::fprintf(stderr, "mcnd step %4zu %-12s %8.1f us\n", i, tl[i].first, 1e3 * ms);
        }
        for (auto& kv : acc)
            std::fprintf(stderr, "mcnd timeline %-10s %8.3f ms  (%d x %.1f us)\n", kv.first.c_str(), kv.second.first,
                         kv.second.second, 1e3 * kv.second.first / kv.second.second);
        for (auto& t : tl) cudaEventDestroy(t.second);
    }

    PivRec* h_rec = (PivRec*)B->hpin;
    K1Err* h_err = (K1Err*)((char*)B->hpin + align_up((size_t)n * sizeof(PivRec), 64));
    CUDA_TRY(cudaMemcpyAsync(h_rec, recs, (size_t)n * sizeof(PivRec), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(h_err, err, sizeof(K1Err), cudaMemcpyDeviceToHost, st));
    e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return fail(MCND_ECUDA, "blocked condensation: %s", cudaGetErrorString(e));
    if (st != st_caller) {  // the caller's later work is ordered after ours
        CUDA_TRY(cudaEventRecord(B->ev_out, st));
        CUDA_TRY(cudaStreamWaitEvent(st_caller, B->ev_out, 0));
    }
    drain.armed = false;  // every stream is idle: st synchronised, side and cpy joined into it
    float ms = 0.f;
    cudaEventElapsedTime(&ms, B->ev0, B->ev1);
    out->device_ms = ms;
    out->torn_reads = h_err->torn;
    if (h_err->nonfinite) return fail(MCND_EINVAL, "matrix entries must be finite (no NaN/Inf)");
    if (h_err->error)
        return fail(MCND_EDEVICE, "device timeout waiting for pivot %u [%u g=%u s=%u i=%u tags %x %x want %x G/r=%u]",
                    h_err->err_step, h_err->dbg[0], h_err->dbg[1], h_err->dbg[2], h_err->dbg[3], h_err->dbg[4],
                    h_err->dbg[5], h_err->dbg[6], h_err->dbg[7]);
    int64_t sing = -1;
    for (int64_t t = 0; t < n; ++t) {
        if (h_rec[t].flag != epoch || h_rec[t].l < 0) { sing = t; break; }
        if (pivots_out) pivots_out[t] = h_rec[t].v;
        if (cols_out) cols_out[t] = h_rec[t].l;
    }
    if (sing >= 0) {
        out->sign = 0; out->singular = 1; out->log_abs = -INFINITY; out->singular_step = sing; out->steps = sing;
        return MCND_OK;
    }
    double log_acc = 0.0;
    int sign_acc = 1;
    for (int64_t t = 0; t < n - 1; ++t) {
        const int64_t m = n - t;
        const double v = h_rec[t].v;
        log_acc += std::log(std::fabs(v));
        const int swap_parity = (h_rec[t].l != m - 1) ? -1 : 1;
        const int parity = ((m - 1) % 2) ? -1 : 1;  // k_pos = 0 (top-to-bottom)
        sign_acc *= (v > 0 ? 1 : -1) * swap_parity * parity;
    }
    const double vf = h_rec[n - 1].v;
    out->sign = sign_acc * (vf > 0 ? 1 : -1);
    out->log_abs = log_acc + std::log(std::fabs(vf));
    out->steps = n - 1;
    return MCND_OK;
}

// ---- multi-GPU (one process per GPU) ----
struct DistHandle {
    int32_t rank = 0, world = 1;
    int64_t n_max = 0;
    GroupLayout GL;             // layout for n_max (identical on every rank)
    Buffers B;                  // this rank's own buffers (workspace = IPC-exported allocation)
    void* meta = nullptr;
    size_t meta_bytes = 0;
    void* peer_base[kMaxGroups] = {};
    bool connected = false;
    uint32_t epoch = 0;
};

// ---- multi-GPU blocked condensation: the per-rank engine (SURVEY.md §8(e) "K2:
// one broadcast per panel of W").  One rank holds a contiguous block of rows x all
// n columns.  The host schedule (dist.py) gives each panel pair to the rank with
// the most live rows (its topmost 128 live rows; north_star (3)); that rank
// factors the pair (mg_pair), the pair's W, Wp and gather descriptor are broadcast
// (NCCL, by the host), and every rank applies the rank-128 update to its own live
// rows (mg_trailing).  The last rows are gathered to one rank and finished by K1
// (mg_tail).  Kernels are exactly the single-GPU K2 kernels.
struct MgHandle {
    int device = 0, sms = 0;
    int64_t n = 0, lr = 0, ld = 0;
    void* mem = nullptr;
    size_t bytes = 0;
    double* ws = nullptr;
    double* wit = nullptr;
    PivRec* recs = nullptr;
    double* L = nullptr;       // [2][lr][128]
    K2Gather* gp = nullptr;    // [2]
    ulonglong2 *cand = nullptr, *wrec = nullptr, *colb = nullptr, *lastb = nullptr;
    K1Err* err = nullptr;
    unsigned* abort = nullptr;
    int32_t* d_int = nullptr;  // iota[max(n,lr)] | never[lr] | init deal ptr[G0+1] rows[lr]
    int64_t g0 = 1;
    void* tail_mem = nullptr;  // tail metadata (iota, deal) + records
    size_t tail_bytes = 0;
    void* hpin = nullptr;
    size_t hpin_bytes = 0;
    uint32_t epoch = 0;
    // native driver (mcnd_mg_logdet): the group, its NCCL communicator and the pair buffers
    int32_t world = 1, rank = 0;
    ncclComm_t comm = nullptr;
    bool use_comm = false;                      // broadcasts even with one rank (test hook)
    // host transport (tests: ranks sharing one GPU over gloo): the collectives go through
    // these callbacks on pinned staging buffers instead of NCCL
    int (*host_bcast)(void* buf, int64_t bytes, int32_t root) = nullptr;
    int (*host_allgather)(const void* send, void* recv, int64_t bytes) = nullptr;
    void* hs_send = nullptr; size_t hs_send_bytes = 0;
    void* hs_recv = nullptr; size_t hs_recv_bytes = 0;
    cudaStream_t crit = nullptr, side = nullptr, cst = nullptr;
    cudaEvent_t ev_pair[2] = {}, ev_bc[2] = {}, ev_trc[2] = {}, ev_trs[2] = {}, ev_side = nullptr, ev_crit = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    void* pmem = nullptr;                       // W[2] | Wp[2] | descriptor[2] | tail buffers | record gather
    size_t pbytes = 0;
    std::vector<unsigned char> hbuf;            // host copies of the gathered records
};

int mg_create(int64_t n, int64_t lr, MgHandle** out) {
    if (n < 1 || lr < 0 || lr > n) return fail(MCND_EINVAL, "mg_create: bad sizes n=%lld rows=%lld", (long long)n, (long long)lr);
    auto* h = new MgHandle();
    cudaGetDevice(&h->device);
    cudaDeviceGetAttribute(&h->sms, cudaDevAttrMultiProcessorCount, h->device);
    h->n = n;
    h->lr = lr;
    h->ld = (int64_t)align_up((size_t)n, 16);
    const int64_t b = kK2B, lrr = std::max<int64_t>(lr, 1);
    h->g0 = std::max<int64_t>(1, std::min<int64_t>(h->sms, lrr));
    if ((lrr + h->g0 - 1) / h->g0 > kK1MaxRowsPerCta) { delete h; return fail(MCND_EINVAL, "mg_create: %lld rows too many", (long long)lr); }
    if (n > (int64_t)kKPMaxCw * std::min<int64_t>(h->sms, kKPMaxG)) {  // the owner's panel spans all n columns
        delete h;
        return fail(MCND_EINVAL, "mg_create: n=%lld too large for the panel kernel (at most %d columns per SM)",
                    (long long)n, kKPMaxCw);
    }
    size_t off = 0;
    auto take = [&](size_t by) { size_t o = off; off = align_up(off + by, 256); return o; };
    const size_t o_ws = take((size_t)lrr * h->ld * sizeof(double));
    const size_t o_wit = take((size_t)lrr * sizeof(double));
    const size_t o_rec = take((size_t)n * sizeof(PivRec));
    const size_t o_L = take((size_t)2 * lrr * 2 * b * sizeof(double));
    const size_t o_gp = take(2 * sizeof(K2Gather));
    const size_t o_cand = take((size_t)64 * kKPMaxG * sizeof(ulonglong2));
    const size_t o_wrec = take((size_t)64 * kKPMaxG * sizeof(ulonglong2));
    const size_t o_colb = take((size_t)64 * kKPMaxG * 64 * sizeof(ulonglong2));
    const size_t o_lastb = take(kLastBufBytes);
    const size_t o_ctl = take(sizeof(K1Err) + 16);
    const int64_t ni = std::max<int64_t>(n, lrr);
    const size_t n_int = (size_t)(ni + lrr + (h->g0 + 1) + lrr);
    const size_t o_int = take(n_int * sizeof(int32_t));
    if (cudaMalloc(&h->mem, off) != cudaSuccess) {
        cudaGetLastError();
        delete h;
        return fail(MCND_ECUDA, "mg_create: cudaMalloc(%zu) failed", off);
    }
    h->bytes = off;
    char* base = (char*)h->mem;
    h->ws = (double*)(base + o_ws);
    h->wit = (double*)(base + o_wit);
    h->recs = (PivRec*)(base + o_rec);
    h->L = (double*)(base + o_L);
    h->gp = (K2Gather*)(base + o_gp);
    h->cand = (ulonglong2*)(base + o_cand);
    h->wrec = (ulonglong2*)(base + o_wrec);
    h->colb = (ulonglong2*)(base + o_colb);
    h->lastb = (ulonglong2*)(base + o_lastb);
    h->err = (K1Err*)(base + o_ctl);
    h->abort = (unsigned*)(base + o_ctl + sizeof(K1Err));
    h->d_int = (int32_t*)(base + o_int);
    std::vector<int32_t> hi(n_int);
    int32_t* iota = hi.data();
    int32_t* never = iota + ni;
    int32_t* iptr = never + lrr;
    int32_t* irows = iptr + (h->g0 + 1);
    for (int64_t i = 0; i < ni; ++i) iota[i] = (int32_t)i;
    for (int64_t i = 0; i < lrr; ++i) never[i] = kNever;
    iptr[0] = 0;
    for (int64_t c = 0; c < h->g0; ++c) iptr[c + 1] = iptr[c] + (int32_t)((lr - c + h->g0 - 1) / h->g0);
    std::vector<int32_t> fill(iptr, iptr + h->g0);
    for (int64_t i = 0; i < lr; ++i) irows[fill[(size_t)(i % h->g0)]++] = (int32_t)i;
    if (cudaMemcpy(h->d_int, hi.data(), n_int * sizeof(int32_t), cudaMemcpyHostToDevice) != cudaSuccess) {
        cudaFree(h->mem);
        delete h;
        return fail(MCND_ECUDA, "mg_create: metadata upload failed");
    }
    *out = h;
    return MCND_OK;
}

// copy + initial witness + finiteness of the local rows (K1 with no steps)
int mg_load(MgHandle* h, const double* src, int64_t lds, cudaStream_t st) {
    if (!src && h->lr > 0) return fail(MCND_EINVAL, "mg_load: null rows");
    if (lds < h->n) return fail(MCND_EINVAL, "mg_load: row stride %lld < n", (long long)lds);
    h->epoch = h->epoch + 1 + (h->epoch + 1 == 0 ? 1 : 0);
    CUDA_TRY(cudaMemsetAsync(h->recs, 0, (size_t)h->n * sizeof(PivRec), st));
    CUDA_TRY(cudaMemsetAsync(h->err, 0, sizeof(K1Err) + 16, st));
    CUDA_TRY(cudaMemsetAsync(h->cand, 0, (size_t)((char*)h->lastb + kLastBufBytes - (char*)h->cand), st));
    if (h->lr == 0) return MCND_OK;
    const int64_t ni = std::max<int64_t>(h->n, h->lr);
    K1Params p{};
    p.src[0] = src;
    p.src_row0[0] = 0;
    p.lds = lds;
    p.ws[0] = h->ws;
    p.row_wit[0] = h->wit;
    p.ld = h->ld;
    p.n = (int32_t)h->lr;
    p.n_groups = 1;
    p.n_local_groups = 1;
    p.epoch = h->epoch;
    p.err = h->err;
    p.chunk = (int32_t)std::min<int64_t>((int64_t)align_up((size_t)h->n, 2), kK1MaxChunk);
    p.timeout_ns = 20ull * 1000000000ull;
    p.abort_flag = h->abort;
    p.ncol0 = (int32_t)h->n;
    p.n_steps = 0;
    p.seq = h->d_int;
    p.row_pstep = h->d_int + ni;
    p.cta_row_ptr = h->d_int + ni + h->lr;
    p.cta_rows = p.cta_row_ptr + (h->g0 + 1);
    p.ctas_per_group = (int32_t)h->g0;
    p.rec[0] = h->recs;
    cudaError_t e = k1_launch(p, false, st);
    if (e != cudaSuccess) return fail(MCND_ECUDA, "mg_load: %s", cudaGetErrorString(e));
    return MCND_OK;
}

// m_split: the active width the column chunks split (the pair's first panel's for both)
KPParams mg_kp(MgHandle* h, int64_t lr0, int64_t t, int64_t m, K2Gather* gp, double* W, int64_t ldw,
               int64_t m_split = -1) {
    const int64_t b = kK2B;
    const int64_t m_act = m;
    if (m_split > 0) m = m_split;
    const int64_t cols = kp_cols_for(m), cap = std::max<int64_t>(256, cols);
    int64_t G = std::min<int64_t>({(int64_t)h->sms, env_long("MCND_KP_MAXG", kKPMaxG), (int64_t)kKPMaxG,
                                   std::max<int64_t>((m + cap - 1) / cap, m / cols)});
    int64_t cw = 0;
    for (;; --G) {
        cw = (int64_t)align_up((size_t)((m + G - 1) / G), 2);
        if (G == 1 || m - (G - 1) * cw >= b) break;
    }
    KPParams kp{};
    kp.ws = h->ws;
    kp.ld = h->ld;
    kp.row0 = (int32_t)lr0;
    kp.m = (int32_t)m_act;
    kp.G = (int32_t)G;
    kp.cw = (int32_t)cw;
    kp.wit = h->wit;
    kp.rec = h->recs + t;
    kp.epoch = h->epoch;
    kp.tag0 = kp_tag0(t);  // slots cleared by mg_load
    kp.W = W;
    kp.ldw = ldw;
    kp.pan = gp;
    kp.abort = h->abort;
    kp.cand = h->cand;
    kp.wrec = h->wrec;
    kp.colbuf = h->colb;
    kp.lastbuf = h->lastb;
    kp.err = h->err;
    kp.timeout_ns = 20ull * 1000000000ull;
    return kp;
}

// owner of a panel pair: local rows lr0..lr0+127 are the pair, m the active width,
// t the global index of its first pivot.  Outputs W (128 x (m-128) in the final
// layout; row stride ldw >= m-64, even: W_k is m-64 wide before the pair prep), Wp
// (64 x 64) and the pair's gather descriptor; pivot records to recs[t .. t+127].
int mg_pair(MgHandle* h, int64_t lr0, int64_t t, int64_t m, double* W, int64_t ldw, double* Wp, K2Gather* gpair,
            cudaStream_t st) {
    const int64_t b = kK2B;
    if (lr0 < 0 || lr0 + 2 * b > h->lr || m < 2 * b + 1 || m > h->n || t < 0 || t + 2 * b > h->n || ldw < m - b ||
        (ldw & 1) || !W ||
        !Wp || !gpair)
        return fail(MCND_EINVAL, "mg_pair: bad arguments (lr0=%lld m=%lld t=%lld)", (long long)lr0, (long long)m,
                    (long long)t);
    K2Gather* gp0 = h->gp;
    K2Gather* gp1 = h->gp + 1;
    const KPParams kp = mg_kp(h, lr0, t, m, gp0, W, ldw);
    cudaError_t e = cudaSuccess;
    const int64_t pair = t / (2 * b);
    unsigned* const bars = reinterpret_cast<unsigned*>(h->lastb + 64 * 64);
    if (pair < kPPBars) {
        // both panels in one launch on the same CTAs and column chunks (as blocked_dev)
        KPParams kp1 = mg_kp(h, lr0 + b, t + b, m - b, gp1, W + b * ldw, ldw, m);
        kp1.r1_g0 = gp0; kp1.r1_W = W; kp1.r1_ldw = ldw;  // + the first panel's update of these rows
        kp1.pp_g0 = gp0; kp1.pp_W = W; kp1.pp_ldw = ldw; kp1.pp_Wp = Wp; kp1.pp_gpair = gpair; kp1.pp_m = (int32_t)m;
        kp1.pp_bar = bars + pair;
        kp1.half_bar = bars + kPPBars + pair;
        e = panel_launch(kp, st, &kp1);
    } else {
        e = kp_launch(kp, st);
        if (e == cudaSuccess) {
            KPParams kp1 = mg_kp(h, lr0 + b, t + b, m - b, gp1, W + b * ldw, ldw);
            kp1.r1_g0 = gp0; kp1.r1_W = W; kp1.r1_ldw = ldw;
            kp1.pp_g0 = gp0; kp1.pp_W = W; kp1.pp_ldw = ldw; kp1.pp_Wp = Wp; kp1.pp_gpair = gpair; kp1.pp_m = (int32_t)m;
            e = kp_launch(kp1, st);  // + the pair prep in its CTA 0 (no barrier counter left)
        }
    }
    if (e != cudaSuccess) return fail(MCND_ECUDA, "mg_pair: %s", cudaGetErrorString(e));
    return MCND_OK;
}

// every rank: gather + L correction + rank-128 update of local rows [lr0, lr0+rows)
// by a pair of active width m (W, Wp, gpair as produced by mg_pair, possibly on
// another rank); par selects the L buffer (alternate it per pair).
int mg_trailing(MgHandle* h, int64_t lr0, int64_t rows, int64_t m, const double* W, int64_t ldw, const double* Wp,
                const K2Gather* gpair, int32_t sm_budget, int32_t par, cudaStream_t st) {
    const int64_t b = kK2B;
    if (rows == 0) return MCND_OK;
    if (lr0 < 0 || rows < 0 || lr0 + rows > h->lr || m < 2 * b + 1 || m > h->n || !W || !Wp || !gpair || ldw < m - b ||
        (ldw & 1))
        return fail(MCND_EINVAL, "mg_trailing: bad arguments");
    // L rows are indexed by local row: concurrent calls on disjoint rows never collide
    double* L = h->L + (size_t)(par & 1) * std::max<int64_t>(h->lr, 1) * 2 * b + (size_t)lr0 * 2 * b;
    cudaError_t e = k2_gather_lcorr(h->ws, h->ld, (int32_t)lr0, (int32_t)rows, gpair, L, Wp, h->abort, st);
    if (e == cudaSuccess)
        e = k2_gemm(h->ws, h->ld, (int32_t)lr0, (int32_t)rows, (int32_t)(m - 2 * b), 128, L, 2 * b, W, ldw, h->wit,
                    h->abort, st, sm_budget);
    if (e != cudaSuccess) return fail(MCND_ECUDA, "mg_trailing: %s", cudaGetErrorString(e));
    return MCND_OK;
}

// local rows [lr0, lr0+rows): their first mt columns (row stride ldo) and witnesses
int mg_export(MgHandle* h, int64_t lr0, int64_t rows, int64_t mt, double* out, int64_t ldo, double* wit_out,
              cudaStream_t st) {
    if (rows == 0) return MCND_OK;
    if (lr0 < 0 || lr0 + rows > h->lr || mt < 1 || mt > h->n || ldo < mt || !out || !wit_out)
        return fail(MCND_EINVAL, "mg_export: bad arguments");
    CUDA_TRY(cudaMemcpy2DAsync(out, (size_t)ldo * sizeof(double), h->ws + lr0 * h->ld, (size_t)h->ld * sizeof(double),
                               (size_t)mt * sizeof(double), (size_t)rows, cudaMemcpyDeviceToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(wit_out, h->wit + lr0, (size_t)rows * sizeof(double), cudaMemcpyDeviceToDevice, st));
    return MCND_OK;
}

// the gathered last mt rows (row stride ldr, in place) with their carried witnesses:
// K1 condenses them top to bottom; records (mt x 16 B) and the error word to the host
int mg_tail(MgHandle* h, double* rows, int64_t ldr, const double* wit, int64_t mt, cudaStream_t st, void* h_recs,
            uint32_t* h_err) {
    if (mt < 1 || ldr < mt || (ldr & 1) || !rows || !wit || !h_recs) return fail(MCND_EINVAL, "mg_tail: bad arguments");
    const int64_t Gt = std::max<int64_t>(1, std::min<int64_t>(h->sms, mt));
    if ((mt + Gt - 1) / Gt > kK1MaxRowsPerCta) return fail(MCND_EINVAL, "mg_tail: %lld rows too many", (long long)mt);
    size_t off = 0;
    auto take = [&](size_t by) { size_t o = off; off = align_up(off + by, 256); return o; };
    const size_t o_int = take((size_t)(mt + Gt + 1 + mt) * sizeof(int32_t));
    const size_t o_rec = take((size_t)mt * sizeof(PivRec));
    const size_t o_wit = take((size_t)mt * sizeof(double));
    const size_t o_err = take(sizeof(K1Err));
    int rc = ensure_dev(&h->tail_mem, &h->tail_bytes, off);
    if (rc) return rc;
    rc = ensure_pinned(&h->hpin, &h->hpin_bytes, (size_t)(mt + Gt + 1 + mt) * sizeof(int32_t) + 64);
    if (rc) return rc;
    char* base = (char*)h->tail_mem;
    int32_t* hi = (int32_t*)h->hpin;
    int32_t* iota = hi;
    int32_t* tptr = iota + mt;
    int32_t* trows = tptr + Gt + 1;
    for (int64_t i = 0; i < mt; ++i) iota[i] = (int32_t)i;
    tptr[0] = 0;
    for (int64_t c = 0; c < Gt; ++c) tptr[c + 1] = tptr[c] + (int32_t)((mt - c + Gt - 1) / Gt);
    std::vector<int32_t> fill(tptr, tptr + Gt);
    for (int64_t i = 0; i < mt; ++i) trows[fill[(size_t)(i % Gt)]++] = (int32_t)i;
    CUDA_TRY(cudaMemcpyAsync(base + o_int, hi, (size_t)(mt + Gt + 1 + mt) * sizeof(int32_t), cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemsetAsync(base + o_rec, 0, (size_t)mt * sizeof(PivRec), st));
    CUDA_TRY(cudaMemsetAsync(base + o_err, 0, sizeof(K1Err), st));
    const int32_t* d_iota = (const int32_t*)(base + o_int);
    K1Params p{};
    p.ws[0] = rows;
    p.row_wit[0] = (double*)(base + o_wit);
    p.ld = ldr;
    p.n = (int32_t)mt;
    p.n_groups = 1;
    p.n_local_groups = 1;
    p.epoch = h->epoch;
    p.err = (K1Err*)(base + o_err);
    p.chunk = (int32_t)std::min<int64_t>((int64_t)align_up((size_t)mt, 2), kK1MaxChunk);
    p.timeout_ns = 20ull * 1000000000ull;
    p.abort_flag = nullptr;
    p.in_place = 1;
    p.wit_in = wit;
    p.ncol0 = (int32_t)mt;
    p.n_steps = (int32_t)(mt - 1);
    p.seq = d_iota;
    p.row_pstep = d_iota;
    p.pstep_offset = 0;
    p.cta_row_ptr = d_iota + mt;
    p.cta_rows = p.cta_row_ptr + Gt + 1;
    p.ctas_per_group = (int32_t)Gt;
    p.rec[0] = (PivRec*)(base + o_rec);
    cudaError_t e = k1_launch(p, false, st);
    if (e != cudaSuccess) return fail(MCND_ECUDA, "mg_tail: %s", cudaGetErrorString(e));
    CUDA_TRY(cudaMemcpyAsync(h_recs, base + o_rec, (size_t)mt * sizeof(PivRec), cudaMemcpyDeviceToHost, st));
    K1Err he{};
    CUDA_TRY(cudaMemcpyAsync(&he, base + o_err, sizeof(K1Err), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    if (h_err) { h_err[0] = he.error; h_err[1] = he.err_step; h_err[2] = he.nonfinite; }
    return MCND_OK;
}

// this rank's pivot records (n x 16 B, global step index) and error word (error,
// step, nonfinite); synchronises the stream
int mg_records(MgHandle* h, void* h_recs, uint32_t* h_err, cudaStream_t st) {
    if (!h_recs) return fail(MCND_EINVAL, "mg_records: null output");
    CUDA_TRY(cudaMemcpyAsync(h_recs, h->recs, (size_t)h->n * sizeof(PivRec), cudaMemcpyDeviceToHost, st));
    K1Err he{};
    CUDA_TRY(cudaMemcpyAsync(&he, h->err, sizeof(K1Err), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    if (h_err) { h_err[0] = he.error; h_err[1] = he.err_step; h_err[2] = he.nonfinite; h_err[3] = h->epoch; }
    return MCND_OK;
}


// ---- native multi-GPU blocked driver (mcnd_mg_logdet) -------------------------------------
// The whole per-pair schedule of one rank in C++ (it was a Python loop: 37.8 ms per C3 call at
// world 1 against 31.0 ms for the single-GPU path): panel pairs from the rank with the most live
// rows (north_star (3)), W / Wp / the gather descriptor broadcast with NCCL on a communication
// stream that waits only for the pair and for the buffer's previous users, the owner's look-ahead
// (next critical rows first on a high-priority stream, the rest on a low-priority one), the tail
// gathered with one all-gather and finished by K1, the pivot records all-gathered and folded.
// NCCL is resolved at run time (dlopen of libnccl.so.2, the copy torch loaded if any), so the
// library has no link-time dependency on it and one-rank runs need none.
struct NcclApi {
    bool ok = false;
    ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*groupStart)() = nullptr;
    ncclResult_t (*groupEnd)() = nullptr;
    const char* (*errStr)(ncclResult_t) = nullptr;
};
const NcclApi& mg_nccl() {
    static const NcclApi api = [] {
        NcclApi a;
        void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!lib) return a;
        a.getUniqueId = (decltype(a.getUniqueId))dlsym(lib, "ncclGetUniqueId");
        a.commInitRank = (decltype(a.commInitRank))dlsym(lib, "ncclCommInitRank");
        a.commDestroy = (decltype(a.commDestroy))dlsym(lib, "ncclCommDestroy");
        a.broadcast = (decltype(a.broadcast))dlsym(lib, "ncclBroadcast");
        a.allGather = (decltype(a.allGather))dlsym(lib, "ncclAllGather");
        a.groupStart = (decltype(a.groupStart))dlsym(lib, "ncclGroupStart");
        a.groupEnd = (decltype(a.groupEnd))dlsym(lib, "ncclGroupEnd");
        a.errStr = (decltype(a.errStr))dlsym(lib, "ncclGetErrorString");
        a.ok = a.getUniqueId && a.commInitRank && a.commDestroy && a.broadcast && a.allGather && a.groupStart &&
               a.groupEnd && a.errStr;
        return a;
    }();
    return api;
}
#define NCCL_TRY(expr)                                                                           \
    do {                                                                                         \
        ncclResult_t _r = (expr);                                                                \
        if (_r != ncclSuccess) return fail(MCND_ENCCL, "%s: %s", #expr, mg_nccl().errStr(_r));   \
    } while (0)

// dist.blocked_schedule: contiguous blocks (plan_blocks, runtime.py:33-44); each pair (128
// rows) from the rank with the most live rows (ties -> lowest rank) as its topmost 128 live
// rows; kpos = live rows of the ranks before it (runtime.py:158-160)
struct MgPair { int32_t o; int64_t lr0, t, m, kpos; };
struct MgSchedule {
    std::vector<int64_t> start, len, top, live;
    std::vector<MgPair> pairs;
    int64_t t_tail = 0;
};
MgSchedule mg_schedule(int64_t n, int32_t world, int64_t tail) {
    MgSchedule S;
    const int64_t base = n / world, extra = n % world;
    for (int32_t w = 0, s0 = 0; w < world; ++w) {
        S.start.push_back(s0);
        S.len.push_back(base + (w < extra ? 1 : 0));
        s0 += (int32_t)S.len.back();
    }
    S.live = S.len;
    S.top.assign(world, 0);
    const int64_t b2 = 2 * kK2B;
    for (int64_t t = 0;; t += b2) {
        const int64_t m = n - t;
        int32_t o = 0;
        for (int32_t r = 1; r < world; ++r) if (S.live[r] > S.live[o]) o = r;
        if (S.live[o] < b2 || m - b2 < std::max<int64_t>(tail, 2)) { S.t_tail = t; break; }
        int64_t kpos = 0;
        for (int32_t r = 0; r < o; ++r) kpos += S.live[r];
        S.pairs.push_back({o, S.top[o], t, m, kpos});
        S.live[o] -= b2;
        S.top[o] += b2;
    }
    return S;
}

int mg_attach(MgHandle* h, int32_t world, int32_t rank, const void* id, int32_t force_comm) {
    if (world < 1 || rank < 0 || rank >= world) return fail(MCND_EINVAL, "mg_attach: bad rank %d of %d", rank, world);
    if (h->comm) { mg_nccl().commDestroy(h->comm); h->comm = nullptr; }
    h->world = world;
    h->rank = rank;
    h->use_comm = world > 1 || force_comm != 0;
    if (h->use_comm) {
        if (!mg_nccl().ok) return fail(MCND_ENCCL, "libnccl.so.2 not found (needed for %d ranks)", world);
        if (!id) return fail(MCND_EINVAL, "mg_attach: null NCCL id");
        ncclUniqueId uid;
        std::memcpy(&uid, id, sizeof(uid));
        NCCL_TRY(mg_nccl().commInitRank(&h->comm, world, uid, rank));
    }
    if (!h->crit) {
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        CUDA_TRY(cudaStreamCreateWithPriority(&h->crit, cudaStreamNonBlocking, hi));
        CUDA_TRY(cudaStreamCreateWithPriority(&h->side, cudaStreamNonBlocking, lo));
        CUDA_TRY(cudaStreamCreateWithFlags(&h->cst, cudaStreamNonBlocking));
        for (int i = 0; i < 2; ++i)
            for (cudaEvent_t* ev : {&h->ev_pair[i], &h->ev_bc[i], &h->ev_trc[i], &h->ev_trs[i]})
                CUDA_TRY(cudaEventCreateWithFlags(ev, cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&h->ev_side, cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&h->ev_crit, cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreate(&h->ev0));
        CUDA_TRY(cudaEventCreate(&h->ev1));
    }
    return MCND_OK;
}

void mg_release_native(MgHandle* h) {
    if (h->comm && mg_nccl().ok) mg_nccl().commDestroy(h->comm);
    h->comm = nullptr;
    if (h->pmem) cudaFree(h->pmem);
    h->pmem = nullptr;
    if (h->hs_send) cudaFreeHost(h->hs_send);
    if (h->hs_recv) cudaFreeHost(h->hs_recv);
    h->hs_send = h->hs_recv = nullptr;
    for (int i = 0; i < 2; ++i)
        for (cudaEvent_t ev : {h->ev_pair[i], h->ev_bc[i], h->ev_trc[i], h->ev_trs[i]}) if (ev) cudaEventDestroy(ev);
    for (cudaEvent_t ev : {h->ev_side, h->ev_crit, h->ev0, h->ev1}) if (ev) cudaEventDestroy(ev);
    for (cudaStream_t s : {h->crit, h->side, h->cst}) if (s) cudaStreamDestroy(s);
    h->crit = h->side = h->cst = nullptr;
}

int mg_logdet(MgHandle* h, const double* rows, int64_t lds, int64_t tail_rows, cudaStream_t cur, mcnd_logdet* out) {
    clear_out(out);
    if (!h->crit) { int rc = mg_attach(h, 1, 0, nullptr, 0); if (rc) return rc; }
    const int64_t n = h->n, b = kK2B;
    const int32_t world = h->world, rank = h->rank;
    const int64_t tail = std::max<int64_t>(2, tail_rows > 0 ? tail_rows : 64);  // rows finished by K1
    const MgSchedule S = mg_schedule(n, world, tail);
    if (S.len[rank] != h->lr)
        return fail(MCND_EINVAL, "mg_logdet: rank %d holds %lld rows, the plan gives it %lld", rank, (long long)h->lr,
                    (long long)S.len[rank]);
    auto ldw_of = [](int64_t m) { return (m - 64 + 1) / 2 * 2; };
    // pair buffers, tail buffers, record gather (sized for this n and world)
    const int64_t mt = n - S.t_tail, ldr = (mt + 1) / 2 * 2;
    int64_t rmax = 1;
    for (int64_t v : S.live) rmax = std::max(rmax, v);
    size_t off = 0;
    auto take = [&](size_t by) { size_t o = off; off = align_up(off + by, 256); return o; };
    const size_t o_W = take((size_t)2 * 128 * (n - 63) * sizeof(double));
    const size_t o_Wp = take((size_t)2 * b * b * sizeof(double));
    const size_t o_gp = take(2 * sizeof(K2Gather));
    const size_t o_buf = take((size_t)rmax * ldr * sizeof(double));
    const size_t o_wbuf = take((size_t)rmax * sizeof(double));
    const size_t o_gbuf = take((size_t)world * rmax * ldr * sizeof(double));
    const size_t o_gwbuf = take((size_t)world * rmax * sizeof(double));
    const size_t o_trows = take((size_t)mt * ldr * sizeof(double));
    const size_t o_twit = take((size_t)mt * sizeof(double));
    const size_t o_errs = take(16);
    const size_t o_grec = take((size_t)world * n * sizeof(PivRec));
    const size_t o_gerr = take((size_t)world * 16);
    int rc = ensure_dev(&h->pmem, &h->pbytes, off);
    if (rc) return rc;
    char* pb = (char*)h->pmem;
    double* W[2] = {(double*)(pb + o_W), (double*)(pb + o_W) + 128 * (n - 63)};
    double* Wp[2] = {(double*)(pb + o_Wp), (double*)(pb + o_Wp) + b * b};
    K2Gather* gp[2] = {(K2Gather*)(pb + o_gp), (K2Gather*)(pb + o_gp) + 1};
    cudaStream_t crit = h->crit, side = h->side, cst = h->cst;
    const NcclApi& nc = mg_nccl();
    const bool host_tx = h->host_bcast != nullptr;
    // the collectives: NCCL on the library's communicator, or (tests) host callbacks
    auto bcast = [&](void* d, size_t bytes, int32_t root, cudaStream_t s) -> int {
        if (!host_tx) {
            NCCL_TRY(nc.broadcast(d, d, bytes, ncclUint8, root, h->comm, s));
            return MCND_OK;
        }
        int r = ensure_pinned(&h->hs_send, &h->hs_send_bytes, bytes);
        if (r) return r;
        CUDA_TRY(cudaMemcpyAsync(h->hs_send, d, bytes, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        if (h->host_bcast(h->hs_send, (int64_t)bytes, root)) return fail(MCND_ENCCL, "host broadcast failed");
        CUDA_TRY(cudaMemcpyAsync(d, h->hs_send, bytes, cudaMemcpyHostToDevice, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        return MCND_OK;
    };
    auto allgather = [&](const void* d_send, void* d_recv, size_t bytes, cudaStream_t s) -> int {
        if (!host_tx) {
            NCCL_TRY(nc.allGather(d_send, d_recv, bytes, ncclUint8, h->comm, s));
            return MCND_OK;
        }
        int r = ensure_pinned(&h->hs_send, &h->hs_send_bytes, bytes);
        if (!r) r = ensure_pinned(&h->hs_recv, &h->hs_recv_bytes, bytes * (size_t)world);
        if (r) return r;
        CUDA_TRY(cudaMemcpyAsync(h->hs_send, d_send, bytes, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        if (h->host_allgather(h->hs_send, h->hs_recv, (int64_t)bytes)) return fail(MCND_ENCCL, "host all-gather failed");
        CUDA_TRY(cudaMemcpyAsync(d_recv, h->hs_recv, bytes * (size_t)world, cudaMemcpyHostToDevice, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        return MCND_OK;
    };
    auto group = [&](bool start) -> int {
        if (host_tx) return MCND_OK;
        NCCL_TRY(start ? nc.groupStart() : nc.groupEnd());
        return MCND_OK;
    };

    CUDA_TRY(cudaEventRecord(h->ev0, cur));
    CUDA_TRY(cudaStreamWaitEvent(crit, h->ev0, 0));
    CUDA_TRY(cudaStreamWaitEvent(side, h->ev0, 0));
    rc = mg_load(h, rows, lds, crit);
    if (rc) return rc;
    int64_t nl = 1;
    std::vector<int64_t> live = S.len, top(world, 0);
    const auto& pairs = S.pairs;
    auto launch_pair = [&](size_t q) -> int {
        const MgPair& P = pairs[q];
        int r = mg_pair(h, P.lr0, P.t, P.m, W[q & 1], ldw_of(P.m), Wp[q & 1], gp[q & 1], crit);
        if (r) return r;
        CUDA_TRY(cudaEventRecord(h->ev_pair[q & 1], crit));
        nl += (P.t / (2 * kK2B) < kPPBars) ? 1 : 2;  // one launch for both panels (mg_pair)
        return MCND_OK;
    };
    auto trailing = [&](int64_t r0, int64_t nrows, size_t q, bool on_side) -> int {
        nl += 2;
        return mg_trailing(h, r0, nrows, pairs[q].m, W[q & 1], ldw_of(pairs[q].m), Wp[q & 1], gp[q & 1],
                           on_side ? -1 : 0, (int32_t)(q & 1), on_side ? side : crit);
    };
    if (!pairs.empty() && pairs[0].o == rank && (rc = launch_pair(0))) return rc;
    bool side_pending = false;
    for (size_t q = 0; q < pairs.size(); ++q) {
        const MgPair& P = pairs[q];
        const int64_t ldw = ldw_of(P.m);
        if (h->use_comm) {
            // the broadcast waits only for the pair (owner) and for the buffer's previous users
            // (pair q-2's updates on this rank)
            if (rank == P.o) CUDA_TRY(cudaStreamWaitEvent(cst, h->ev_pair[q & 1], 0));
            if (q >= 2) {
                CUDA_TRY(cudaStreamWaitEvent(cst, h->ev_trc[q & 1], 0));
                CUDA_TRY(cudaStreamWaitEvent(cst, h->ev_trs[q & 1], 0));
            }
            if ((rc = group(true)) || (rc = bcast(W[q & 1], (size_t)128 * ldw * sizeof(double), P.o, cst)) ||
                (rc = bcast(Wp[q & 1], (size_t)b * b * sizeof(double), P.o, cst)) ||
                (rc = bcast(gp[q & 1], sizeof(K2Gather), P.o, cst)) || (rc = group(false)))
                return rc;
            CUDA_TRY(cudaEventRecord(h->ev_bc[q & 1], cst));
            CUDA_TRY(cudaStreamWaitEvent(crit, h->ev_bc[q & 1], 0));
            CUDA_TRY(cudaStreamWaitEvent(side, h->ev_bc[q & 1], 0));
        } else {
            CUDA_TRY(cudaStreamWaitEvent(side, h->ev_pair[q & 1], 0));  // the side update reads the pair's output
        }
        live[P.o] -= 2 * b;
        top[P.o] += 2 * b;
        // look-ahead: the next owner updates the 128 rows it contributes next on the high-priority
        // stream and factors them at once (its broadcast can start), the rest on the low-priority
        // stream meanwhile, released after the critical rows (single-GPU schedule)
        const int32_t nxt = (q + 1 < pairs.size()) ? pairs[q + 1].o : -1;
        const int64_t r0 = top[rank], rows_r = live[rank];
        if (side_pending) {  // rows about to be touched on crit were last updated on side
            CUDA_TRY(cudaStreamWaitEvent(crit, h->ev_side, 0));
            side_pending = false;
        }
        if (nxt == rank && rows_r > 2 * b) {
            if ((rc = trailing(r0, 2 * b, q, false))) return rc;
            CUDA_TRY(cudaEventRecord(h->ev_crit, crit));
            if ((rc = launch_pair(q + 1))) return rc;
            CUDA_TRY(cudaStreamWaitEvent(side, h->ev_crit, 0));
            if ((rc = trailing(r0 + 2 * b, rows_r - 2 * b, q, true))) return rc;
            CUDA_TRY(cudaEventRecord(h->ev_side, side));
            side_pending = true;
        } else {
            if (rows_r > 0 && (rc = trailing(r0, rows_r, q, false))) return rc;
            if (nxt == rank && (rc = launch_pair(q + 1))) return rc;
        }
        CUDA_TRY(cudaEventRecord(h->ev_trc[q & 1], crit));
        CUDA_TRY(cudaEventRecord(h->ev_trs[q & 1], side));
    }
    CUDA_TRY(cudaEventRecord(h->ev_side, side));
    CUDA_TRY(cudaStreamWaitEvent(crit, h->ev_side, 0));
    CUDA_TRY(cudaEventRecord(h->ev_crit, crit));
    CUDA_TRY(cudaStreamWaitEvent(cur, h->ev_crit, 0));
    // tail: every rank's remaining rows (first mt columns) in rank order = global order
    double* buf = (double*)(pb + o_buf);
    double* wbuf = (double*)(pb + o_wbuf);
    double* gbuf = (double*)(pb + o_gbuf);
    double* gwbuf = (double*)(pb + o_gwbuf);
    double* trows = (double*)(pb + o_trows);
    double* twit = (double*)(pb + o_twit);
    if (live[rank] > 0 && (rc = mg_export(h, top[rank], live[rank], mt, buf, ldr, wbuf, cur))) return rc;
    if (h->use_comm) {
        if ((rc = group(true)) || (rc = allgather(buf, gbuf, (size_t)rmax * ldr * sizeof(double), cur)) ||
            (rc = allgather(wbuf, gwbuf, (size_t)rmax * sizeof(double), cur)) || (rc = group(false)))
            return rc;
    } else {
        gbuf = buf;
        gwbuf = wbuf;
    }
    for (int32_t r = 0, row = 0; r < world; row += (int32_t)live[r], ++r) {
        if (live[r] == 0) continue;
        CUDA_TRY(cudaMemcpyAsync(trows + (size_t)row * ldr, gbuf + (size_t)r * rmax * ldr,
                                 (size_t)live[r] * ldr * sizeof(double), cudaMemcpyDeviceToDevice, cur));
        CUDA_TRY(cudaMemcpyAsync(twit + row, gwbuf + (size_t)r * rmax, (size_t)live[r] * sizeof(double),
                                 cudaMemcpyDeviceToDevice, cur));
    }
    std::vector<PivRec> trec((size_t)mt);
    uint32_t terr[4] = {0, 0, 0, 0};
    if ((rc = mg_tail(h, trows, ldr, twit, mt, cur, trec.data(), terr))) return rc;
    ++nl;
    // every rank's pivot records and error words {error, step, nonfinite, epoch}
    uint32_t* errs = (uint32_t*)(pb + o_errs);
    PivRec* grec = (PivRec*)(pb + o_grec);
    uint32_t* gerr = (uint32_t*)(pb + o_gerr);
    const uint32_t epoch_h[1] = {h->epoch};
    CUDA_TRY(cudaMemcpyAsync(errs, h->err, 3 * sizeof(uint32_t), cudaMemcpyDeviceToDevice, cur));
    CUDA_TRY(cudaMemcpyAsync(errs + 3, epoch_h, sizeof(uint32_t), cudaMemcpyHostToDevice, cur));
    if (h->use_comm) {
        if ((rc = group(true)) || (rc = allgather(h->recs, grec, (size_t)n * sizeof(PivRec), cur)) ||
            (rc = allgather(errs, gerr, 16, cur)) || (rc = group(false)))
            return rc;
    } else {
        grec = h->recs;
        gerr = errs;
    }
    h->hbuf.resize((size_t)world * (n * sizeof(PivRec) + 16));
    PivRec* hrec = (PivRec*)h->hbuf.data();
    uint32_t* herr = (uint32_t*)(h->hbuf.data() + (size_t)world * n * sizeof(PivRec));
    CUDA_TRY(cudaMemcpyAsync(hrec, grec, (size_t)world * n * sizeof(PivRec), cudaMemcpyDeviceToHost, cur));
    CUDA_TRY(cudaMemcpyAsync(herr, gerr, (size_t)world * 16, cudaMemcpyDeviceToHost, cur));
    CUDA_TRY(cudaEventRecord(h->ev1, cur));
    CUDA_TRY(cudaStreamSynchronize(cur));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, h->ev0, h->ev1);
    out->device_ms = ms;
    out->launches = nl;
    for (int32_t r = 0; r < world; ++r)
        if (herr[4 * r + 2] || terr[2]) return fail(MCND_EINVAL, "matrix entries must be finite (no NaN/Inf)");
    for (int32_t r = 0; r < world; ++r)
        if (herr[4 * r] || terr[0])
            return fail(MCND_EDEVICE, "multi-GPU blocked: device timeout (rank %d step %u, tail step %u)", r,
                        herr[4 * r + 1], terr[1]);
    // fold: the reference's sign / log bookkeeping (condense.py:124-128, 159-160) in step order
    int sign = 1;
    double log_acc = 0.0;
    int64_t steps = 0;
    auto singular = [&](int64_t at) {
        out->sign = 0; out->singular = 1; out->log_abs = -INFINITY; out->singular_step = at; out->steps = at;
        return MCND_OK;
    };
    for (const MgPair& P : pairs) {
        const PivRec* ro = hrec + (size_t)P.o * n;
        const uint32_t ep = herr[4 * P.o + 3];
        for (int64_t s = 0; s < 2 * b; ++s, ++steps) {
            const PivRec& rr = ro[P.t + s];
            if (rr.flag != ep || rr.l < 0) return singular(steps);
            const int64_t ms_ = P.m - s;
            sign *= (rr.v > 0 ? 1 : -1) * (rr.l != ms_ - 1 ? -1 : 1) * (((P.kpos + ms_ - 1) & 1) ? -1 : 1);
            log_acc += std::log(std::fabs(rr.v));
        }
    }
    for (int64_t j = 0; j < mt; ++j, ++steps) {
        const PivRec& rr = trec[(size_t)j];
        if (rr.flag != h->epoch || rr.l < 0) return singular(steps);
        const int64_t mj = mt - j;
        if (j < mt - 1) sign *= (rr.v > 0 ? 1 : -1) * (rr.l != mj - 1 ? -1 : 1) * (((mj - 1) & 1) ? -1 : 1);
        else sign *= rr.v > 0 ? 1 : -1;
        log_acc += std::log(std::fabs(rr.v));
    }
    out->sign = sign;
    out->log_abs = log_acc;
    out->steps = n - 1;
    return MCND_OK;
}

}  // namespace
}  // namespace mcnd

using namespace mcnd;

extern "C" {

int mcnd_logdet_condensation_dev(const double* d_a, int64_t n, int64_t lda, const int64_t* pivot_sequence,
                                 int64_t pivot_sequence_len, uint32_t flags, void* stream, mcnd_logdet* out,
                                 double* pivots_out, int32_t* cols_out) {
    if (!out) return fail(MCND_EINVAL, "null out");
    clear_out(out);
    if (int rc = check_shape(d_a, n, lda)) return rc;  // argument errors before touching a device
    int code = MCND_OK;
    Buffers* B = buffers_for_current(&code);
    if (!B) return code;
    std::lock_guard<std::mutex> lk(B->mu);
    return serial_dev(d_a, n, lda, pivot_sequence, pivot_sequence_len, flags, (cudaStream_t)stream, out,
                      pivots_out, cols_out);
}

int mcnd_logdet_condensation(const double* h_a, int64_t n, int64_t lda, const int64_t* pivot_sequence,
                             int64_t pivot_sequence_len, uint32_t flags, void* stream, mcnd_logdet* out,
                             double* pivots_out, int32_t* cols_out) {
    if (!out) return fail(MCND_EINVAL, "null out");
    clear_out(out);
    int rc = check_shape(h_a, n, lda);
    if (rc) return rc;
    int code = MCND_OK;
    Buffers* B = buffers_for_current(&code);
    if (!B) return code;
    std::lock_guard<std::mutex> lk(B->mu);
    const double* d_a = nullptr;
    rc = stage_input(*B, h_a, n, n, lda, (cudaStream_t)stream, &d_a);
    if (rc) return rc;
    return serial_dev(d_a, n, n, pivot_sequence, pivot_sequence_len, flags, (cudaStream_t)stream, out,
                      pivots_out, cols_out);
}

int mcnd_mc_parallel_dev(const double* d_a, int64_t n, int64_t lda, int32_t p, uint32_t flags, void* stream,
                         mcnd_logdet* out, mcnd_comm_stats* stats, int64_t* payload_entries,
                         int64_t* row_updates, int32_t* owners_out) {
    if (!out) return fail(MCND_EINVAL, "null out");
    clear_out(out);
    if (int rc = check_shape(d_a, n, lda)) return rc;  // argument errors before touching a device
    int code = MCND_OK;
    Buffers* B = buffers_for_current(&code);
    if (!B) return code;
    std::lock_guard<std::mutex> lk(B->mu);
    return parallel_dev(d_a, n, lda, p, flags, (cudaStream_t)stream, out, stats, payload_entries, row_updates,
                        owners_out);
}

int mcnd_mc_parallel(const double* h_a, int64_t n, int64_t lda, int32_t p, uint32_t flags, void* stream,
                     mcnd_logdet* out, mcnd_comm_stats* stats, int64_t* payload_entries, int64_t* row_updates,
                     int32_t* owners_out) {
    if (!out) return fail(MCND_EINVAL, "null out");
    clear_out(out);
    int rc = check_shape(h_a, n, lda);
    if (rc) return rc;
    int code = MCND_OK;
    Buffers* B = buffers_for_current(&code);
    if (!B) return code;
    std::lock_guard<std::mutex> lk(B->mu);
    const double* d_a = nullptr;
    CUDA_TRY(cudaEventRecord(B->ev_h0, (cudaStream_t)stream));
    rc = stage_input(*B, h_a, n, n, lda, (cudaStream_t)stream, &d_a);
    if (rc) return rc;
    CUDA_TRY(cudaEventRecord(B->ev_h1, (cudaStream_t)stream));
    rc = parallel_dev(d_a, n, n, p, flags, (cudaStream_t)stream, out, stats, payload_entries, row_updates,
                      owners_out);
    float h2d_ms = 0.f;  // the matrix reaching the device is part of the scatter (runtime.py:138-143)
    if (rc == MCND_OK && stats && cudaEventElapsedTime(&h2d_ms, B->ev_h0, B->ev_h1) == cudaSuccess)
        stats->scatter_seconds += (double)h2d_ms * 1e-3;
    return rc;
}

/* debug (not part of the ABI header): panel-launch spans of the calls since the last read */
int mcnd_debug_kp_spans(unsigned long long* out, int max_spans) {
    // both panel kernels' spans, in time order
    const int a = mcnd::kp_debug_spans(out, max_spans);
    if (a < 0) return a;
    const int b = mcnd::kc_debug_spans(out + 2 * (size_t)a, max_spans - a);
    if (b < 0) return b;
    std::vector<std::pair<unsigned long long, unsigned long long>> v((size_t)(a + b));
    for (int i = 0; i < a + b; ++i) v[(size_t)i] = {out[2 * i], out[2 * i + 1]};
    std::sort(v.begin(), v.end());
    for (int i = 0; i < a + b; ++i) { out[2 * i] = v[(size_t)i].first; out[2 * i + 1] = v[(size_t)i].second; }
    return a + b;
}

int mcnd_logdet_blocked_dev(const double* d_a, int64_t n, int64_t lda, uint32_t flags, void* stream,
                            mcnd_logdet* out, double* pivots_out, int32_t* cols_out) {
    if (!out) return fail(MCND_EINVAL, "null out");
    clear_out(out);
    if (int rc = check_shape(d_a, n, lda)) return rc;  // argument errors before touching a device
    int code = MCND_OK;
    Buffers* B = buffers_for_current(&code);
    if (!B) return code;
    std::lock_guard<std::mutex> lk(B->mu);
    return blocked_dev(d_a, n, lda, flags, (cudaStream_t)stream, out, pivots_out, cols_out);
}

int mcnd_logdet_blocked(const double* h_a, int64_t n, int64_t lda, uint32_t flags, void* stream, mcnd_logdet* out,
                        double* pivots_out, int32_t* cols_out) {
    if (!out) return fail(MCND_EINVAL, "null out");
    clear_out(out);
    int rc = check_shape(h_a, n, lda);
    if (rc) return rc;
    int code = MCND_OK;
    Buffers* B = buffers_for_current(&code);
    if (!B) return code;
    std::lock_guard<std::mutex> lk(B->mu);
    // staged inside: streamed by row chunks when h_a is pinned (overlaps the first pairs)
    return blocked_dev(nullptr, n, lda, flags, (cudaStream_t)stream, out, pivots_out, cols_out, h_a);
}

int32_t mcnd_blocked_panel(void) { return kK2B; }

int mcnd_logdet_lu_dev(const double* d_a, int64_t n, int64_t lda, const double* d_row_witness, uint32_t flags,
                       void* stream, mcnd_logdet* out, double* pivots_out, int32_t* rows_out) {
    if (!out) return fail(MCND_EINVAL, "null out");
    clear_out(out);
    if (int rc = check_shape(d_a, n, lda)) return rc;
    int code = MCND_OK;
    Buffers* B = buffers_for_current(&code);
    if (!B) return code;
    std::lock_guard<std::mutex> lk(B->mu);
    return ge_dev(d_a, n, lda, d_row_witness, flags, (cudaStream_t)stream, out, pivots_out, rows_out);
}

int mcnd_logdet_lu(const double* h_a, int64_t n, int64_t lda, const double* h_row_witness, uint32_t flags,
                   void* stream, mcnd_logdet* out, double* pivots_out, int32_t* rows_out) {
    if (!out) return fail(MCND_EINVAL, "null out");
    clear_out(out);
    if (int rc = check_shape(h_a, n, lda)) return rc;
    int code = MCND_OK;
    Buffers* B = buffers_for_current(&code);
    if (!B) return code;
    std::lock_guard<std::mutex> lk(B->mu);
    const double* d_a = nullptr;
    int rc = stage_input(*B, h_a, n, n, lda, (cudaStream_t)stream, &d_a);
    if (rc) return rc;
    return ge_dev(d_a, n, n, nullptr, flags, (cudaStream_t)stream, out, pivots_out, rows_out, h_row_witness);
}

int mcnd_fold_mc_parallel(int64_t n, int32_t p, const double* piv_vals, const int32_t* piv_cols,
                          int64_t singular_at, const double* rem, const double* rem_wit, mcnd_logdet* out,
                          mcnd_comm_stats* stats, int64_t* payload_entries, int64_t* row_updates) {
    if (!out) return fail(MCND_EINVAL, "null out");
    clear_out(out);
    if (p < 1 || p > n) return fail(MCND_EINVAL, "invalid plan: need 1 <= p <= n, got p=%d, n=%lld", p, (long long)n);
    if (stats) std::memset(stats, 0, sizeof(*stats));
    return fold_parallel(n, p, piv_vals, piv_cols, singular_at, rem, rem_wit, out, stats, payload_entries,
                         row_updates);
}

int32_t mcnd_dist_ipc_handle_bytes(void) { return (int32_t)sizeof(cudaIpcMemHandle_t); }

int mcnd_dist_create(int32_t rank, int32_t world, int64_t n_max, void** handle, void* ipc_out) {
    if (!handle || !ipc_out) return fail(MCND_EINVAL, "null handle/ipc_out");
    if (world < 1 || world > kMaxGroups || rank < 0 || rank >= world)
        return fail(MCND_EINVAL, "need 1 <= world <= %d and 0 <= rank < world", kMaxGroups);
    if (n_max < world) return fail(MCND_EINVAL, "n_max < world");
    auto* h = new DistHandle();
    h->rank = rank;
    h->world = world;
    h->n_max = n_max;
    h->GL = group_layout(n_max, n_max);
    int dev = 0;
    cudaGetDevice(&dev);
    int rc = init_buffers(h->B, dev);
    if (rc) { delete h; return rc; }
    rc = ensure_dev(&h->B.dws, &h->B.dws_bytes, h->GL.bytes);
    if (rc) { delete h; return rc; }
    if (cudaMemset(h->B.dws, 0, h->GL.bytes) != cudaSuccess) { delete h; return fail(MCND_ECUDA, "cudaMemset"); }
    h->meta_bytes = meta_bytes_for(n_max, n_max, (int64_t)h->B.sms);
    if (cudaMalloc(&h->meta, h->meta_bytes) != cudaSuccess) { delete h; return fail(MCND_ECUDA, "cudaMalloc meta"); }
    cudaIpcMemHandle_t ipc;
    cudaError_t e = cudaIpcGetMemHandle(&ipc, h->B.dws);
    if (e != cudaSuccess) { delete h; return fail(MCND_ECUDA, "cudaIpcGetMemHandle: %s", cudaGetErrorString(e)); }
    std::memcpy(ipc_out, &ipc, sizeof(ipc));
    if (cudaDeviceSynchronize() != cudaSuccess) { delete h; return fail(MCND_ECUDA, "cudaDeviceSynchronize"); }
    *handle = h;
    return MCND_OK;
}

int mcnd_dist_connect(void* handle, const void* ipc_all) {
    auto* h = (DistHandle*)handle;
    if (!h || !ipc_all) return fail(MCND_EINVAL, "null handle");
    for (int32_t r = 0; r < h->world; ++r) {
        if (r == h->rank) { h->peer_base[r] = h->B.dws; continue; }
        cudaIpcMemHandle_t ipc;
        std::memcpy(&ipc, (const char*)ipc_all + (size_t)r * sizeof(ipc), sizeof(ipc));
        cudaError_t e = cudaIpcOpenMemHandle(&h->peer_base[r], ipc, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) return fail(MCND_ECUDA, "cudaIpcOpenMemHandle(rank %d): %s", r, cudaGetErrorString(e));
    }
    h->connected = true;
    return MCND_OK;
}

int mcnd_dist_mc_parallel(void* handle, const double* d_rows, int64_t n, int64_t lda, uint32_t flags, void* stream,
                          double* piv_vals, int32_t* piv_cols, int64_t* singular_at, double* rem_row,
                          double* rem_wit, double* device_ms) {
    auto* h = (DistHandle*)handle;
    if (!h || !h->connected) return fail(MCND_EINVAL, "dist handle not connected");
    if (n != h->n_max) return fail(MCND_EINVAL, "n (%lld) must equal the handle's n_max (%lld)", (long long)n,
                                   (long long)h->n_max);
    if (!d_rows || lda < n) return fail(MCND_EINVAL, "bad local rows");
    const int32_t P = h->world;
    cudaStream_t st = (cudaStream_t)stream;
    const Blocks blk = plan_blocks(n, P);
    K1Run run;
    run.n = n;
    std::vector<int32_t> owner;
    round_robin(blk, &run.seq, &owner);
    run.steps = (int64_t)run.seq.size();
    const GroupLayout& GL = h->GL;
    K1Launch L;
    L.n = n;
    L.lda = lda;
    L.n_groups = P;
    L.group0 = h->rank;
    L.n_local = 1;
    L.cpg = (int32_t)std::max<int64_t>(1, std::min<int64_t>(h->B.sms, blk.len[(size_t)h->rank]));
    L.sys = true;
    L.epoch = ++h->epoch;
    L.reset_records = false;
    L.timeout_ns = 60ull * 1000000000ull;
    for (int32_t g = 0; g < P; ++g) {
        char* gb = (char*)h->peer_base[g];
        L.ws[g] = (double*)gb;
        L.rec[g] = (PivRec*)(gb + GL.o_rec);
    }
    L.wit[0] = (double*)((char*)h->B.dws + GL.o_wit);
    L.src[0] = d_rows;
    L.src_row0[0] = blk.start[(size_t)h->rank];
    L.row_group.assign((size_t)n, 0);
    for (int64_t r = 0; r < n; ++r) L.row_group[(size_t)r] = blk.group_of(r);
    L.d_meta = h->meta;
    L.meta_bytes = h->meta_bytes;
    int rc = k1_execute(h->B, L, (flags & MCND_FLAG_FAST) != 0, st, run);
    if (rc) return rc;
    const int64_t k = run.singular_at >= 0 ? run.singular_at + 1 : run.steps;
    for (int64_t t = 0; t < k; ++t) { piv_vals[t] = run.piv_val[(size_t)t]; piv_cols[t] = run.piv_col[(size_t)t]; }
    *singular_at = run.singular_at;
    const int64_t r = blk.start[(size_t)h->rank] + blk.len[(size_t)h->rank] - 1;  // my last live row
    CUDA_TRY(cudaMemcpy(rem_row, (double*)h->B.dws + r * GL.ld, (size_t)P * sizeof(double), cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(rem_wit, L.wit[0] + r, sizeof(double), cudaMemcpyDeviceToHost));
    if (device_ms) *device_ms = run.device_ms;
    return MCND_OK;
}

void mcnd_dist_destroy(void* handle) {
    auto* h = (DistHandle*)handle;
    if (!h) return;
    cudaDeviceSynchronize();
    for (int32_t r = 0; r < h->world; ++r)
        if (r != h->rank && h->peer_base[r]) cudaIpcCloseMemHandle(h->peer_base[r]);
    if (h->meta) cudaFree(h->meta);
    if (h->B.dws) cudaFree(h->B.dws);
    if (h->B.hpin) cudaFreeHost(h->B.hpin);
    if (h->B.ev0) cudaEventDestroy(h->B.ev0);
    if (h->B.ev1) cudaEventDestroy(h->B.ev1);
    delete h;
}

int mcnd_logdet_batched_dev(const double* d_a, int64_t batch, int64_t n, int64_t stride, uint32_t flags,
                            void* stream, int32_t* d_sign, double* d_log_abs, double* d_pivots,
                            uint32_t* d_nonfinite) {
    if (batch < 0 || n < 1 || n > 128) return fail(MCND_EINVAL, "batched kernel needs 1 <= n <= 128 (got %lld)", (long long)n);
    if (stride < n * n) return fail(MCND_EINVAL, "stride < n*n");
    if (batch > 0 && (!d_a || !d_sign || !d_log_abs)) return fail(MCND_EINVAL, "null pointer");
    cudaError_t e = k3_launch(d_a, batch, n, stride, (flags & MCND_FLAG_FAST) != 0, d_sign, d_log_abs, d_pivots,
                              d_nonfinite, (cudaStream_t)stream);
    if (e != cudaSuccess) return fail(MCND_ECUDA, "batched kernel: %s", cudaGetErrorString(e));
    return MCND_OK;
}

int mcnd_logdet_batched(const double* h_a, int64_t batch, int64_t n, int64_t stride, uint32_t flags, void* stream,
                        int32_t* h_sign, double* h_log_abs) {
    if (batch < 0 || n < 1 || n > 128) return fail(MCND_EINVAL, "batched kernel needs 1 <= n <= 128 (got %lld)", (long long)n);
    if (stride < n * n) return fail(MCND_EINVAL, "stride < n*n");
    if (batch == 0) return MCND_OK;
    int code = MCND_OK;
    Buffers* B = buffers_for_current(&code);
    if (!B) return code;
    std::lock_guard<std::mutex> lk(B->mu);
    cudaStream_t st = (cudaStream_t)stream;
    const size_t in_bytes = (size_t)batch * stride * sizeof(double);
    const size_t o_sign = align_up((size_t)batch * sizeof(double), 256);
    const size_t o_flag = o_sign + align_up((size_t)batch * sizeof(int32_t), 256);
    int rc = ensure_dev(&B->din, &B->din_bytes, in_bytes);
    if (rc) return rc;
    rc = ensure_dev(&B->dws, &B->dws_bytes, o_flag + 256);
    if (rc) return rc;
    rc = ensure_pinned(&B->hpin, &B->hpin_bytes, 256);
    if (rc) return rc;
    double* d_log = (double*)B->dws;
    int32_t* d_sign = (int32_t*)((char*)B->dws + o_sign);
    unsigned* d_flag = (unsigned*)((char*)B->dws + o_flag);
    CUDA_TRY(cudaMemsetAsync(d_flag, 0, sizeof(unsigned), st));
    CUDA_TRY(cudaMemcpyAsync(B->din, h_a, in_bytes, cudaMemcpyHostToDevice, st));
    cudaError_t e = k3_launch((const double*)B->din, batch, n, stride, (flags & MCND_FLAG_FAST) != 0, d_sign, d_log,
                              nullptr, d_flag, st);
    if (e != cudaSuccess) return fail(MCND_ECUDA, "batched kernel: %s", cudaGetErrorString(e));
    CUDA_TRY(cudaMemcpyAsync(h_log_abs, d_log, (size_t)batch * sizeof(double), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(h_sign, d_sign, (size_t)batch * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(B->hpin, d_flag, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    if (*(unsigned*)B->hpin) return fail(MCND_EINVAL, "matrix entries must be finite (no NaN/Inf)");
    return MCND_OK;
}

const char* mcnd_last_error(void) { return g_err.c_str(); }

int32_t mcnd_version(void) { return 110; }

int32_t mcnd_k1_grid(void) {
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

void mcnd_release_workspace(void) {
    std::lock_guard<std::mutex> lk(g_mu);
    int cur = 0;
    cudaGetDevice(&cur);
    for (auto& b : g_bufs) {
        std::lock_guard<std::mutex> lb(b.mu);  // (must not race a call on that device)
        cudaSetDevice(b.device);
        if (b.dws) cudaFree(b.dws);
        if (b.din) cudaFree(b.din);
        if (b.dge) cudaFree(b.dge);
        if (b.hpin) cudaFreeHost(b.hpin);
        if (b.ev0) cudaEventDestroy(b.ev0);
        if (b.ev1) cudaEventDestroy(b.ev1);
    }
    cudaSetDevice(cur);
    g_bufs.clear();
}


/* ---- multi-GPU blocked condensation, per-rank engine (see mcnd_b200.h) ---- */
int mcnd_mg_create(int64_t n, int64_t local_rows, void** handle) {
    if (!handle) return fail(MCND_EINVAL, "null handle");
    MgHandle* h = nullptr;
    int rc = mg_create(n, local_rows, &h);
    *handle = h;
    return rc;
}
int mcnd_mg_load(void* handle, const double* d_rows, int64_t lds, void* stream) {
    if (!handle) return fail(MCND_EINVAL, "null handle");
    return mg_load((MgHandle*)handle, d_rows, lds, (cudaStream_t)stream);
}
int mcnd_mg_pair(void* handle, int64_t lr0, int64_t t, int64_t m, double* d_W, int64_t ldw, double* d_Wp,
                 void* d_gather, void* stream) {
    if (!handle) return fail(MCND_EINVAL, "null handle");
    return mg_pair((MgHandle*)handle, lr0, t, m, d_W, ldw, d_Wp, (K2Gather*)d_gather, (cudaStream_t)stream);
}
int mcnd_mg_trailing(void* handle, int64_t lr0, int64_t rows, int64_t m, const double* d_W, int64_t ldw,
                     const double* d_Wp, const void* d_gather, int32_t sm_budget, int32_t par, void* stream) {
    if (!handle) return fail(MCND_EINVAL, "null handle");
    return mg_trailing((MgHandle*)handle, lr0, rows, m, d_W, ldw, d_Wp, (const K2Gather*)d_gather, sm_budget, par,
                       (cudaStream_t)stream);
}
int mcnd_mg_export(void* handle, int64_t lr0, int64_t rows, int64_t mt, double* d_out, int64_t ldo, double* d_wit,
                   void* stream) {
    if (!handle) return fail(MCND_EINVAL, "null handle");
    return mg_export((MgHandle*)handle, lr0, rows, mt, d_out, ldo, d_wit, (cudaStream_t)stream);
}
int mcnd_mg_tail(void* handle, double* d_rows, int64_t ldr, const double* d_wit, int64_t mt, void* stream,
                 void* h_recs, uint32_t* h_err) {
    if (!handle) return fail(MCND_EINVAL, "null handle");
    return mg_tail((MgHandle*)handle, d_rows, ldr, d_wit, mt, (cudaStream_t)stream, h_recs, h_err);
}
int mcnd_mg_records(void* handle, void* h_recs, uint32_t* h_err, void* stream) {
    if (!handle) return fail(MCND_EINVAL, "null handle");
    return mg_records((MgHandle*)handle, h_recs, h_err, (cudaStream_t)stream);
}
int64_t mcnd_mg_gather_bytes(void) { return (int64_t)sizeof(K2Gather); }
int64_t mcnd_mg_ld(void* handle) { return handle ? ((MgHandle*)handle)->ld : 0; }
int32_t mcnd_nccl_id_bytes(void) { return (int32_t)sizeof(ncclUniqueId); }
int mcnd_nccl_unique_id(void* id_out) {
    if (!id_out) return fail(MCND_EINVAL, "null id");
    if (!mg_nccl().ok) return fail(MCND_ENCCL, "libnccl.so.2 not found");
    ncclUniqueId uid;
    NCCL_TRY(mg_nccl().getUniqueId(&uid));
    std::memcpy(id_out, &uid, sizeof(uid));
    return MCND_OK;
}
int mcnd_mg_attach(void* handle, int32_t world, int32_t rank, const void* nccl_id, int32_t force_comm) {
    if (!handle) return fail(MCND_EINVAL, "null handle");
    return mg_attach((MgHandle*)handle, world, rank, nccl_id, force_comm);
}
int mcnd_mg_attach_host(void* handle, int32_t world, int32_t rank, int (*bcast)(void*, int64_t, int32_t),
                        int (*allgather)(const void*, void*, int64_t)) {
    if (!handle || !bcast || !allgather) return fail(MCND_EINVAL, "null handle / callback");
    if (world < 1 || rank < 0 || rank >= world) return fail(MCND_EINVAL, "mg_attach_host: bad rank %d of %d", rank, world);
    int rc = mg_attach((MgHandle*)handle, 1, 0, nullptr, 0);  // the streams and events, no NCCL
    if (rc) return rc;
    auto* h = (MgHandle*)handle;
    h->world = world;
    h->rank = rank;
    h->use_comm = true;
    h->host_bcast = bcast;
    h->host_allgather = allgather;
    return MCND_OK;
}
int mcnd_mg_logdet(void* handle, const double* d_rows, int64_t lds, int64_t tail, void* stream, mcnd_logdet* out) {
    if (!handle || !out) return fail(MCND_EINVAL, "null handle/out");
    return mg_logdet((MgHandle*)handle, d_rows, lds, tail, (cudaStream_t)stream, out);
}
int64_t mcnd_mg_schedule(int64_t n, int32_t world, int64_t tail, int64_t* pairs_out, int64_t max_pairs) {
    if (n < 1 || world < 1 || world > n) return -1;
    const MgSchedule S = mg_schedule(n, world, tail);
    for (size_t q = 0; q < S.pairs.size() && (int64_t)q < max_pairs && pairs_out; ++q) {
        const MgPair& P = S.pairs[q];
        int64_t* o = pairs_out + 5 * q;
        o[0] = P.o; o[1] = P.lr0; o[2] = P.t; o[3] = P.m; o[4] = P.kpos;
    }
    return (int64_t)S.pairs.size();
}

int mcnd_mg_destroy(void* handle) {
    auto* h = (MgHandle*)handle;
    if (!h) return MCND_OK;
    mg_release_native(h);
    cudaFree(h->mem);
    if (h->tail_mem) cudaFree(h->tail_mem);
    if (h->hpin) cudaFreeHost(h->hpin);
    delete h;
    return MCND_OK;
}

}  // extern "C"

// Host runtime + C ABI (include/mcnd_b200.h).
//
// Everything the reference does on the host around the hot loop lives here,
// in native code: argument validation (matrix.py:32-48, condense.py:85-86,
// runtime.py:35-36), the pivot schedule (condense.py:147-152 top-to-bottom or
// a caller sequence; runtime.py:153-156 round-robin block owners), the exact
// sign bookkeeping (condense.py:125-128, runtime.py:179-182), the sequential
// log sum (condense.py:124; runtime.py:114-120 rank-ordered reduce), the p x p
// elimination tail of the block-row driver (runtime.py:206-219 ->
// gauss.py:34-68) and the communication accounting (runtime.py:47-66,
// 82-90).  The GPU does all O(N^3) work; the host touches O(N) numbers.
//
// Compiled with -ffp-contract=off: the tail LU must round exactly like numpy.
#include <cuda_runtime.h>
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
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

// ---- cached device/pinned buffers (one set per device; calls are serialised) ----
struct Buffers {
    int device = -1;
    void* dws = nullptr;   size_t dws_bytes = 0;    // condensation workspace
    void* din = nullptr;   size_t din_bytes = 0;    // H2D staging for host-input calls
    void* hpin = nullptr;  size_t hpin_bytes = 0;   // pinned metadata / result staging
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    int sms = 0;
};
std::mutex g_mu;
std::deque<Buffers> g_bufs;

Buffers* buffers_for_current(int* code) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) { *code = fail(MCND_ECUDA, "cudaGetDevice: %s", cudaGetErrorString(e)); return nullptr; }
    for (auto& b : g_bufs) if (b.device == dev) return &b;
    Buffers b;
    b.device = dev;
    cudaDeviceGetAttribute(&b.sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaEventCreate(&b.ev0) != cudaSuccess || cudaEventCreate(&b.ev1) != cudaSuccess) {
        *code = fail(MCND_ECUDA, "cudaEventCreate failed");
        return nullptr;
    }
    g_bufs.push_back(b);
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

// ---- K1 plan and run ----
struct K1Run {
    // inputs
    int64_t n = 0;
    int64_t steps = 0;              // S
    std::vector<int32_t> seq;       // S (+1 if a final 1x1 pivot is published)
    // outputs
    std::vector<double> piv_val;    // seq.size()
    std::vector<int32_t> piv_col;
    std::vector<double> row_wit;    // n (only when want_wit)
    int64_t singular_at = -1;       // pivot index with failed witness test
    double device_ms = 0.0;
};

// Runs the persistent condensation on device matrix d_a.  If keep_rows is
// non-null, copies rows keep_rows[i] (first keep_cols columns) of the final
// workspace to keep_out (row-major).
int k1_run(Buffers& B, const double* d_a, int64_t n, int64_t lda, bool fast, cudaStream_t st,
           K1Run& run, bool want_wit, const std::vector<int32_t>* keep_rows, int64_t keep_cols,
           std::vector<double>* keep_out) {
    const int64_t S = run.steps;
    const int64_t npiv = (int64_t)run.seq.size();
    const int64_t ld = (int64_t)align_up((size_t)n, 16);
    int64_t G = std::min<int64_t>(B.sms, n);
    if (const char* eg = std::getenv("MCND_K1_GRID")) {  // test knob: fewer CTAs, more rows per CTA
        const long v = std::strtol(eg, nullptr, 10);
        if (v > 0) G = std::min<int64_t>(G, v);
    }
    if (G < 1) G = 1;
    if ((n + G - 1) / G > kK1MaxRowsPerCta)
        return fail(MCND_EINVAL, "n=%lld exceeds the single-GPU limit (%d rows per SM)", (long long)n,
                    kK1MaxRowsPerCta);

    // pivot index of every row, rows dealt cyclically to CTAs in pivot order
    std::vector<int32_t> pstep((size_t)n, kNever);
    for (int64_t t = 0; t < npiv; ++t) pstep[(size_t)run.seq[(size_t)t]] = (int32_t)t;
    std::vector<int32_t> order;
    order.reserve((size_t)n);
    for (int64_t t = 0; t < npiv; ++t) order.push_back(run.seq[(size_t)t]);
    for (int64_t r = 0; r < n; ++r) if (pstep[(size_t)r] == kNever) order.push_back((int32_t)r);
    std::vector<int32_t> row_ptr((size_t)G + 1, 0), rows((size_t)n);
    for (int64_t g = 0; g < G; ++g) row_ptr[(size_t)g + 1] = row_ptr[(size_t)g] + (int32_t)((n - g + G - 1) / G);
    {
        std::vector<int32_t> fill(row_ptr.begin(), row_ptr.end() - 1);
        for (int64_t i = 0; i < n; ++i) rows[(size_t)fill[(size_t)(i % G)]++] = order[(size_t)i];
    }

    // device workspace layout
    const size_t npv = (size_t)std::max<int64_t>(npiv, 1);
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off = align_up(off + bytes, 256); return o; };
    const size_t o_mat = take((size_t)n * ld * sizeof(double));
    const size_t o_int = take((npv + (size_t)n + (size_t)G + 1 + (size_t)n) * sizeof(int32_t));
    const size_t o_pv = take(npv * sizeof(double));
    const size_t o_pw = take(npv * sizeof(double));
    const size_t o_pc = take(npv * sizeof(int32_t));
    const size_t o_rw = take((size_t)n * sizeof(double));
    const size_t o_ctl = take(sizeof(K1Ctrl));
    int rc = ensure_dev(&B.dws, &B.dws_bytes, off);
    if (rc) return rc;
    char* base = (char*)B.dws;

    const size_t n_int = npv + (size_t)n + (size_t)G + 1 + (size_t)n;
    const size_t h_need = std::max(n_int * sizeof(int32_t),
                                   npv * (sizeof(double) + sizeof(int32_t)) + sizeof(K1Ctrl) + 64);
    rc = ensure_pinned(&B.hpin, &B.hpin_bytes, std::max(h_need, (size_t)n * sizeof(double)) + 256);
    if (rc) return rc;
    int32_t* hi = (int32_t*)B.hpin;
    std::memset(hi, 0, npv * sizeof(int32_t));
    std::memcpy(hi, run.seq.data(), (size_t)npiv * sizeof(int32_t));
    std::memcpy(hi + npv, pstep.data(), (size_t)n * sizeof(int32_t));
    std::memcpy(hi + npv + n, row_ptr.data(), ((size_t)G + 1) * sizeof(int32_t));
    std::memcpy(hi + npv + n + G + 1, rows.data(), (size_t)n * sizeof(int32_t));
    CUDA_TRY(cudaMemcpyAsync(base + o_int, hi, n_int * sizeof(int32_t), cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemsetAsync(base + o_ctl, 0, sizeof(K1Ctrl), st));

    K1Params p{};
    p.src = d_a;
    p.lds = lda;
    p.ws = (double*)(base + o_mat);
    p.ld = ld;
    p.n = (int32_t)n;
    p.n_steps = (int32_t)S;
    int32_t* di = (int32_t*)(base + o_int);
    p.seq = di;
    p.row_pstep = di + npv;
    p.cta_row_ptr = di + npv + n;
    p.cta_rows = di + npv + n + G + 1;
    p.piv_val = (double*)(base + o_pv);
    p.piv_wit = (double*)(base + o_pw);
    p.piv_col = (int32_t*)(base + o_pc);
    p.row_wit = (double*)(base + o_rw);
    p.ctrl = (K1Ctrl*)(base + o_ctl);
    p.chunk = (int32_t)std::min<int64_t>(align_up((size_t)n, 2), kK1MaxChunk);
    if (const char* ec = std::getenv("MCND_K1_CHUNK")) {  // test knob: force multi-chunk staging
        const long v = std::strtol(ec, nullptr, 10);
        if (v >= 2 && v <= kK1MaxChunk) p.chunk = (int32_t)std::min<int64_t>(p.chunk, v & ~1L);
    }
    p.timeout_ns = 20ull * 1000000000ull;

    CUDA_TRY(cudaEventRecord(B.ev0, st));
    cudaError_t e = k1_launch(p, (int)G, fast, st);
    if (e != cudaSuccess) return fail(MCND_ECUDA, "condensation kernel launch: %s", cudaGetErrorString(e));
    CUDA_TRY(cudaEventRecord(B.ev1, st));

    // results -> pinned host
    char* hp = (char*)B.hpin;
    double* h_pv = (double*)hp;
    int32_t* h_pc = (int32_t*)(hp + npv * sizeof(double));
    K1Ctrl* h_ctl = (K1Ctrl*)(hp + align_up(npv * (sizeof(double) + sizeof(int32_t)), 16));
    CUDA_TRY(cudaMemcpyAsync(h_pv, base + o_pv, npv * sizeof(double), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(h_pc, base + o_pc, npv * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(h_ctl, base + o_ctl, sizeof(K1Ctrl), cudaMemcpyDeviceToHost, st));
    if (want_wit) {
        run.row_wit.resize((size_t)n);
        CUDA_TRY(cudaMemcpyAsync(run.row_wit.data(), base + o_rw, (size_t)n * sizeof(double),
                                 cudaMemcpyDeviceToHost, st));
    }
    if (keep_rows && keep_out) {
        keep_out->assign(keep_rows->size() * (size_t)keep_cols, 0.0);
        for (size_t i = 0; i < keep_rows->size(); ++i)
            CUDA_TRY(cudaMemcpyAsync(keep_out->data() + i * keep_cols,
                                     p.ws + (int64_t)(*keep_rows)[i] * ld, (size_t)keep_cols * sizeof(double),
                                     cudaMemcpyDeviceToHost, st));
    }
    e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return fail(MCND_ECUDA, "condensation kernel: %s", cudaGetErrorString(e));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, B.ev0, B.ev1);
    run.device_ms = ms;
    if (h_ctl->error)
        return fail(MCND_EDEVICE, "device timeout waiting for pivot %u (published %u)", h_ctl->err_step,
                    h_ctl->published);
    run.piv_val.assign(h_pv, h_pv + npiv);
    run.piv_col.assign(h_pc, h_pc + npiv);
    run.singular_at = -1;
    const unsigned pub = h_ctl->published;
    for (int64_t t = 0; t < npiv; ++t) {
        if (run.piv_col[(size_t)t] < 0) { run.singular_at = t; break; }
    }
    if (run.singular_at < 0 && (int64_t)pub != npiv)
        return fail(MCND_EDEVICE, "protocol error: %u of %lld pivots published", pub, (long long)npiv);
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
    rc = k1_run(*B, d_a, n, lda, (flags & MCND_FLAG_FAST) != 0, st, run, false, nullptr, 0, nullptr);
    if (rc) return rc;
    out->device_ms = run.device_ms;
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

int parallel_dev(const double* d_a, int64_t n, int64_t lda, int32_t p, uint32_t flags, cudaStream_t st,
                 mcnd_logdet* out, mcnd_comm_stats* stats, int64_t* payload_out, int64_t* row_updates_out,
                 int32_t* owners_out) {
    clear_out(out);
    if (stats) std::memset(stats, 0, sizeof(*stats));
    int rc = check_shape(d_a, n, lda);
    if (rc) return rc;
    if (p < 1 || p > n) return fail(MCND_EINVAL, "invalid plan: need 1 <= p <= n, got p=%d, n=%lld", p, (long long)n);
    int code = MCND_OK;
    Buffers* B = buffers_for_current(&code);
    if (!B) return code;

    // plan_blocks (runtime.py:33-44) and the round-robin owner schedule (runtime.py:153-156)
    std::vector<int64_t> start((size_t)p), len((size_t)p), consumed((size_t)p, 0);
    {
        const int64_t base = n / p, extra = n % p;
        int64_t s0 = 0;
        for (int32_t w = 0; w < p; ++w) {
            start[(size_t)w] = s0;
            len[(size_t)w] = base + (w < extra ? 1 : 0);
            s0 += len[(size_t)w];
        }
    }
    K1Run run;
    run.n = n;
    std::vector<int32_t> owner;
    for (;;) {
        bool any = false;
        for (int32_t w = 0; w < p; ++w) any |= (len[(size_t)w] - consumed[(size_t)w] > 1);
        if (!any) break;
        for (int32_t w = 0; w < p; ++w) {
            if (len[(size_t)w] - consumed[(size_t)w] <= 1) continue;
            run.seq.push_back((int32_t)(start[(size_t)w] + consumed[(size_t)w]));
            owner.push_back(w);
            consumed[(size_t)w] += 1;
        }
    }
    run.steps = (int64_t)run.seq.size();  // n - p
    std::vector<int32_t> rem_rows((size_t)p);
    for (int32_t w = 0; w < p; ++w) rem_rows[(size_t)w] = (int32_t)(start[(size_t)w] + consumed[(size_t)w]);
    std::vector<double> rem;
    rc = k1_run(*B, d_a, n, lda, (flags & MCND_FLAG_FAST) != 0, st, run, true, &rem_rows, p, &rem);
    if (rc) return rc;
    out->device_ms = run.device_ms;

    const int64_t S = run.steps;
    const int64_t done = run.singular_at >= 0 ? run.singular_at : S;
    // accounting (runtime.py:82-90, 185-197)
    std::vector<int64_t> cons((size_t)p, 0), row_upd((size_t)p, 0);
    int64_t bbytes = 0, scalar = 0;
    std::vector<double> local_logs((size_t)p, 0.0);
    Fenwick live(n);
    int sign = 1;
    for (int64_t t = 0; t < done; ++t) {
        const int32_t w = owner[(size_t)t];
        const int64_t m = n - t, last = m - 1;
        const double v = run.piv_val[(size_t)t];
        const int64_t r = run.seq[(size_t)t];
        local_logs[(size_t)w] += std::log(std::fabs(v));
        cons[(size_t)w] += 1;
        const int64_t k_pos = live.prefix(r);
        live.remove(r);
        const int swap_parity = (run.piv_col[(size_t)t] != last) ? -1 : 1;
        const int parity = ((k_pos + m - 1) % 2) ? -1 : 1;
        sign *= (v > 0 ? 1 : -1) * swap_parity * parity;
        bbytes += 8 * last + 8;
        if (payload_out) payload_out[t] = last;
        for (int32_t u = 0; u < p; ++u) {
            const int64_t lv = len[(size_t)u] - cons[(size_t)u];
            row_upd[(size_t)u] += lv;
            scalar += lv * last;
        }
    }
    if (owners_out) for (int64_t t = 0; t < S; ++t) owners_out[t] = owner[(size_t)t];
    if (row_updates_out) for (int32_t u = 0; u < p; ++u) row_updates_out[u] = row_upd[(size_t)u];
    if (stats) {
        stats->broadcasts = done + (run.singular_at >= 0 ? 1 : 0);
        stats->broadcast_bytes = bbytes + (run.singular_at >= 0 ? 1 : 0);
        stats->pivot_search_msgs = 0;
        stats->scalar_updates = scalar;
        stats->aborted_step = run.singular_at;
    }
    out->steps = done;
    if (run.singular_at >= 0) {
        out->sign = 0;
        out->singular = 1;
        out->log_abs = -INFINITY;
        out->singular_step = run.singular_at;
        return MCND_OK;
    }
    // gather -> reduce_sum -> LU tail (runtime.py:209-219)
    std::vector<double> fw((size_t)p);
    for (int32_t w = 0; w < p; ++w) fw[(size_t)w] = run.row_wit[(size_t)rem_rows[(size_t)w]];
    double total = 0.0;
    for (int32_t w = 0; w < p; ++w) total += local_logs[(size_t)w];
    int32_t rs = 0;
    double rl = 0.0;
    logdet_lu_host(rem, p, fw, &rs, &rl);
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

}  // namespace
}  // namespace mcnd

using namespace mcnd;

extern "C" {

int mcnd_logdet_condensation_dev(const double* d_a, int64_t n, int64_t lda, const int64_t* pivot_sequence,
                                 int64_t pivot_sequence_len, uint32_t flags, void* stream, mcnd_logdet* out,
                                 double* pivots_out, int32_t* cols_out) {
    if (!out) return fail(MCND_EINVAL, "null out");
    std::lock_guard<std::mutex> lk(g_mu);
    return serial_dev(d_a, n, lda, pivot_sequence, pivot_sequence_len, flags, (cudaStream_t)stream, out,
                      pivots_out, cols_out);
}

int mcnd_logdet_condensation(const double* h_a, int64_t n, int64_t lda, const int64_t* pivot_sequence,
                             int64_t pivot_sequence_len, uint32_t flags, void* stream, mcnd_logdet* out,
                             double* pivots_out, int32_t* cols_out) {
    if (!out) return fail(MCND_EINVAL, "null out");
    int rc = check_shape(h_a, n, lda);
    if (rc) return rc;
    std::lock_guard<std::mutex> lk(g_mu);
    int code = MCND_OK;
    Buffers* B = buffers_for_current(&code);
    if (!B) return code;
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
    std::lock_guard<std::mutex> lk(g_mu);
    return parallel_dev(d_a, n, lda, p, flags, (cudaStream_t)stream, out, stats, payload_entries, row_updates,
                        owners_out);
}

int mcnd_mc_parallel(const double* h_a, int64_t n, int64_t lda, int32_t p, uint32_t flags, void* stream,
                     mcnd_logdet* out, mcnd_comm_stats* stats, int64_t* payload_entries, int64_t* row_updates,
                     int32_t* owners_out) {
    if (!out) return fail(MCND_EINVAL, "null out");
    int rc = check_shape(h_a, n, lda);
    if (rc) return rc;
    std::lock_guard<std::mutex> lk(g_mu);
    int code = MCND_OK;
    Buffers* B = buffers_for_current(&code);
    if (!B) return code;
    const double* d_a = nullptr;
    rc = stage_input(*B, h_a, n, n, lda, (cudaStream_t)stream, &d_a);
    if (rc) return rc;
    return parallel_dev(d_a, n, n, p, flags, (cudaStream_t)stream, out, stats, payload_entries, row_updates,
                        owners_out);
}

int mcnd_logdet_batched_dev(const double* d_a, int64_t batch, int64_t n, int64_t stride, uint32_t flags,
                            void* stream, int32_t* d_sign, double* d_log_abs, double* d_pivots) {
    if (batch < 0 || n < 1 || n > 128) return fail(MCND_EINVAL, "batched kernel needs 1 <= n <= 128 (got %lld)", (long long)n);
    if (stride < n * n) return fail(MCND_EINVAL, "stride < n*n");
    if (batch > 0 && (!d_a || !d_sign || !d_log_abs)) return fail(MCND_EINVAL, "null pointer");
    cudaError_t e = k3_launch(d_a, batch, n, stride, (flags & MCND_FLAG_FAST) != 0, d_sign, d_log_abs, d_pivots,
                              (cudaStream_t)stream);
    if (e != cudaSuccess) return fail(MCND_ECUDA, "batched kernel: %s", cudaGetErrorString(e));
    return MCND_OK;
}

int mcnd_logdet_batched(const double* h_a, int64_t batch, int64_t n, int64_t stride, uint32_t flags, void* stream,
                        int32_t* h_sign, double* h_log_abs) {
    if (batch < 0 || n < 1 || n > 128) return fail(MCND_EINVAL, "batched kernel needs 1 <= n <= 128 (got %lld)", (long long)n);
    if (stride < n * n) return fail(MCND_EINVAL, "stride < n*n");
    if (batch == 0) return MCND_OK;
    std::lock_guard<std::mutex> lk(g_mu);
    int code = MCND_OK;
    Buffers* B = buffers_for_current(&code);
    if (!B) return code;
    cudaStream_t st = (cudaStream_t)stream;
    const size_t in_bytes = (size_t)batch * stride * sizeof(double);
    const size_t out_bytes = align_up((size_t)batch * sizeof(double), 256) + (size_t)batch * sizeof(int32_t);
    int rc = ensure_dev(&B->din, &B->din_bytes, in_bytes);
    if (rc) return rc;
    rc = ensure_dev(&B->dws, &B->dws_bytes, out_bytes);
    if (rc) return rc;
    double* d_log = (double*)B->dws;
    int32_t* d_sign = (int32_t*)((char*)B->dws + align_up((size_t)batch * sizeof(double), 256));
    CUDA_TRY(cudaMemcpyAsync(B->din, h_a, in_bytes, cudaMemcpyHostToDevice, st));
    cudaError_t e = k3_launch((const double*)B->din, batch, n, stride, (flags & MCND_FLAG_FAST) != 0, d_sign, d_log,
                              nullptr, st);
    if (e != cudaSuccess) return fail(MCND_ECUDA, "batched kernel: %s", cudaGetErrorString(e));
    CUDA_TRY(cudaMemcpyAsync(h_log_abs, d_log, (size_t)batch * sizeof(double), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(h_sign, d_sign, (size_t)batch * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    return MCND_OK;
}

const char* mcnd_last_error(void) { return g_err.c_str(); }

int32_t mcnd_version(void) { return 100; }

int32_t mcnd_k1_grid(void) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    return k1_max_grid(dev);
}

void mcnd_release_workspace(void) {
    std::lock_guard<std::mutex> lk(g_mu);
    for (auto& b : g_bufs) {
        int cur = 0;
        cudaGetDevice(&cur);
        cudaSetDevice(b.device);
        if (b.dws) cudaFree(b.dws);
        if (b.din) cudaFree(b.din);
        if (b.hpin) cudaFreeHost(b.hpin);
        if (b.ev0) cudaEventDestroy(b.ev0);
        if (b.ev1) cudaEventDestroy(b.ev1);
        cudaSetDevice(cur);
    }
    g_bufs.clear();
}

}  // extern "C"

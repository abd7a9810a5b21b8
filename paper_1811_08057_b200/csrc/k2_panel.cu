// K2 panel factorisation, column-distributed and shared-memory resident.
//
// The b = 64 panel rows x m active columns are split by COLUMN chunks over G
// co-resident CTAs (one per SM, cooperative launch); each CTA keeps its
// 64 x cw chunk in shared memory for the whole panel.  Per pivot s (the
// reference's rule, condense.py:82-131, applied to panel row s):
//
//   1. every CTA publishes its chunk's argmax of row s (ties -> lowest column)
//      with that column's 64 values and its running |.| max of row s; the owner
//      of the last active column also publishes that column.  Every value
//      travels in a 16-byte {value, tag} record written with one store, so the
//      readers simply poll the records: no fences, no arrival counters;
//   2. every CTA reduces the G proposals identically -> (v, l), witness test
//      (condense.py:90), then fetches the winner's column and the last column;
//   3. every CTA applies the step to its chunk: column exchange l <- m_s-1 on
//      ALL 64 rows (finished rows stay in the current layout), row s scaled by
//      true division (its u_s), rows > s get the rank-1 update with the two
//      roundings of condense.py:118 and their running maxima; the threads of
//      row s+1 produce the next candidate on the fly.
//
// Because finished rows follow every column exchange, the winner column of
// step s also carries T[t][s] = u_t(p_s) for t < s, and at the end the chunk
// holds U in the FINAL layout.  Column s of T^{-1} is formed as soon as column s
// of T arrives (off the critical path, one row per thread), so W = T^{-1} U at the
// end is a register-blocked product written straight to global.  CTA 0 derives the panel-start column
// of each pivot and the <= b moved columns for the trailing-row gather.
#include <algorithm>
#include <cstdint>
#include <climits>
#include "mcnd_internal.h"
#include "k2_pair_prep.cuh"

namespace mcnd {
namespace {

constexpr int kB = kK2B;
#ifndef KP_THREADS
#define KP_THREADS 512
#endif
constexpr int kThreads = KP_THREADS;
constexpr int kTPR = kThreads / kK2B;  // threads per panel row in the load pass (8 or 16)
constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ bool beats(double av, int ai, double bv, int bi) {
    const double fa = fabs(av), fb = fabs(bv);
    return fa > fb || (fa == fb && ai < bi);
}

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Record = two 8-byte words {tag:16 | aux:16 | hi32(value)}, {tag:16 | aux:16 | lo32(value)}
// written with ONE 16-byte store and polled with relaxed gpu-scope loads.  Each 8-byte
// word is single-copy atomic on its own, so a reader that finds the wanted tag in BOTH
// words holds the value and aux of that store -- whatever the atomicity of the 16-byte
// access as a whole.  A torn read (one word of this store, one stale) shows a tag
// mismatch in one word, is counted and re-polled: deterministic, no hash.  A slot's tag
// (the pivot's global step + 1, < 65535: n <= kKPMaxCw * kKPMaxG) is unique within a call
// and the slots are cleared per call.  aux carries a candidate position (< 2^16 - 1).
using Rec = ulonglong2;
__device__ __forceinline__ Rec pack(double v, unsigned tag, int aux) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    const unsigned a16 = (aux == INT_MAX) ? 0xffffu : ((unsigned)aux & 0xffffu);
    const unsigned long long hdr = ((unsigned long long)(tag & 0xffffu) << 48) | ((unsigned long long)a16 << 32);
    return make_ulonglong2(hdr | (b >> 32), hdr | (b & 0xffffffffull));
}
__device__ __forceinline__ double val_of(Rec r) {
    return __longlong_as_double((long long)(((r.x & 0xffffffffull) << 32) | (r.y & 0xffffffffull)));
}
// Candidate record: word 0's aux = the candidate position, word 1's aux = a power-of-two
// upper bound of the CTA's running max of the pivot row (its biased exponent + 1), so the
// witness test (condense.py:90) needs no second record on the critical path: |v| above
// 1e-12 x the bound proves the pivot regular; otherwise (only near singularity) the exact
// maxima are read from the WREC records.
__device__ __forceinline__ Rec pack_cand(double v, unsigned tag, int pos, double rowmax) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    const unsigned a16 = (pos == INT_MAX) ? 0xffffu : ((unsigned)pos & 0xffffu);
    const unsigned e16 = (unsigned)((unsigned long long)__double_as_longlong(rowmax) >> 52) & 0x7ffu;
    const unsigned long long t = (unsigned long long)(tag & 0xffffu) << 48;
    return make_ulonglong2(t | ((unsigned long long)a16 << 32) | (b >> 32),
                           t | ((unsigned long long)e16 << 32) | (b & 0xffffffffull));
}
__device__ __forceinline__ unsigned rowmax_exp_of(Rec r) { return (unsigned)(r.y >> 32) & 0xffffu; }
// 2^(e - 1022) > every double with biased exponent e (e = 0: 2^-1022 bounds the subnormals)
__device__ __forceinline__ double exp_bound(unsigned e) {
    return __longlong_as_double((long long)((unsigned long long)(e + 1u) << 52));
}
__device__ __forceinline__ unsigned tag_of(Rec r) { return (unsigned)(r.x >> 48); }
__device__ __forceinline__ int aux_of(Rec r) {
    const unsigned a16 = (unsigned)(r.x >> 32) & 0xffffu;
    return a16 == 0xffffu ? INT_MAX : (int)a16;
}
__device__ __forceinline__ bool rec_ok(Rec r, unsigned tag, unsigned* torn) {
    const unsigned t = tag & 0xffffu;
    const bool a = (unsigned)(r.x >> 48) == t, b = (unsigned)(r.y >> 48) == t;
    if (a && b) return true;
    if (a != b) atomicAdd(torn, 1u);  // one word of this store, one stale: re-polled
    return false;
}
// Record traffic goes through L2 with relaxed gpu-scope accesses.  The polling loads
// MUST be asm volatile: a plain __ldcg in a spin loop may legally be hoisted by the
// compiler (it was, depending on the surrounding code), hanging the panel.
__device__ __forceinline__ void put(Rec* p, Rec v) {
    asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(v.x), "l"(v.y) : "memory");
}
__device__ __forceinline__ Rec get(const Rec* p) {
    Rec v;
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ Rec get1(const Rec* p) { return __ldcg(p); }  // one-shot read (never in a spin loop)

// x / v correctly rounded (= __ddiv_rn) from r = RN(1/v): q0 = RN(x r), e = x - q0 v (exact,
// one FMA), q = RN(q0 + e r) (Markstein's final step; exact for operands whose quotient and
// residual stay in the normal range, guaranteed here by |x|, |v| in [2^-500, 2^500)); three
// dependent FP64 operations instead of the division's iteration.  Other operands: IEEE division.
__device__ __forceinline__ double div_rn_rcp(double x, double v, double r) {
    const unsigned ex = (unsigned)(((unsigned long long)__double_as_longlong(x) >> 52) & 0x7ffu);
    const unsigned ev = (unsigned)(((unsigned long long)__double_as_longlong(v) >> 52) & 0x7ffu);
    if (ex - 523u < 1000u && ev - 523u < 1000u) {
        const double q0 = __dmul_rn(x, r);
        const double e = __fma_rn(-q0, v, x);
        return __fma_rn(e, r, q0);
    }
    return __ddiv_rn(x, v);
}

// Exact warp max of non-negative 64-bit patterns (|double| bits order like the values).
__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
    const unsigned hi = (unsigned)(v >> 32), lo = (unsigned)v;
    const unsigned mh = __reduce_max_sync(kFull, hi);
    const unsigned ml = __reduce_max_sync(kFull, hi == mh ? lo : 0u);
    return ((unsigned long long)mh << 32) | ml;
}
__device__ __forceinline__ unsigned long long abs_bits(double x) {
    return (unsigned long long)__double_as_longlong(x) & 0x7fffffffffffffffull;
}


// Race stress (test builds only: MCND_BUILD_DEFINES="MCND_JITTER=1"): pseudo-random sleeps of up
// to ~2 us at the protocol's hand-off points, so a read that is not properly ordered after its
// write would see stale data (wrong pivots) or time out.  The parity tests then run unchanged.
#ifndef MCND_JITTER
#define MCND_JITTER 0
#endif
__device__ __forceinline__ void jitter(unsigned salt) {
#if MCND_JITTER
    unsigned long long c;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
    unsigned x = (unsigned)c * 2654435761u ^ (blockIdx.x * 40503u + threadIdx.x * 9176u + salt * 7919u);
    x ^= x >> 15; x *= 2246822519u; x ^= x >> 13;
    if ((x & 7u) == 0u) __nanosleep(x % 2048u);
#else
    (void)salt;
#endif
}

// Span log of the panel launches (CTA 0: globaltimer at entry and exit), read by
// mcnd_debug_kp_spans() for schedule analysis; two stores per panel.
__device__ unsigned long long g_kp_span[4096][2];
__device__ unsigned g_kp_span_n;

#ifndef KP_TRACE
#define KP_TRACE 0  // microbenchmark knob: record per-step phase timestamps of CTA 0
#endif
#if KP_TRACE
__device__ unsigned long long g_kp_trace[64][16];
__device__ unsigned long long g_kp_gt[64][kKPMaxG][4];  // per CTA (globaltimer): poll done, fetch done, published
#define KP_GT(s, k) do { if (threadIdx.x == 0) g_kp_gt[s][blockIdx.x][k] = globaltimer(); } while (0)
#define KP_MARK(s, k) do { if (blockIdx.x == 0 && threadIdx.x == 0) g_kp_trace[s][k] = clock64(); } while (0)
#define KP_MARKT(s, k, t) do { if (blockIdx.x == 0 && threadIdx.x == (t)) g_kp_trace[s][k] = clock64(); } while (0)
#else
#define KP_MARKT(s, k, t) do { } while (0)
#define KP_MARK(s, k) do { } while (0)
#define KP_GT(s, k) do { } while (0)
#endif

// KPER: candidate records per lane of the reducing warp (G <= 32 * KPER).  One launch runs
// `halves` panels: the first of a pair and -- halves = 2 -- the second one (p1: its r1
// prologue applies the first panel's update, its epilogue the pair prep) on the same CTAs
// and column chunks, one grid barrier between them: no second launch (it waited ~11 us per
// pair for SMs the overlapped GEMM had taken), the second panel's rows load meanwhile.
template <int KPER>
__global__ void __launch_bounds__(kThreads, 1) kp_panel_kernel(const KPParams p0, const KPParams p1, const int halves) {
    extern __shared__ __align__(16) double S[];  // [kB][cw]
    __shared__ double sTi[kB][kB + 1];  // T^{-1}, built one column per step
    __shared__ double s_mult2[2][kB], s_last2[2][kB];  // by step parity: warp 0 fetches step s
                                                       // while the bulk of step s-1 still reads
    __shared__ double s_rmax[kB], s_rmax2[kB];
    __shared__ double s_wit0[kB];  // witnesses the panel rows carry in (constant during the panel)
    __shared__ double s_lv[8], s_lm[8];
    __shared__ int s_li[8];
    __shared__ int s_l[kB];
    __shared__ double s_cv, s_win_v, s_win_w, s_win_r;
    __shared__ int s_cpos, s_win_l, s_win_g, s_stop;
    __shared__ PairPrepSmem s_pp;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    bool bail = false;  // singular / protocol stop: no second half
    for (int half = 0; half < halves; ++half) {
        const KPParams& p = half ? p1 : p0;
        const int g = blockIdx.x, G = p.G, cw = p.cw, m = p.m;
        const int lo = g * cw;
        const int wc = max(0, min(cw, m - lo));  // my columns at panel start
        const unsigned long long t_start = globaltimer();
        KP_MARK(0, 8);
        unsigned span_slot = 0;
        if (g == 0 && tid == 0) {
            span_slot = atomicAdd(&g_kp_span_n, 1u) & 4095u;
            g_kp_span[span_slot][0] = t_start;
        }
        if (*(volatile const unsigned*)p.abort) return;  // uniform: set only by earlier launches
        // Record slots: [step][CTA] history in global memory (L2), reused by every panel
        // (the tags tell the panels apart)
        auto CAND = [&](int s, int h) -> Rec* { return p.cand + s * G + h; };
        auto WREC = [&](int s, int h) -> Rec* { return p.wrec + s * G + h; };
        auto LAST = [&](int s, int r) -> Rec* { return p.lastbuf + s * kB + r; };
        auto COL = [&](int s, int h, int r) -> Rec* { return p.colbuf + ((int64_t)s * G + h) * kB + r; };

        // ---- load my chunk of the 64 panel rows; running max per row; candidate of row 0
        for (int r = warp; r < kB; r += kThreads / 32) {  // row per warp, 16-byte loads (ld, lo, cw even)
            const double* src = p.ws + (int64_t)(p.row0 + r) * p.ld + lo;
            for (int c = 2 * lane; c < wc; c += 64) {
                if (c + 1 < wc) {
                    const unsigned d = (unsigned)__cvta_generic_to_shared(S + r * cw + c);
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src + c) : "memory");
                } else {
                    S[r * cw + c] = __ldcg(src + c);
                }
            }
        }
        for (int e = tid; e < kB * (kB + 1); e += kThreads) {
            const int t = e / (kB + 1), j = e - t * (kB + 1);
            sTi[t][j] = (t == j) ? 1.0 : 0.0;
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        if (tid == 0) s_stop = 0;
        if (tid < kB) s_wit0[tid] = p.wit[p.row0 + tid];
        if (g == 0 && tid == 0) p.pan->n_moved = 0;
        __syncthreads();
        if (half > 0) {
            // every CTA through the first panel (its W columns, CTA 0's descriptor) before the
            // second reads them; this CTA's own rows were loaded above, meanwhile
            if (tid == 0) {
                __threadfence();
                atomicAdd(p.half_bar, 1u);
                unsigned v;
                for (;;) {
                    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p.half_bar) : "memory");
                    if (v >= (unsigned)G) break;
                    if (globaltimer() - t_start > p.timeout_ns) {
                        atomicExch(&p.err->error, 1u);
                        atomicExch(&p.err->err_step, (unsigned)p.row0);
                        s_stop = 1;
                        break;
                    }
                }
            }
            __syncthreads();
            if (s_stop) return;
        }
        if (p.r1_g0) {
            // ---- the pair's first panel applied to these rows (replaces the gather + GEMM
            //      launches): NL = -A[rows, P0] (staged in sTi's storage), the moved columns,
            //      then S += NL * W0 with the GEMM's k order (bitwise the DMMA update)
            const K2Gather* g0 = p.r1_g0;
            for (int e = tid; e < kB * kB; e += kThreads) {
                const int r = e >> 6, k = e & 63;
                sTi[r][k] = -__ldcg(p.ws + (int64_t)(p.row0 + r) * p.ld + __ldg(&g0->P[k]));
            }
            const int nm = __ldg(&g0->n_moved);
            for (int e = tid; e < kB * nm; e += kThreads) {
                const int r = e / nm, j = e - r * nm;
                const int c = __ldg(&g0->moved_c[j]);
                if (c >= lo && c < lo + wc)
                    S[r * cw + (c - lo)] = __ldcg(p.ws + (int64_t)(p.row0 + r) * p.ld + __ldg(&g0->moved_src[j]));
            }
            __syncthreads();
            const double* W0 = p.r1_W + lo;
            {
                // on the FP64 tensor cores (mma.sync.m8n8k4.f64, k ascending: the trailing GEMM's
                // arithmetic): warp w owns the 8-column tiles w, w + 16, ... (two at a time) for
                // all 64 rows, so every W0 element is read from L2 once per CTA
                const int gq = lane >> 2, qq = lane & 3;
                const int ntiles = (wc + 7) >> 3;
                constexpr int kNW = kThreads / 32;
                for (int tp = warp; tp < ntiles; tp += 2 * kNW) {
                    const int tl[2] = {tp, tp + kNW};
                    double acc[8][2][2];
    #pragma unroll
                    for (int i = 0; i < 8; ++i)
    #pragma unroll
                        for (int t = 0; t < 2; ++t) {
                            const int c = tl[t] * 8 + 2 * qq;
                            const double* sp = S + (8 * i + gq) * cw + c;
                            acc[i][t][0] = (c < wc) ? sp[0] : 0.0;
                            acc[i][t][1] = (c + 1 < wc) ? sp[1] : 0.0;
                        }
                    constexpr int kPF = 4;  // W0 k-steps in a register ring
                    double bq[kPF][2];
    #pragma unroll
                    for (int s4 = 0; s4 < kPF; ++s4)
    #pragma unroll
                        for (int t = 0; t < 2; ++t) {
                            const int c = tl[t] * 8 + gq;
                            bq[s4][t] = (c < wc) ? __ldg(W0 + (int64_t)(4 * s4 + qq) * p.r1_ldw + c) : 0.0;
                        }
                    for (int k0 = 0; k0 < kB; k0 += 4 * kPF) {
    #pragma unroll
                        for (int s4 = 0; s4 < kPF; ++s4) {
                            const int k = k0 + 4 * s4;
    #pragma unroll
                            for (int i = 0; i < 8; ++i) {
                                const double av = sTi[8 * i + gq][k + qq];
    #pragma unroll
                                for (int t = 0; t < 2; ++t)
                                    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                                        : "+d"(acc[i][t][0]), "+d"(acc[i][t][1]) : "d"(av), "d"(bq[s4][t]));
                            }
                            if (k + 4 * kPF < kB) {
    #pragma unroll
                                for (int t = 0; t < 2; ++t) {
                                    const int c = tl[t] * 8 + gq;
                                    bq[s4][t] = (c < wc) ? __ldg(W0 + (int64_t)(k + 4 * kPF + qq) * p.r1_ldw + c) : 0.0;
                                }
                            }
                        }
                    }
    #pragma unroll
                    for (int i = 0; i < 8; ++i)
    #pragma unroll
                        for (int t = 0; t < 2; ++t) {
                            const int c = tl[t] * 8 + 2 * qq;
                            double* const sp = S + (8 * i + gq) * cw + c;
                            if (c < wc) sp[0] = acc[i][t][0];
                            if (c + 1 < wc) sp[1] = acc[i][t][1];
                        }
                }
            }
            __syncthreads();
            for (int e = tid; e < kB * (kB + 1); e += kThreads) {
                const int t = e / (kB + 1), j = e - t * (kB + 1);
                sTi[t][j] = (t == j) ? 1.0 : 0.0;
            }
            __syncthreads();
        }
        {
            const int r = tid / kTPR, j = tid % kTPR;  // 64 rows x kTPR threads
            const unsigned hm = ((1u << kTPR) - 1u) << (lane & (32 - kTPR));
            double mx = 0.0, bv = 0.0;
            int bi = INT_MAX;
            for (int c = j; c < wc; c += kTPR) {
                const double x = S[r * cw + c];
                mx = fmax(mx, fabs(x));
                if (r == 0 && beats(x, lo + c, bv, bi)) { bv = x; bi = lo + c; }
            }
    #pragma unroll
            for (int o = kTPR / 2; o; o >>= 1) {
                mx = fmax(mx, __shfl_xor_sync(hm, mx, o));
                const double ov = __shfl_xor_sync(hm, bv, o);
                const int oi = __shfl_xor_sync(hm, bi, o);
                if (beats(ov, oi, bv, bi)) { bv = ov; bi = oi; }
            }
            if (j == 0) { s_rmax[r] = mx; s_rmax2[r] = 0.0; }
            if (r == 0 && j == 0) { s_cv = bv; s_cpos = bi; }
        }
        __syncthreads();

        // ---- publish the proposal for pivot 0 (row 0's candidate from the load pass)
        if (tid < kB) {
            const int pos = s_cpos;
            put(COL(0, g, tid), pack(pos != INT_MAX ? S[tid * cw + (pos - lo)] : 0.0, p.tag0, 0));
            if (lo <= m - 1 && m - 1 < lo + wc) put(LAST(0, tid), pack(S[tid * cw + (m - 1 - lo)], p.tag0, 0));
            if (tid == 0) put(CAND(0, g), pack_cand(s_cv, p.tag0, pos, s_rmax[0]));
            if (tid == 1) put(WREC(0, g), pack(s_rmax[0], p.tag0, 0));
        }

        KP_MARK(0, 9);
        // E's per-lane running maxima of its rows (row ew + 14k in slot k), kept across steps
        constexpr int kEWarps = (kThreads - 64) / 32;                  // bulk warps
        constexpr int kERows = (kB + kEWarps - 1) / kEWarps;          // rows per bulk warp
        unsigned long long emax[kERows];
    #pragma unroll
        for (int k = 0; k < kERows; ++k) emax[k] = 0ull;
        for (int s = 0; s < kB; ++s) {
            const int ms = m - s;  // active width before pivot s
            const unsigned tag = p.tag0 + (unsigned)s;
            double* const s_mult = s_mult2[s & 1];
            double* const s_last = s_last2[s & 1];
            KP_MARK(s, 0);
            // ---- A. reduce the G proposals for pivot s: warp 0 polls all tagged records
            if (warp == 0) {
                constexpr int kPer = KPER;
                Rec c[kPer];
                unsigned need = 0;  // bit k: record lane + 32k still missing
    #pragma unroll
                for (int k = 0; k < kPer; ++k)
                    if (lane + 32 * k < G) need |= 1u << k;
                jitter(3u);
                for (unsigned it = 0;; ++it) {
    #pragma unroll
                    for (int k = 0; k < kPer; ++k)
                        if (need & (1u << k)) c[k] = get(CAND(s, lane + 32 * k));
    #pragma unroll
                    for (int k = 0; k < kPer; ++k)
                        if ((need & (1u << k)) && rec_ok(c[k], tag, &p.err->torn))
                            need &= ~(1u << k);
                    if (__all_sync(kFull, need == 0)) break;
                    if ((it & 7u) == 7u && globaltimer() - t_start > p.timeout_ns) {
    #ifdef KP_DEBUG
                        for (int k = 0; k < kPer; ++k)
                            if (need & (1u << k))
                                printf("KP timeout A: g=%d s=%d row0=%d m=%d G=%d cw=%d waiting rec %d: cand tag %x wrec tag %x want %x\n",
                                       g, s, p.row0, m, G, cw, lane + 32 * k, tag_of(c[k]), tag_of(w[k]), tag);
    #endif
                        {
                            const unsigned nb = __ballot_sync(kFull, need != 0);
                            if (lane == (int)(__ffs(nb) - 1) && atomicCAS(&p.err->dbg[0], 0u, 1u) == 0u) {
                                const int k = __ffs(need) - 1;
                                unsigned t4 = 0u, t5 = 0u;  // static indexing only: keeps c/w in registers
    #pragma unroll
                                for (int kk = 0; kk < kPer; ++kk)
                                    if (kk == k) { t4 = tag_of(c[kk]); t5 = 0u; }
                                p.err->dbg[1] = (unsigned)g; p.err->dbg[2] = (unsigned)s; p.err->dbg[3] = (unsigned)(lane + 32 * k);
                                p.err->dbg[4] = t4; p.err->dbg[5] = t5; p.err->dbg[6] = tag;
                                p.err->dbg[7] = (unsigned)G;
                            }
                        }
                        if (lane == 0) {
                            atomicExch(&p.err->error, 1u);
                            atomicExch(&p.err->err_step, (unsigned)(p.row0 + s));
                            s_stop = 1;
                        }
                        break;
                    }
                }
                if (s > 0) KP_MARK(s, 8);
                KP_GT(s, 0);
                // exact argmax of |value| (ties -> lowest column) and the bound of the running row
                // maxima: per-lane scan, then redux on the 64-bit |x| patterns
                unsigned long long kb = 0ull;
                unsigned eb = 0u;
                int bi = INT_MAX, bg = 0;
                double bv = 0.0;
    #pragma unroll
                for (int k = 0; k < kPer; ++k) {
                    const int h = lane + 32 * k;
                    if (h < G) {
                        const double xv = val_of(c[k]);
                        const unsigned long long xb = abs_bits(xv);
                        const int xi = aux_of(c[k]);
                        if (xb > kb || (xb == kb && xi < bi)) { kb = xb; bi = xi; bv = xv; bg = h; }
                        eb = max(eb, rowmax_exp_of(c[k]));
                    }
                }
                const unsigned long long mb = warp_max_u64(kb);
                const unsigned wi = __reduce_min_sync(kFull, kb == mb ? (unsigned)bi : 0xffffffffu);
                const int src = __ffs(__ballot_sync(kFull, kb == mb && (unsigned)bi == wi)) - 1;
                bv = __shfl_sync(kFull, bv, src);
                bi = __shfl_sync(kFull, bi, src);
                bg = __shfl_sync(kFull, bg, src);
                double bw = fmax(exp_bound(__reduce_max_sync(kFull, eb)), s_wit0[s]);
                double rcp = 0.0;
                if (!(fabs(bv) > kSingularRtol * bw)) {
                    // near-singular: the exact running maxima decide (condense.py:90)
                    unsigned long long wb = 0ull;
    #pragma unroll
                    for (int k = 0; k < kPer; ++k) {
                        const int h = lane + 32 * k;
                        if (h >= G) continue;
                        Rec w = get(WREC(s, h));
                        while (!rec_ok(w, tag, &p.err->torn) && globaltimer() - t_start <= p.timeout_ns) w = get(WREC(s, h));
                        wb = max(wb, abs_bits(val_of(w)));
                    }
                    bw = fmax(__longlong_as_double((long long)warp_max_u64(wb)), s_wit0[s]);
                }
                // the winner's column (multipliers of rows > s, T entries of rows < s) and the
                // last active column: fetched right here by warp 0, two rows per lane
                if (s > 0) KP_MARK(s, 9);
                if (fabs(bv) > kSingularRtol * bw) {
                    // all four records in flight at once (one round trip); first a plain L2 read
                    // (usually already there), strong re-polls only for what had not arrived
                    Rec cm[2], cl[2];
    #pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        cm[h] = get1(COL(s, bg, lane + 32 * h));
                        cl[h] = get1(LAST(s, lane + 32 * h));
                    }
                    rcp = __drcp_rn(bv);  // while the fetch is in flight
    #pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int r = lane + 32 * h;
                        while (!rec_ok(cm[h], tag, &p.err->torn) || !rec_ok(cl[h], tag, &p.err->torn)) {
                            if (globaltimer() - t_start > p.timeout_ns) {
    #ifdef KP_DEBUG
                                printf("KP timeout col: g=%d s=%d row0=%d m=%d G=%d r=%d bg=%d bi=%d coltag %x lasttag %x want %x\n",
                                       g, s, p.row0, m, G, r, bg, bi, tag_of(cm[h]), tag_of(cl[h]), tag);
    #endif
                                if (atomicCAS(&p.err->dbg[0], 0u, 2u) == 0u) {
                                    p.err->dbg[1] = (unsigned)g; p.err->dbg[2] = (unsigned)s; p.err->dbg[3] = (unsigned)bg;
                                    p.err->dbg[4] = tag_of(cm[h]); p.err->dbg[5] = tag_of(cl[h]); p.err->dbg[6] = tag;
                                    p.err->dbg[7] = (unsigned)r;
                                }
                                atomicExch(&p.err->error, 1u);
                                atomicExch(&p.err->err_step, (unsigned)(p.row0 + s));
                                s_stop = 1;
                                break;
                            }
                            cm[h] = get(COL(s, bg, r));
                            cl[h] = get(LAST(s, r));
                        }
                        s_mult[r] = val_of(cm[h]);
                        s_last[r] = val_of(cl[h]);
                    }
                }
                if (s > 0) KP_MARK(s, 10);
                KP_GT(s, 1);
                if (lane == 0) {
                    s_win_r = rcp;
                    s_win_v = bv;
                    s_win_l = bi;
                    s_win_g = bg;
                    s_win_w = bw;
                }
            }
            __syncthreads();
            KP_MARK(s, 1);
            if (s_stop) { bail = true; goto finish; }
            const double v = s_win_v;
            const int l = s_win_l;
            if (!(fabs(v) > kSingularRtol * s_win_w)) {  // condense.py:90 -> singular
                if (g == 0 && tid == 0) {
                    p.rec[s].v = v;
                    p.rec[s].l = -1;
                    p.rec[s].flag = p.epoch;
                    atomicExch(p.abort, 1u);
                }
                bail = true;
                goto finish;
            }
            const int wn = max(0, min(wc, ms - 1 - lo));  // my active columns after the step
            KP_MARK(s, 7);
            // ---- B+D1. warps 0-7: row s scaled by true division (condense.py:110) with the
            //      column exchange (condense.py:104-107) folded in, and -- lookahead -- row s+1
            //      updated from it, its running max and the next candidate, published at once.
            //      The next 2 warps meanwhile: the exchange on the other rows, the T^{-1} column, the record.
            constexpr int kLA = 64;   // publishing threads (D2)
    #ifndef KP_D1
    #define KP_D1 256
    #endif
            constexpr int kD1 = KP_D1;  // row s / s+1 threads (<= 256)
            const int lx = (l >= lo && l - lo < wn) ? l - lo : -1;  // exchange target, local
            const bool last_step = (s + 1 == kB);
            const unsigned tag1 = tag + 1u;
            if (tid < kD1) {
                double* const rs = S + s * cw;
                double* const row = S + (s + 1) * cw;
                const double mu = last_step ? 0.0 : s_mult[s + 1];
                const double rv = s_win_r;
                // the row max IS |candidate|: one exact argmax (ties -> lowest column) via redux
                unsigned long long bb = 0ull;
                double bv = 0.0;
                int bi = INT_MAX;
                for (int c = tid; c < wn; c += kD1) {
                    const double q = div_rn_rcp(c == lx ? s_last[s] : rs[c], v, rv);
                    rs[c] = q;
                    if (!last_step) {
                        const double y = __dsub_rn(c == lx ? s_last[s + 1] : row[c], __dmul_rn(mu, q));
                        row[c] = y;
                        const unsigned long long yb = abs_bits(y);
                        if (bi == INT_MAX || yb > bb) { bb = yb; bv = y; bi = lo + c; }
                    }
                }
                KP_MARK(s, 3);
                if (!last_step) {
                    const unsigned long long mb = warp_max_u64(bb);
                    const int wi = (int)__reduce_min_sync(kFull, bb == mb ? (unsigned)bi : 0xffffffffu);
                    if (bb == mb && bi == wi) { s_lv[warp] = bv; s_li[warp] = bi; s_lm[warp] = fabs(bv); }
                    if (lane == 0 && wi == INT_MAX) { s_lv[warp] = 0.0; s_li[warp] = INT_MAX; s_lm[warp] = 0.0; }
                    asm volatile("bar.sync 1, %0;" ::"n"(kD1));
                    KP_MARK(s, 5);
                    // the D1 warps' results combined by warp 0 (exact redux argmax, ties -> lowest column)
                    double v0 = 0.0, m0 = 0.0;
                    int i0 = INT_MAX;
                    if (warp == 0) {
                        const bool has = lane < kD1 / 32;
                        const double lv = has ? s_lv[lane] : 0.0, lm = has ? s_lm[lane] : 0.0;
                        const int li = has ? s_li[lane] : INT_MAX;
                        const unsigned long long kb = (li == INT_MAX) ? 0ull : abs_bits(lv);
                        const unsigned long long mb = warp_max_u64(kb);
                        i0 = (int)__reduce_min_sync(kFull, kb == mb ? (unsigned)li : 0xffffffffu);
                        const int src = __ffs(__ballot_sync(kFull, kb == mb && li == i0)) - 1;
                        v0 = __shfl_sync(kFull, lv, src < 0 ? 0 : src);
                        if (i0 == INT_MAX) v0 = 0.0;
                        m0 = __longlong_as_double((long long)warp_max_u64((unsigned long long)__double_as_longlong(lm)));
                    }
                    if (tid == 0) {
                        s_cv = v0;
                        s_cpos = i0;
                        const double rm = fmax(fmax(s_rmax[s + 1], s_rmax2[s + 1]), m0);
                        s_rmax[s + 1] = rm;
                        // proposal of pivot s+1 goes out now; its column follows in D2
                        jitter(1u);
                        put(WREC(s + 1, g), pack(rm, tag1, 0));
                        put(CAND(s + 1, g), pack_cand(v0, tag1, i0, rm));
                        KP_MARK(s, 6);
                        KP_GT(s + 1, 2);
                    }
                }
            } else if (tid < kD1 + kB) {
                const int r = tid - kD1;
                if (lx >= 0 && r != s && r != s + 1) S[r * cw + lx] = s_last[r];
                if (r < s) {  // T[t][s] = u_t(p_s) (t < s) arrives now: column s of T^{-1}, row r by thread r
                    double acc = 0.0;
                    for (int j = r; j < s; ++j) acc = fma(sTi[r][j], s_mult[j], acc);
                    sTi[r][s] = -acc;
                }
                if (r == 0) {
                    s_l[s] = l;
                    if (g == 0) {
                        p.rec[s].v = v;
                        p.rec[s].l = l;
                        p.rec[s].flag = p.epoch;
                    }
                }
            }
            __syncthreads();
            KP_MARK(s, 2);
            if (last_step) break;
            const double* us = S + s * cw;
            jitter(4u);
            const int pos = s_cpos;                                   // candidate column of pivot s+1
            const int pc = (pos != INT_MAX) ? pos - lo : -1;          // local
            const int lc = (ms - 2 >= lo && ms - 2 - lo < wn) ? ms - 2 - lo : -1;  // new last column, local
            if (tid < kLA) {
                // ---- D2. publish the candidate column of pivot s+1 (one row per thread): rows > s+1 get
                //          columns pc / lc updated here (E skips them); their maxima go to
                //          s_rmax2 (single writer, no atomics)
                const int r = tid;
                const double mu = s_mult[r];
                double* row = S + r * cw;
                double mx = 0.0, xc = 0.0, xl = 0.0;
                if (pc >= 0) {
                    xc = row[pc];
                    if (r > s + 1) { xc = __dsub_rn(xc, __dmul_rn(mu, us[pc])); row[pc] = xc; mx = fabs(xc); }
                }
                if (lc >= 0) {
                    if (lc == pc) xl = xc;
                    else {
                        xl = row[lc];
                        if (r > s + 1) { xl = __dsub_rn(xl, __dmul_rn(mu, us[lc])); row[lc] = xl; mx = fmax(mx, fabs(xl)); }
                    }
                    put(LAST(s + 1, r), pack(xl, tag1, 0));
                }
                jitter(2u);
                put(COL(s + 1, g, r), pack(xc, tag1, 0));
                if (r > s + 1) s_rmax2[r] = fmax(s_rmax2[r], mx);
            } else {
                // ---- E. bulk (warps 2..15): rows > s+1, all columns except pc / lc, with the
                //         reference's two roundings (condense.py:118).  Row r belongs to warp
                //         2 + (r mod 14) for the whole panel, so each lane keeps its running
                //         |.| maximum of the row in a register across steps; the warp folds it
                //         into s_rmax once, at the step after which the row is next (D1 reads
                //         it) -- no per-step reductions or shared atomics.  Each lane does two
                //         adjacent columns per 16-byte access (one unrolled pass of 4 covers 256).
                const int ew = warp - kLA / 32;  // 0..13
    #pragma unroll
                for (int k = 0; k < kERows; ++k) {
                    const int r = ew + kEWarps * k;
                    if (r < s + 2 || r >= kB) continue;  // warp-uniform
                    const double mu = s_mult[r];
                    double* row = S + r * cw;
                    unsigned long long mb = emax[k];
                    auto seg = [&](int c) {  // two adjacent columns, one 16-byte access
                        if (c < wn) {
                            const double2 x = *reinterpret_cast<const double2*>(row + c);
                            const double2 pv = *reinterpret_cast<const double2*>(us + c);
                            double2 y;
                            y.x = __dsub_rn(x.x, __dmul_rn(mu, pv.x));
                            y.y = __dsub_rn(x.y, __dmul_rn(mu, pv.y));  // c+1 may be a dropped column: harmless
                            if (c != pc && c + 1 != pc && c != lc && c + 1 != lc) {
                                *reinterpret_cast<double2*>(row + c) = y;
                                mb = max(mb, max(abs_bits(y.x), c + 1 < wn ? abs_bits(y.y) : 0ull));
                            } else {
                                // pc / lc belong to D2, which is updating them right now: never write
                                // them back (not even unchanged), element-wise stores only
                                if (c != pc && c != lc) { row[c] = y.x; mb = max(mb, abs_bits(y.x)); }
                                if (c + 1 < wn && c + 1 != pc && c + 1 != lc) { row[c + 1] = y.y; mb = max(mb, abs_bits(y.y)); }
                            }
                        }
                    };
    #pragma unroll
                    for (int j = 0; j < 4; ++j) seg(64 * j + 2 * lane);
    #pragma unroll 1
                    for (int j = 4; 64 * j < wn; ++j) seg(64 * j + 2 * lane);  // chunks wider than 256 columns
                    emax[k] = mb;
                }
                // row s+2 is D1's row at the next step: fold its lane maxima now
                const int rn = s + 2;
                if (rn < kB && rn % kEWarps == ew) {
                    unsigned long long v = 0ull;
    #pragma unroll
                    for (int k = 0; k < kERows; ++k)
                        if (ew + kEWarps * k == rn) v = emax[k];
                    v = warp_max_u64(v);
                    if (lane == 0) {
                        unsigned long long* sr = reinterpret_cast<unsigned long long*>(s_rmax) + rn;
                        *sr = max(*sr, v);
                    }
                }
            }
            KP_MARK(s, 4);
            KP_MARKT(s, 12, 64);   // E done, warp 2
            KP_MARKT(s, 13, 480);  // E done, warp 15
            KP_MARKT(s, 14, 32);   // D2 done, warp 1
        }
        __syncthreads();

        KP_MARK(0, 10);
        // ---- W = T^{-1} U on my final columns (T unit upper triangular)
        {
        const int wf = max(0, min(wc, m - kB - lo));
        {
            // W = T^{-1} U on the FP64 tensor cores (mma.sync.m8n8k4.f64; A = T^{-1}, B = U, the
            // chunk itself), straight to global.  Warp w owns the 8-column tiles w, w + 16, ...
            // (two at a time) for all 64 rows; row block mb joins at its diagonal (k0 >= 8 mb):
            // the terms below the diagonal are zero and leave the accumulator at +0, so every
            // element is the FMA chain of the loop below (bitwise, kp_bench W checksums)
            const int gq = lane >> 2, qq = lane & 3;
            const int ntiles = (wf + 7) >> 3;
            constexpr int kNW = kThreads / 32;
            for (int tp = warp; tp < ntiles; tp += 2 * kNW) {
                const int tl[2] = {tp, tp + kNW};
                double acc[8][2][2];
    #pragma unroll
                for (int i = 0; i < 8; ++i)
    #pragma unroll
                    for (int t = 0; t < 2; ++t) { acc[i][t][0] = 0.0; acc[i][t][1] = 0.0; }
    #pragma unroll
                for (int k0 = 0; k0 < kB; k0 += 4) {
                    double bv[2];
    #pragma unroll
                    for (int t = 0; t < 2; ++t) {
                        const int c = tl[t] * 8 + gq;
                        bv[t] = (c < wf) ? S[(k0 + qq) * cw + c] : 0.0;
                    }
    #pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        if (8 * i <= k0 + 3) {  // compile-time after unrolling
                            const double av = sTi[8 * i + gq][k0 + qq];
    #pragma unroll
                            for (int t = 0; t < 2; ++t)
                                asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                                    : "+d"(acc[i][t][0]), "+d"(acc[i][t][1]) : "d"(av), "d"(bv[t]));
                        }
                    }
                }
    #pragma unroll
                for (int i = 0; i < 8; ++i)
    #pragma unroll
                    for (int t = 0; t < 2; ++t) {
                        const int c = tl[t] * 8 + 2 * qq;
                        double* const wr = p.W + (int64_t)(8 * i + gq) * p.ldw + lo + c;
                        if (c + 1 < wf) *reinterpret_cast<double2*>(wr) = make_double2(acc[i][t][0], acc[i][t][1]);
                        else if (c < wf) wr[0] = acc[i][t][0];
                    }
            }
        }
        KP_MARK(1, 11);
        // ---- panel-start column of each pivot and the moved final columns (CTA 0)
        if (g == 0 && tid < kB) {
            const int s = tid;
            int pos = s_l[s];
            for (int j = s - 1; j >= 0; --j) pos = (pos == s_l[j]) ? (m - j - 1) : pos;
            p.pan->P[s] = pos;
            p.pan->l[s] = s_l[s];
            const int c = s_l[s];
            bool first = c < m - kB;
            for (int t = 0; t < s && first; ++t) first = (s_l[t] != c);  // dedupe
            if (first) {
                int q = c;
                for (int t = kB - 1; t >= 0; --t) q = (q == s_l[t]) ? (m - t - 1) : q;
                if (q != c) {
                    const int k = atomicAdd(&p.pan->n_moved, 1);
                    p.pan->moved_c[k] = c;
                    p.pan->moved_src[k] = q;
                }
            }
        }
        if (p.pp_g0 && p.pp_bar) {
            // pair prep spread over every CTA: (a) a slice of Wp[s][s'] = -W_k[s][P1[s']] with
            // P1 derived from this CTA's own pivot list, CTA 0 meanwhile the composite
            // descriptor; one grid barrier (every Wp read of W_k done); (b) a slice of W_k's
            // moved columns, from the descriptor CTA 0 published (k2_pair_prep.cuh, same values)
            __shared__ int s_P1[kB];
            if (tid < kB) {
                int pos = s_l[tid];
                for (int j = tid - 1; j >= 0; --j) pos = (pos == s_l[j]) ? (m - j - 1) : pos;
                s_P1[tid] = pos;
            }
            __syncthreads();
            {
                const int e0 = (int)((int64_t)kB * kB * g / G), e1 = (int)((int64_t)kB * kB * (g + 1) / G);
                for (int e = e0 + tid; e < e1; e += kThreads) {
                    const int sr = e / kB, sp = e % kB;
                    p.pp_Wp[e] = -__ldcg(p.pp_W + (int64_t)sr * p.pp_ldw + s_P1[sp]);  // negated, as pair_prep_body
                }
            }
            if (g == 0) {
                __syncthreads();
                pair_prep_desc<kThreads>(p.pp_g0, p.pan, p.pp_m, p.pp_gpair, s_pp, tid);
            }
            __syncthreads();
            if (tid == 0) {
                __threadfence();
                atomicAdd(p.pp_bar, 1u);
                unsigned v;
                for (;;) {
                    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p.pp_bar) : "memory");
                    if (v >= (unsigned)G) break;
                    if (globaltimer() - t_start > p.timeout_ns) {
                        atomicExch(&p.err->error, 1u);
                        atomicExch(&p.err->err_step, (unsigned)(p.row0 + kB - 1));
                        break;
                    }
                }
            }
            __syncthreads();
            {
                const int nm1 = __ldcg(&p.pan->n_moved), wf2 = p.pp_m - 2 * kB;
                const int tot = kB * nm1;
                const int e0 = (int)((int64_t)tot * g / G), e1 = (int)((int64_t)tot * (g + 1) / G);
                for (int e = e0 + tid; e < e1; e += kThreads) {
                    const int sr = e / nm1, k = e % nm1;
                    const int c = __ldcg(&p.pan->moved_c[k]);
                    if (c < wf2) p.pp_W[(int64_t)sr * p.pp_ldw + c] = __ldcg(p.pp_W + (int64_t)sr * p.pp_ldw + __ldcg(&p.pan->moved_src[k]));
                }
            }
        } else if (p.pp_g0 && g == 0) {  // pair prep right here: this CTA's descriptor is final
            __syncthreads();
            pair_prep_body<kThreads>(p.pp_g0, p.pan, p.pp_m, p.pp_W, p.pp_ldw, p.pp_Wp, p.pp_gpair, s_pp, tid);
        }
        }
        KP_MARK(0, 11);
        if (g == 0 && tid == 0) g_kp_span[span_slot][1] = globaltimer();
finish:;
        if (bail) return;
        __syncthreads();  // the W epilogue's reads of S / sTi / s_l before the next half reloads them
    }
}

}  // namespace

int kp_debug_spans(unsigned long long* out, int max_spans) {
    unsigned n = 0;
    if (cudaMemcpyFromSymbol(&n, g_kp_span_n, sizeof(n)) != cudaSuccess) return -1;
    const int k = (int)std::min<unsigned>(std::min<unsigned>(n, 4096u), (unsigned)max_spans);
    if (k > 0 && cudaMemcpyFromSymbol(out, g_kp_span, (size_t)k * 2 * sizeof(unsigned long long)) != cudaSuccess) return -1;
    const unsigned zero = 0;
    cudaMemcpyToSymbol(g_kp_span_n, &zero, sizeof(zero));
    return k;
}

size_t kp_smem_bytes(int cw) { return (size_t)kB * cw * sizeof(double); }

cudaError_t kp_launch(const KPParams& p, cudaStream_t s, const KPParams* second) {
    const size_t smem = kp_smem_bytes(p.cw);
    if (p.cw < 2 || (p.cw & 1) || p.cw > kKPMaxCw || p.G < 1 || p.G > kKPMaxG) return cudaErrorInvalidValue;
    if (p.tag0 < 1 || p.tag0 + kB >= 0xffffu) return cudaErrorInvalidValue;  // 16-bit record tags
    if (second && (second->G != p.G || second->cw != p.cw || !second->half_bar || second->tag0 + kB >= 0xffffu))
        return cudaErrorInvalidValue;  // the pair runs on the same CTAs and chunks
    const void* fn = p.G <= 32   ? (const void*)kp_panel_kernel<1>
                     : p.G <= 64 ? (const void*)kp_panel_kernel<2>
                     : p.G <= 96 ? (const void*)kp_panel_kernel<3>
                                 : (const void*)kp_panel_kernel<kKPMaxG / 32>;
    // set on every launch: the attribute is per device (context), calls may alternate devices
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    KPParams p0 = p, p1 = second ? *second : p;
    int halves = second ? 2 : 1;
    void* args[] = {&p0, &p1, &halves};
    return cudaLaunchCooperativeKernel(fn, dim3(p.G), dim3(kThreads), args, smem, s);
}

}  // namespace mcnd

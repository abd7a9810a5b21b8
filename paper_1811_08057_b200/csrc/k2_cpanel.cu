// K2 panel factorisation, cluster-resident (thread-block cluster + distributed shared memory).
//
// The column-distributed panel kernel of k2_panel.cu pays two L2 round trips per pivot
// between ~45 CTAs (3.2 us per pivot at C3).  Here the 64 panel rows x m active columns
// live in the shared memory of ONE thread-block cluster (C <= 16 CTAs, m <= C * 400) and the
// 64 pivots are taken in 8 micro-panels of 8 rows:
//
//   * inside a micro-panel the 8 rows live in REGISTERS of 4 "chain" warps (1-3 consecutive
//     columns per thread: lane order = column order).  Per pivot
//     (the reference's rule, condense.py:82-131, on micro-panel row i): warp argmax (redux),
//     CTA argmax, then ONE hop: every CTA sends its {candidate, column, the candidate column's
//     8 entries} (and the owner of the last active column that column's 8 entries) to every
//     CTA of the cluster with st.async (DSMEM stores that complete a transaction count on the
//     receiver's mbarrier); every CTA reduces the C records identically, takes the column
//     exchange (condense.py:104-107) and the update of the 8 rows (condense.py:110-118, the
//     reference's roundings) in registers.  No L2 traffic, no polling.
//   * at the micro-panel boundary the other 56 rows take the 8 pivots at once, in the W form
//     of the trailing update: row <- row o pi - row[P8] * W8 with W8 = T8^{-1} U8.  Finished
//     rows are kept as rows of W (not U), for which the same formula is exactly the block
//     recurrence of W = T^{-1} U -- so finished and future rows take one uniform rank-8 update
//     and the chunk holds the panel's W at the end (no T^{-1}, no epilogue product).  Only the
//     next micro-panel's 8 rows are updated on the critical path; the other 48 follow on the
//     8 non-chain warps while the next micro-panel's chain runs.  The 8 multiplier columns and
//     the 8 topmost columns (the sources of moved columns) cross CTAs through L2 around one
//     cluster barrier, published by a helper warp while the chain runs.
//   * the chunk's rows come in and the W rows go out as bulk copies (cp.async.bulk, the TMA
//     engine); descriptors stay in shared memory, the pair's composite descriptor is built from
//     direct-address column maps in the dead chunk.
//
// Same KPParams, outputs (W, pivot records, gather descriptor, pair prep) and pair launch
// (both panels of a pair in one launch, the second applying the first's update to its rows
// in its prologue) as kp_launch.  The witness test (condense.py:90) uses an upper bound of
// the running row maxima within 2^-20 (their high 32 bits + 1); the blocked path is
// tolerance-parity, its pivot values differ from the reference's in the last bits anyway.
#include <algorithm>
#include <cstdint>
#include <climits>
#include <cstddef>
#include <type_traits>
#include "mcnd_internal.h"

namespace mcnd {
namespace {

constexpr int kB = kK2B;
constexpr int kR = 8;            // micro-panel rows
constexpr int kThreads = 384;  // 4 chain warps + 8 more for the bulk phases; 170 registers per thread
constexpr int kWarps = kThreads / 32;
constexpr unsigned kFull = 0xffffffffu;
constexpr int kRecWords = 10;    // {value, col | maxhi << 32, the candidate column's 8 entries}

#ifndef KC_TRACE
#define KC_TRACE 0
#endif
#if KC_TRACE
__device__ unsigned long long g_kc_trace[64][16];  // per step: phase timestamps of CTA 0 thread 0
__device__ unsigned long long g_kc_tb[8][8];
__device__ unsigned long long g_kc_th[2][16];
#define KC_MARKH(h, k) do { if (blockIdx.x == 0 && threadIdx.x == 0) g_kc_th[h][k] = clock64(); } while (0)
#define KC_MARK(s, k) do { if (blockIdx.x == 0 && threadIdx.x == 0) g_kc_trace[s][k] = clock64(); } while (0)
#define KC_MARKB(j, k) do { if (blockIdx.x == 0 && threadIdx.x == 0) g_kc_tb[j][k] = clock64(); } while (0)
#else
#define KC_MARK(s, k) do { } while (0)
#define KC_MARKB(j, k) do { } while (0)
#define KC_MARKH(h, k) do { } while (0)
#endif

// Span log of the panels (CTA 0: globaltimer at the start and end of every panel), read by
// mcnd_debug_kp_spans() together with the column-distributed kernel's
__device__ unsigned long long g_kc_span[4096][2];
__device__ unsigned g_kc_span_n;

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned long long abs_bits(double x) {
    return (unsigned long long)__double_as_longlong(x) & 0x7fffffffffffffffull;
}
__device__ __forceinline__ unsigned hi_abs(double x) { return (unsigned)(abs_bits(x) >> 32); }

// Race stress (test builds only: MCND_BUILD_DEFINES="MCND_JITTER=1", scripts/race_stress.sh):
// pseudo-random sleeps of up to ~2 us at the hand-off points, so a read that is not properly
// ordered after its write sees stale data (wrong pivots) or times out
#ifndef MCND_JITTER
#define MCND_JITTER 0
#endif
__device__ __forceinline__ void jitter(unsigned salt) {
#if MCND_JITTER
    unsigned long long c;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
    unsigned x = (unsigned)c * 2654435761u ^ (blockIdx.x * 40503u + (threadIdx.x >> 5) * 9176u + salt * 7919u);
    x ^= x >> 15; x *= 2246822519u; x ^= x >> 13;
    if ((x & 7u) == 0u) __nanosleep(x % 2048u);
#else
    (void)salt;
#endif
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t cta) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(cta));
    return r;
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
    return ok != 0;
}
// 16 bytes into a peer CTA's shared memory, completing 16 bytes of its mbarrier's transaction count
__device__ __forceinline__ void st_async_v2(uint32_t raddr, unsigned long long a, unsigned long long b, uint32_t rbar) {
    asm volatile("st.async.weak.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];"
                 ::"r"(raddr), "l"(a), "l"(b), "r"(rbar) : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned cluster_ctarank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

// Shared-memory accesses of the per-pivot path go through explicit ld/st.shared on a base address
// held in a register: in a cluster launch the compiler forms shared addresses from the CTA's rank
// in the cluster (S2R SR_CgaCtaId) and re-reads that special register at every use -- ~100+ cycles
// each, several times per pivot (measured: phases of ~40 instructions took ~400 cycles).
__device__ __forceinline__ uint32_t opaque_u32(uint32_t v) {
    asm volatile("mov.u32 %0, %0;" : "+r"(v));
    return v;
}
__device__ __forceinline__ ulonglong2 lds_v2(uint32_t a) {
    ulonglong2 v;
    asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long lds_u64(uint32_t a) {
    unsigned long long v;
    asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ unsigned lds_u32(uint32_t a) {
    unsigned v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void sts_v2(uint32_t a, unsigned long long x, unsigned long long y) {
    asm volatile("st.shared.v2.u64 [%0], {%1, %2};" ::"r"(a), "l"(x), "l"(y) : "memory");
}
__device__ __forceinline__ void sts_u64(uint32_t a, unsigned long long x) {
    asm volatile("st.shared.u64 [%0], %1;" ::"r"(a), "l"(x) : "memory");
}
__device__ __forceinline__ void sts_u32(uint32_t a, unsigned x) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(x) : "memory");
}
__device__ __forceinline__ unsigned long long d2u(double x) { return (unsigned long long)__double_as_longlong(x); }
__device__ __forceinline__ double u2d(unsigned long long x) { return __longlong_as_double((long long)x); }

struct KCSmem {
    double NL[kB][16 + 4];                       // r1 prologue staging: one k-block of 16 of -A[rows, P0]; +4: conflict-free A fragments
    unsigned long long rcv[2][16][kRecWords];    // per step parity: one record per CTA
    unsigned long long rxl[2][kR];               // per step parity: the last active column's 8 entries
    unsigned long long bar[2];                   // mbarriers (step parity)
    unsigned long long bar_ld;                   // mbarrier of the bulk row load (one phase per panel)
    double L[kB][kR];                            // boundary: the multiplier columns of the other rows
    double T8[kR][kR];                           // micro-panel T (strict upper part)
    ulonglong2 wrec[8];                          // per chain warp: {|candidate| bits, column}
    double wx[8][kR];                            // per chain warp: the candidate column's 8 entries
    double xl[kR];
    unsigned rmaxhi[kB];                         // per row: high word of the chunk's running max |.|
    double wit0[kB];
    int l[kB];
    int P8[kR], mc[kR], ms[kR];
    int bail;
    K2Gather d0, d1;                             // the pair's first descriptor, this panel's
    K2Gather gp;                                 // the pair's composite descriptor
    int cnt[4];
};

constexpr int kChainWarps = 5;  // 160 chain threads x <= 3 columns: chunks up to 480 columns
constexpr int kChainThreads = 32 * kChainWarps;

struct KCChain {
    int g, C, cw, wc, lo, m, dst, part;
    uint32_t r_rcv, r_rxl, r_bar, l_bar, sb;
    unsigned exp_bytes;
    unsigned long long t_start, timeout_ns;
    PivRec* rec;
    unsigned* abort;
    K1Err* err;
    uint32_t epoch;
    int row0;
};

// One micro-panel (rows r0 .. r0+7 of the panel) on the 4 chain warps: thread t owns the columns
// NC t .. NC t + NC - 1 of the chunk, their 8 entries in registers.  At exit the rows'
// slots in the chunk hold W8 = T8^{-1} U8 (the micro-panel's rows of W).
// One micro-panel (rows r0 .. r0+7 of the panel) on the 4 chain warps: thread t owns the columns
// NC t .. NC t + NC - 1 of the chunk, their 8 entries in registers.  At exit the rows'
// slots in the chunk hold W8 = T8^{-1} U8 (the micro-panel's rows of W).  Roles besides the
// common path: warp 0 sends the CTA's record, warp 1 keeps T8, warp 2 runs the witness test and
// writes the pivot records.
template <int NC>
__device__ __forceinline__ void kc_chain(KCSmem& sm, double* __restrict__ S, const KCChain& cc, const int r0,
                                         unsigned& gs, bool& stopped) {
    const int t = (int)opaque_u32(threadIdx.x), lane = t & 31, warp = t >> 5;
    const int cw = cc.cw, lo = cc.lo, m = cc.m, C = cc.C;
    double x[NC][kR];
    int col[NC];
    bool own[NC];
#pragma unroll
    for (int u = 0; u < NC; ++u) {
        // NC CONSECUTIVE columns per thread: lane order = column order, so "ties -> lowest column"
        // is "lowest lane" at every level of the argmax (no conditional tie-break code)
        own[u] = NC * t + u < cc.wc;
        col[u] = lo + NC * t + u;
#pragma unroll
        for (int i = 0; i < kR; ++i) x[u][i] = own[u] ? S[(r0 + i) * cw + NC * t + u] : 0.0;
    }
    // a row's state at its micro-panel start joins its witness (with its state at the panel load;
    // the states in between are not tracked: witnesses only matter near singularity)
#pragma unroll
    for (int i = 0; i < kR; ++i) {
        unsigned h = 0u;
#pragma unroll
        for (int u = 0; u < NC; ++u) h = max(h, hi_abs(x[u][i]));
        h = __reduce_max_sync(kFull, h);
        if (lane == 0) atomicMax(&sm.rmaxhi[r0 + i], h);
    }
    bool dead = false;  // (warp 2) a pivot of this micro-panel failed the witness test: the remaining
                        // exchanges still run (uniform control flow), the boundary drops their results
    const uint32_t sb = cc.sb;  // &sm in the shared window, opaque to the compiler
#define KC_OFF(f) ((uint32_t)offsetof(KCSmem, f))
#pragma unroll
    for (int i = 0; i < kR; ++i) {
        const int s = r0 + i;
        const int ms = m - s;  // active width before pivot s
        const unsigned par = gs & 1u, ph = (gs >> 1) & 1u;
        ++gs;
        KC_MARK(s, 0);
        // ---- my best column, then the warp's (exact; ties -> lowest column): one redux on the high
        //      words, the full comparison only when several lanes share the top word
        unsigned long long bits = 0ull;
        int bc = INT_MAX;
#pragma unroll
        for (int u = 0; u < NC; ++u) {
            const unsigned long long b = abs_bits(x[u][i]);
            if (own[u] && col[u] < ms && (bc == INT_MAX || b > bits)) { bits = b; bc = col[u]; }
        }
        const bool has = bc != INT_MAX;
        KC_MARK(s, 13);
        // exact 64-bit argmax, branch-free: redux on the high words, on the low words among the top,
        // ballot; the lowest lane of the ballot is the lowest column
        const unsigned bh = has ? (unsigned)(bits >> 32) : 0u, bl = (unsigned)bits;
        const unsigned mh = __reduce_max_sync(kFull, bh);
        const unsigned ml = __reduce_max_sync(kFull, (has && bh == mh) ? bl : 0u);
        const unsigned ball = __ballot_sync(kFull, has && bh == mh && bl == ml);
        KC_MARK(s, 14);
        jitter(1u);
        {
            // the winner lane publishes {|candidate|, column} and the column's 8 entries (a warp
            // without active columns: an invalid record from lane 0)
            const int wl = ball ? (int)(__ffs(ball) - 1) : 0;
            if (lane == wl) {
                const uint32_t aw = sb + KC_OFF(wrec) + warp * 16, ax = sb + KC_OFF(wx) + warp * (kR * 8);
                sts_v2(aw, ball ? bits : 0ull, (unsigned long long)(unsigned)(ball ? bc : INT_MAX));
#pragma unroll
                for (int u = 0; u < NC; ++u)
                    if (NC == 1 || col[u] == bc) {
#pragma unroll
                        for (int k = 0; k < kR; k += 2) sts_v2(ax + k * 8, d2u(x[u][k]), d2u(x[u][k + 1]));
                    }
            }
            // the owner of the last active column publishes it
            if (ms - 1 - lo >= NC * t && ms - 1 - lo < NC * t + NC) {
#pragma unroll
                for (int u = 0; u < NC; ++u)
                    if (own[u] && col[u] == ms - 1) {
#pragma unroll
                        for (int k = 0; k < kR; k += 2) sts_v2(sb + KC_OFF(xl) + k * 8, d2u(x[u][k]), d2u(x[u][k + 1]));
                    }
            }
        }
        KC_MARK(s, 15);
        asm volatile("bar.sync 1, %0;" ::"n"(kChainThreads) : "memory");
        KC_MARK(s, 1);
        if (warp == 0) {
            // ---- CTA argmax over the 4 warps' winners (lanes 0..3, redux), the record to every CTA
            ulonglong2 rw = make_ulonglong2(0ull, 0x7fffffffull);
            if (lane < kChainWarps) rw = lds_v2(sb + KC_OFF(wrec) + lane * 16);
            const unsigned rmh = lds_u32(sb + KC_OFF(rmaxhi) + s * 4);
            const unsigned wh = (unsigned)(rw.x >> 32), wlo = (unsigned)rw.x;
            const bool wok = (unsigned)rw.y != 0x7fffffffu;
            const unsigned wmh = __reduce_max_sync(kFull, wok ? wh : 0u);
            const unsigned wml = __reduce_max_sync(kFull, (wok && wh == wmh) ? wlo : 0u);
            const unsigned wbal = __ballot_sync(kFull, wok && wh == wmh && wlo == wml);
            const int ww = wbal ? (int)(__ffs(wbal) - 1) : 0;
            const ulonglong2 rbest = lds_v2(sb + KC_OFF(wrec) + ww * 16);
            const unsigned long long b0 = rbest.x;
            const int c0 = (int)(unsigned)rbest.y;
            KC_MARK(s, 8);
            jitter(2u);
            if (cc.dst < C) {
                // words: 0 value, 1 col | maxhi << 32, 2..9 the column's 8 entries
                const uint32_t bb = cc.r_bar + par * 8;
                const uint32_t a = cc.r_rcv + par * (16 * kRecWords * 8);
                const uint32_t ax = sb + KC_OFF(wx) + ww * (kR * 8);
                if (cc.part == 0) {
                    const unsigned maxhi = max(rmh, (unsigned)(b0 >> 32));
                    const ulonglong2 e0 = lds_v2(ax), e1 = lds_v2(ax + 16);
                    const unsigned long long vi = lds_u64(ax + i * 8);
                    KC_MARK(s, 9);
                    st_async_v2(a, vi, (unsigned long long)(unsigned)c0 | ((unsigned long long)maxhi << 32), bb);
                    st_async_v2(a + 16, e0.x, e0.y, bb);
                    st_async_v2(a + 32, e1.x, e1.y, bb);
                } else {
                    const ulonglong2 e2 = lds_v2(ax + 32), e3 = lds_v2(ax + 48);
                    st_async_v2(a + 48, e2.x, e2.y, bb);
                    st_async_v2(a + 64, e3.x, e3.y, bb);
                }
                if (lo <= ms - 1 && ms - 1 < lo + cc.wc) {  // I own the last active column
                    const uint32_t al = cc.r_rxl + par * (kR * 8) + cc.part * 32;
                    const ulonglong2 y0 = lds_v2(sb + KC_OFF(xl) + cc.part * 32), y1 = lds_v2(sb + KC_OFF(xl) + cc.part * 32 + 16);
                    st_async_v2(al, y0.x, y0.y, bb);
                    st_async_v2(al + 16, y1.x, y1.y, bb);
                }
            }
            KC_MARK(s, 10);
            if (lane == 0) mbar_arrive_expect_tx(cc.l_bar + par * 8, cc.exp_bytes);
        }
        KC_MARK(s, 2);
        // ---- every record of pivot s has arrived
        jitter(3u);
        if (!stopped) {
            unsigned spins = 0;
            while (!mbar_try_wait(cc.l_bar + par * 8, ph)) {
                if ((++spins & 63u) == 0u) {
                    if (globaltimer() - cc.t_start > cc.timeout_ns || *(volatile unsigned*)&cc.err->error) {
                        atomicExch(&cc.err->error, 1u);
                        atomicExch(&cc.err->err_step, (unsigned)(cc.row0 + s));
                        stopped = true;
                        break;
                    }
                }
            }
        }
        KC_MARK(s, 3);
        // ---- the cluster's argmax (ties -> lowest column = lowest CTA); every lane < C also forms
        //      the reciprocal of its record's value while the reduction runs
        double v, rcp;
        int l;
        unsigned hi1;
        uint32_t arec;  // the winner's record
        const uint32_t arcv = sb + KC_OFF(rcv) + par * (16 * kRecWords * 8);
        {
            const bool hl = lane < C;
            ulonglong2 r = make_ulonglong2(0ull, 0x7fffffffull);
            if (hl) r = lds_v2(arcv + lane * (kRecWords * 8));
            const int c = (int)(unsigned)r.y;
            const bool ok = c != INT_MAX;
            const double vl = u2d(r.x);
            KC_MARK(s, 11);
            const double rl = __drcp_rn(ok ? vl : 1.0);
            const unsigned long long b = r.x & 0x7fffffffffffffffull;
            const unsigned h2 = ok ? (unsigned)(b >> 32) : 0u, l2 = (unsigned)b;
            const unsigned mh2 = __reduce_max_sync(kFull, h2);
            const unsigned ml2 = __reduce_max_sync(kFull, (ok && h2 == mh2) ? l2 : 0u);
            const unsigned bal2 = __ballot_sync(kFull, ok && h2 == mh2 && l2 == ml2);
            const int gw = bal2 ? (int)(__ffs(bal2) - 1) : 0;
            KC_MARK(s, 12);
            arec = arcv + gw * (kRecWords * 8);
            const ulonglong2 rbest = lds_v2(arec);
            rcp = __shfl_sync(kFull, rl, gw);
            v = u2d(rbest.x);
            l = (int)(unsigned)rbest.y;
            hi1 = hl ? (unsigned)(r.y >> 32) : 0u;
        }
        KC_MARK(s, 4);
        jitter(4u);
        // the multipliers of rows > i (the winner column's entries), the last column if I take it
        unsigned long long mu[kR];
#pragma unroll
        for (int k = (i + 1) & ~1; k < kR; k += 2) {
            const ulonglong2 q2 = lds_v2(arec + 16 + k * 8);
            mu[k] = q2.x;
            mu[k + 1] = q2.y;
        }
        if (i + 1 < kR && ((i + 1) & 1)) mu[i + 1] = lds_u64(arec + 16 + (i + 1) * 8);
        if (warp == 1) {
            if (lane < i) sts_u64(sb + KC_OFF(T8) + (lane * kR + i) * 8, lds_u64(arec + 16 + lane * 8));
        } else if (warp == 2) {
            // witness test (condense.py:90) against an upper bound of the running row max; the records
            const unsigned bound_hi = __reduce_max_sync(kFull, hi1);
            const double bound = fmax(bound_hi >= 0x7fefffffu ? 1.7976931348623157e308 : u2d((unsigned long long)(bound_hi + 1u) << 32),
                                      u2d(lds_u64(sb + KC_OFF(wit0) + s * 8)));
            const bool singular = !dead && !stopped && !(fabs(v) > kSingularRtol * bound);
            if (lane == 0 && !dead) {
                sts_u32(sb + KC_OFF(l) + s * 4, (unsigned)l);
                if (cc.g == 0) {
                    cc.rec[s].v = v;
                    cc.rec[s].l = singular ? -1 : l;
                    cc.rec[s].flag = cc.epoch;
                    if (singular) atomicExch(cc.abort, 1u);
                }
                if (singular) sts_u32(sb + KC_OFF(bail), 1u);
            }
            dead = dead || singular;
        }
        // ---- the step in registers: column exchange, row i scaled, rows > i updated.  Dropped and
        //      foreign columns are computed along (their values are never used): no per-column
        //      branches; one branch picks the division: x / v correctly rounded from rcp = RN(1/v)
        //      (Markstein: q0 = RN(x rcp), e = x - q0 v exact, q = RN(q0 + e rcp); operands in
        //      [2^-500, 2^500), as k2_panel.cu) when every live operand of the thread is in range,
        //      IEEE division otherwise
        if (l != ms - 1 && l - lo >= NC * t && l - lo < NC * t + NC) {
#pragma unroll
            for (int u = 0; u < NC; ++u)
                if (col[u] == l) {
#pragma unroll
                    for (int k = 0; k < kR; k += 2) {
                        const ulonglong2 q2 = lds_v2(sb + KC_OFF(rxl) + par * (kR * 8) + k * 8);
                        x[u][k] = u2d(q2.x);
                        x[u][k + 1] = u2d(q2.y);
                    }
                }
        }
        {
            bool inr = ((unsigned)((d2u(v) >> 52) & 0x7ffu) - 523u) < 1000u;
#pragma unroll
            for (int u = 0; u < NC; ++u)  // (a dropped or foreign column never forces the slow path)
                inr = inr && (!(own[u] && col[u] < ms - 1) || (((unsigned)((d2u(x[u][i]) >> 52) & 0x7ffu) - 523u) < 1000u));
            double q[NC];
            if (inr) {
#pragma unroll
                for (int u = 0; u < NC; ++u) {
                    const double q0 = __dmul_rn(x[u][i], rcp);
                    const double e = __fma_rn(-q0, v, x[u][i]);
                    q[u] = __fma_rn(e, rcp, q0);
                }
            } else {
#pragma unroll
                for (int u = 0; u < NC; ++u) q[u] = __ddiv_rn(x[u][i], v);
            }
#pragma unroll
            for (int u = 0; u < NC; ++u) {
                x[u][i] = q[u];
#pragma unroll
                for (int k = i + 1; k < kR; ++k) x[u][k] = __dsub_rn(x[u][k], __dmul_rn(u2d(mu[k]), q[u]));
            }
        }
        KC_MARK(s, 5);
    }
#undef KC_OFF
    // ---- W8 = T8^{-1} U8 for my columns, into the micro-panel's rows of the chunk
    asm volatile("bar.sync 1, %0;" ::"n"(kChainThreads) : "memory");  // T8 complete (warp 1 wrote it)
#pragma unroll
    for (int u = 0; u < NC; ++u) {
        double w[kR];
#pragma unroll
        for (int a = kR - 1; a >= 0; --a) {
            double acc = x[u][a];
#pragma unroll
            for (int k = a + 1; k < kR; ++k) acc = __fma_rn(-sm.T8[a][k], w[k], acc);
            w[a] = acc;
        }
        if (own[u]) {
#pragma unroll
            for (int a = 0; a < kR; ++a) S[(r0 + a) * cw + NC * t + u] = w[a];
        }
    }
}

__device__ __forceinline__ void kc_copy_desc(K2Gather* dst, const K2Gather* src, int tid) {
    constexpr int kWords = (int)(sizeof(K2Gather) / sizeof(int32_t));
    for (int i = tid; i < kWords; i += kThreads)
        reinterpret_cast<int32_t*>(dst)[i] = reinterpret_cast<const int32_t*>(src)[i];
}

// Rank-8 update of the four rows rb .. rb+3 of the chunk by the micro-panel at rows r0 .. r0+7
// (whose slots hold W8): row <- row - L[row, 0:8] W8, columns c0, c0 + cstep, ... < wa.
__device__ __forceinline__ void kc_update4(double* __restrict__ S, const KCSmem& sm, const int cw, const int r0,
                                           const int rb, const int c0, const int cstep, const int wa) {
    double lq[4][kR];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int k = 0; k < kR; ++k) lq[u][k] = -sm.L[rb + u][k];
    for (int c = c0; c < wa; c += cstep) {
        double w8[kR], acc[4];
#pragma unroll
        for (int k = 0; k < kR; ++k) w8[k] = S[(r0 + k) * cw + c];
#pragma unroll
        for (int u = 0; u < 4; ++u) acc[u] = S[(rb + u) * cw + c];
#pragma unroll
        for (int k = 0; k < kR; ++k)
#pragma unroll
            for (int u = 0; u < 4; ++u) acc[u] = __fma_rn(lq[u][k], w8[k], acc[u]);
#pragma unroll
        for (int u = 0; u < 4; ++u) S[(rb + u) * cw + c] = acc[u];
    }
}

template <int NC>
__global__ void __launch_bounds__(kThreads, 1) kc_panel_kernel(const KPParams p0, const KPParams p1, const int halves) {
    extern __shared__ __align__(16) double S[];  // [kB][cw]
    __shared__ __align__(16) KCSmem sm;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = (int)cluster_ctarank();
    const unsigned long long t_start = globaltimer();
    if (tid == 0) {
        mbar_init(smem_u32(&sm.bar[0]), 1);
        mbar_init(smem_u32(&sm.bar[1]), 1);
        mbar_init(smem_u32(&sm.bar_ld), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        sm.bail = 0;
    }
    cluster_sync_all();
    unsigned gs = 0;  // exchange counter of this launch (mbarrier parity / phase)
    bool stopped = false;  // this thread timed out in an exchange: no more waits, the call fails

    for (int half = 0; half < halves; ++half) {
        const KPParams& p = half ? p1 : p0;
        const int C = p.G, cw = p.cw, m = p.m;
        const int lo = g * cw;
        const int wc = max(0, min(cw, m - lo));  // my columns at panel start
        if (*(volatile const unsigned*)p.abort) break;  // uniform: set only by earlier launches
        unsigned span_slot = 0;
        if (g == 0 && tid == 0) {
            span_slot = atomicAdd(&g_kc_span_n, 1u) & 4095u;
            g_kc_span[span_slot][0] = globaltimer();
        }
        double* const gcol = reinterpret_cast<double*>(p.colbuf);  // [micro-panel parity][multiplier | top columns][8][64]

        KC_MARKH(half, 0);
        // ---- load my chunk of the 64 panel rows: one bulk copy (TMA engine, cp.async.bulk) per
        //      row, issued by 64 threads, completing a transaction count on an mbarrier (rows are
        //      16-byte aligned: ld and the chunk offset are even; an odd last column goes by hand)
        const bool al_in = ((reinterpret_cast<uintptr_t>(p.ws) & 15u) == 0) && ((p.ld & 1) == 0);
        const bool al_out = ((reinterpret_cast<uintptr_t>(p.W) & 15u) == 0) && ((p.ldw & 1) == 0);
        {
            // (rows not 16-byte aligned -- never from this library's workspaces -- go element-wise)
            const unsigned rb = al_in ? (unsigned)(wc & ~1) * 8u : 0u;  // bytes per row through the bulk copy
            if (tid == 0) mbar_arrive_expect_tx(smem_u32(&sm.bar_ld), rb * kB);
            if (!al_in)
                for (int e = tid; e < kB * wc; e += kThreads) {
                    const int r = e / wc, c = e - r * wc;
                    S[r * cw + c] = __ldcg(p.ws + (int64_t)(p.row0 + r) * p.ld + lo + c);
                }
            if (tid < kB) {
                const double* src = p.ws + (int64_t)(p.row0 + tid) * p.ld + lo;
                if (rb)
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                                 ::"r"(smem_u32(S + tid * cw)), "l"(src), "r"(rb), "r"(smem_u32(&sm.bar_ld)) : "memory");
                if (al_in && (wc & 1)) S[tid * cw + wc - 1] = __ldcg(src + wc - 1);
            }
            while (!mbar_try_wait(smem_u32(&sm.bar_ld), (unsigned)half & 1u)) {
                if (globaltimer() - t_start > p.timeout_ns) {
                    atomicExch(&p.err->error, 1u);
                    atomicExch(&p.err->err_step, (unsigned)p.row0);
                    break;
                }
            }
        }
        if (tid < kB) {
            sm.wit0[tid] = p.wit[p.row0 + tid];
            sm.rmaxhi[tid] = 0u;
            sm.l[tid] = -2;  // "pivot not taken yet" (the publisher warp polls these)
        }
        __syncthreads();
        KC_MARKH(half, 1);
        if (half > 0) cluster_sync_all();  // the first panel's W and descriptor are complete
        KC_MARKH(half, 2);
        if (p.r1_g0) {
            // ---- the pair's first panel applied to these rows: NL = -A[rows, P0], the moved
            //      columns, then S += NL * W0 on the FP64 tensor cores, k ascending (the trailing
            //      GEMM's arithmetic; same code as k2_panel.cu)
            // (the first panel's descriptor is in shared memory: kept from the first half of this
            //  launch, or staged here; every gather below then has all its loads in flight)
            if (half == 0) {
                for (int i = tid; i < (int)(sizeof(K2Gather) / sizeof(int32_t)); i += kThreads)
                    reinterpret_cast<int32_t*>(&sm.d0)[i] = __ldcg(reinterpret_cast<const int32_t*>(p.r1_g0) + i);
                __syncthreads();
            }
            const K2Gather& g0 = sm.d0;
            const double* const rows = p.ws + (int64_t)p.row0 * p.ld;
            // NL = -A[rows, P0] in registers: thread t gathers column k = t mod 64 of rows t/64,
            // t/64 + 6, ... (all loads in flight); the staging buffer holds one k-block of 16 at a
            // time (the shared memory a full 64 x 64 staging would take goes to the chunk: 400
            // instead of 352 columns per CTA), so the thread stores its values in the pass of its
            // k-block
            constexpr int kNLper = (kB * kB + kThreads - 1) / kThreads;  // 11
            static_assert(kThreads % kB == 0, "a thread's gathered elements share their column");
            double nlv[kNLper];
#pragma unroll
            for (int u = 0; u < kNLper; ++u) {
                const int e = tid + u * kThreads;
                nlv[u] = (e < kB * kB) ? __ldcg(rows + (int64_t)(e >> 6) * p.ld + g0.P[e & 63]) : 0.0;
            }
            const int nm = g0.n_moved;
            for (int e0 = tid; e0 < kB * nm; e0 += 4 * kThreads) {
                double v[4];
                int at[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int e = e0 + u * kThreads;
                    at[u] = -1;
                    v[u] = 0.0;
                    if (e < kB * nm) {
                        const int r = e / nm, j = e - r * nm;
                        const int c = g0.moved_c[j];
                        if (c >= lo && c < lo + wc) {
                            at[u] = r * cw + (c - lo);
                            v[u] = __ldcg(rows + (int64_t)r * p.ld + g0.moved_src[j]);
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (at[u] >= 0) S[at[u]] = v[u];
            }
            KC_MARKH(half, 3);
            // S += NL * W0 on the FP64 tensor cores (mma.sync.m8n8k4.f64), k ascending (the trailing
            // GEMM's arithmetic), in 4 passes of 16 k: warp w owns the 8-column tiles w, w + 12, ...
            // two at a time for all 64 rows (one A fragment feeds both)
            const double* W0 = p.r1_W + lo;
            const int gq = lane >> 2, qq = lane & 3;
            const int ntiles = (wc + 7) >> 3;
            // (two copies of the loop body, with and without the second tile: a predicate around
            //  mma.sync makes the compiler bracket every DMMA with WARPSYNC)
            // Rounds of 24 tiles (two per warp); inside a round the 4 k-block passes run with the
            // accumulators in registers (the chunk's tiles are read and written once).  Three copies
            // of the round body -- two tiles, one tile, no tile (barriers and staging only) -- since
            // a predicate around mma.sync makes the compiler bracket every DMMA with WARPSYNC.
            auto stage = [&](const int k0) {
                __syncthreads();  // (the previous pass is done with the staging)
                if (((tid & 63) >> 4) == (k0 >> 4)) {
#pragma unroll
                    for (int u = 0; u < kNLper; ++u) {
                        const int e = tid + u * kThreads;
                        if (e < kB * kB) sm.NL[e >> 6][e & 15] = -nlv[u];
                    }
                }
                __syncthreads();
            };
            auto round = [&](const int tp, auto nt_c) {
                constexpr int NT = decltype(nt_c)::value;
                if constexpr (NT == 0) {
                    for (int k0 = 0; k0 < kB; k0 += 16) stage(k0);
                } else {
                    const int tl[2] = {tp, tp + kWarps};
                    auto load_bq = [&](const int k0, double (&bv)[4][NT]) {
#pragma unroll
                        for (int s4 = 0; s4 < 4; ++s4)
#pragma unroll
                            for (int t = 0; t < NT; ++t) {
                                const int c = tl[t] * 8 + gq;
                                bv[s4][t] = (c < wc) ? __ldcg(W0 + (int64_t)(k0 + 4 * s4 + qq) * p.r1_ldw + c) : 0.0;
                            }
                    };
                    double bq[4][NT];
                    load_bq(0, bq);
                    double acc[8][NT][2];
#pragma unroll
                    for (int i = 0; i < 8; ++i)
#pragma unroll
                        for (int t = 0; t < NT; ++t) {
                            const int c = tl[t] * 8 + 2 * qq;
                            const double* sp = S + (8 * i + gq) * cw + c;
                            acc[i][t][0] = (c < wc) ? sp[0] : 0.0;
                            acc[i][t][1] = (c + 1 < wc) ? sp[1] : 0.0;
                        }
                    for (int k0 = 0; k0 < kB; k0 += 16) {
                        stage(k0);
                        double bn[4][NT];
                        if (k0 + 16 < kB) load_bq(k0 + 16, bn);  // the next pass's W0 rows meanwhile
#pragma unroll
                        for (int s4 = 0; s4 < 4; ++s4) {
                            double av[8];
#pragma unroll
                            for (int i = 0; i < 8; ++i) av[i] = sm.NL[8 * i + gq][4 * s4 + qq];
#pragma unroll
                            for (int i = 0; i < 8; ++i)
#pragma unroll
                                for (int t = 0; t < NT; ++t)
                                    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                                        : "+d"(acc[i][t][0]), "+d"(acc[i][t][1]) : "d"(av[i]), "d"(bq[s4][t]));
                        }
                        if (k0 + 16 < kB) {
#pragma unroll
                            for (int s4 = 0; s4 < 4; ++s4)
#pragma unroll
                                for (int t = 0; t < NT; ++t) bq[s4][t] = bn[s4][t];
                        }
                    }
#pragma unroll
                    for (int i = 0; i < 8; ++i)
#pragma unroll
                        for (int t = 0; t < NT; ++t) {
                            const int c = tl[t] * 8 + 2 * qq;
                            double* const sp = S + (8 * i + gq) * cw + c;
                            if (c < wc) sp[0] = acc[i][t][0];
                            if (c + 1 < wc) sp[1] = acc[i][t][1];
                        }
                }
            };
            __syncthreads();  // the moved columns are in the chunk
            const int rounds = (ntiles + 2 * kWarps - 1) / (2 * kWarps);  // CTA-uniform
            for (int rd = 0; rd < rounds; ++rd) {
                const int tp = warp + rd * 2 * kWarps;
                if (tp + kWarps < ntiles) round(tp, std::integral_constant<int, 2>{});
                else if (tp < ntiles) round(tp, std::integral_constant<int, 1>{});
                else round(tp, std::integral_constant<int, 0>{});
            }
            __syncthreads();
        }
        KC_MARKH(half, 4);
        // ---- running row maxima of my chunk (high words: an upper bound within 2^-20)
        for (int r = warp; r < kB; r += kWarps) {
            unsigned h = 0u;
            for (int c = lane; c < wc; c += 32) h = max(h, hi_abs(S[r * cw + c]));
            h = __reduce_max_sync(kFull, h);
            if (lane == 0) sm.rmaxhi[r] = h;
        }
        __syncthreads();

        // remote addresses of my record slot / the last-column slot / the barriers in the CTA this
        // lane sends to (warp 0: lanes 2c, 2c+1 -> CTA c)
        KCChain cc;
        cc.g = g; cc.C = C; cc.cw = cw; cc.wc = wc; cc.lo = lo; cc.m = m;
        cc.dst = lane >> 1; cc.part = lane & 1;
        cc.r_rcv = 0; cc.r_rxl = 0; cc.r_bar = 0;
        if (warp == 0 && cc.dst < C) {
            cc.r_rcv = mapa(smem_u32(&sm.rcv[0][g][0]), (uint32_t)cc.dst);
            cc.r_rxl = mapa(smem_u32(&sm.rxl[0][0]), (uint32_t)cc.dst);
            cc.r_bar = mapa(smem_u32(&sm.bar[0]), (uint32_t)cc.dst);
        }
        cc.sb = opaque_u32(smem_u32(&sm));
        cc.l_bar = cc.sb + (uint32_t)offsetof(KCSmem, bar);
        cc.exp_bytes = (unsigned)(C * kRecWords * 8 + kR * 8);
        cc.t_start = t_start; cc.timeout_ns = p.timeout_ns;
        cc.rec = p.rec; cc.abort = p.abort; cc.err = p.err; cc.epoch = p.epoch; cc.row0 = p.row0;

        for (int j = 0; j < kB / kR; ++j) {
            const int r0 = j * kR;
            KC_MARKB(j, 0);
            if (warp < kChainWarps) {
                // ================= the micro-panel: 8 pivots, rows in registers (4 warps)
                kc_chain<NC>(sm, S, cc, r0, gs, stopped);
                KC_MARKB(j, 1);
                // ---- the micro-panel-start positions of the 8 pivot columns and the columns whose
                //      content moved (the composition of the 8 exchanges), identically in every CTA
                if (tid < kR) {
                    const int k = tid;
                    int lv[kR];  // the 8 pivot positions in registers: the chains below are select-only
#pragma unroll
                    for (int tt = 0; tt < kR; ++tt) lv[tt] = sm.l[r0 + tt];
                    int c = lv[0];
#pragma unroll
                    for (int tt = 1; tt < kR; ++tt) c = (tt == k) ? lv[tt] : c;
                    int pos = c, q = c;
                    bool first = c < m - r0 - kR;
#pragma unroll
                    for (int tt = kR - 1; tt >= 0; --tt) {
                        q = (q == lv[tt]) ? (m - (r0 + tt) - 1) : q;
                        if (tt < k) {
                            pos = (pos == lv[tt]) ? (m - (r0 + tt) - 1) : pos;
                            first = first && (lv[tt] != c);
                        }
                    }
                    sm.P8[k] = pos;
                    sm.mc[k] = (first && q != c) ? c : -1;
                    sm.ms[k] = q;
                }
            } else {
                // the other warps meanwhile, off the critical path: (1) the previous micro-panel's
                // update of the rows the chain does not hold (12 blocks of four rows: all but the
                // previous and the current micro-panel's)
                if (j > 0) {
                    const int jp = j - 1;
                    const int wa = max(0, min(wc, m - jp * kR - kR - lo));
                    for (int q = warp - kChainWarps; q < 12; q += kWarps - kChainWarps) {
                        const int grp = q < 2 * jp ? q : q + 2;          // skips the current micro-panel's blocks ...
                        const int rb = 4 * (grp < 2 * jp ? grp : grp + 2);  // ... and the previous one's
                        kc_update4(S, sm, cw, jp * kR, rb, lane, 32, wa);
                    }
                }
                asm volatile("bar.sync 3, %0;" ::"n"(kThreads - kChainThreads) : "memory");  // (1) done in this CTA
                // (2) one warp publishes what the boundary exchanges, as soon as it exists: the 8
                //     topmost active columns (the only possible sources of moved columns) now, the
                //     multiplier column of pivot k as soon as the chain has taken it -- so the
                //     boundary's cluster barrier finds the stores long complete
                if (warp == kChainWarps) {
                    double* const gc = gcol + (j & 1) * (2 * kR * kB);
                    double* const gt = gc + kR * kB;
                    const int ms0 = m - r0;
#pragma unroll
                    for (int tt = 0; tt < kR; ++tt) {
                        const int P = ms0 - kR + tt;
                        if (P >= lo && P < lo + wc) {
#pragma unroll
                            for (int h = 0; h < 2; ++h) {
                                const int r = lane + 32 * h;
                                if (r < r0 || r >= r0 + kR) gt[tt * kB + r] = S[r * cw + (P - lo)];
                            }
                        }
                    }
                    int lv[kR];
#pragma unroll
                    for (int k = 0; k < kR; ++k) {
                        int v;
                        for (;;) {
                            v = *(volatile int*)&sm.l[r0 + k];
                            if (v != -2 || *(volatile int*)&sm.bail) break;
                            __nanosleep(64);
                        }
                        lv[k] = v;
                        int pos = v;
#pragma unroll
                        for (int tt = kR - 1; tt >= 0; --tt)
                            if (tt < k) pos = (pos == lv[tt]) ? (m - (r0 + tt) - 1) : pos;
                        if (v >= 0 && pos >= lo && pos < lo + wc) {
#pragma unroll
                            for (int h = 0; h < 2; ++h) {
                                const int r = lane + 32 * h;
                                if (r < r0 || r >= r0 + kR) gc[k * kB + r] = S[r * cw + (pos - lo)];
                            }
                        }
                    }
                }
            }
            __syncthreads();
            if (sm.bail) goto finish;
            // ---- boundary: the 8 multiplier columns and the moved columns of the other 56 rows
            //      cross the cluster through L2 (published during the chain, above) around one
            //      cluster barrier
            cluster_sync_all();
            KC_MARKB(j, 2);
            jitter(6u);
            {
                const double* const gc = gcol + (j & 1) * (2 * kR * kB);
                const double* const gt = gc + kR * kB;
                const int ms0 = m - r0;
                for (int e = tid; e < kR * kB; e += kThreads) {
                    const int k = e >> 6, r = e & 63;
                    if (r < r0 || r >= r0 + kR) {
                        sm.L[r][k] = __ldcg(gc + k * kB + r);
                        const int c = sm.mc[k];
                        if (c >= lo && c < lo + wc) S[r * cw + (c - lo)] = __ldcg(gt + (sm.ms[k] - (ms0 - kR)) * kB + r);
                    }
                }
            }
            __syncthreads();
            KC_MARKB(j, 3);
            // ---- the other 56 rows: row <- row - L[row, 0:8] W8 (finished rows are rows of W,
            //      future rows panel rows: one formula; W8 read from the micro-panel's own rows of
            //      the chunk), in blocks of four rows (a block never straddles the 8-aligned
            //      micro-panels).  Only the NEXT micro-panel's 8 rows are on the critical path: all
            //      warps take them now (column slices), the other 48 rows follow on the non-chain
            //      warps while the next micro-panel runs.  The last boundary updates all 56 here.
            {
                const int wa = max(0, min(wc, m - r0 - kR - lo));  // my active columns after the micro-panel
                if (j + 1 < kB / kR) {
                    const int rb = (r0 + kR) + 4 * (warp & 1);
                    kc_update4(S, sm, cw, r0, rb, (warp >> 1) * 32 + lane, 32 * (kWarps / 2), wa);
                } else {
                    for (int grp = warp; grp < 14; grp += kWarps) kc_update4(S, sm, cw, r0, 4 * grp, lane, 32, wa);
                }
            }
            __syncthreads();
            KC_MARKB(j, 4);
        }

        KC_MARKH(half, 5);
        // ---- the chunk holds W in the final layout: out (columns < m - 64), one bulk store per row
        //      (shared -> global through the TMA engine; the generic-proxy writes of the chunk are
        //      fenced into the async proxy first)
        {
            const int wf = max(0, min(wc, m - kB - lo));
            const unsigned rb = al_out ? (unsigned)(wf & ~1) * 8u : 0u;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncthreads();
            if (!al_out)
                for (int e = tid; e < kB * wf; e += kThreads) {
                    const int r = e / wf, c = e - r * wf;
                    p.W[(int64_t)r * p.ldw + lo + c] = S[r * cw + c];
                }
            if (tid < kB) {
                double* const dstw = p.W + (int64_t)tid * p.ldw + lo;
                if (rb)
                    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                                 ::"l"(dstw), "r"(smem_u32(S + tid * cw)), "r"(rb) : "memory");
                if (al_out && (wf & 1)) dstw[wf - 1] = S[tid * cw + wf - 1];
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
        }
        KC_MARKH(half, 6);
        // ---- the panel's gather descriptor: panel-start column of each pivot and the final columns
        //      whose content moved (the composition of the 64 exchanges), by every CTA in shared
        //      memory (the pair prep below needs it everywhere); CTA 0 publishes it
        {
            K2Gather& d1 = sm.d1;
            int c = 0, q = 0, pre = 0;
            bool flag = false;
            if (tid < kB) {
                const int s = tid;
                c = sm.l[s];
                int pos = c;
                q = c;
                bool first = c < m - kB;
#pragma unroll 8
                for (int j = kB - 1; j >= 0; --j) {
                    const int lj = sm.l[j];
                    q = (q == lj) ? (m - j - 1) : q;
                    if (j < s) {
                        pos = (pos == lj) ? (m - j - 1) : pos;
                        first = first && (lj != c);
                    }
                }
                d1.P[s] = pos;
                d1.l[s] = c;
                flag = first && q != c;
                const unsigned ball = __ballot_sync(kFull, flag);
                pre = __popc(ball & ((1u << lane) - 1u));
                if (lane == 0) sm.cnt[warp] = __popc(ball);
            }
            __syncthreads();
            if (tid < kB && flag) {
                const int k = pre + (warp ? sm.cnt[0] : 0);
                d1.moved_c[k] = c;
                d1.moved_src[k] = q;
            }
            if (tid == 0) d1.n_moved = sm.cnt[0] + sm.cnt[1];
            // the W rows are out (complete in global memory: the barriers below publish them; the
            // chunk may be reused)
            if (tid < kB) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
            __syncthreads();
            if (g == 0) kc_copy_desc(p.pan, &d1, tid);
        }
        if (p.pp_g0) {
            // ---- pair prep spread over the cluster: (a) a slice of Wp[s][s'] = -W_k[s][P1[s']];
            //      the pair's composite descriptor (every CTA in shared memory, CTA 0 publishes it;
            //      one thread per entry, deterministic order); one cluster barrier (every Wp read
            //      of W_k done); (b) a slice of W_k's moved columns
            const K2Gather& d0 = sm.d0;
            const K2Gather& d1 = sm.d1;
            if (half == 0) {  // (a second panel launched on its own: the first descriptor from memory)
                for (int i = tid; i < (int)(sizeof(K2Gather) / sizeof(int32_t)); i += kThreads)
                    reinterpret_cast<int32_t*>(&sm.d0)[i] = __ldcg(reinterpret_cast<const int32_t*>(p.pp_g0) + i);
                __syncthreads();
            }
            {
                const int e0 = (int)((int64_t)kB * kB * g / C), e1 = (int)((int64_t)kB * kB * (g + 1) / C);
                for (int e = e0 + tid; e < e1; e += kThreads) {
                    const int sr = e / kB, sp = e % kB;
                    p.pp_Wp[e] = -__ldcg(p.pp_W + (int64_t)sr * p.pp_ldw + d1.P[sp]);
                }
            }
            KC_MARKH(half, 7);
            if (g == 0) {
                // (the chunk is dead after the W output: it holds two direct-address maps, final
                //  column -> source column of each panel, so every lookup is one load)
                const int wf = p.pp_m - 2 * kB;
                int* const map0 = reinterpret_cast<int*>(S);   // panel k   : width pp_m
                int* const map1 = map0 + p.pp_m;               // panel k+1 : width pp_m - 64
                for (int i = tid; i < 2 * p.pp_m; i += kThreads) map0[i] = -1;
                __syncthreads();
                if (tid < d0.n_moved) map0[d0.moved_c[tid]] = d0.moved_src[tid];
                if (tid >= 2 * kB && tid - 2 * kB < d1.n_moved) map1[d1.moved_c[tid - 2 * kB]] = d1.moved_src[tid - 2 * kB];
                __syncthreads();
                auto pi0 = [&](int x) { const int r = map0[x]; return r < 0 ? x : r; };
                auto pi1 = [&](int x) { const int r = map1[x]; return r < 0 ? x : r; };
                if (tid < kB) {
                    sm.gp.P[tid] = d0.P[tid];
                    sm.gp.P[kB + tid] = pi0(d1.P[tid]);
                    sm.gp.l[tid] = d1.l[tid];
                }
                // candidate moved columns: targets of either panel inside the final width (the
                // first panel's only when the second does not also move them)
                int c = 0, src = 0, pre = 0;
                bool flag = false;
                if (tid < 2 * kB) {
                    const int n1 = d1.n_moved, n0 = d0.n_moved;
                    bool valid = false;
                    if (tid < n1) {
                        c = d1.moved_c[tid];
                        valid = c < wf;
                    } else if (tid - n1 < n0) {
                        c = d0.moved_c[tid - n1];
                        valid = c < wf && map1[c] < 0;
                    }
                    if (valid) {
                        src = pi0(pi1(c));
                        flag = src != c;
                    }
                    const unsigned ball = __ballot_sync(kFull, flag);
                    pre = __popc(ball & ((1u << lane) - 1u));
                    if (lane == 0) sm.cnt[warp] = __popc(ball);
                }
                __syncthreads();
                if (tid < 2 * kB && flag) {
                    int k = pre;
                    for (int w = 0; w < warp; ++w) k += sm.cnt[w];
                    sm.gp.moved_c[k] = c;
                    sm.gp.moved_src[k] = src;
                }
                if (tid == 0) sm.gp.n_moved = sm.cnt[0] + sm.cnt[1] + sm.cnt[2] + sm.cnt[3];
                __syncthreads();
                kc_copy_desc(p.pp_gpair, &sm.gp, tid);
            }
            KC_MARKH(half, 8);
            __threadfence();
            cluster_sync_all();
            KC_MARKH(half, 9);
            {
                const int nm1 = d1.n_moved, wf2 = p.pp_m - 2 * kB;
                const int tot = kB * nm1;
                const int e0 = (int)((int64_t)tot * g / C), e1 = (int)((int64_t)tot * (g + 1) / C);
                for (int e = e0 + tid; e < e1; e += kThreads) {
                    const int sr = e / nm1, k = e % nm1;
                    const int c = d1.moved_c[k];
                    if (c < wf2) p.pp_W[(int64_t)sr * p.pp_ldw + c] = __ldcg(p.pp_W + (int64_t)sr * p.pp_ldw + d1.moved_src[k]);
                }
            }
        }
        if (half + 1 < halves) {  // the second panel's prologue and pair prep read this descriptor
            __syncthreads();
            kc_copy_desc(&sm.d0, &sm.d1, tid);
        }
        KC_MARKH(half, 10);
        if (g == 0 && tid == 0) g_kc_span[span_slot][1] = globaltimer();
        __threadfence();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // (the next half's bulk load overwrites the chunk)
        __syncthreads();  // S / sm.l reads done before the next half reloads them
    }
finish:
    cluster_sync_all();  // no CTA leaves while a peer may still address its shared memory
}

}  // namespace

#if KC_TRACE
void kc_debug_trace(unsigned long long* steps, unsigned long long* bounds) {
    cudaMemcpyFromSymbol(steps, g_kc_trace, sizeof(g_kc_trace));
    cudaMemcpyFromSymbol(bounds, g_kc_tb, sizeof(g_kc_tb));
}
void kc_debug_trace_halves(unsigned long long* halves) { cudaMemcpyFromSymbol(halves, g_kc_th, sizeof(g_kc_th)); }
#endif

int kc_debug_spans(unsigned long long* out, int max_spans) {
    unsigned n = 0;
    if (cudaMemcpyFromSymbol(&n, g_kc_span_n, sizeof(n)) != cudaSuccess) return -1;
    const int k = (int)std::min<unsigned>(std::min<unsigned>(n, 4096u), (unsigned)max_spans);
    if (k > 0 && cudaMemcpyFromSymbol(out, g_kc_span, (size_t)k * 2 * sizeof(unsigned long long)) != cudaSuccess) return -1;
    const unsigned zero = 0;
    cudaMemcpyToSymbol(g_kc_span_n, &zero, sizeof(zero));
    return k;
}

size_t kc_smem_bytes(int cw) { return (size_t)kB * cw * sizeof(double); }

// Cluster size and chunk width for active width m (0: the cluster kernel does not take it)
int kc_plan(int64_t m, int* cw_out) {
    const int cmax = kc_max_cluster();
    if (cmax < 2 || m < 2 * kB || m > (int64_t)cmax * kKCMaxCw) return 0;
    int C = cmax;
    while (C > 2 && m <= (int64_t)(C / 2) * 128) C /= 2;  // at least ~128 columns per CTA
    int cw = (int)((m + C - 1) / C);
    cw = (cw + 31) / 32 * 32;
    if (cw > kKCMaxCw) cw = (int)(((m + C - 1) / C + 1) / 2 * 2);
    if (cw > kKCMaxCw) return 0;
    *cw_out = cw;
    return C;
}

// Largest cluster (16, 8, 4, 2; 0: none) the current device can co-schedule with the kernel's
// largest footprint (400 columns per CTA), probed once per device: a device or partition without
// 16 free SMs in one GPC takes smaller clusters, or the column-distributed kernel.
int kc_max_cluster() {
    constexpr int kMaxDev = 64;
    static int cache[kMaxDev] = {};  // 0: not probed, -1: none
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) return 0;
    if (cache[dev]) return cache[dev] < 0 ? 0 : cache[dev];
    auto fn = kc_panel_kernel<3>;
    const size_t smem = kc_smem_bytes(kKCMaxCw);
    int best = -1;
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) == cudaSuccess &&
        cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess) {
        for (int C = kKCMaxC; C >= 2; C /= 2) {
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(C);
            cfg.blockDim = dim3(kThreads);
            cfg.dynamicSmemBytes = smem;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = (unsigned)C;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            int n = 0;
            if (cudaOccupancyMaxActiveClusters(&n, fn, &cfg) == cudaSuccess && n >= 1) {
                best = C;
                break;
            }
        }
    }
    (void)cudaGetLastError();
    cache[dev] = best;
    return best < 0 ? 0 : best;
}

cudaError_t kc_launch(const KPParams& p, cudaStream_t s, const KPParams* second) {
    const size_t smem = kc_smem_bytes(p.cw);
    if (p.cw < 2 || (p.cw & 1) || p.cw > kKCMaxCw || p.G < 1 || p.G > kKCMaxC || (int64_t)p.G * p.cw < p.m)
        return cudaErrorInvalidValue;
    if (second && (second->G != p.G || second->cw != p.cw)) return cudaErrorInvalidValue;
    const int nc = (p.cw + kChainThreads - 1) / kChainThreads;  // columns per chain thread
    auto fn = nc <= 1 ? kc_panel_kernel<1> : nc == 2 ? kc_panel_kernel<2> : kc_panel_kernel<3>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if (p.G > 8) {
        e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(p.G);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)p.G;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const KPParams q0 = p, q1 = second ? *second : p;
    const int halves = second ? 2 : 1;
    return cudaLaunchKernelEx(&cfg, fn, q0, q1, halves);
}

}  // namespace mcnd

// K1: persistent, barrier-free matrix-condensation kernel for sm_100a.
//
// Restates condense_step / logdet_condensation (mcnd/condense.py:82-160) and
// the block-row worker update of mc_parallel (mcnd/runtime.py:157-203) as ONE
// cooperative launch with one 1024-thread CTA per SM.
//
// Data layout (HBM): the caller's rows are copied once into a workspace of
// n rows x ld doubles (ld = n rounded up to 16, so every row starts on a
// 128-byte line).  Condensation is IN PLACE and never moves rows: step s
// drops the pivot row, and the column exchange l <-> m-1 of condense.py:104-107
// is folded into the read pattern (column l of the result reads old column
// m-1), so the active block is always columns [0, m) of the live rows.
//
// Work split: rows are dealt cyclically to CTAs in pivot order, so the live
// rows (a suffix of the pivot order) stay balanced for any pivot sequence
// (the paper's arbitrary-pivot-row property).  Each CTA
// updates only its own rows, so the only cross-CTA data is the pivot row.
//
// Dataflow instead of grid barriers: the CTA that owns the pivot row of step
// s+1 updates that row FIRST in step s, reduces its argmax (ties -> lowest
// column, condense.py:88), runs the witness test (condense.py:90), writes the
// scaled, column-permuted pivot row (condense.py:110-111) into the row's slot
// of every group's workspace -- the "broadcast" of runtime.py:185, done as
// stores into peer memory over NVLink when groups are other GPUs -- and then
// release-stores the pivot record's flag.  Every CTA waits only for "pivot s
// published" before step s, so pivot selection runs one step ahead of the bulk
// update (lookahead) and there is no grid- or job-wide barrier anywhere.
//
// Arithmetic: parity mode uses __dmul_rn then __dsub_rn (two roundings, exactly
// numpy's `sub -= col[:,None]*prow`, condense.py:118) and true division for
// the pivot row; fast mode uses one FMA.  The running row witness
// (condense.py:120-122) is fused into the same pass as a per-segment warp max
// folded into shared memory with a 64-bit atomicMax on the bit pattern.  The
// finiteness check of matrix.py:39-40 is fused into the prologue copy.
#include <cstdint>
#include <climits>
#include "mcnd_internal.h"

namespace mcnd {
namespace {

constexpr int kThreads = kK1Threads;
constexpr int kWarps = kThreads / 32;
constexpr int kU = 4;                   // double2 per lane per segment
constexpr int kSegPairs = 32 * kU;      // 128 pairs = 256 doubles = 2 KB per warp segment
constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ unsigned ld_acquire_flag(const uint32_t* p, bool sys) {
    unsigned v;
    if (sys) asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    else asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_flag(uint32_t* p, unsigned v, bool sys) {
    if (sys) asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
    else asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
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

#ifndef K1_POLL_SLEEP
#define K1_POLL_SLEEP 32  // ns between flag polls
#endif

template <bool kFast>
__device__ __forceinline__ double upd(double x, double mult, double p) {
    if (kFast) return fma(-mult, p, x);
    return __dsub_rn(x, __dmul_rn(mult, p));
}

// GE mode breaks ties by the original row id of the column (gauss.py:49-52 takes the first
// maximum in the original row order), condensation by the column position (condense.py:88).
__device__ __forceinline__ int tie_key(const K1Params& p, int c) { return p.ge_ids ? __ldcg(p.ge_ids + c) : c; }

// (value, column) argmax order: larger |value| wins, ties -> lower column.
__device__ __forceinline__ bool beats(double av, int ai, double bv, int bi) {
    double fa = fabs(av), fb = fabs(bv);
    return fa > fb || (fa == fb && ai < bi);
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(kFull, v, o));
    return v;
}

struct Smem {
    int rows[kK1MaxRowsPerCta];
    int pstep[kK1MaxRowsPerCta];
    unsigned long long wit[kK1MaxRowsPerCta];  // non-negative doubles as u64 (order-preserving)
    double mult[kK1MaxRowsPerCta];             // a[r][l]   (multiplier, old pivot column)
    double last[kK1MaxRowsPerCta];             // a[r][m-1] (moves into column l)
    double red_v[kWarps + 1];
    double red_w[kWarps + 1];
    int red_i[kWarps + 1];
    int step_l;
    int win_pos;  // GE mode: column position of the winning (value, original id)
};

// Whole-CTA reduction of (argmax value, column) and witness max.  Every thread
// returns the CTA result.  Exact: |x| compared as its 64-bit pattern (redux.sync
// on the high then the low word), ties -> lowest column, as beats() orders them.
__device__ __forceinline__ unsigned long long abs_bits(double x) {
    return (unsigned long long)__double_as_longlong(x) & 0x7fffffffffffffffull;
}
__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
    const unsigned hi = (unsigned)(v >> 32), lo = (unsigned)v;
    const unsigned mh = __reduce_max_sync(kFull, hi);
    const unsigned ml = __reduce_max_sync(kFull, hi == mh ? lo : 0u);
    return ((unsigned long long)mh << 32) | ml;
}
__device__ __forceinline__ void warp_argmax(double& v, int& i, unsigned long long& w) {
    const unsigned long long kb = abs_bits(v);
    const unsigned long long mb = warp_max_u64(kb);
    const unsigned wi = __reduce_min_sync(kFull, kb == mb ? (unsigned)i : 0xffffffffu);
    const int src = __ffs(__ballot_sync(kFull, kb == mb && (unsigned)i == wi)) - 1;
    v = __shfl_sync(kFull, v, src);
    i = __shfl_sync(kFull, i, src);
    w = warp_max_u64(w);
}
__device__ __forceinline__ void cta_reduce(Smem& sm, double& v, int& i, double& w) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long wb = abs_bits(w);
    warp_argmax(v, i, wb);
    if (lane == 0) { sm.red_v[warp] = v; sm.red_i[warp] = i; sm.red_w[warp] = __longlong_as_double((long long)wb); }
    __syncthreads();
    if (warp == 0) {
        v = lane < kWarps ? sm.red_v[lane] : 0.0;
        i = lane < kWarps ? sm.red_i[lane] : INT_MAX;
        wb = lane < kWarps ? abs_bits(sm.red_w[lane]) : 0ull;
        warp_argmax(v, i, wb);
        if (lane == 0) { sm.red_v[kWarps] = v; sm.red_i[kWarps] = i; sm.red_w[kWarps] = __longlong_as_double((long long)wb); }
    }
    __syncthreads();
    v = sm.red_v[kWarps]; i = sm.red_i[kWarps]; w = sm.red_w[kWarps];
}

// Publish pivot t of global row `row` (active width m_pub; its values are final
// in this group's workspace and visible CTA-wide).  Writes the scaled pivot
// row prow[c] = row[sigma(c)] / v, c < m_pub-1, into that row's slot of every
// group's workspace (the row is dead after pivot t, so nobody else ever
// touches those slots), then the record, then the release flag.  Whole CTA.
__device__ void publish(const K1Params& p, Smem& sm, int g, int row, int t, int m_pub, double v, int l,
                        double wit) {
    // condense.py:90; GE mode: gauss.py:55-58 (exact zero, or the caller's row witness)
    const bool singular = p.ge_ids ? (v == 0.0 || (p.ge_rowwit && fabs(v) <= kSingularRtol * p.ge_rowwit[p.ge_ids[l]]))
                                   : !(fabs(v) > kSingularRtol * wit);
    const unsigned long long t_pub = threadIdx.x == 0 ? globaltimer() : 0ull;  // CommStats.comm_seconds
    const int wp = m_pub - 1;
    const bool sys = p.sys_scope != 0;
    double* own = p.ws[g] + (int64_t)row * p.ld;
    jitter(5u);
    if (!singular && wp > 0) {
        const double ylast = own[wp];
        for (int c = threadIdx.x; c < wp; c += kThreads) {
            const double y = __ddiv_rn((c == l) ? ylast : own[c], v);  // condense.py:110 (true division)
            for (int h = 0; h < p.n_groups; ++h) p.ws[h][(int64_t)row * p.ld + c] = y;
        }
    }
    if (sys) __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        // GE mode: the exchange l <- m-1 moves that column's row id too (ordered before the
        // flag release, so the next publisher sees the new layout)
        if (p.ge_ids && wp > 0 && l != wp) p.ge_ids[l] = p.ge_ids[wp];
        for (int h = 0; h < p.n_groups; ++h) {
            p.rec[h][t].v = v;
            // singular: -1 (condensation); GE mode keeps the position as -(l + 2) (its pivot row
            // is reported, as gauss.py's loop reached it)
            p.rec[h][t].l = singular ? (p.ge_ids ? -(l + 2) : -1) : l;
        }
        // single GPU: the gpu-scope release is cumulative over the CTA's row stores
        // (ordered before it by the barrier), no separate fence needed
        if (sys) __threadfence_system();
        jitter(6u);
        for (int h = 0; h < p.n_groups; ++h) st_release_flag(&p.rec[h][t].flag, p.epoch, sys);
        atomicAdd(&p.err->comm_ns, globaltimer() - t_pub);
    }
}

template <bool kFast>
__global__ void __launch_bounds__(kThreads, 1) k1_condense(const K1Params p) {
    extern __shared__ __align__(16) double s_prow[];
    __shared__ Smem sm;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned long long t_k0 = globaltimer();
    const int gl = blockIdx.x / p.ctas_per_group;  // local group
    const int g = p.group0 + gl;                   // global group (worker / rank)
    double* const ws = p.ws[g];
    PivRec* const rec = p.rec[g];
    const bool sys = p.sys_scope != 0;
    const int rbeg = p.cta_row_ptr[blockIdx.x];
    const int nr = p.cta_row_ptr[blockIdx.x + 1] - rbeg;
    for (int i = tid; i < nr; i += kThreads) {
        const int r = p.cta_rows[rbeg + i];
        sm.rows[i] = r;
        sm.pstep[i] = p.row_pstep[r] - p.pstep_offset;
        sm.wit[i] = 0ull;
    }
    __syncthreads();

    if (p.abort_flag && *(volatile const unsigned*)p.abort_flag) return;  // uniform per CTA
    const int ncol0 = p.ncol0;

    // ---- prologue: copy my rows into the workspace, initial witness (condense.py:72-78)
    //      and the finiteness check (matrix.py:39-40).  In panel mode (blocked K2) the
    //      rows are already in place: only the witness is refreshed.
    if (p.in_place) {
        for (int i = warp; i < nr; i += kWarps) {
            const int r = sm.rows[i];
            const double* row = ws + (int64_t)r * p.ld;
            double wm = 0.0;
            for (int c = lane; c < ncol0; c += 32) wm = fmax(wm, fabs(row[c]));
            wm = fmax(warp_max(wm), p.wit_in[r]);
            if (lane == 0) sm.wit[i] = (unsigned long long)__double_as_longlong(wm);
        }
    } else {
        constexpr int kSeg = 256;
        const int nseg = (ncol0 + kSeg - 1) / kSeg;
        const int total = nr * nseg;
        bool bad = false;
        for (int j = warp; j < total; j += kWarps) {
            const int i = j / nseg, sg = j - i * nseg;
            const int r = sm.rows[i];
            const double* src = p.src[gl] + (r - p.src_row0[gl]) * p.lds;
            double* dst = ws + (int64_t)r * p.ld;
            const int c0 = sg * kSeg + lane;
            double x[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int c = c0 + 32 * k;
                x[k] = (c < ncol0) ? __ldg(src + c) : 0.0;
            }
            double wm = 0.0;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int c = c0 + 32 * k;
                if (c < ncol0) {
                    dst[c] = x[k];
                    wm = fmax(wm, fabs(x[k]));
                    bad |= !isfinite(x[k]);
                }
            }
            wm = warp_max(wm);
            if (lane == 0) atomicMax(&sm.wit[i], (unsigned long long)__double_as_longlong(wm));
        }
        if (__any_sync(kFull, bad) && lane == 0) atomicOr(&p.err->nonfinite, 1u);
    }
    __syncthreads();
    if (tid == 0 && !p.in_place) atomicMax(&p.err->scatter_ns, globaltimer() - t_k0);  // CommStats.scatter_seconds

    // ---- pivot 0 (its row was just copied by this CTA)
    if (nr > 0 && sm.pstep[0] == 0) {
        double* rowp = ws + (int64_t)sm.rows[0] * p.ld;
        double bv = 0.0, bw = 0.0;
        int bi = INT_MAX;
        int bp = INT_MAX;  // position of the local best (GE: bi is its original id)
        for (int c = tid; c < ncol0; c += kThreads) {
            const double x = rowp[c];
            const int key = tie_key(p, c);
            if (beats(x, key, bv, bi)) { bv = x; bi = key; bp = c; }
        }
        const int lbi = bi;
        const double lbv = bv;
        cta_reduce(sm, bv, bi, bw);
        if (p.ge_ids) {  // the one thread holding the winner knows its position
            if (lbi == bi && abs_bits(lbv) == abs_bits(bv)) sm.win_pos = bp;
            __syncthreads();
            bi = sm.win_pos;
        }
        publish(p, sm, g, sm.rows[0], 0, ncol0, bv, bi, __longlong_as_double((long long)sm.wit[0]));
    }

    int start = 0;  // first live local row
    for (int s = 0; s < p.n_steps; ++s) {
        const int m = ncol0 - s, w = m - 1;
        // ---- wait for pivot s
        if (tid == 0) {
            int l = -2;
            const unsigned long long t0 = globaltimer();
            for (;;) {
                if (ld_acquire_flag(&rec[s].flag, sys) == p.epoch) {
                    l = *(volatile const int32_t*)&rec[s].l;
                    break;
                }
                if (*(volatile unsigned*)&p.err->error) break;
                if (globaltimer() - t0 > p.timeout_ns) {
                    atomicExch(&p.err->error, 1u);
                    atomicExch(&p.err->err_step, (unsigned)s);
                    break;
                }
                if (K1_POLL_SLEEP) __nanosleep(K1_POLL_SLEEP);
            }
            sm.step_l = l;
        }
        __syncthreads();
        const int l = sm.step_l;
        if (l < 0) break;  // singular (-1) or error (-2): everybody stops
        while (start < nr && sm.pstep[start] <= s) ++start;

        // ---- stage multipliers / last column of my live rows, and chunk 0 of the pivot row
        const double* prow_g = ws + (int64_t)__ldg(p.seq + s) * p.ld;
        for (int i = start + tid; i < nr; i += kThreads) {
            const double* rp = ws + (int64_t)sm.rows[i] * p.ld;
            sm.mult[i] = rp[l];
            sm.last[i] = rp[w];
        }
        const int cw0 = w < p.chunk ? w : p.chunk;
        for (int c = tid; c < cw0; c += kThreads) s_prow[c] = __ldcg(prow_g + c);
        if (tid == 0 && (cw0 & 1)) s_prow[cw0] = 0.0;
        __syncthreads();

        int bulk_first = start;
        // ---- lookahead: I own the next pivot row -> update it first with the whole CTA
        if (start < nr && sm.pstep[start] == s + 1) {
            bulk_first = start + 1;
            double* rowp = ws + (int64_t)sm.rows[start] * p.ld;
            const double mult = sm.mult[start], lastv = sm.last[start];
            const int npairs = (w + 1) >> 1;
            double bv = 0.0, bw = 0.0;
            int bi = INT_MAX, bp = INT_MAX;  // GE mode: bi = original id, bp = its position
            for (int pj = tid; pj < npairs; pj += kThreads) {
                const int c = 2 * pj;
                double2 x = *reinterpret_cast<const double2*>(rowp + c);
                if (c == l) x.x = lastv;
                if (c + 1 == l) x.y = lastv;
                double p0, p1;
                if (c < cw0) { p0 = s_prow[c]; p1 = s_prow[c + 1]; }
                else { p0 = __ldcg(prow_g + c); p1 = (c + 1 < w) ? __ldcg(prow_g + c + 1) : 0.0; }
                double2 y;
                y.x = upd<kFast>(x.x, mult, p0);
                y.y = upd<kFast>(x.y, mult, p1);
                *reinterpret_cast<double2*>(rowp + c) = y;
                const int k0 = tie_key(p, c);
                if (beats(y.x, k0, bv, bi)) { bv = y.x; bi = k0; bp = c; }
                bw = fmax(bw, fabs(y.x));
                if (c + 1 < w) {
                    const int k1 = tie_key(p, c + 1);
                    if (beats(y.y, k1, bv, bi)) { bv = y.y; bi = k1; bp = c + 1; }
                    bw = fmax(bw, fabs(y.y));
                }
            }
            const int lbi = bi;
            const double lbv = bv;
            cta_reduce(sm, bv, bi, bw);
            if (p.ge_ids) {
                if (lbi == bi && abs_bits(lbv) == abs_bits(bv)) sm.win_pos = bp;
                __syncthreads();
                bi = sm.win_pos;
            }
            const double wit = fmax(__longlong_as_double((long long)sm.wit[start]), bw);
            publish(p, sm, g, sm.rows[start], s + 1, w, bv, bi, wit);
            if (tid == 0) sm.wit[start] = (unsigned long long)__double_as_longlong(wit);
        }

        jitter(7u);
        // ---- bulk update of my other live rows, chunk by chunk
        for (int c0 = 0; c0 < w; c0 += p.chunk) {
            const int cend = (c0 + p.chunk < w) ? c0 + p.chunk : w;
            if (c0 > 0) {
                __syncthreads();
                const int clen = cend - c0;
                for (int c = tid; c < clen; c += kThreads) s_prow[c] = __ldcg(prow_g + c0 + c);
                if (tid == 0 && (clen & 1)) s_prow[clen] = 0.0;
                __syncthreads();
            }
            const int npairs = (cend - c0 + 1) >> 1;
            const int nseg = (npairs + kSegPairs - 1) / kSegPairs;
            const int total = (nr - bulk_first) * nseg;
            for (int j = warp; j < total; j += kWarps) {
                const int ii = j / nseg, sg = j - ii * nseg;
                const int i = bulk_first + ii;
                double* rowp = ws + (int64_t)sm.rows[i] * p.ld + c0;
                const double mult = sm.mult[i], lastv = sm.last[i];
                const int pj0 = sg * kSegPairs + lane;
                double2 x[kU];
#pragma unroll
                for (int k = 0; k < kU; ++k) {
                    const int pj = pj0 + 32 * k;
                    if (pj < npairs) x[k] = *reinterpret_cast<const double2*>(rowp + 2 * pj);
                }
                double wm = 0.0;
#pragma unroll
                for (int k = 0; k < kU; ++k) {
                    const int pj = pj0 + 32 * k;
                    if (pj < npairs) {
                        const int c = c0 + 2 * pj;
                        if (c == l) x[k].x = lastv;
                        if (c + 1 == l) x[k].y = lastv;
                        const double2 pv = *reinterpret_cast<const double2*>(s_prow + 2 * pj);
                        double2 y;
                        y.x = upd<kFast>(x[k].x, mult, pv.x);
                        y.y = upd<kFast>(x[k].y, mult, pv.y);
                        *reinterpret_cast<double2*>(rowp + 2 * pj) = y;
                        wm = fmax(wm, fabs(y.x));
                        if (c + 1 < w) wm = fmax(wm, fabs(y.y));
                    }
                }
                wm = warp_max(wm);
                if (lane == 0) atomicMax(&sm.wit[i], (unsigned long long)__double_as_longlong(wm));
            }
        }
        __syncthreads();  // smem (prow chunk, mult/last) is restaged next step
    }

    __syncthreads();
    for (int i = tid; i < nr; i += kThreads)
        p.row_wit[gl][sm.rows[i]] = __longlong_as_double((long long)sm.wit[i]);
}

// out[c][r] = a[r][c] (n x n, out row stride ldo): 32 x 32 tiles through shared memory,
// coalesced on both sides.  The GE mode runs K1 on the transpose (gauss.py's column pivots
// become K1's row pivots; the arithmetic is the same, see mcnd_logdet_lu).
__global__ void __launch_bounds__(256) transpose_kernel(const double* __restrict__ a, int64_t n, int64_t lda,
                                                        double* __restrict__ out, int64_t ldo) {
    __shared__ double t[32][33];
    const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
#pragma unroll
    for (int k = 0; k < 32; k += 8) {
        const int64_t r = r0 + ty + k, c = c0 + tx;
        if (r < n && c < n) t[ty + k][tx] = a[r * lda + c];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 32; k += 8) {
        const int64_t r = c0 + ty + k, c = r0 + tx;  // out row = a column
        if (r < n && c < n) out[r * ldo + c] = t[tx][ty + k];
    }
}

}  // namespace

cudaError_t transpose_launch(const double* a, int64_t n, int64_t lda, double* out, int64_t ldo, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    const unsigned nb = (unsigned)((n + 31) / 32);
    transpose_kernel<<<dim3(nb, nb), 256, 0, s>>>(a, n, lda, out, ldo);
    return cudaGetLastError();
}

size_t k1_smem_bytes(int chunk) { return (size_t)(chunk + 2) * sizeof(double); }

cudaError_t k1_launch(const K1Params& p, bool fast, cudaStream_t s) {
    const size_t smem = k1_smem_bytes(p.chunk);
    const void* fn = fast ? (const void*)k1_condense<true> : (const void*)k1_condense<false>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kThreads, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    K1Params pc = p;
    void* args[] = {&pc};
    const int grid = p.n_local_groups * p.ctas_per_group;
    // Cooperative launch guarantees co-residency of all CTAs, which the
    // publish/wait dataflow between CTAs relies on.
    return cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kThreads), args, smem, s);
}

}  // namespace mcnd

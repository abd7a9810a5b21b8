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
// holds U in the FINAL layout: W = T^{-1} U is a back substitution in shared
// memory, written straight to global.  CTA 0 derives the panel-start column
// of each pivot and the <= b moved columns for the trailing-row gather.
#include <cstdint>
#include <climits>
#include "mcnd_internal.h"

namespace mcnd {
namespace {

constexpr int kB = kK2B;
constexpr int kThreads = 1024;
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

__device__ __forceinline__ double2 pack(double v, unsigned tag, int aux) {
    return make_double2(v, __longlong_as_double((long long)(((unsigned long long)tag << 32) | (unsigned)aux)));
}
__device__ __forceinline__ unsigned tag_of(double2 r) {
    return (unsigned)((unsigned long long)__double_as_longlong(r.y) >> 32);
}
__device__ __forceinline__ int aux_of(double2 r) { return (int)(unsigned)__double_as_longlong(r.y); }
__device__ __forceinline__ void put(double2* p, double2 v) { __stcg(p, v); }
__device__ __forceinline__ double2 get(const double2* p) { return __ldcg(p); }

#ifndef KP_TRACE
#define KP_TRACE 0  // microbenchmark knob: record per-step phase timestamps of CTA 0
#endif
#if KP_TRACE
__device__ unsigned long long g_kp_trace[64][8];
#define KP_MARK(s, k) do { if (blockIdx.x == 0 && threadIdx.x == 0) g_kp_trace[s][k] = clock64(); } while (0)
#else
#define KP_MARK(s, k) do { } while (0)
#endif

__global__ void __launch_bounds__(kThreads, 1) kp_panel_kernel(const KPParams p) {
    extern __shared__ __align__(16) double S[];  // [kB][cw]
    __shared__ double sT[kB][kB + 1];
    __shared__ double s_mult2[2][kB], s_last2[2][kB];  // by step parity: warp 0 fetches step s
                                                       // while the bulk of step s-1 still reads
    __shared__ double s_rmax[kB], s_rmax2[kB];
    __shared__ double s_lv[4], s_lm[4];
    __shared__ int s_li[4];
    __shared__ int s_l[kB];
    __shared__ double s_cv, s_win_v, s_win_w;
    __shared__ int s_cpos, s_win_l, s_win_g, s_stop;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = blockIdx.x, G = p.G, cw = p.cw, m = p.m;
    const int lo = g * cw;
    const int wc = max(0, min(cw, m - lo));  // my columns at panel start
    const unsigned long long t_start = globaltimer();
    if (*(volatile const unsigned*)p.abort) return;

    // ---- load my chunk of the 64 panel rows; running max per row; candidate of row 0
    for (int e = tid; e < kB * wc; e += kThreads) {
        const int r = e / wc, c = e - r * wc;
        S[r * cw + c] = p.ws[(int64_t)(p.row0 + r) * p.ld + lo + c];
    }
    if (tid == 0) s_stop = 0;
    if (g == 0 && tid == 0) p.pan->n_moved = 0;
    __syncthreads();
    {
        const int r = tid >> 4, j = tid & 15;  // 64 rows x 16 threads (half warps)
        const unsigned hm = 0xffffu << (lane & 16);
        double mx = 0.0, bv = 0.0;
        int bi = INT_MAX;
        for (int c = j; c < wc; c += 16) {
            const double x = S[r * cw + c];
            mx = fmax(mx, fabs(x));
            if (r == 0 && beats(x, lo + c, bv, bi)) { bv = x; bi = lo + c; }
        }
#pragma unroll
        for (int o = 8; o; o >>= 1) {
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
        put(p.colbuf + (int64_t)g * kB + tid, pack(pos != INT_MAX ? S[tid * cw + (pos - lo)] : 0.0, p.tag0, 0));
        if (lo <= m - 1 && m - 1 < lo + wc) put(p.lastbuf + tid, pack(S[tid * cw + (m - 1 - lo)], p.tag0, 0));
        if (tid == 0) put(p.cand + g, pack(s_cv, p.tag0, pos));
        if (tid == 1) put(p.wrec + g, pack(s_rmax[0], p.tag0, 0));
    }

    for (int s = 0; s < kB; ++s) {
        const int ms = m - s;  // active width before pivot s
        const unsigned tag = p.tag0 + (unsigned)s;
        double* const s_mult = s_mult2[s & 1];
        double* const s_last = s_last2[s & 1];
        KP_MARK(s, 0);
        // ---- A. reduce the G proposals for pivot s: warp 0 polls all tagged records
        if (warp == 0) {
            constexpr int kPer = kKPMaxG / 32;
            double2 c[kPer], w[kPer];
            unsigned need = 0;  // bit k: record lane + 32k still missing
#pragma unroll
            for (int k = 0; k < kPer; ++k)
                if (lane + 32 * k < G) need |= 1u << k;
            for (;;) {
#pragma unroll
                for (int k = 0; k < kPer; ++k)
                    if (need & (1u << k)) {
                        c[k] = get(p.cand + s * G + lane + 32 * k);
                        w[k] = get(p.wrec + s * G + lane + 32 * k);
                    }
#pragma unroll
                for (int k = 0; k < kPer; ++k)
                    if ((need & (1u << k)) && tag_of(c[k]) == tag && tag_of(w[k]) == tag) need &= ~(1u << k);
                if (__all_sync(kFull, need == 0)) break;
                if (globaltimer() - t_start > p.timeout_ns) {
                    if (lane == 0) {
                        atomicExch(&p.err->error, 1u);
                        atomicExch(&p.err->err_step, (unsigned)(p.row0 + s));
                        s_stop = 1;
                    }
                    break;
                }
            }
            double bv = 0.0, bw = 0.0;
            int bi = INT_MAX, bg = 0;
#pragma unroll
            for (int k = 0; k < kPer; ++k) {
                const int h = lane + 32 * k;
                if (h < G) {
                    if (beats(c[k].x, aux_of(c[k]), bv, bi)) { bv = c[k].x; bi = aux_of(c[k]); bg = h; }
                    bw = fmax(bw, w[k].x);
                }
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                const double ov = __shfl_xor_sync(kFull, bv, o);
                const int oi = __shfl_xor_sync(kFull, bi, o);
                const int og = __shfl_xor_sync(kFull, bg, o);
                const double ow = __shfl_xor_sync(kFull, bw, o);
                if (beats(ov, oi, bv, bi)) { bv = ov; bi = oi; bg = og; }
                bw = fmax(bw, ow);
            }
            bw = fmax(bw, p.wit[p.row0 + s]);
            // the winner's column (multipliers of rows > s, T entries of rows < s) and the
            // last active column: fetched right here by warp 0, two rows per lane
            if (fabs(bv) > kSingularRtol * bw) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int r = lane + 32 * h;
                    const double2* pm = p.colbuf + ((int64_t)s * G + bg) * kB + r;
                    const double2* pl = p.lastbuf + s * kB + r;
                    double2 cm = get(pm), cl = get(pl);
                    while (tag_of(cm) != tag || tag_of(cl) != tag) {
                        if (globaltimer() - t_start > p.timeout_ns) {
                            atomicExch(&p.err->error, 1u);
                            s_stop = 1;
                            break;
                        }
                        cm = get(pm);
                        cl = get(pl);
                    }
                    s_mult[r] = cm.x;
                    s_last[r] = cl.x;
                }
            }
            if (lane == 0) {
                s_win_v = bv;
                s_win_l = bi;
                s_win_g = bg;
                s_win_w = bw;
            }
        }
        __syncthreads();
        KP_MARK(s, 1);
        if (s_stop) return;
        const double v = s_win_v;
        const int l = s_win_l;
        if (!(fabs(v) > kSingularRtol * s_win_w)) {  // condense.py:90 -> singular
            if (g == 0 && tid == 0) {
                p.rec[s].v = v;
                p.rec[s].l = -1;
                p.rec[s].flag = p.epoch;
                atomicExch(p.abort, 1u);
            }
            return;
        }
        const int wn = max(0, min(wc, ms - 1 - lo));  // my active columns after the step
        KP_MARK(s, 7);
        // ---- B. column exchange (condense.py:104-107): position l takes the last column
        //         on every row (one element per row); row s scaled by true division
        //         (condense.py:110); T column; the pivot record
        if (tid < kB) {
            if (l >= lo && l - lo < wn) S[tid * cw + (l - lo)] = (tid == s) ? __ddiv_rn(s_last[s], v) : s_last[tid];
            if (tid < s) sT[tid][s] = s_mult[tid];  // T[t][s] = u_t(p_s), t < s
        }
        for (int c = tid; c < wn; c += kThreads)
            if (lo + c != l) S[s * cw + c] = __ddiv_rn(S[s * cw + c], v);
        if (g == 0 && tid == 0) {
            p.rec[s].v = v;
            p.rec[s].l = l;
            p.rec[s].flag = p.epoch;
        }
        if (tid == 0) s_l[s] = l;
        __syncthreads();
        KP_MARK(s, 2);
        KP_MARK(s, 3);
        if (s + 1 == kB) break;
        const double* us = S + s * cw;
        // ---- D1. lookahead (warps 0-3): update row s+1, its running max, next candidate
        constexpr int kLA = 64;   // publishing threads (D2)
        constexpr int kD1 = 128;  // row s+1 update threads
        if (tid < kD1) {
            const double mu = s_mult[s + 1];
            double* row = S + (s + 1) * cw;
            double mx = 0.0, bv = 0.0;
            int bi = INT_MAX;
            for (int c = tid; c < wn; c += kD1) {
                const double y = __dsub_rn(row[c], __dmul_rn(mu, us[c]));
                row[c] = y;
                mx = fmax(mx, fabs(y));
                if (beats(y, lo + c, bv, bi)) { bv = y; bi = lo + c; }
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                mx = fmax(mx, __shfl_xor_sync(kFull, mx, o));
                const double ov = __shfl_xor_sync(kFull, bv, o);
                const int oi = __shfl_xor_sync(kFull, bi, o);
                if (beats(ov, oi, bv, bi)) { bv = ov; bi = oi; }
            }
            if (lane == 0) { s_lv[warp] = bv; s_li[warp] = bi; s_lm[warp] = mx; }
            asm volatile("bar.sync 1, %0;" ::"n"(kD1));
            if (tid == 0) {
                double v0 = s_lv[0], m0 = s_lm[0];
                int i0 = s_li[0];
#pragma unroll
                for (int k = 1; k < kD1 / 32; ++k) {
                    if (beats(s_lv[k], s_li[k], v0, i0)) { v0 = s_lv[k]; i0 = s_li[k]; }
                    m0 = fmax(m0, s_lm[k]);
                }
                s_cv = v0;
                s_cpos = i0;
                s_rmax[s + 1] = fmax(fmax(s_rmax[s + 1], s_rmax2[s + 1]), m0);
            }
        }
        __syncthreads();
        KP_MARK(s, 5);
        const int pos = s_cpos;                                   // candidate column of pivot s+1
        const int pc = (pos != INT_MAX) ? pos - lo : -1;          // local
        const int lc = (ms - 2 >= lo && ms - 2 - lo < wn) ? ms - 2 - lo : -1;  // new last column, local
        const unsigned tag1 = tag + 1u;
        if (tid < kLA) {
            // ---- D2. publish pivot s+1's proposal (one row per thread): rows > s+1 get
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
                put(p.lastbuf + (s + 1) * kB + r, pack(xl, tag1, 0));
            }
            put(p.colbuf + ((int64_t)(s + 1) * G + g) * kB + r, pack(xc, tag1, 0));
            if (r > s + 1) s_rmax2[r] = fmax(s_rmax2[r], mx);
            if (r == 1) put(p.wrec + (s + 1) * G + g, pack(s_rmax[s + 1], tag1, 0));
            if (r == 0) put(p.cand + (s + 1) * G + g, pack(s_cv, tag1, pos));
            KP_MARK(s, 6);
        } else {
            // ---- E. bulk (warps 2..31): rows > s+1, all columns except pc / lc, with the
            //         reference's two roundings (condense.py:118); per-row maxima by a
            //         two-segment warp reduction
            const int total = (kB - 2 - s) * wn;
            constexpr int kBulk = kThreads - kLA;
            for (int e0 = tid - kLA - lane; e0 < total; e0 += kBulk) {
                const int e = e0 + lane;
                double mx = 0.0;
                int r = INT_MAX;
                if (e < total) {
                    r = s + 2 + e / wn;
                    const int c = e - (r - s - 2) * wn;
                    if (c != pc && c != lc) {
                        const double y = __dsub_rn(S[r * cw + c], __dmul_rn(s_mult[r], us[c]));
                        S[r * cw + c] = y;
                        mx = fabs(y);
                    }
                }
                const int ra = __shfl_sync(kFull, r, 0);
                double ma = (r == ra) ? mx : 0.0, mb = (r == ra) ? 0.0 : mx;
#pragma unroll
                for (int o = 16; o; o >>= 1) {
                    ma = fmax(ma, __shfl_xor_sync(kFull, ma, o));
                    mb = fmax(mb, __shfl_xor_sync(kFull, mb, o));
                }
                const int rb = __shfl_sync(kFull, r, 31);
                if (lane == 0)
                    atomicMax(reinterpret_cast<unsigned long long*>(s_rmax) + ra,
                              (unsigned long long)__double_as_longlong(ma));
                if (lane == 31 && rb != ra && rb != INT_MAX)
                    atomicMax(reinterpret_cast<unsigned long long*>(s_rmax) + rb,
                              (unsigned long long)__double_as_longlong(mb));
            }
        }
        KP_MARK(s, 4);
    }
    __syncthreads();

    // ---- W = T^{-1} U on my final columns (T unit upper triangular), right-looking
    const int wf = max(0, min(wc, m - kB - lo));
    for (int s = kB - 1; s >= 1; --s) {
        for (int e = tid; e < s * wf; e += kThreads) {
            const int t = e / wf, c = e - t * wf;
            S[t * cw + c] = fma(-sT[t][s], S[s * cw + c], S[t * cw + c]);
        }
        __syncthreads();
    }
    for (int e = tid; e < kB * wf; e += kThreads) {
        const int t = e / wf, c = e - t * wf;
        p.W[(int64_t)t * p.ldw + lo + c] = S[t * cw + c];
    }
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
}

}  // namespace

size_t kp_smem_bytes(int cw) { return (size_t)kB * cw * sizeof(double); }

cudaError_t kp_launch(const KPParams& p, cudaStream_t s) {
    const size_t smem = kp_smem_bytes(p.cw);
    cudaError_t e = cudaFuncSetAttribute(kp_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    KPParams pc = p;
    void* args[] = {&pc};
    return cudaLaunchCooperativeKernel((const void*)kp_panel_kernel, dim3(p.G), dim3(kThreads), args, smem, s);
}

}  // namespace mcnd

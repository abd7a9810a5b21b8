// K2: blocked rank-b condensation (b = 64) with the trailing update on FP64
// tensor cores (sm_100a DMMA via mma.sync.m8n8k4.f64 -- tcgen05 has no f64 kind).
//
// The paper leaves block condensation to future work; the
// unblocked step it generalises is condense_step (mcnd/condense.py:95-131).
// Per panel of b pivot rows (top-to-bottom order, identical pivot rule):
//
//   1-3. panel factorisation (k2_panel.cu): the unblocked steps on the b panel
//      rows, column-distributed over all SMs with the panel in shared memory,
//      so every panel pivot is chosen by the reference's rule (argmax |.|,
//      ties -> lowest column, witness test).  It also yields T[t][s] = u_t(p_s)
//      (unit upper triangular), W = T^{-1} U in the final column layout, the
//      panel-start column p_s of every pivot and the <= b final columns whose
//      source moved (composition of the column exchanges of condense.py:104-107);
//   4. k2_gather_fix: per trailing row, L[r, s] = A[r, p_s] (the b multiplier
//      columns), then the moved columns A[r, c] <- A[r, pi(c)];
//   5. k2_gemm: A[R, 0:m-b] -= L W on DMMA, in place, with the running row
//      witness (condense.py:120-122) fused into the epilogue (at panel
//      granularity -- documented weakening for singular inputs).
//
// In exact arithmetic this is the unblocked result: coef_{r,s} (the step-s
// multiplier of row r) satisfies coef T = A[r, P], and the b rank-1 updates
// sum to coef U = A[r, P] T^{-1} U = L W.  Rounding differs (tolerance parity).
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include "mcnd_internal.h"

namespace mcnd {
namespace {

constexpr int kMaxDevices = 64;
int device_sms(int dev) {  // SM count per device (cached; calls are serialised by the host runtime)
    static int cache[kMaxDevices] = {};
    if (dev < 0 || dev >= kMaxDevices) return 148;
    if (!cache[dev]) cudaDeviceGetAttribute(&cache[dev], cudaDevAttrMultiProcessorCount, dev);
    return cache[dev] > 0 ? cache[dev] : 148;
}


// One warp per trailing row: L[r, 0:K] = A[r, P], then the moved columns.
template <int K>
__global__ void k2_gather_fix_kernel(double* __restrict__ ws, int64_t ld, int32_t rbase, int32_t nrows,
                                     const K2Gather* __restrict__ gp, double* __restrict__ L,
                                     const unsigned* __restrict__ abort) {
    if (*(volatile const unsigned*)abort) return;
    const int lane = threadIdx.x & 31;
    const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (i >= nrows) return;
    double* row = ws + (int64_t)(rbase + i) * ld;
    constexpr int KL = K / 32;
    double x[KL];
#pragma unroll
    for (int k = 0; k < KL; ++k) x[k] = row[gp->P[lane + 32 * k]];
    const int nm = gp->n_moved;
    double v[KL];
#pragma unroll
    for (int k = 0; k < KL; ++k) v[k] = (lane + 32 * k < nm) ? row[gp->moved_src[lane + 32 * k]] : 0.0;
    __syncwarp();
#pragma unroll
    for (int k = 0; k < KL; ++k) L[(int64_t)i * K + lane + 32 * k] = -x[k];  // stored negated: C + L W
#pragma unroll
    for (int k = 0; k < KL; ++k)
        if (lane + 32 * k < nm) row[gp->moved_c[lane + 32 * k]] = v[k];
}

// Pair gather fused with the L correction: per trailing row (one warp),
// NL = -A[r, P[0:128]] and the moved columns fixed as in k2_gather_fix_kernel<128>,
// then NL[64:128] += NL[0:64] * Wp (Wp = -W_k[:, P_{k+1}], staged in shared memory)
// as 64 sequential FMAs per output -- replacing the separate 64-wide GEMM launch.
constexpr int kGLThreads = 256;
__global__ void __launch_bounds__(kGLThreads) k2_gather_lcorr_kernel(double* __restrict__ ws, int64_t ld, int32_t rbase,
                                                                     int32_t nrows, const K2Gather* __restrict__ gp,
                                                                     double* __restrict__ L, int64_t ldl,
                                                                     const double* __restrict__ Wp,
                                                                     const unsigned* __restrict__ abort) {
    __shared__ double sWp[64 * 64];
    if (*(volatile const unsigned*)abort) return;
    const int lane = threadIdx.x & 31;
    const int stride = gridDim.x * (kGLThreads / 32);
    int i = blockIdx.x * (kGLThreads / 32) + (threadIdx.x >> 5);
    // the descriptor, Wp and this warp's first row are all requested before anything waits
    const int nm = gp->n_moved;
    int pk[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) pk[k] = gp->P[lane + 32 * k];
    const int mc0 = lane < nm ? gp->moved_c[lane] : 0, ms0 = lane < nm ? gp->moved_src[lane] : 0;
    const int mc1 = lane + 32 < nm ? gp->moved_c[lane + 32] : 0, ms1 = lane + 32 < nm ? gp->moved_src[lane + 32] : 0;
    const int mc2 = lane + 64 < nm ? gp->moved_c[lane + 64] : 0, ms2 = lane + 64 < nm ? gp->moved_src[lane + 64] : 0;
    const int mc3 = lane + 96 < nm ? gp->moved_c[lane + 96] : 0, ms3 = lane + 96 < nm ? gp->moved_src[lane + 96] : 0;
    double x[4], v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;
    auto gather = [&](int r) {
        const double* row = ws + (int64_t)(rbase + r) * ld;
#pragma unroll
        for (int k = 0; k < 4; ++k) x[k] = row[pk[k]];
        v0 = lane < nm ? row[ms0] : 0.0;
        v1 = lane + 32 < nm ? row[ms1] : 0.0;
        v2 = lane + 64 < nm ? row[ms2] : 0.0;
        v3 = lane + 96 < nm ? row[ms3] : 0.0;
    };
    if (i < nrows) gather(i);
    {   // Wp staged with all 16 loads per thread in flight (one L2 round trip, not 16)
        constexpr int kPer = 64 * 64 / kGLThreads;
        double w[kPer];
#pragma unroll
        for (int u = 0; u < kPer; ++u) w[u] = __ldg(Wp + threadIdx.x + kGLThreads * u);
#pragma unroll
        for (int u = 0; u < kPer; ++u) sWp[threadIdx.x + kGLThreads * u] = w[u];
    }
    __syncthreads();
    for (; i < nrows; i += stride) {
        double* row = ws + (int64_t)(rbase + i) * ld;
        __syncwarp();
        if (lane < nm) row[mc0] = v0;
        if (lane + 32 < nm) row[mc1] = v1;
        if (lane + 64 < nm) row[mc2] = v2;
        if (lane + 96 < nm) row[mc3] = v3;
        const double n00 = -x[0], n01 = -x[1];
        // four independent FMA chains per output (k even / odd of each half), summed at the end
        double a10 = -x[2], a11 = -x[3], b10 = 0.0, b11 = 0.0, c10 = 0.0, c11 = 0.0, d10 = 0.0, d11 = 0.0;
#pragma unroll 8
        for (int k = 0; k < 32; k += 2) {
            const double e0 = __shfl_sync(0xffffffffu, n00, k), e1 = __shfl_sync(0xffffffffu, n00, k + 1);
            a10 = fma(e0, sWp[k * 64 + lane], a10);
            a11 = fma(e0, sWp[k * 64 + lane + 32], a11);
            b10 = fma(e1, sWp[(k + 1) * 64 + lane], b10);
            b11 = fma(e1, sWp[(k + 1) * 64 + lane + 32], b11);
        }
#pragma unroll 8
        for (int k = 0; k < 32; k += 2) {
            const double e0 = __shfl_sync(0xffffffffu, n01, k), e1 = __shfl_sync(0xffffffffu, n01, k + 1);
            c10 = fma(e0, sWp[(k + 32) * 64 + lane], c10);
            c11 = fma(e0, sWp[(k + 32) * 64 + lane + 32], c11);
            d10 = fma(e1, sWp[(k + 33) * 64 + lane], d10);
            d11 = fma(e1, sWp[(k + 33) * 64 + lane + 32], d11);
        }
        const double n10 = (a10 + b10) + (c10 + d10), n11 = (a11 + b11) + (c11 + d11);
        if (i + stride < nrows) gather(i + stride);  // the next row's loads overlap the stores below
        double* Lr = L + (int64_t)i * ldl;
        Lr[lane] = n00;
        Lr[lane + 32] = n01;
        Lr[lane + 64] = n10;
        Lr[lane + 96] = n11;
    }
}


// ---- DMMA GEMM: C[M x N2] (rows rbase.., in ws) += NL[M x K] * W[K x N2], K = 64 or 128, where
// NL = -L is stored negated by the gather so the DMMA operands carry no negation (keeps the
// A-operand register reuse cache usable) ----
constexpr int BM = 64, BN = 128;             // tile rows / cols
constexpr int LDWS = BN + 4;                 // = 4 (mod 16): the B fragment (lanes 4q+g) hits 16 distinct bank pairs per half-warp

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}

// zero-filling form: src_bytes = 0 writes 16 zero bytes and reads nothing
__device__ __forceinline__ void cp_async16_zf(void* smem, const void* gmem, bool valid) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(gmem), "r"(valid ? 16 : 0) : "memory");
}

// ---- multistage variant: 2 CTAs per SM, K consumed in stages of 16 through a
// 4-deep cp.async ring (CUTLASS-style multistage mainloop).  The C tile is loaded
// into the accumulators at the start of each tile: its latency is hidden by the
// other CTA on the SM, so a CTA-wide barrier never idles the whole SM's tensor
// pipe.  Persistent over a contiguous, row-block-major tile range per CTA so the
// witness maxima are flushed once per row block.
constexpr int MS_BK = 16, MS_ST = 4;          // K per stage, ring depth
constexpr int MS_LDL = MS_BK + 4;             // 20 doubles: conflict-free A fragments
constexpr int MS_STAGE = BM * MS_LDL + MS_BK * LDWS;

// SUB = 2: a "fat" CTA of two independent 256-thread sub-CTAs (own smem ring, own named
// barrier) that fills a whole SM, so a grid of B fat CTAs occupies exactly B SMs and
// leaves the rest free for the panel kernel running concurrently on another stream.
// BNT: tile width, 128 (8 warps, 2 x 4 of 32 x 32) or 64 (4 warps, 2 x 2): the narrow tiles
// double the CTA count of a short (critical-path) update so more SMs share it.
template <int K, int SUB, int BNT = BN>
__global__ void __launch_bounds__(64 * (BNT / 32) * SUB, 2 / SUB) k2_gemm_ms_kernel(double* __restrict__ ws, int64_t ld, int32_t rbase,
                                                                   int32_t M, int32_t N2, const double* __restrict__ L,
                                                                   int64_t ldl, const double* __restrict__ W, int64_t ldw,
                                                                   unsigned long long* __restrict__ wit,
                                                                   const unsigned* __restrict__ abort) {
    constexpr int KS = K / MS_BK;  // stages per tile
    constexpr int WN = BNT / 32, NJ = 4, NTH = 64 * WN;  // warps in N, 8x8 tiles per warp in N, threads
    constexpr int LDW_T = BNT + 4, STAGE_T = BM * MS_LDL + MS_BK * LDW_T;
    extern __shared__ __align__(16) double sh_all[];
    if (*(volatile const unsigned*)abort) return;
    const int sub = SUB == 2 ? (int)(threadIdx.x >= NTH) : 0;
    double* const sh = sh_all + sub * (MS_ST * STAGE_T);
    auto sync = [&]() {
        if constexpr (SUB == 1) __syncthreads();
        else asm volatile("bar.sync %0, %1;" ::"r"(1 + sub), "n"(NTH) : "memory");
    };
    const int tid = (int)threadIdx.x - sub * NTH, lane = tid & 31, warp = tid >> 5;
    const int wm = warp / WN, wn = warp % WN;
    const int g = lane >> 2, q = lane & 3;
    const int ntn = (N2 + BNT - 1) / BNT, ntm = (M + BM - 1) / BM;
    const int64_t T = (int64_t)ntn * ntm;
    const int64_t vb = (int64_t)blockIdx.x * SUB + sub, vg = (int64_t)gridDim.x * SUB;
    const int64_t t_begin = T * vb / vg, t_end = T * (vb + 1) / vg;
    if (t_begin >= t_end) return;
    const int64_t nst = (t_end - t_begin) * KS;

    auto load_stage = [&](int64_t j) {
        if (j < nst) {
            const int64_t t = t_begin + j / KS;
            const int kk = (int)(j % KS) * MS_BK;
            const int row0 = (int)(t / ntn) * BM, col0 = (int)(t % ntn) * BNT;
            double* ls = sh + (int)(j % MS_ST) * STAGE_T;
            double* wsm = ls + BM * MS_LDL;
            for (int i = tid; i < BM * (MS_BK / 2); i += NTH) {
                const int r = i / (MS_BK / 2), c2 = i % (MS_BK / 2);
                double* dst = ls + r * MS_LDL + 2 * c2;
                if (row0 + r < M) cp_async16(dst, L + (int64_t)(row0 + r) * ldl + kk + 2 * c2);
                else { dst[0] = 0.0; dst[1] = 0.0; }
            }
            for (int i = tid; i < MS_BK * (BNT / 2); i += NTH) {
                const int k = i / (BNT / 2), c2 = i % (BNT / 2);
                const int col = col0 + 2 * c2;
                double* dst = wsm + k * LDW_T + 2 * c2;
                if (col < N2) cp_async16(dst, W + (int64_t)(kk + k) * ldw + col);
                else { dst[0] = 0.0; dst[1] = 0.0; }
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");  // (possibly empty) group keeps the count
    };

    // C tiles are pulled into L2 ahead of use (the first at entry, each next one
    // mid-way through the current tile): the accumulator load then hits L2
    auto prefetch_c = [&](int64_t t) {
        const int row0 = (int)(t / ntn) * BM, col0 = (int)(t % ntn) * BNT;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int r = row0 + wm * 32 + i * 8 + g;
            if (r < M && q == 0) {
                const double* crow = ws + (int64_t)(rbase + r) * ld + col0 + wn * 32;
                asm volatile("prefetch.global.L2 [%0];" ::"l"(crow));
                if (col0 + wn * 32 + 16 < N2) asm volatile("prefetch.global.L2 [%0];" ::"l"(crow + 16));
            }
        }
    };
    prefetch_c(t_begin);
#pragma unroll
    for (int j = 0; j < MS_ST - 1; ++j) load_stage(j);
    double rmx[4] = {0.0, 0.0, 0.0, 0.0};
    double acc[4][NJ][2];
    for (int64_t j = 0; j < nst; ++j) {
        const int64_t t = t_begin + j / KS;
        const int ks = (int)(j % KS);
        const int row0 = (int)(t / ntn) * BM, col0 = (int)(t % ntn) * BNT;
        if (ks == 0) {  // C tile -> accumulators (acc = C - L W)
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int r = row0 + wm * 32 + i * 8 + g;
                const double* crow = ws + (int64_t)(rbase + r) * ld;
#pragma unroll
                for (int jj = 0; jj < NJ; ++jj) {
                    const int c = col0 + wn * 32 + jj * 8 + 2 * q;
                    if (r < M && c < N2) {
                        const double2 v = __ldcs(reinterpret_cast<const double2*>(crow + c));
                        acc[i][jj][0] = v.x;
                        acc[i][jj][1] = v.y;
                    } else {
                        acc[i][jj][0] = 0.0;
                        acc[i][jj][1] = 0.0;
                    }
                }
            }
        }
        if (ks == KS / 2 && t + 1 < t_end) prefetch_c(t + 1);
        asm volatile("cp.async.wait_group %0;" ::"n"(MS_ST - 2) : "memory");
        sync();  // stage j landed; buffer (j-1) % MS_ST is free
        load_stage(j + MS_ST - 1);
        const double* ls = sh + (int)(j % MS_ST) * STAGE_T;
        const double* wsm = ls + BM * MS_LDL;
#pragma unroll
        for (int k0 = 0; k0 < MS_BK; k0 += 4) {
            double a[4], b[NJ];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = ls[(wm * 32 + i * 8 + g) * MS_LDL + k0 + q];
#pragma unroll
            for (int jj = 0; jj < NJ; ++jj) b[jj] = wsm[(k0 + q) * LDW_T + wn * 32 + jj * 8 + g];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int jj = 0; jj < NJ; ++jj) dmma(acc[i][jj][0], acc[i][jj][1], a[i], b[jj]);
        }
        if (ks != KS - 1) continue;
        const int bm = (int)(t / ntn);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int r = row0 + wm * 32 + i * 8 + g;
            double* crow = ws + (int64_t)(rbase + r) * ld;
#pragma unroll
            for (int jj = 0; jj < NJ; ++jj) {
                const int c = col0 + wn * 32 + jj * 8 + 2 * q;
                if (r < M && c < N2) {
                    if (c + 1 < N2) {
                        __stcs(reinterpret_cast<double2*>(crow + c), make_double2(acc[i][jj][0], acc[i][jj][1]));
                        rmx[i] = fmax(rmx[i], fmax(fabs(acc[i][jj][0]), fabs(acc[i][jj][1])));
                    } else {
                        crow[c] = acc[i][jj][0];
                        rmx[i] = fmax(rmx[i], fabs(acc[i][jj][0]));
                    }
                }
            }
        }
        const bool flush = (t + 1 == t_end) || ((int)((t + 1) / ntn) != bm);
        if (flush && wit) {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                double mx = rmx[i];
                mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
                mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
                const int r = row0 + wm * 32 + i * 8 + g;
                if (q == 0 && r < M) atomicMax(wit + rbase + r, (unsigned long long)__double_as_longlong(mx));
                rmx[i] = 0.0;
            }
        }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
}

// ---- 4-warp variant: 64 x 128 tiles, 2 x 2 warps of 32 x 64 (32 DMMA per 12 fragment
// loads), fragments double-buffered across k-steps and across stages, one barrier per
// stage.  Two CTAs per SM with one warp per SM sub-partition each: every warp alone can
// keep its sub-partition's DMMA pipe busy, so the stall of one CTA (C-tile load,
// epilogue, barrier) is covered by the other.  Same arithmetic as k2_gemm_ms_kernel
// (acc starts at C, DMMA k-steps in k order): bitwise the same result.
constexpr int W4_THREADS = 128;
// WN = warps in N: 2 -> 64 x 128 tiles, 128 threads (the trailing update); 1 -> 64 x 64 tiles,
// 64 threads (the short critical-path update: twice the CTAs)
// U: stages per iteration of the (not unrolled) stage loop -- 2 in the persistent grid (the
// compiler keeps the accumulators in place across the pair: 28.15 -> 28.67 TF at n = 16384,
// scripts/micro/gemm_w5.cu), 1 for one tile per CTA (2 is 0.5 % slower there)
// K = 256 (a group of two pairs): W rows 0..127 from W, rows 128..255 from W1 (same ldw).
template <int K, int S, int WN = 2, int BK = MS_BK, int U = 1>
__global__ void __launch_bounds__(64 * WN, 2) k2_gemm_w4_kernel(double* __restrict__ ws, int64_t ld, int32_t rbase,
                                                                    int32_t M, int32_t N2, const double* __restrict__ L,
                                                                    int64_t ldl, const double* __restrict__ W, int64_t ldw,
                                                                    unsigned long long* __restrict__ wit,
                                                                    const unsigned* __restrict__ abort,
                                                                    const double* __restrict__ W1 = nullptr) {
    constexpr int KS = K / BK, LDA = BK + 4;
    constexpr int MI = 4, NJ = 8;  // warp tile 32 x 64
    constexpr int NTH = 64 * WN, BNW = 64 * WN, LDW = BNW + 4, STG = BM * LDA + BK * LDW;
    constexpr int LR = BM * (BK / 2) / NTH;     // L chunks per thread (rows NTH/(BK/2) apart)
    constexpr int WR = BK * (BNW / 2) / NTH;    // W chunks per thread (rows 2 apart)
    extern __shared__ __align__(16) double sh[];
    if (*(volatile const unsigned*)abort) return;
    const int tid = (int)threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp / WN, wn = warp % WN;
    const int g = lane >> 2, q = lane & 3;
    const int ntn = (N2 + BNW - 1) / BNW, ntm = (M + BM - 1) / BM;
    const int T = ntn * ntm;  // < 2^31 tiles for any n the panel kernel accepts
    const int t_begin = (int)((int64_t)T * blockIdx.x / gridDim.x), t_end = (int)((int64_t)T * (blockIdx.x + 1) / gridDim.x);
    if (t_begin >= t_end) return;

    // Loader state (advanced incrementally: no divisions per stage).  Per thread: L rows
    // tid/8 + (NTH/8)u (u < LR), 16-byte chunk tid%8; W rows tid/(BNW/2) + 2u (u < 8), chunk
    // tid%(BNW/2); out-of-range chunks are zero-filled.
    const int ra = tid / (BK / 2), ca = 2 * (tid % (BK / 2)), kb = tid / (BNW / 2), cb = 2 * (tid % (BNW / 2));
    int l_t = t_begin, l_ks = 0, l_slot = 0;
    const double* l_src = nullptr;  // L + row(u = 0) * ldl + kk + ca
    const double* w_src = nullptr;  // W + (kk + kb) * ldw + col
    const double* w_src1 = nullptr; // W1 + (kk - 128 + kb) * ldw + col (K = 256)
    unsigned l_ok = 0;              // bit u: row u in range; bit 4: column chunk in range
    auto l_tile = [&]() {
        const int row0 = (l_t / ntn) * BM, col0 = (l_t % ntn) * BNW;
        l_ok = 0;
#pragma unroll
        for (int u = 0; u < LR; ++u) l_ok |= (unsigned)(row0 + ra + (NTH / (BK / 2)) * u < M) << u;
        const bool okc = col0 + cb < N2;
        l_ok |= (unsigned)okc << 16;
        l_src = L + (int64_t)(row0 + ra) * ldl + ca;
        w_src = W + (int64_t)kb * ldw + (okc ? col0 + cb : 0);
        if constexpr (K > 128) w_src1 = W1 + (int64_t)kb * ldw + (okc ? col0 + cb : 0);
    };
    auto load_next = [&]() {  // one stage -> slot l_slot, then advance
        if (l_t < t_end) {
            double* ls = sh + l_slot * STG;
            double* wsm = ls + BM * LDA;
            const int kk = l_ks * BK;
#pragma unroll
            for (int u = 0; u < LR; ++u) {
                const bool ok = (l_ok >> u) & 1u;
                cp_async16_zf(ls + (ra + (NTH / (BK / 2)) * u) * LDA + ca, ok ? l_src + (int64_t)((NTH / (BK / 2)) * u) * ldl + kk : L, ok);
            }
            const bool okc = (l_ok >> 16) & 1u;
            const double* wsrc = (K > 128 && kk >= 128) ? w_src1 + (int64_t)(kk - 128) * ldw : w_src + (int64_t)kk * ldw;
#pragma unroll
            for (int u = 0; u < WR; ++u) cp_async16_zf(wsm + (kb + 2 * u) * LDW + cb, wsrc + (int64_t)(2 * u) * ldw, okc);
            if (++l_ks == KS) {
                l_ks = 0;
                if (++l_t < t_end) l_tile();
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");  // (possibly empty) group keeps the count
        l_slot = l_slot + 1 == S ? 0 : l_slot + 1;
    };
    auto prefetch_c = [&](int row0, int col0) {
#pragma unroll
        for (int i = 0; i < MI; ++i) {
            const int r = row0 + wm * 32 + i * 8 + g;
            const int c = col0 + wn * 64 + q * 16;  // the warp's 64 columns of row r: four 128-byte lines
            if (r < M && c < N2) asm volatile("prefetch.global.L2 [%0];" ::"l"(ws + (int64_t)(rbase + r) * ld + c));
        }
    };
    double a[2][MI], b[2][NJ];
    auto load_frags = [&](int buf, int slot, int k0) {
        const double* ls = sh + slot * STG;
        const double* wsm = ls + BM * LDA;
#pragma unroll
        for (int i = 0; i < MI; ++i) a[buf][i] = ls[(wm * 32 + i * 8 + g) * LDA + k0 + q];
#pragma unroll
        for (int jj = 0; jj < NJ; ++jj) b[buf][jj] = wsm[(k0 + q) * LDW + wn * 64 + jj * 8 + g];
    };
    double acc[MI][NJ][2];
    auto load_c = [&](int row0, int col0) {  // C tile -> accumulators (acc = C - L W)
        const bool full = row0 + BM <= M && col0 + BNW <= N2;
#pragma unroll
        for (int i = 0; i < MI; ++i) {
            const int r = row0 + wm * 32 + i * 8 + g;
            const double* crow = ws + (int64_t)(rbase + r) * ld + col0 + wn * 64 + 2 * q;
#pragma unroll
            for (int jj = 0; jj < NJ; ++jj) {
                if (full || (r < M && col0 + wn * 64 + jj * 8 + 2 * q < N2)) {
                    const double2 v = __ldcs(reinterpret_cast<const double2*>(crow + jj * 8));
                    acc[i][jj][0] = v.x;
                    acc[i][jj][1] = v.y;
                } else {
                    acc[i][jj][0] = 0.0;
                    acc[i][jj][1] = 0.0;
                }
            }
        }
    };

    l_tile();
    int t = t_begin, row0 = (t / ntn) * BM, col0 = (t % ntn) * BNW;
    prefetch_c(row0, col0);
#pragma unroll
    for (int j = 0; j < S; ++j) load_next();
    load_c(row0, col0);  // in flight together with the first stages
    asm volatile("cp.async.wait_group %0;" ::"n"(S - 1) : "memory");
    __syncthreads();
    load_frags(0, 0, 0);
    double rmx[MI] = {0.0, 0.0, 0.0, 0.0};
    int c_slot = 0;
    for (;;) {
#pragma unroll U
        for (int ks = 0; ks < KS; ++ks) {
            if (ks == KS / 2 && t + 1 < t_end) {
                const int tn = t + 1;
                prefetch_c((tn / ntn) * BM, (tn % ntn) * BNW);
            }
            const int n_slot = c_slot + 1 == S ? 0 : c_slot + 1;
            const bool more = ks + 1 < KS || t + 1 < t_end;
#pragma unroll
            for (int kq = 0; kq < BK / 4; ++kq) {
                if (kq == BK / 4 - 1) {
                    // the next stage landed; every warp is done reading this one (its last
                    // fragments are in registers), so its slot takes the stage S ahead
                    asm volatile("cp.async.wait_group %0;" ::"n"(S - 2) : "memory");
                    __syncthreads();
                    load_next();
                    if (more) load_frags((kq + 1) & 1, n_slot, 0);
                } else {
                    load_frags((kq + 1) & 1, c_slot, 4 * (kq + 1));
                }
#pragma unroll
                for (int i = 0; i < MI; ++i)
#pragma unroll
                    for (int jj = 0; jj < NJ; ++jj) dmma(acc[i][jj][0], acc[i][jj][1], a[kq & 1][i], b[kq & 1][jj]);
            }
            c_slot = n_slot;
        }
        // epilogue: store the tile, fold the row maxima
        const bool full = row0 + BM <= M && col0 + BNW <= N2;
#pragma unroll
        for (int i = 0; i < MI; ++i) {
            const int r = row0 + wm * 32 + i * 8 + g;
            double* crow = ws + (int64_t)(rbase + r) * ld;
#pragma unroll
            for (int jj = 0; jj < NJ; ++jj) {
                const int c = col0 + wn * 64 + jj * 8 + 2 * q;
                if (full || (r < M && c + 1 < N2)) {
                    __stcs(reinterpret_cast<double2*>(crow + c), make_double2(acc[i][jj][0], acc[i][jj][1]));
                    rmx[i] = fmax(rmx[i], fmax(fabs(acc[i][jj][0]), fabs(acc[i][jj][1])));
                } else if (r < M && c < N2) {
                    crow[c] = acc[i][jj][0];
                    rmx[i] = fmax(rmx[i], fabs(acc[i][jj][0]));
                }
            }
        }
        const int prow0 = row0;
        ++t;
        if (t < t_end) {
            row0 = (t / ntn) * BM;
            col0 = (t % ntn) * BNW;
        }
        if ((t == t_end || row0 != prow0) && wit) {
#pragma unroll
            for (int i = 0; i < MI; ++i) {
                double mx = rmx[i];
                mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
                mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
                const int r = prow0 + wm * 32 + i * 8 + g;
                if (q == 0 && r < M) atomicMax(wit + rbase + r, (unsigned long long)__double_as_longlong(mx));
                rmx[i] = 0.0;
            }
        }
        if (t == t_end) break;
        load_c(row0, col0);
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
}

// ---- a group of two pairs (a, b = a + 1) applied to the rows past b's next pair as ONE
// rank-256 update (the GEMM at K = 256 runs ~9 % faster than two K = 128 updates: per-tile
// C traffic and pipeline fill are amortised over twice the k-steps).  With the rows still in
// the state before a (a's column moves applied by a's gather), b's multipliers need a's update
// of b's pivot columns:  NL_b = lcorr_b(-(x + NL_a W_a[:, P_b])) = lcorr_b(-x) + NL_a Wx,
// Wx = lcorr_b applied to the columns of -W_a[:, P_b] (built here, 128 x 128), and W_a's
// columns take b's column moves (fixed in place once every per-pair user of W_a is done).
__global__ void k2_group_wx_kernel(const double* __restrict__ Wa, int64_t ldw, const K2Gather* __restrict__ gb,
                                   const double* __restrict__ Wpb, double* __restrict__ Wx, const unsigned* __restrict__ abort) {
    __shared__ double t[128];
    if (*(volatile const unsigned*)abort) return;  // a singular panel left no descriptor
    const int j = blockIdx.x, k = threadIdx.x;
    t[k] = -Wa[(int64_t)j * ldw + gb->P[k]];
    __syncthreads();
    double v = t[k];
    if (k >= 64)
        for (int i = 0; i < 64; ++i) v = fma(t[i], Wpb[i * 64 + (k - 64)], v);
    Wx[j * 128 + k] = v;
}

__global__ void k2_group_wfix_kernel(double* __restrict__ Wa, int64_t ldw, const K2Gather* __restrict__ gb,
                                     const unsigned* __restrict__ abort) {
    if (*(volatile const unsigned*)abort) return;
    const int j = blockIdx.x, k = threadIdx.x;
    if (k < gb->n_moved) {  // sources (dropped columns) and destinations are disjoint
        double* const row = Wa + (int64_t)j * ldw;
        row[gb->moved_c[k]] = row[gb->moved_src[k]];
    }
}

}  // namespace

cudaError_t k2_group_prep(double* Wa, int64_t ldw, const K2Gather* gb, const double* Wpb, double* Wx,
                          const unsigned* abort, cudaStream_t s) {
    k2_group_wx_kernel<<<128, 128, 0, s>>>(Wa, ldw, gb, Wpb, Wx, abort);
    k2_group_wfix_kernel<<<128, 128, 0, s>>>(Wa, ldw, gb, abort);
    return cudaGetLastError();
}

cudaError_t k2_gather_fix(double* ws, int64_t ld, int32_t rbase, int32_t nrows, int32_t K, const K2Gather* gp,
                          double* L, const unsigned* abort, cudaStream_t s) {
    if (nrows <= 0) return cudaSuccess;
    const int warps = 8;
    const dim3 grid((nrows + warps - 1) / warps);
    if (K != 64) return cudaErrorInvalidValue;  // the pair path gathers with k2_gather_lcorr
    k2_gather_fix_kernel<64><<<grid, warps * 32, 0, s>>>(ws, ld, rbase, nrows, gp, L, abort);
    return cudaGetLastError();
}

cudaError_t k2_gather_lcorr(double* ws, int64_t ld, int32_t rbase, int32_t nrows, const K2Gather* gp, double* L,
                            const double* Wp, const unsigned* abort, cudaStream_t s, int64_t ldl) {
    if (nrows <= 0) return cudaSuccess;
    int dev = 0;
    cudaGetDevice(&dev);
    const int sms = device_sms(dev);
    const int per = kGLThreads / 32;
    const int grid = (int)std::min<int64_t>(((int64_t)nrows + per - 1) / per, 4 * (int64_t)sms);
    k2_gather_lcorr_kernel<<<grid, kGLThreads, 0, s>>>(ws, ld, rbase, nrows, gp, L, ldl, Wp, abort);
    return cudaGetLastError();
}


cudaError_t k2_gemm(double* ws, int64_t ld, int32_t rbase, int32_t M, int32_t N2, int32_t K, const double* L,
                    int64_t ldl, const double* W, int64_t ldw, double* row_wit, const unsigned* abort, cudaStream_t s,
                    int sm_budget, const double* W1) {
    if (M <= 0 || N2 <= 0) return cudaSuccess;
    if (K != 64 && K != 128 && !(K == 256 && W1)) return cudaErrorInvalidValue;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const int sms = device_sms(dev);
    // shared-memory opt-in: a per-device (context) attribute, set once per device
    static bool attr_done[kMaxDevices] = {};
    const int sm4 = (int)(3 * MS_STAGE * sizeof(double));
    const int smn = (int)((size_t)MS_ST * (BM * MS_LDL + MS_BK * (64 + 4)) * sizeof(double));
    if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
    if (!attr_done[dev]) {
        if ((e = cudaFuncSetAttribute(k2_gemm_w4_kernel<64, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm4)) != cudaSuccess ||
            (e = cudaFuncSetAttribute(k2_gemm_w4_kernel<128, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm4)) != cudaSuccess ||
            (e = cudaFuncSetAttribute(k2_gemm_w4_kernel<128, 3, 2, MS_BK, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm4)) != cudaSuccess ||
            (e = cudaFuncSetAttribute(k2_gemm_w4_kernel<256, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm4)) != cudaSuccess ||
            (e = cudaFuncSetAttribute(k2_gemm_w4_kernel<256, 3, 2, MS_BK, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm4)) != cudaSuccess ||
            (e = cudaFuncSetAttribute(k2_gemm_ms_kernel<128, 1, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smn)) != cudaSuccess)
            return e;
        attr_done[dev] = true;
    }
    auto* w = reinterpret_cast<unsigned long long*>(row_wit);
    if (sm_budget == 0 && M <= 2 * BM && K == 128) {
        // a short critical-path update (the next pair's 128 rows): 64 x 64 tiles, twice the
        // CTAs of the 64 x 128 kernel, so more SMs share it (measured faster than the 4-warp
        // kernel with 64-wide tiles: 24.6 vs 25.1 us at m = 8000, and inside C3/C5)
        const int64_t tiles_n = (int64_t)((N2 + 63) / 64) * ((M + BM - 1) / BM);
        k2_gemm_ms_kernel<128, 1, 64><<<(int)tiles_n, 128, smn, s>>>(ws, ld, rbase, M, N2, L, ldl, W, ldw, w, abort);
        return cudaGetLastError();
    }
    // 4-warp kernel (64 x 128 tiles, 32 x 64 warp tiles).  An overlapped (side, sm_budget < 0)
    // update runs one tile per CTA, so SMs go back to the next panel tile by tile, unless it is
    // more than 40 waves of 2 CTAs per SM: then the GEMM, not the panel chain, bounds the pair
    // and a persistent grid (no per-CTA pipeline fill) is faster.  Critical-stream updates
    // (sm_budget >= 0) always run persistent.
    const int64_t tiles = (int64_t)((N2 + BN - 1) / BN) * ((M + BM - 1) / BM);
    const bool one_tile = sm_budget < 0 && tiles * K <= 40 * 2 * (int64_t)sms * 128;
    const int g4 = (int)(one_tile ? tiles : std::min<int64_t>(tiles, 2 * (int64_t)sms));
    if (K == 256) {
        if (one_tile) k2_gemm_w4_kernel<256, 3><<<g4, W4_THREADS, sm4, s>>>(ws, ld, rbase, M, N2, L, ldl, W, ldw, w, abort, W1);
        else k2_gemm_w4_kernel<256, 3, 2, MS_BK, 2><<<g4, W4_THREADS, sm4, s>>>(ws, ld, rbase, M, N2, L, ldl, W, ldw, w, abort, W1);
    } else if (K == 64) k2_gemm_w4_kernel<64, 3><<<g4, W4_THREADS, sm4, s>>>(ws, ld, rbase, M, N2, L, ldl, W, ldw, w, abort);
    else if (one_tile) k2_gemm_w4_kernel<128, 3><<<g4, W4_THREADS, sm4, s>>>(ws, ld, rbase, M, N2, L, ldl, W, ldw, w, abort);
    else k2_gemm_w4_kernel<128, 3, 2, MS_BK, 2><<<g4, W4_THREADS, sm4, s>>>(ws, ld, rbase, M, N2, L, ldl, W, ldw, w, abort);
    return cudaGetLastError();
}

}  // namespace mcnd

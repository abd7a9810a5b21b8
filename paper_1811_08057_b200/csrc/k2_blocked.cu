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
#include "mcnd_internal.h"

namespace mcnd {
namespace {

constexpr int kB = kK2B;

// One warp per trailing row.
__global__ void k2_gather_fix_kernel(double* __restrict__ ws, int64_t ld, int32_t rbase, int32_t nrows,
                                     const K2Panel* __restrict__ pan, double* __restrict__ L,
                                     const unsigned* __restrict__ abort) {
    if (*(volatile const unsigned*)abort) return;
    const int lane = threadIdx.x & 31;
    const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (i >= nrows) return;
    double* row = ws + (int64_t)(rbase + i) * ld;
    const double x0 = row[pan->p[lane]];
    const double x1 = row[pan->p[lane + 32]];
    __syncwarp();
    L[(int64_t)i * kB + lane] = x0;
    L[(int64_t)i * kB + lane + 32] = x1;
    const int nm = pan->n_moved;
    double v = 0.0;
    if (lane < nm) v = row[pan->moved_src[lane]];
    double v2 = 0.0;
    if (lane + 32 < nm) v2 = row[pan->moved_src[lane + 32]];
    __syncwarp();
    if (lane < nm) row[pan->moved_c[lane]] = v;
    if (lane + 32 < nm) row[pan->moved_c[lane + 32]] = v2;
}

// ---- DMMA GEMM: C[M x N2] (rows rbase.., in ws) -= L[M x 64] * W[64 x N2] ----
constexpr int BM = 64, BN = 128, BK = kB;
constexpr int LDLS = BK + 4;   // padded smem strides (conflict-free fragment loads)
constexpr int LDWS = BN + 8;
#ifndef MCND_GEMM_VARIANT
#define MCND_GEMM_VARIANT 0  // microbenchmark knob: 1 = no C traffic, 2 = operands loaded once
#endif
constexpr int kGThreads = 512;  // 16 warps: 2 (M) x 8 (N), warp tile 32 x 16
constexpr int WN = 8, WTN = 16, NJ = WTN / 8;

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}

// Persistent: one CTA per SM walks a contiguous range of 64 x 128 output tiles
// (row-block major, so L is reused and W streams from L2).  Software pipeline
// per tile: operands of tile t+1 go to the other shared-memory buffer with
// cp.async and the C fragments of tile t+1 are loaded into registers while the
// DMMAs of tile t run; stores are fire-and-forget.  Row maxima (witness) are
// kept in registers and flushed with one atomicMax per row-block change.
__global__ void __launch_bounds__(kGThreads, 1) k2_gemm_kernel(double* __restrict__ ws, int64_t ld, int32_t rbase,
                                                               int32_t M, int32_t N2, const double* __restrict__ L,
                                                               const double* __restrict__ W, int64_t ldw,
                                                               unsigned long long* __restrict__ wit,
                                                               const unsigned* __restrict__ abort) {
    extern __shared__ __align__(16) double sh[];
    if (*(volatile const unsigned*)abort) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp / WN, wn = warp % WN;
    const int g = lane >> 2, q = lane & 3;
    const int ntn = (N2 + BN - 1) / BN, ntm = (M + BM - 1) / BM;
    const int64_t T = (int64_t)ntn * ntm;
    const int64_t t_begin = T * blockIdx.x / gridDim.x, t_end = T * (blockIdx.x + 1) / gridDim.x;
    if (t_begin >= t_end) return;

    auto Ls = [&](int buf) { return sh + buf * (BM * LDLS + BK * LDWS); };
    auto Ws = [&](int buf) { return sh + buf * (BM * LDLS + BK * LDWS) + BM * LDLS; };
    auto load_operands = [&](int64_t t, int buf) {
        const int row0 = (int)(t / ntn) * BM, col0 = (int)(t % ntn) * BN;
        double* ls = Ls(buf);
        double* wsm = Ws(buf);
        for (int i = tid; i < BM * (BK / 2); i += kGThreads) {
            const int r = i / (BK / 2), c2 = i % (BK / 2);
            double* dst = ls + r * LDLS + 2 * c2;
            if (row0 + r < M) cp_async16(dst, L + (int64_t)(row0 + r) * BK + 2 * c2);
            else { dst[0] = 0.0; dst[1] = 0.0; }
        }
        for (int i = tid; i < BK * (BN / 2); i += kGThreads) {
            const int k = i / (BN / 2), c2 = i % (BN / 2);
            const int col = col0 + 2 * c2;
            double* dst = wsm + k * LDWS + 2 * c2;
            if (col < N2) cp_async16(dst, W + (int64_t)k * ldw + col);
            else { dst[0] = 0.0; dst[1] = 0.0; }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    double cn[4][NJ][2];
    auto load_c = [&](int64_t t) {
        const int row0 = (int)(t / ntn) * BM, col0 = (int)(t % ntn) * BN;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int r = row0 + wm * 32 + i * 8 + g;
            const double* crow = ws + (int64_t)(rbase + r) * ld;
#pragma unroll
            for (int j = 0; j < NJ; ++j) {
                const int c = col0 + wn * WTN + j * 8 + 2 * q;
                if (MCND_GEMM_VARIANT != 1 && MCND_GEMM_VARIANT != 4 && r < M && c < N2) {
                    const double2 v = __ldcs(reinterpret_cast<const double2*>(crow + c));
                    cn[i][j][0] = v.x;
                    cn[i][j][1] = v.y;
                } else {
                    cn[i][j][0] = 0.0;
                    cn[i][j][1] = 0.0;
                }
            }
        }
    };

    load_operands(t_begin, 0);
    load_c(t_begin);
    double rmx[4] = {0.0, 0.0, 0.0, 0.0};
    for (int64_t t = t_begin; t < t_end; ++t) {
        const int buf = (int)((t - t_begin) & 1);
        const int bm = (int)(t / ntn);
        const int row0 = bm * BM, col0 = (int)(t % ntn) * BN;
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads();
        double acc[4][NJ][2];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < NJ; ++j) { acc[i][j][0] = cn[i][j][0]; acc[i][j][1] = cn[i][j][1]; }
        if (t + 1 < t_end) {
            if (MCND_GEMM_VARIANT != 2 || t == t_begin) load_operands(t + 1, buf ^ 1);
            load_c(t + 1);
        }
        const double* ls = Ls(buf);
        const double* wsm = Ws(buf);
#pragma unroll 4
        for (int k0 = 0; k0 < BK; k0 += 4) {
            double a[4], b[NJ];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = -ls[(wm * 32 + i * 8 + g) * LDLS + k0 + q];
#pragma unroll
            for (int j = 0; j < NJ; ++j) b[j] = wsm[(k0 + q) * LDWS + wn * WTN + j * 8 + g];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < NJ; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
        }
        // epilogue: store, fold |.| into the per-row maxima
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int r = row0 + wm * 32 + i * 8 + g;
            double* crow = ws + (int64_t)(rbase + r) * ld;
#pragma unroll
            for (int j = 0; j < NJ; ++j) {
                const int c = col0 + wn * WTN + j * 8 + 2 * q;
                if (MCND_GEMM_VARIANT == 1 || MCND_GEMM_VARIANT == 3)
                    rmx[i] = fmax(rmx[i], fabs(acc[i][j][0] + acc[i][j][1]));
                if (MCND_GEMM_VARIANT != 1 && MCND_GEMM_VARIANT != 3 && r < M && c < N2) {
                    if (c + 1 < N2) {
                        __stcs(reinterpret_cast<double2*>(crow + c), make_double2(acc[i][j][0], acc[i][j][1]));
                        rmx[i] = fmax(rmx[i], fmax(fabs(acc[i][j][0]), fabs(acc[i][j][1])));
                    } else {
                        crow[c] = acc[i][j][0];
                        rmx[i] = fmax(rmx[i], fabs(acc[i][j][0]));
                    }
                }
            }
        }
        const bool flush = (t + 1 == t_end) || ((int)((t + 1) / ntn) != bm);
        if (flush) {
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
}

}  // namespace

cudaError_t k2_gather_fix(double* ws, int64_t ld, int32_t rbase, int32_t nrows, const K2Panel* pan, double* L,
                          const unsigned* abort, cudaStream_t s) {
    if (nrows <= 0) return cudaSuccess;
    const int warps = 8;
    k2_gather_fix_kernel<<<(nrows + warps - 1) / warps, warps * 32, 0, s>>>(ws, ld, rbase, nrows, pan, L, abort);
    return cudaGetLastError();
}

cudaError_t k2_gemm(double* ws, int64_t ld, int32_t rbase, int32_t M, int32_t N2, const double* L, const double* W,
                    int64_t ldw, double* row_wit, const unsigned* abort, cudaStream_t s) {
    if (M <= 0 || N2 <= 0) return cudaSuccess;
    const size_t smem = (size_t)2 * (BM * LDLS + BK * LDWS) * sizeof(double);
    static int sms = 0;
    if (!sms) {
        cudaError_t e = cudaFuncSetAttribute(k2_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const int64_t tiles = (int64_t)((N2 + BN - 1) / BN) * ((M + BM - 1) / BM);
    const int grid = (int)std::min<int64_t>(tiles, sms);
    k2_gemm_kernel<<<grid, kGThreads, smem, s>>>(ws, ld, rbase, M, N2, L, W, ldw,
                                                 reinterpret_cast<unsigned long long*>(row_wit), abort);
    return cudaGetLastError();
}

}  // namespace mcnd

// K2: blocked rank-b condensation (b = 64) with the trailing update on FP64
// tensor cores (sm_100a DMMA via mma.sync.m8n8k4.f64 -- tcgen05 has no f64 kind).
//
// The paper leaves block condensation to future work; the
// unblocked step it generalises is condense_step (mcnd/condense.py:95-131).
// Per panel of b pivot rows (top-to-bottom order, identical pivot rule):
//
//   1. panel factorisation: K1 restricted to the b panel rows (k1_condense.cu,
//      in-place mode) -- exactly the unblocked steps on those rows, so every
//      panel pivot is chosen by the reference's rule (argmax |.|, ties -> lowest
//      column, witness test); row t of the panel ends up holding the scaled
//      pivot row u_t in the column layout of step t+1;
//   2. k2_bookkeep: from the b pivot positions l_t, the panel-start column p_s
//      of every pivot and T[t][s] = u_t(p_s) (unit upper triangular);
//   3. k2_make_w: for every final column c (width m-b), its source column pi(c)
//      (the composition of the b column exchanges of condense.py:104-107) and
//      W[:, c] = T^{-1} U[:, c] by back substitution; columns whose source moved
//      are listed (<= b of them);
//   4. k2_gather_fix: per trailing row, L[r, s] = A[r, p_s] (the b multiplier
//      columns), then the moved columns A[r, c] <- A[r, pi(c)];
//   5. k2_gemm: A[R, 0:m-b] -= L W on DMMA, in place, with the running row
//      witness (condense.py:120-122) fused into the epilogue (at panel
//      granularity -- documented weakening for singular inputs).
//
// In exact arithmetic this is the unblocked result: coef_{r,s} (the step-s
// multiplier of row r) satisfies coef T = A[r, P], and the b rank-1 updates
// sum to coef U = A[r, P] T^{-1} U = L W.  Rounding differs (tolerance parity).
#include <cstdint>
#include "mcnd_internal.h"

namespace mcnd {
namespace {

constexpr int kB = kK2B;

__global__ void k2_bookkeep_kernel(const PivRec* __restrict__ rec, uint32_t epoch, const double* __restrict__ ws,
                                   int64_t ld, int32_t row0, int32_t m, K2Panel* __restrict__ pan,
                                   unsigned* __restrict__ abort) {
    __shared__ int s_l[kB];
    __shared__ int s_bad;
    const int s = threadIdx.x;
    if (*(volatile unsigned*)abort) return;
    if (s == 0) s_bad = 0;
    __syncthreads();
    const PivRec r = rec[s];
    const bool ok = (r.flag == epoch) && (r.l >= 0);
    if (!ok) atomicOr(&s_bad, 1);
    s_l[s] = r.l;
    __syncthreads();
    if (s_bad) {
        if (s == 0) *abort = 1u;
        return;
    }
    pan->l[s] = s_l[s];
    if (s == 0) pan->n_moved = 0;
    // position of pivot s's column, walked back from layout s to layout 0
    int pos = s_l[s];
    for (int t = 0; t < kB; ++t) pan->T[t][s] = (t == s) ? 1.0 : 0.0;
    for (int j = s - 1; j >= 0; --j) {
        pan->T[j][s] = ws[(int64_t)(row0 + j) * ld + pos];  // u_j lives in layout j+1
        pos = (pos == s_l[j]) ? (m - j - 1) : pos;           // sigma_j
    }
    pan->p[s] = pos;
}

// One thread per final column; W in registers (64 doubles).
constexpr int kWThreads = 128;
__global__ void __launch_bounds__(kWThreads) k2_make_w_kernel(const double* __restrict__ ws, int64_t ld,
                                                               int32_t row0, int32_t m, K2Panel* __restrict__ pan,
                                                               double* __restrict__ W, int64_t ldw,
                                                               const unsigned* __restrict__ abort) {
    __shared__ double sT[kB][kB + 1];
    __shared__ int s_l[kB];
    if (*(volatile const unsigned*)abort) return;
    for (int i = threadIdx.x; i < kB * kB; i += kWThreads) sT[i / kB][i % kB] = pan->T[i / kB][i % kB];
    for (int i = threadIdx.x; i < kB; i += kWThreads) s_l[i] = pan->l[i];
    __syncthreads();
    const int n2 = m - kB;
    const int c = blockIdx.x * kWThreads + threadIdx.x;
    if (c >= n2) return;
    double w[kB];
    int pos = c;
#pragma unroll
    for (int t = kB - 1; t >= 0; --t) {
        w[t] = __ldg(ws + (int64_t)(row0 + t) * ld + pos);  // u_t at final column c (layout t+1)
        pos = (pos == s_l[t]) ? (m - t - 1) : pos;
    }
    if (pos != c) {  // source column moved (it lies in the tail [m-b, m))
        const int k = atomicAdd(&pan->n_moved, 1);
        pan->moved_c[k] = c;
        pan->moved_src[k] = pos;
    }
    // back substitution T W = U (T unit upper triangular)
#pragma unroll
    for (int t = kB - 2; t >= 0; --t) {
        double acc = w[t];
#pragma unroll
        for (int s = t + 1; s < kB; ++s) acc = fma(-sT[t][s], w[s], acc);
        w[t] = acc;
    }
#pragma unroll
    for (int t = 0; t < kB; ++t) W[(int64_t)t * ldw + c] = w[t];
}

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
constexpr int kGThreads = 256;  // 8 warps: 2 (M) x 4 (N), warp tile 32 x 32

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}

__global__ void __launch_bounds__(kGThreads, 2) k2_gemm_kernel(double* __restrict__ ws, int64_t ld, int32_t rbase,
                                                               int32_t M, int32_t N2, const double* __restrict__ L,
                                                               const double* __restrict__ W, int64_t ldw,
                                                               unsigned long long* __restrict__ wit,
                                                               const unsigned* __restrict__ abort) {
    extern __shared__ __align__(16) double sh[];
    double* Ls = sh;                 // [BM][LDLS]
    double* Ws = sh + BM * LDLS;     // [BK][LDWS]
    if (*(volatile const unsigned*)abort) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp >> 2, wn = warp & 3;
    const int g = lane >> 2, q = lane & 3;
    const int row0 = blockIdx.y * BM, col0 = blockIdx.x * BN;

    // operands -> smem (async)
    for (int i = tid; i < BM * (BK / 2); i += kGThreads) {
        const int r = i / (BK / 2), c2 = i % (BK / 2);
        double* dst = Ls + r * LDLS + 2 * c2;
        if (row0 + r < M) cp_async16(dst, L + (int64_t)(row0 + r) * BK + 2 * c2);
        else { dst[0] = 0.0; dst[1] = 0.0; }
    }
    for (int i = tid; i < BK * (BN / 2); i += kGThreads) {
        const int k = i / (BN / 2), c2 = i % (BN / 2);
        const int col = col0 + 2 * c2;
        double* dst = Ws + k * LDWS + 2 * c2;
        if (col < N2) cp_async16(dst, W + (int64_t)k * ldw + col);
        else { dst[0] = 0.0; dst[1] = 0.0; }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");

    // C fragments -> registers (accumulate in place: acc = C - L W)
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int r = row0 + wm * 32 + i * 8 + g;
        const double* crow = ws + (int64_t)(rbase + r) * ld;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int c = col0 + wn * 32 + j * 8 + 2 * q;
            if (r < M && c < N2) {
                const double2 v = *reinterpret_cast<const double2*>(crow + c);
                acc[i][j][0] = v.x;
                acc[i][j][1] = v.y;
            } else {
                acc[i][j][0] = 0.0;
                acc[i][j][1] = 0.0;
            }
        }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();

#pragma unroll 4
    for (int k0 = 0; k0 < BK; k0 += 4) {
        double a[4], b[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = -Ls[(wm * 32 + i * 8 + g) * LDLS + k0 + q];
#pragma unroll
        for (int j = 0; j < 4; ++j) b[j] = Ws[(k0 + q) * LDWS + wn * 32 + j * 8 + g];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }

    // epilogue: store + per-row witness max
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int r = row0 + wm * 32 + i * 8 + g;
        double* crow = ws + (int64_t)(rbase + r) * ld;
        double mx = 0.0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int c = col0 + wn * 32 + j * 8 + 2 * q;
            if (r < M && c < N2) {
                if (c + 1 < N2) {
                    *reinterpret_cast<double2*>(crow + c) = make_double2(acc[i][j][0], acc[i][j][1]);
                    mx = fmax(mx, fmax(fabs(acc[i][j][0]), fabs(acc[i][j][1])));
                } else {
                    crow[c] = acc[i][j][0];
                    mx = fmax(mx, fabs(acc[i][j][0]));
                }
            }
        }
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
        if (q == 0 && r < M) atomicMax(wit + rbase + r, (unsigned long long)__double_as_longlong(mx));
    }
}

}  // namespace

cudaError_t k2_bookkeep(const PivRec* rec, uint32_t epoch, const double* ws, int64_t ld, int32_t row0, int32_t m,
                        K2Panel* pan, unsigned* abort, cudaStream_t s) {
    k2_bookkeep_kernel<<<1, kB, 0, s>>>(rec, epoch, ws, ld, row0, m, pan, abort);
    return cudaGetLastError();
}

cudaError_t k2_make_w(const double* ws, int64_t ld, int32_t row0, int32_t m, K2Panel* pan, double* W, int64_t ldw,
                      const unsigned* abort, cudaStream_t s) {
    const int n2 = m - kB;
    if (n2 <= 0) return cudaSuccess;
    k2_make_w_kernel<<<(n2 + kWThreads - 1) / kWThreads, kWThreads, 0, s>>>(ws, ld, row0, m, pan, W, ldw, abort);
    return cudaGetLastError();
}

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
    const size_t smem = (size_t)(BM * LDLS + BK * LDWS) * sizeof(double);
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(k2_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    dim3 grid((N2 + BN - 1) / BN, (M + BM - 1) / BM);
    k2_gemm_kernel<<<grid, kGThreads, smem, s>>>(ws, ld, rbase, M, N2, L, W, ldw,
                                                 reinterpret_cast<unsigned long long*>(row_wit), abort);
    return cudaGetLastError();
}

}  // namespace mcnd

// K3: batched condensation log-determinant, one CTA per small matrix.
//
// Same step as condense_step (mcnd/condense.py:95-131) with the default
// top-to-bottom pivot order, but the whole n x n matrix (n <= 128) lives in
// shared memory for all n-1 steps: HBM is touched once to load each matrix
// and once to store (sign, log|det|).  The reference has no batched entry
// point; its oracle is a loop of logdet_condensation.
//
// Per step: warp 0 takes the argmax of the pivot row (ties -> lowest column),
// runs the witness test and writes the scaled, column-permuted pivot row to
// smem; then each warp owns whole rows, so the in-place hazard on the
// multiplier column is resolved inside the warp (all lanes read their
// operands before any lane writes, __syncwarp in between).  Per-row witness
// maxima are warp reductions (no atomics).  log|det| is accumulated in step
// order by one thread at the end (device log(), so |d log| stays within the
// north_star tolerance; the per-step pivots are also emitted so a host can
// recompute the bitwise-reference sum when it wants to).
#include <cstdint>
#include <climits>
#include "mcnd_internal.h"

namespace mcnd {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr unsigned kFull = 0xffffffffu;
constexpr int kMaxPerLane = 4;  // n <= 128 -> at most 4 columns per lane

template <bool kFast>
__device__ __forceinline__ double upd(double x, double mult, double p) {
    if (kFast) return fma(-mult, p, x);
    return __dsub_rn(x, __dmul_rn(mult, p));
}

template <bool kFast>
__global__ void __launch_bounds__(kThreads) k3_batched(const double* __restrict__ a, int n, int64_t stride,
                                                       int32_t* __restrict__ sign_out,
                                                       double* __restrict__ log_out,
                                                       double* __restrict__ piv_out) {
    extern __shared__ __align__(16) double sh[];
    double* A = sh;                 // n x n, row stride n
    double* wit = A + n * n;        // n
    double* prow = wit + n;         // n
    double* piv = prow + n;         // n  pivot values
    int* pcol = reinterpret_cast<int*>(piv + n);  // n pivot columns
    __shared__ int s_l;
    __shared__ int s_sing;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const double* src = a + (int64_t)blockIdx.x * stride;
    const int nn = n * n;
    for (int e = tid; e < nn; e += kThreads) A[e] = __ldg(src + e);
    if (tid == 0) s_sing = 0;
    __syncthreads();
    // initial witness (condense.py:78), warp per row
    for (int r = warp; r < n; r += kWarps) {
        double wm = 0.0;
        for (int c = lane; c < n; c += 32) wm = fmax(wm, fabs(A[r * n + c]));
#pragma unroll
        for (int o = 16; o; o >>= 1) wm = fmax(wm, __shfl_xor_sync(kFull, wm, o));
        if (lane == 0) wit[r] = wm;
    }
    __syncthreads();

    for (int s = 0; s < n - 1; ++s) {
        const int m = n - s, w = m - 1;
        const double* rk = A + s * n;  // pivot row = top live row
        if (warp == 0) {
            double bv = 0.0;
            int bi = INT_MAX;
            for (int c = lane; c < m; c += 32) {
                const double x = rk[c];
                const double fx = fabs(x), fb = fabs(bv);
                if (fx > fb || (fx == fb && c < bi)) { bv = x; bi = c; }
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                const double ov = __shfl_xor_sync(kFull, bv, o);
                const int oi = __shfl_xor_sync(kFull, bi, o);
                const double fo = fabs(ov), fb = fabs(bv);
                if (fo > fb || (fo == fb && oi < bi)) { bv = ov; bi = oi; }
            }
            const bool singular = !(fabs(bv) > kSingularRtol * wit[s]);
            if (!singular) {
                const double ylast = rk[w];
                for (int c = lane; c < w; c += 32) prow[c] = __ddiv_rn(c == bi ? ylast : rk[c], bv);
            }
            if (lane == 0) {
                piv[s] = bv;
                pcol[s] = bi;
                s_l = bi;
                if (singular) s_sing = 1;
            }
        }
        __syncthreads();
        if (s_sing) break;
        const int l = s_l;
        for (int r = s + 1 + warp; r < n; r += kWarps) {
            double* rr = A + r * n;
            const double mult = rr[l], lastv = rr[w];
            double x[kMaxPerLane];
#pragma unroll
            for (int k = 0; k < kMaxPerLane; ++k) {
                const int c = lane + 32 * k;
                x[k] = (c < w) ? (c == l ? lastv : rr[c]) : 0.0;
            }
            __syncwarp();
            double wm = 0.0;
#pragma unroll
            for (int k = 0; k < kMaxPerLane; ++k) {
                const int c = lane + 32 * k;
                if (c < w) {
                    const double y = upd<kFast>(x[k], mult, prow[c]);
                    rr[c] = y;
                    wm = fmax(wm, fabs(y));
                }
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) wm = fmax(wm, __shfl_xor_sync(kFull, wm, o));
            if (lane == 0) wit[r] = fmax(wit[r], wm);
        }
        __syncthreads();
    }
    if (tid == 0) {
        int32_t sign = 0;
        double la = -INFINITY;
        if (!s_sing) {
            const double v = A[(n - 1) * n];
            if (fabs(v) > kSingularRtol * wit[n - 1]) {
                piv[n - 1] = v;
                pcol[n - 1] = 0;
                int sg = 1;
                double acc = 0.0;
                for (int s = 0; s < n - 1; ++s) {
                    const int m = n - s;
                    const double pv = piv[s];
                    acc += log(fabs(pv));
                    const int swap = (pcol[s] != m - 1) ? -1 : 1;
                    const int par = ((m - 1) & 1) ? -1 : 1;  // k_pos = 0 (top-to-bottom)
                    sg *= (pv > 0 ? 1 : -1) * swap * par;
                }
                sign = sg * (v > 0 ? 1 : -1);
                la = acc + log(fabs(v));
            } else {
                piv[n - 1] = v;
            }
        }
        sign_out[blockIdx.x] = sign;
        log_out[blockIdx.x] = la;
    }
    if (piv_out) {
        __syncthreads();
        for (int s = tid; s < n; s += kThreads) piv_out[(int64_t)blockIdx.x * n + s] = piv[s];
    }
}

}  // namespace

cudaError_t k3_launch(const double* a, int64_t batch, int64_t n, int64_t stride, bool fast,
                      int32_t* sign, double* log_abs, double* pivots, cudaStream_t s) {
    if (n < 1 || n > 32 * kMaxPerLane || batch < 0) return cudaErrorInvalidValue;
    if (batch == 0) return cudaSuccess;
    const size_t smem = (size_t)(n * n + 3 * n) * sizeof(double) + (size_t)n * sizeof(int) + 16;
    const void* fn = fast ? (const void*)k3_batched<true> : (const void*)k3_batched<false>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if (fast)
        k3_batched<true><<<(unsigned)batch, kThreads, smem, s>>>(a, (int)n, stride, sign, log_abs, pivots);
    else
        k3_batched<false><<<(unsigned)batch, kThreads, smem, s>>>(a, (int)n, stride, sign, log_abs, pivots);
    return cudaGetLastError();
}

}  // namespace mcnd

// K3: batched condensation log-determinant, one WARP per small matrix.
//
// Same step as condense_step (mcnd/condense.py:95-131) with the default
// top-to-bottom pivot order and the reference's arithmetic (true division for
// the pivot row, product then difference for the update), so the pivots are
// bitwise the reference's.  The whole n x n matrix (n <= 128) lives in shared
// memory (row stride n+1: conflict-free for both row and column walks) for all
// n-1 steps: HBM is touched once to load each matrix and once to store
// (sign, log|det|).  The reference has no batched entry point; its oracle is a
// loop of logdet_condensation.
//
// One warp owns one matrix, so there is no block-level synchronisation at all.
// Each lane owns whole rows (see k3_batched_warp); the argmax of the pivot row
// is an exact 64-bit max reduction done as two 32-bit warp reductions
// (redux.sync on the high word, then on the low word of the lanes holding the
// high-word maximum) -- non-negative doubles order like their bit patterns.
// |x| is taken by clearing the sign bit (integer pipe), leaving the FP64 pipe
// with exactly the two operations per element the reference performs.  log|det| is accumulated in step order by one lane
// (device log(): within the north_star tolerance; the pivots themselves can
// be returned for a bitwise check).
#include <cstdint>
#include <climits>
#include "mcnd_internal.h"

namespace mcnd {
namespace {

constexpr unsigned kFull = 0xffffffffu;

template <bool kFast>
__device__ __forceinline__ double upd(double x, double mult, double p) {
    if (kFast) return fma(-mult, p, x);
    return __dsub_rn(x, __dmul_rn(mult, p));
}

__device__ __forceinline__ unsigned long long abs_bits(double x) {
    return (unsigned long long)__double_as_longlong(x) & 0x7fffffffffffffffull;
}

// Exact warp max of non-negative 64-bit patterns.
__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
    const unsigned hi = (unsigned)(v >> 32), lo = (unsigned)v;
    const unsigned mh = __reduce_max_sync(kFull, hi);
    const unsigned ml = __reduce_max_sync(kFull, hi == mh ? lo : 0u);
    return ((unsigned long long)mh << 32) | ml;
}

// Warp argmax of |x| (bit patterns), ties -> lowest column.
__device__ __forceinline__ int warp_argmax(unsigned long long a, int idx) {
    const unsigned long long m = warp_max_u64(a);
    return (int)__reduce_min_sync(kFull, a == m ? (unsigned)idx : 0xffffffffu);
}

// Two warps per matrix (kWPM): lane i of the pair owns rows i, i+64, ... (NR of
// them) and updates them entirely by itself (no cross-lane hazard on the
// multiplier column, no synchronisation inside the update), keeping their
// running maxima in shared memory.  Per step the first warp scans the pivot
// row (2..4 columns per lane, exact warp argmax), runs the witness test and
// writes the scaled pivot row; two named barriers per step order the pair.
constexpr int kWPM = 2;
constexpr int kTPM = 32 * kWPM;  // threads per matrix

template <bool kFast, int NR>
__global__ void k3_batched_warp(const double* __restrict__ a, int n, int64_t stride, int64_t batch,
                                int32_t* __restrict__ sign_out, double* __restrict__ log_out,
                                double* __restrict__ piv_out, unsigned* __restrict__ nonfinite) {
    extern __shared__ __align__(16) double sh[];
    const int lane = threadIdx.x & 31;
    const int mat = threadIdx.x / kTPM;            // matrix slot in this CTA
    const int li = threadIdx.x % kTPM;             // lane within the matrix
    const bool lead = li < 32;                     // first warp of the pair
    const int64_t b = (int64_t)blockIdx.x * (blockDim.x / kTPM) + mat;
    if (b >= batch) return;                        // uniform for the pair
    const int ld = n + 1;  // odd stride: lanes walking different rows hit different banks
    double* A = sh + (size_t)mat * (n * ld + 4 * n + 4);
    double* prow = A + n * ld;          // scaled pivot row of the current step
    double* piv = prow + n;             // pivot values
    double* wit = piv + n;              // running row maxima
    int* pcol = reinterpret_cast<int*>(wit + n);  // pivot columns
    double* ctl = reinterpret_cast<double*>(pcol + n + (n & 1));  // [v, l, stop]
    const int bar = 1 + mat;
    const double* src = a + b * stride;

    // load (coalesced rows; 8 rows in flight per thread, no index division)
    for (int r0 = 0; r0 < n; r0 += 8) {
        double x[8][NR];
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int k = 0; k < NR; ++k) {
                const int r = r0 + u, c = li + kTPM * k;
                x[u][k] = (r < n && c < n) ? __ldg(src + (int64_t)r * n + c) : 0.0;
            }
        bool bad = false;
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int k = 0; k < NR; ++k) {
                const int r = r0 + u, c = li + kTPM * k;
                if (r < n && c < n) {
                    A[r * ld + c] = x[u][k];
                    bad |= !isfinite(x[u][k]);
                }
            }
        if (bad && nonfinite) atomicOr(nonfinite, 1u);  // matrix.py:39-40, checked on device
    }
    asm volatile("bar.sync %0, %1;" ::"r"(bar), "n"(kTPM));
    // initial witness of my rows (condense.py:78)
#pragma unroll
    for (int k = 0; k < NR; ++k) {
        const int r = li + kTPM * k;
        if (r < n) {
            double mx = 0.0;
            for (int c = 0; c < n; ++c) mx = fmax(mx, fabs(A[r * ld + c]));
            wit[r] = mx;
        }
    }

    int sign = 1;
    bool stopped = false;
    for (int s = 0; s < n - 1; ++s) {
        const int m = n - s, w = m - 1;
        asm volatile("bar.sync %0, %1;" ::"r"(bar), "n"(kTPM));  // row s final, witnesses current
        if (lead) {
            const double* rk = A + s * ld;
            unsigned long long best = 0ull;
            int bi = INT_MAX;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int c = lane + 32 * k;
                if (c < m) {
                    const unsigned long long ab = abs_bits(rk[c]);
                    if (bi == INT_MAX || ab > best) { best = ab; bi = c; }
                }
            }
            const int l = warp_argmax(best, bi);  // ties -> lowest column (condense.py:88)
            const double v = rk[l];
            const bool singular = !(fabs(v) > kSingularRtol * wit[s]);  // condense.py:90
            if (!singular) {
                const double ylast = rk[w];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int c = lane + 32 * k;
                    if (c < w) prow[c] = __ddiv_rn(c == l ? ylast : rk[c], v);
                }
            }
            if (lane == 0) {
                piv[s] = v;
                pcol[s] = singular ? -1 : l;
                ctl[0] = v;
                ctl[1] = singular ? -1.0 : (double)l;
                if (!singular) sign *= (v > 0 ? 1 : -1) * (l != w ? -1 : 1) * ((w & 1) ? -1 : 1);  // k_pos = 0
            }
        }
        asm volatile("bar.sync %0, %1;" ::"r"(bar), "n"(kTPM));  // pivot row + (v, l) published
        const int l = (int)ctl[1];
        if (l < 0) { stopped = true; break; }  // singular: uniform for the pair
        // my live rows: rank-1 update in place (condense.py:118) + running maxima (:120-122)
        double mult[NR], mx[NR];
        double* rr[NR];
        bool live[NR];
#pragma unroll
        for (int k = 0; k < NR; ++k) {
            const int r = li + kTPM * k;
            live[k] = r > s && r < n;
            rr[k] = A + (live[k] ? r : s) * ld;
            mult[k] = live[k] ? rr[k][l] : 0.0;
            if (live[k]) rr[k][l] = rr[k][w];  // column exchange (mult already read)
            mx[k] = 0.0;
        }
#pragma unroll 4
        for (int c = 0; c < w; ++c) {
            const double pc = prow[c];
#pragma unroll
            for (int k = 0; k < NR; ++k) {
                if (live[k]) {
                    const double y = upd<kFast>(rr[k][c], mult[k], pc);
                    rr[k][c] = y;
                    mx[k] = fmax(mx[k], fabs(y));
                }
            }
        }
#pragma unroll
        for (int k = 0; k < NR; ++k)
            if (live[k]) wit[li + kTPM * k] = fmax(wit[li + kTPM * k], mx[k]);
    }
    asm volatile("bar.sync %0, %1;" ::"r"(bar), "n"(kTPM));
    if (li == 0) {
        int32_t sg = 0;
        double la = -INFINITY;
        if (!stopped) {
            const double v = A[(n - 1) * ld];
            piv[n - 1] = v;
            pcol[n - 1] = 0;
            if (fabs(v) > kSingularRtol * wit[n - 1]) {
                sg = sign * (v > 0 ? 1 : -1);
                double acc = 0.0;
                for (int t = 0; t < n; ++t) acc += log(fabs(piv[t]));
                la = acc;
            }
        }
        sign_out[b] = sg;
        log_out[b] = sg == 0 ? -INFINITY : la;
    }
    if (piv_out) {
        asm volatile("bar.sync %0, %1;" ::"r"(bar), "n"(kTPM));
        for (int t = li; t < n; t += kTPM) piv_out[b * n + t] = piv[t];
    }
}

// The blocked path's tail: the last mt <= 128 rows x mt columns of the workspace (rows row0 ..,
// row stride ldw) condensed to the end by ONE pair of warps with the same step as above -- the
// arithmetic of K1's in-place tail (bitwise: same pivots, same records), at ~0.3 us per step
// instead of the 148-CTA kernel's ~3.9 us (its per-step cost is the inter-CTA publication, which
// a 64 x 64 block does not need).  Witnesses start from the carried-in running maxima; every
// pivot goes out as a PivRec {v, l (-1: failed the witness test), epoch}, the final 1 x 1 last.
template <bool kFast, int TPM>
__global__ void __launch_bounds__(TPM) k3_tail_kernel(const double* __restrict__ ws, int64_t ldw, int row0, int n,
                                                       const double* __restrict__ wit_in, PivRec* __restrict__ rec,
                                                       uint32_t epoch, const unsigned* __restrict__ abort) {
    extern __shared__ __align__(16) double sh[];
    if (abort && *(volatile const unsigned*)abort) return;
    const int lane = threadIdx.x & 31, li = threadIdx.x;
    const bool lead = li < 32;
    const int ld = n + 1 + (n & 1);  // odd: threads walking different rows hit different banks
    double* A = sh;
    double* prow = A + n * ld;
    double* wit = prow + n;
    double* ctl = wit + n;  // [l]
    for (int r = 0; r < n; ++r)
        for (int c = li; c < n; c += TPM) A[r * ld + c] = __ldcg(ws + (int64_t)(row0 + r) * ldw + c);
    for (int r = li; r < n; r += TPM) wit[r] = wit_in[row0 + r];
    for (int s = 0; s < n - 1; ++s) {
        const int m = n - s, w = m - 1;
        __syncthreads();  // row s final, witnesses current
        if (lead) {
            const double* rk = A + s * ld;
            unsigned long long best = 0ull;
            int bi = INT_MAX;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int c = lane + 32 * k;
                if (c < m) {
                    const unsigned long long ab = abs_bits(rk[c]);
                    if (bi == INT_MAX || ab > best) { best = ab; bi = c; }
                }
            }
            const int l = warp_argmax(best, bi);  // ties -> lowest column (condense.py:88)
            const double v = rk[l];
            const bool singular = !(fabs(v) > kSingularRtol * wit[s]);  // condense.py:90
            if (!singular) {
                const double ylast = rk[w];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int c = lane + 32 * k;
                    if (c < w) prow[c] = __ddiv_rn(c == l ? ylast : rk[c], v);
                }
            }
            if (lane == 0) {
                rec[s].v = v;
                rec[s].l = singular ? -1 : l;
                rec[s].flag = epoch;
                ctl[0] = singular ? -1.0 : (double)l;
            }
        }
        __syncthreads();  // pivot row + l published
        const int l = (int)ctl[0];
        if (l < 0) return;  // singular: uniform
        constexpr int NR = 1;  // one row per thread (n <= TPM)
        double mult[NR], mx[NR];
        double* rr[NR];
        bool live[NR];
#pragma unroll
        for (int k = 0; k < NR; ++k) {
            const int r = li + TPM * k;
            live[k] = r > s && r < n;
            rr[k] = A + (live[k] ? r : s) * ld;
            mult[k] = live[k] ? rr[k][l] : 0.0;
            if (live[k]) rr[k][l] = rr[k][w];  // column exchange (mult already read)
            mx[k] = 0.0;
        }
#pragma unroll 4
        for (int c = 0; c < w; ++c) {
            const double pc = prow[c];
#pragma unroll
            for (int k = 0; k < NR; ++k) {
                if (live[k]) {
                    const double y = upd<kFast>(rr[k][c], mult[k], pc);
                    rr[k][c] = y;
                    mx[k] = fmax(mx[k], fabs(y));
                }
            }
        }
#pragma unroll
        for (int k = 0; k < NR; ++k)
            if (live[k]) wit[li + TPM * k] = fmax(wit[li + TPM * k], mx[k]);
    }
    __syncthreads();
    if (li == 0) {  // the final 1 x 1 (condense.py:153-158)
        const double v = A[(n - 1) * ld];
        rec[n - 1].v = v;
        rec[n - 1].l = (fabs(v) > kSingularRtol * wit[n - 1]) ? 0 : -1;
        rec[n - 1].flag = epoch;
    }
}

}  // namespace

cudaError_t k3_tail_launch(const double* ws, int64_t ldw, int32_t row0, int32_t n, bool fast, const double* wit_in,
                           PivRec* rec, uint32_t epoch, const unsigned* abort, cudaStream_t s) {
    if (n < 1 || n > 128) return cudaErrorInvalidValue;
    const size_t smem = (size_t)(n * (n + 1 + (n & 1)) + 2 * n + 2) * sizeof(double);
    cudaError_t e;
#define MCND_K3T(F, T)                                                                                  \
    e = cudaFuncSetAttribute(k3_tail_kernel<F, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    if (e != cudaSuccess) return e;                                                                     \
    k3_tail_kernel<F, T><<<1, T, smem, s>>>(ws, ldw, row0, n, wit_in, rec, epoch, abort);
    if (n <= 64) {
        if (fast) { MCND_K3T(true, 64) } else { MCND_K3T(false, 64) }
    } else {
        if (fast) { MCND_K3T(true, 128) } else { MCND_K3T(false, 128) }
    }
#undef MCND_K3T
    return cudaGetLastError();
}

cudaError_t k3_launch(const double* a, int64_t batch, int64_t n, int64_t stride, bool fast,
                      int32_t* sign, double* log_abs, double* pivots, unsigned* nonfinite, cudaStream_t s) {
    if (n < 1 || n > 128 || batch < 0) return cudaErrorInvalidValue;
    if (batch == 0) return cudaSuccess;
    const int mats = n <= 64 ? 2 : 1;  // matrices per CTA (shared-memory bound)
    const size_t per = (size_t)(n * (n + 1) + 4 * n + 4) * sizeof(double);
    const size_t smem = per * mats;
    const dim3 grid((unsigned)((batch + mats - 1) / mats)), block(kTPM * mats);
    cudaError_t e;
#define MCND_K3(F, NR)                                                                                   \
    e = cudaFuncSetAttribute(k3_batched_warp<F, NR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    if (e != cudaSuccess) return e;                                                                      \
    k3_batched_warp<F, NR><<<grid, block, smem, s>>>(a, (int)n, stride, batch, sign, log_abs, pivots, nonfinite);
    if (n <= 64) {
        if (fast) { MCND_K3(true, 1) } else { MCND_K3(false, 1) }
    } else {
        if (fast) { MCND_K3(true, 2) } else { MCND_K3(false, 2) }
    }
#undef MCND_K3
    return cudaGetLastError();
}

}  // namespace mcnd

// Variant of k2_gemm_w4_kernel for register-pressure experiments (PF: mid-tile L2 prefetch of
// the next C tile; WT: witness maxima folded per tile instead of per row block).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xptxas -v -o gemm_w5 gemm_w5.cu -lcublas -lcurand
#include <cstdio>
#include <vector>
#include <cublas_v2.h>
#include <curand.h>
#include "../../paper_1811_08057_b200/csrc/k2_blocked.cu"
namespace mcnd { namespace {
template <int K, int S, int WN = 2, int BK = MS_BK, bool PF = true, bool WT = false, int U = 1, bool CZ = false>
__global__ void __launch_bounds__(64 * WN, 2) k2_gemm_w5_kernel(double* __restrict__ ws, int64_t ld, int32_t rbase,
                                                                    int32_t M, int32_t N2, const double* __restrict__ L,
                                                                    int64_t ldl, const double* __restrict__ W, int64_t ldw,
                                                                    unsigned long long* __restrict__ wit,
                                                                    const unsigned* __restrict__ abort) {
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
            const double* wsrc = w_src + (int64_t)kk * ldw;
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
        if constexpr (CZ) {
#pragma unroll
            for (int i = 0; i < MI; ++i)
#pragma unroll
                for (int jj = 0; jj < NJ; ++jj) { acc[i][jj][0] = 0.0; acc[i][jj][1] = 0.0; }
            return;
        }
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
            if (PF && ks == KS / 2 && t + 1 < t_end) {
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
                    if constexpr (CZ) {
                        const double2 cv = __ldcs(reinterpret_cast<const double2*>(crow + c));
                        acc[i][jj][0] += cv.x;
                        acc[i][jj][1] += cv.y;
                    }
                    __stcs(reinterpret_cast<double2*>(crow + c), make_double2(acc[i][jj][0], acc[i][jj][1]));
                    rmx[i] = fmax(rmx[i], fmax(fabs(acc[i][jj][0]), fabs(acc[i][jj][1])));
                } else if (r < M && c < N2) {
                    if constexpr (CZ) acc[i][jj][0] += crow[c];
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
        if ((WT || t == t_end || row0 != prow0) && wit) {
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

} }

template <class F>
static float timeit(F f, double* ws, const double* ws0, size_t bytes, int reps = 5) {
    f(); f();
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float tot = 0;
    for (int i = 0; i < reps; ++i) {
        cudaMemcpy(ws, ws0, bytes, cudaMemcpyDeviceToDevice);
        cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); tot += ms;
    }
    return tot / reps;
}

int main(int argc, char** argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 16384;
    constexpr int K = 128;
    const int64_t ld = (n + 15) / 16 * 16;
    const size_t bytes = (size_t)n * ld * 8;
    double *ws, *ws0, *ref, *L, *W, *wit, *wit2; unsigned* abort;
    cudaMalloc(&ws, bytes); cudaMalloc(&ws0, bytes); cudaMalloc(&ref, bytes);
    cudaMalloc(&L, (size_t)n * K * 8); cudaMalloc(&W, (size_t)K * ld * 8);
    cudaMalloc(&wit, (size_t)n * 8); cudaMalloc(&wit2, (size_t)n * 8); cudaMalloc(&abort, 4);
    cudaMemset(abort, 0, 4);
    curandGenerator_t gen; curandCreateGenerator(&gen, CURAND_RNG_PSEUDO_DEFAULT);
    curandSetPseudoRandomGeneratorSeed(gen, 5);
    curandGenerateUniformDouble(gen, ws0, bytes / 8);
    curandGenerateUniformDouble(gen, L, (size_t)n * K);
    curandGenerateUniformDouble(gen, W, (size_t)K * ld);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const double fl = 2.0 * n * (double)n * K;
    const int64_t T = (int64_t)((n + mcnd::BM - 1) / mcnd::BM) * ((n + mcnd::BN - 1) / mcnd::BN);
    const size_t sm = (size_t)3 * mcnd::MS_STAGE * 8;
    auto* w1 = reinterpret_cast<unsigned long long*>(wit);
    auto* w2 = reinterpret_cast<unsigned long long*>(wit2);
    cudaFuncSetAttribute(mcnd::k2_gemm_w4_kernel<K, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaMemset(wit, 0, (size_t)n * 8);
    cudaMemcpy(ws, ws0, bytes, cudaMemcpyDeviceToDevice);
    mcnd::k2_gemm_w4_kernel<K, 3><<<2 * sms, mcnd::W4_THREADS, sm>>>(ws, ld, 0, n, n, L, K, W, ld, w1, abort);
    cudaMemcpy(ref, ws, bytes, cudaMemcpyDeviceToDevice);
    std::vector<double> x(bytes / 8), y(bytes / 8);
    std::vector<unsigned long long> wa(n), wb(n);
    cudaMemcpy(wa.data(), wit, n * 8, cudaMemcpyDeviceToHost);
    for (int grid : {(int)T, 2 * sms}) {
        auto f = [&]() { mcnd::k2_gemm_w4_kernel<K, 3><<<grid, mcnd::W4_THREADS, sm>>>(ws, ld, 0, n, n, L, K, W, ld, w1, abort); };
        float t = timeit(f, ws, ws0, bytes);
        printf("w4            grid %6d: %.3f ms %.2f TF\n", grid, t, fl / t / 1e9);
    }
    size_t smv = sm;
    auto variant = [&](auto kern, const char* name) {
        const size_t sm = smv;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        for (int grid : {(int)T, 2 * sms}) {
            auto f = [&]() { kern<<<grid, mcnd::W4_THREADS, sm>>>(ws, ld, 0, n, n, L, K, W, ld, w2, abort); };
            float t = timeit(f, ws, ws0, bytes);
            cudaMemset(wit2, 0, (size_t)n * 8);
            cudaMemcpy(ws, ws0, bytes, cudaMemcpyDeviceToDevice);
            f();
            cudaMemcpy(x.data(), ref, bytes, cudaMemcpyDeviceToHost);
            cudaMemcpy(y.data(), ws, bytes, cudaMemcpyDeviceToHost);
            cudaMemcpy(wb.data(), wit2, n * 8, cudaMemcpyDeviceToHost);
            size_t bad = 0, wbad = 0;
            for (size_t i = 0; i < x.size(); ++i) bad += (x[i] != y[i]);
            for (int i = 0; i < n; ++i) wbad += (wa[i] != wb[i]);
            printf("%-14s grid %6d: %.3f ms %.2f TF  diff %zu wit %zu (%s)\n", name, grid, t, fl / t / 1e9, bad, wbad,
                   cudaGetErrorString(cudaGetLastError()));
        }
    };
    auto variant4 = [&](auto kern, const char* name) { smv = (size_t)4 * mcnd::MS_STAGE * 8; variant(kern, name); smv = sm; };
    variant(mcnd::k2_gemm_w5_kernel<K, 3, 2, 16, true, false, 2>, "w5 u2");
    variant(mcnd::k2_gemm_w5_kernel<K, 3, 2, 16, true, false, 1, true>, "w5 cz");
    variant(mcnd::k2_gemm_w5_kernel<K, 3, 2, 16, true, false, 2, true>, "w5 cz u2");
    return 0;
}

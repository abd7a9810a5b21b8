// Trailing-GEMM variants on random data at the C5 side-update shape (n x n, K = 128):
// k2_gemm_ms_kernel (8 warps of 32 x 32) vs k2_gemm_w4_kernel (4 warps of 32 x 64),
// one tile per CTA and persistent, against cuBLAS DGEMM (C = C - L W) on the same data;
// the two hand-written kernels must agree bitwise.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o gemm_w4 gemm_w4.cu -lcublas -lcurand
#include <cstdio>
#include <vector>
#include <cublas_v2.h>
#include <curand.h>
#include "../../paper_1811_08057_b200/csrc/k2_blocked.cu"

static double* ws0;
template <class F>
static float timeit(F f, double* ws, size_t bytes, int reps = 5) {
    f(); f();
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float tot = 0;
    for (int i = 0; i < reps; ++i) {
        cudaMemcpy(ws, ws0, bytes, cudaMemcpyDeviceToDevice);  // also flushes L2
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
    double *ws, *L, *W, *wit, *out_a; unsigned* abort;
    cudaMalloc(&ws, bytes); cudaMalloc(&ws0, bytes); cudaMalloc(&out_a, bytes);
    cudaMalloc(&L, (size_t)n * K * 8); cudaMalloc(&W, (size_t)K * ld * 8);
    cudaMalloc(&wit, (size_t)n * 8); cudaMalloc(&abort, 4);
    cudaMemset(abort, 0, 4); cudaMemset(wit, 0, (size_t)n * 8);
    curandGenerator_t gen; curandCreateGenerator(&gen, CURAND_RNG_PSEUDO_DEFAULT);
    curandSetPseudoRandomGeneratorSeed(gen, 5);
    curandGenerateUniformDouble(gen, ws0, bytes / 8);
    curandGenerateUniformDouble(gen, L, (size_t)n * K);
    curandGenerateUniformDouble(gen, W, (size_t)K * ld);
    auto* w = reinterpret_cast<unsigned long long*>(wit);
    const int64_t T = (int64_t)((n + mcnd::BM - 1) / mcnd::BM) * ((n + mcnd::BN - 1) / mcnd::BN);
    const double fl = 2.0 * n * (double)n * K;
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);

    const size_t smem_ms = (size_t)mcnd::MS_ST * mcnd::MS_STAGE * 8;
    cudaFuncSetAttribute(mcnd::k2_gemm_ms_kernel<K, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_ms);
    auto ms_one = [&]() { mcnd::k2_gemm_ms_kernel<K, 1><<<(unsigned)T, mcnd::MS_THREADS, smem_ms>>>(ws, ld, 0, n, n, L, K, W, ld, w, abort); };
    float t = timeit(ms_one, ws, bytes);
    printf("ms  one-tile   : %.3f ms %.2f TFLOP/s\n", t, fl / t / 1e9);
    cudaMemcpy(ws, ws0, bytes, cudaMemcpyDeviceToDevice); ms_one(); cudaMemcpy(out_a, ws, bytes, cudaMemcpyDeviceToDevice);

    auto check = [&](const char* name) {
        std::vector<double> x(bytes / 8), y(bytes / 8);
        cudaMemcpy(x.data(), out_a, bytes, cudaMemcpyDeviceToHost);
        cudaMemcpy(y.data(), ws, bytes, cudaMemcpyDeviceToHost);
        size_t bad = 0;
        for (size_t i = 0; i < x.size(); ++i) bad += (x[i] != y[i]);
        printf("    %s: %zu differing doubles (%s)\n", name, bad, cudaGetErrorString(cudaGetLastError()));
    };
    auto run_w4 = [&](auto S_c) {
        constexpr int S = decltype(S_c)::value;
        const size_t sm = (size_t)S * mcnd::MS_STAGE * 8;
        cudaFuncSetAttribute(mcnd::k2_gemm_w4_kernel<K, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        for (int grid : {(int)T, (int)T / 2, (int)T / 4, 2 * sms}) {
            auto f = [&]() { mcnd::k2_gemm_w4_kernel<K, S><<<grid, mcnd::W4_THREADS, sm>>>(ws, ld, 0, n, n, L, K, W, ld, w, abort); };
            float tt = timeit(f, ws, bytes);
            printf("w4 S=%d grid %6d: %.3f ms %.2f TFLOP/s\n", S, grid, tt, fl / tt / 1e9);
            cudaMemcpy(ws, ws0, bytes, cudaMemcpyDeviceToDevice); f(); check("vs ms");
        }
    };
    run_w4(std::integral_constant<int, 3>{});
    {   // K per stage 32 (one barrier per 8 k-steps), 2 stages
        const size_t sm = (size_t)2 * (mcnd::BM * 36 + 32 * mcnd::LDWS) * 8;
        cudaFuncSetAttribute(mcnd::k2_gemm_w4_kernel<K, 2, 2, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        for (int grid : {(int)T, 2 * sms}) {
            auto f = [&]() { mcnd::k2_gemm_w4_kernel<K, 2, 2, 32><<<grid, mcnd::W4_THREADS, sm>>>(ws, ld, 0, n, n, L, K, W, ld, w, abort); };
            float tt = timeit(f, ws, bytes);
            printf("w4 BK=32 S=2 grid %6d: %.3f ms %.2f TFLOP/s\n", grid, tt, fl / tt / 1e9);
            cudaMemcpy(ws, ws0, bytes, cudaMemcpyDeviceToDevice); f(); check("vs ms");
        }
    }

    {   // the critical-path shape: 128 rows x n, 64-wide tiles (8-warp-era kernel vs WN = 1)
        const int M2 = 128;
        const size_t sm64 = (size_t)mcnd::MS_ST * (mcnd::BM * mcnd::MS_LDL + mcnd::MS_BK * (64 + 4)) * 8;
        const size_t sm1 = (size_t)3 * (mcnd::BM * mcnd::MS_LDL + mcnd::MS_BK * (64 + 4)) * 8;
        cudaFuncSetAttribute(mcnd::k2_gemm_ms_kernel<K, 1, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm64);
        cudaFuncSetAttribute(mcnd::k2_gemm_w4_kernel<K, 3, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1);
        const int tn = ((n + 63) / 64) * 2;
        auto f0 = [&]() { mcnd::k2_gemm_ms_kernel<K, 1, 64><<<tn, 128, sm64>>>(ws, ld, 0, M2, n, L, K, W, ld, w, abort); };
        auto f1 = [&]() { mcnd::k2_gemm_w4_kernel<K, 3, 1><<<tn, 64, sm1>>>(ws, ld, 0, M2, n, L, K, W, ld, w, abort); };
        const double fl2 = 2.0 * M2 * (double)n * K;
        float t0 = timeit(f0, ws, bytes, 20), t1 = timeit(f1, ws, bytes, 20);
        printf("128 rows: ms<64-wide> %.1f us (%.2f TF), w4<WN=1> %.1f us (%.2f TF)\n", t0 * 1e3, fl2 / t0 / 1e9, t1 * 1e3, fl2 / t1 / 1e9);
        cudaMemcpy(ws, ws0, bytes, cudaMemcpyDeviceToDevice); f0(); cudaMemcpy(out_a, ws, bytes, cudaMemcpyDeviceToDevice);
        cudaMemcpy(ws, ws0, bytes, cudaMemcpyDeviceToDevice); f1(); check("WN=1 vs ms 64-wide");
    }
    cublasHandle_t h; cublasCreate(&h);
    const double one = 1.0, mone = -1.0;
    // row-major C(n x n, ld) -= L(n x K) W(K x n): column-major C^T = C^T - W^T L^T
    auto cb = [&]() { cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, n, n, K, &mone, W, ld, L, K, &one, ws, ld); };
    t = timeit(cb, ws, bytes);
    printf("cuBLAS DGEMM   : %.3f ms %.2f TFLOP/s\n", t, fl / t / 1e9);
    return 0;
}

// Trailing-GEMM efficiency vs the update rank K (128: the panel pair; 256: two pairs at once):
// k2_gemm_w4_kernel persistent and one tile per CTA, against cuBLAS DGEMM, C = C - L W at n x n.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o gemm_k gemm_k.cu -lcublas -lcurand
#include <cstdio>
#include <cublas_v2.h>
#include <curand.h>
#include "../../paper_1811_08057_b200/csrc/k2_blocked.cu"

template <class F>
static float timeit(F f, double* ws, const double* ws0, size_t bytes, int reps = 5) {
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

template <int K>
static void run(int n, double* ws, double* ws0, double* L, double* W, unsigned long long* w, unsigned* abort, int64_t ld,
                size_t bytes, int sms, cublasHandle_t h) {
    const int64_t T = (int64_t)((n + mcnd::BM - 1) / mcnd::BM) * ((n + mcnd::BN - 1) / mcnd::BN);
    const double fl = 2.0 * n * (double)n * K;
    const size_t sm = (size_t)3 * mcnd::MS_STAGE * 8;
    cudaFuncSetAttribute(mcnd::k2_gemm_w4_kernel<K, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    for (int grid : {(int)T, 2 * sms}) {
        auto f = [&]() { mcnd::k2_gemm_w4_kernel<K, 3><<<grid, mcnd::W4_THREADS, sm>>>(ws, ld, 0, n, n, L, K, W, ld, w, abort); };
        float tt = timeit(f, ws, ws0, bytes);
        printf("K=%d w4 grid %6d: %.3f ms %.2f TFLOP/s (%s)\n", K, grid, tt, fl / tt / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
    const double one = 1.0, mone = -1.0;
    auto cb = [&]() { cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, n, n, K, &mone, W, ld, L, K, &one, ws, ld); };
    float t = timeit(cb, ws, ws0, bytes);
    printf("K=%d cuBLAS      : %.3f ms %.2f TFLOP/s\n", K, t, fl / t / 1e9);
}

int main(int argc, char** argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 16384;
    const int64_t ld = (n + 15) / 16 * 16;
    const size_t bytes = (size_t)n * ld * 8;
    double *ws, *ws0, *L, *W, *wit; unsigned* abort;
    cudaMalloc(&ws, bytes); cudaMalloc(&ws0, bytes);
    cudaMalloc(&L, (size_t)n * 512 * 8); cudaMalloc(&W, (size_t)512 * ld * 8);
    cudaMalloc(&wit, (size_t)n * 8); cudaMalloc(&abort, 4);
    cudaMemset(abort, 0, 4); cudaMemset(wit, 0, (size_t)n * 8);
    curandGenerator_t gen; curandCreateGenerator(&gen, CURAND_RNG_PSEUDO_DEFAULT);
    curandSetPseudoRandomGeneratorSeed(gen, 5);
    curandGenerateUniformDouble(gen, ws0, bytes / 8);
    curandGenerateUniformDouble(gen, L, (size_t)n * 512);
    curandGenerateUniformDouble(gen, W, (size_t)512 * ld);
    auto* w = reinterpret_cast<unsigned long long*>(wit);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cublasHandle_t h; cublasCreate(&h);
    run<128>(n, ws, ws0, L, W, w, abort, ld, bytes, sms, h);
    run<256>(n, ws, ws0, L, W, w, abort, ld, bytes, sms, h);
    run<512>(n, ws, ws0, L, W, w, abort, ld, bytes, sms, h);
    return 0;
}

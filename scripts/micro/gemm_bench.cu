// Microbenchmark of the K2 trailing-update GEMM (C[MxN] -= L[Mx64] W[64xN]) as built
// into the library (k2_blocked.cu is included verbatim), for M = N = argv[1].
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../../paper_1811_08057_b200/csrc/k2_blocked.cu"
#ifndef KK
#define KK 64
#endif
int main(int argc, char** argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 16384;
    const int budget = argc > 2 ? atoi(argv[2]) : 0;  // 0 persistent, -1 one tile per CTA, >0 fat CTAs
    const int64_t ld = (n + 15) / 16 * 16;
    double *ws, *L, *W, *wit;
    unsigned* abort;
    cudaMalloc(&ws, (size_t)n * ld * 8);
    cudaMalloc(&L, (size_t)n * KK * 8);
    cudaMalloc(&W, (size_t)KK * ld * 8);
    cudaMalloc(&wit, (size_t)n * 8);
    cudaMalloc(&abort, 4);
    cudaMemset(abort, 0, 4);
    cudaMemset(ws, 0, (size_t)n * ld * 8);
    cudaMemset(L, 0, (size_t)n * KK * 8);
    cudaMemset(W, 0, (size_t)KK * ld * 8);
    cudaMemset(wit, 0, (size_t)n * 8);
    for (int i = 0; i < 3; ++i) mcnd::k2_gemm(ws, ld, 0, n, n, KK, L, KK, W, ld, wit, abort, 0, budget);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    const int reps = 10;
    for (int i = 0; i < reps; ++i) mcnd::k2_gemm(ws, ld, 0, n, n, KK, L, KK, W, ld, wit, abort, 0, budget);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    const double fl = 2.0 * n * (double)n * KK;
    printf("budget=%d K=%d n=%d gemm %.3f ms  %.1f TFLOP/s  C-traffic %.0f GB/s  err=%s\n", budget, KK, n, ms, fl / ms / 1e9,
           16.0 * n * (double)n / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    return 0;
}

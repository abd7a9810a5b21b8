// The multistage trailing GEMM (k2_gemm_ms_kernel, one tile per CTA) at K = 128..512:
// separates the per-tile C load/store overhead from the DMMA mainloop rate.
#include <cstdio>
#include "../../paper_1811_08057_b200/csrc/k2_blocked.cu"
template <int K>
void run(int n) {
    constexpr int NTH = mcnd::MS_THREADS;
    const int64_t ld = (n + 15) / 16 * 16;
    double *ws, *L, *W, *wit; unsigned* abort;
    cudaMalloc(&ws, (size_t)n * ld * 8); cudaMalloc(&L, (size_t)n * K * 8); cudaMalloc(&W, (size_t)K * ld * 8);
    cudaMalloc(&wit, (size_t)n * 8); cudaMalloc(&abort, 4);
    cudaMemset(abort, 0, 4); cudaMemset(ws, 0, (size_t)n * ld * 8); cudaMemset(L, 0, (size_t)n * K * 8);
    cudaMemset(W, 0, (size_t)K * ld * 8); cudaMemset(wit, 0, (size_t)n * 8);
    const size_t smem = (size_t)mcnd::MS_ST * mcnd::MS_STAGE * sizeof(double);
    cudaFuncSetAttribute(mcnd::k2_gemm_ms_kernel<K, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int64_t T = (int64_t)((n + mcnd::BM - 1) / mcnd::BM) * ((n + mcnd::BN - 1) / mcnd::BN);
    auto launch = [&]() {
        mcnd::k2_gemm_ms_kernel<K, 1><<<(unsigned)T, NTH, smem>>>(ws, ld, 0, n, n, L, K, W, ld,
                                                               reinterpret_cast<unsigned long long*>(wit), abort);
    };
    for (int i = 0; i < 2; ++i) launch();
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int i = 0; i < 5; ++i) launch();
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
    printf("ms kernel NTH=%d K=%d n=%d: %.3f ms %.1f TFLOP/s  %s\n", NTH, K, n, ms, 2.0 * n * (double)n * K / ms / 1e9,
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(ws); cudaFree(L); cudaFree(W); cudaFree(wit); cudaFree(abort);
}
int main() { run<128>(16384); run<256>(16384); run<512>(16384); return 0; }

// Microbenchmark: FP64 vector (non-tensor) throughput on this GPU: DFMA, DMUL+DADD (two roundings).
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(double* out, int iters) {
    double a[8], b = 1.0000001 + threadIdx.x * 1e-9, c = 0.9999999;
    for (int i = 0; i < 8; ++i) a[i] = i * 1e-3 + blockIdx.x * 1e-6;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (MODE == 0) a[i] = fma(a[i], b, c);
            else a[i] = __dsub_rn(a[i], __dmul_rn(b, c));
        }
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += a[i];
    if (s == 1234.5) out[0] = s;
}
template <int MODE>
void run(int threads, int bps) {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out; cudaMalloc(&out, 8);
    int iters = 4096;
    k<MODE><<<sms * bps, threads>>>(out, iters);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<MODE><<<sms * bps, threads>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = (MODE == 0 ? 1.0 : 2.0) * 8.0 * iters * (double)threads * sms * bps;
    printf("mode=%s threads=%d blocks/SM=%d: %.2f T FP64-instr/s = %.1f per clk per SM (at 1.965 GHz)\n",
           MODE == 0 ? "DFMA" : "DMUL+DADD", threads, bps, ops / ms / 1e9, ops / (ms * 1e-3) / sms / 1.965e9);
}
int main() { run<0>(256, 4); run<0>(1024, 2); run<1>(256, 4); run<1>(1024, 2); return 0; }

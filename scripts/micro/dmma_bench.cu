// Microbenchmark: peak DMMA.8x8x4 throughput vs warps per SM and accumulators per warp.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int NACC>
__global__ void k(double* out, int iters) {
    double acc[NACC][2];
    double a = threadIdx.x * 1e-3, b = blockIdx.x * 1e-3;
    for (int i = 0; i < NACC; ++i) { acc[i][0] = 0; acc[i][1] = 0; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < NACC; ++i) dmma(acc[i][0], acc[i][1], a, b);
    }
    double s = 0;
    for (int i = 0; i < NACC; ++i) s += acc[i][0] + acc[i][1];
    if (s == 12345.0) out[0] = s;
}
template <int NACC>
void run(int threads, int blocks_per_sm) {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out; cudaMalloc(&out, 8);
    int iters = 4096 / NACC * 16;
    k<NACC><<<sms * blocks_per_sm, threads>>>(out, iters);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<NACC><<<sms * blocks_per_sm, threads>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 512.0 * NACC * (double)iters * (threads / 32) * sms * blocks_per_sm;
    printf("NACC=%2d threads=%4d blocks/SM=%d warps/SM=%2d : %.1f TFLOP/s\n", NACC, threads, blocks_per_sm,
           threads / 32 * blocks_per_sm, flops / ms / 1e9);
    cudaFree(out);
}
int main() {
    run<16>(128, 1); run<16>(256, 1); run<16>(512, 1); run<16>(1024, 1);
    run<8>(256, 1); run<8>(512, 1); run<4>(512, 1); run<32>(256, 1); run<16>(128, 4); run<8>(1024, 1);
    return 0;
}

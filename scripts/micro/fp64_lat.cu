// Dependent-chain latency of FP64 operations on one thread (cycles per op).
#include <cstdio>
__global__ void k(double* out, double a, double b, int n, long long* cyc) {
    double x = a, y = b;
    long long t0, t1;
    // DFMA chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = fma(x, y, 1e-300);
    t1 = clock64(); cyc[0] = t1 - t0;
    // DADD chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = x + y;
    t1 = clock64(); cyc[1] = t1 - t0;
    // division chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = __ddiv_rn(x, y);
    t1 = clock64(); cyc[2] = t1 - t0;
    // fabs + compare + select chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = (fabs(x) > y) ? x * 0.5 : x + 1.0;
    t1 = clock64(); cyc[3] = t1 - t0;
    // integer 64-bit chain (abs bits compare)
    unsigned long long u = __double_as_longlong(x);
    t0 = clock64();
    for (int i = 0; i < n; ++i) u = ((u & 0x7fffffffffffffffull) > 12345ull) ? (u >> 1) : (u + 3);
    t1 = clock64(); cyc[4] = t1 - t0;
    // shuffle chain (double)
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1) + 1.0;
    t1 = clock64(); cyc[5] = t1 - t0;
    // redux.sync chain
    unsigned r = (unsigned)u;
    t0 = clock64();
    for (int i = 0; i < n; ++i) r = __reduce_max_sync(0xffffffffu, r) + 1u;
    t1 = clock64(); cyc[6] = t1 - t0;
    // shared load-store chain
    __shared__ double sh[64];
    sh[threadIdx.x] = x;
    __syncthreads();
    int j = threadIdx.x;
    t0 = clock64();
    for (int i = 0; i < n; ++i) { double z = sh[j]; j = (int)(z == 12345.0) + threadIdx.x; }
    t1 = clock64(); cyc[7] = t1 - t0;
    // __syncthreads cost (1024 threads)
    t0 = clock64();
    for (int i = 0; i < n; ++i) __syncthreads();
    t1 = clock64(); cyc[8] = t1 - t0;
    out[threadIdx.x] = x + (double)u + r + j;
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 8 * 1024); cudaMalloc(&c, 8 * 16);
    const int n = 1000;
    const char* nm[] = {"dfma", "dadd", "ddiv_rn", "fabs+cmp+sel", "int64 cmp+sel", "shfl+dadd", "redux.max", "lds dep", "syncthreads(1024 thr)"};
    for (int bs : {32, 1024}) {
        k<<<1, bs>>>(o, 1.0000001, 0.9999999, n, c);
        long long h[16]; cudaMemcpy(h, c, 8 * 16, cudaMemcpyDeviceToHost);
        printf("block %d:\n", bs);
        for (int i = 0; i < 9; ++i) printf("  %-22s %.1f cycles/op\n", nm[i], (double)h[i] / n);
    }
    return 0;
}

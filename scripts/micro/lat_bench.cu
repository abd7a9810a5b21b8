// Dependent-chain latencies (cycles) of the operations on the cluster panel kernel's per-pivot path:
// redux.sync, ballot, shfl, DFMA, reciprocal + Markstein division, named barrier with n warps, LDS,
// and the st.async -> mbarrier round trip across a cluster.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 lat_bench.cu -o lat_bench
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k_lat(unsigned long long* out, double dv, unsigned seed) {
    __shared__ double sd[64];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int N = 256;
    unsigned long long t0, t1;
    if (warp == 0) {
        unsigned v = seed + lane;
        t0 = clock64();
#pragma unroll 8
        for (int i = 0; i < N; ++i) v = __reduce_max_sync(0xffffffffu, v + (unsigned)lane);
        t1 = clock64();
        if (lane == 0) { out[0] = (t1 - t0) / N; out[20] = v; }
        v = seed + lane;
        t0 = clock64();
#pragma unroll 8
        for (int i = 0; i < N; ++i) v = __ballot_sync(0xffffffffu, (v >> (lane & 7)) & 1u) + lane;
        t1 = clock64();
        if (lane == 0) { out[1] = (t1 - t0) / N; out[21] = v; }
        v = seed + lane;
        t0 = clock64();
#pragma unroll 8
        for (int i = 0; i < N; ++i) v = __shfl_sync(0xffffffffu, v, (lane + 1) & 31) + 1u;
        t1 = clock64();
        if (lane == 0) { out[2] = (t1 - t0) / N; out[22] = v; }
        double x = dv + lane;
        t0 = clock64();
#pragma unroll 8
        for (int i = 0; i < N; ++i) x = __fma_rn(x, 1.0000001, 1e-9);
        t1 = clock64();
        if (lane == 0) { out[3] = (t1 - t0) / N; out[23] = (unsigned long long)x; }
        x = dv + lane;
        t0 = clock64();
#pragma unroll 8
        for (int i = 0; i < N; ++i) x = __drcp_rn(x) + 1.5;
        t1 = clock64();
        if (lane == 0) { out[4] = (t1 - t0) / N; out[24] = (unsigned long long)x; }
        x = dv + lane;
        t0 = clock64();
#pragma unroll 8
        for (int i = 0; i < N; ++i) x = __ddiv_rn(dv, x) + 1.5;
        t1 = clock64();
        if (lane == 0) { out[5] = (t1 - t0) / N; out[25] = (unsigned long long)x; }
        sd[lane] = (double)((lane + 1) & 31);
        __syncwarp();
        int idx = lane;
        t0 = clock64();
#pragma unroll 8
        for (int i = 0; i < N; ++i) idx = (int)sd[idx];
        t1 = clock64();
        if (lane == 0) { out[6] = (t1 - t0) / N; out[26] = idx; }
        // two dependent redux + ballot (the exact 64-bit argmax)
        unsigned long long b = seed * 2654435761ull + lane;
        t0 = clock64();
#pragma unroll 4
        for (int i = 0; i < N; ++i) {
            const unsigned hi = (unsigned)(b >> 32), lo = (unsigned)b;
            const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
            const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
            const unsigned ball = __ballot_sync(0xffffffffu, hi == mh && lo == ml);
            b = b * 6364136223846793005ull + ball;
        }
        t1 = clock64();
        if (lane == 0) { out[7] = (t1 - t0) / N; out[27] = b; }
    }
    __syncthreads();
    // named barrier among nw warps (all warps of the CTA here)
    t0 = clock64();
    for (int i = 0; i < N; ++i) asm volatile("bar.sync 1, %0;" ::"r"((int)blockDim.x) : "memory");
    t1 = clock64();
    if (threadIdx.x == 0) out[8] = (t1 - t0) / N;
}

// all-to-all st.async exchange across a cluster: every CTA sends 16 bytes to every CTA, waits for all
__global__ void k_xchg(unsigned long long* out, int iters) {
    __shared__ __align__(16) unsigned long long rcv[2][16][2];
    __shared__ unsigned long long bar[2];
    unsigned g, C;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(g));
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(C));
    const int lane = threadIdx.x;
    if (lane == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[1])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    uint32_t r_rcv = 0, r_bar = 0;
    if (lane < (int)C) {
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r_rcv) : "r"(smem_u32(&rcv[0][g][0])), "r"((unsigned)lane));
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r_bar) : "r"(smem_u32(&bar[0])), "r"((unsigned)lane));
    }
    unsigned long long acc = g;
    const unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        const unsigned par = i & 1, ph = (i >> 1) & 1;
        if (lane < (int)C)
            asm volatile("st.async.weak.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];"
                         ::"r"(r_rcv + par * 256), "l"(acc), "l"(acc + 1), "r"(r_bar + par * 8) : "memory");
        if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[par])), "r"(C * 16) : "memory");
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                         : "=r"(ok) : "r"(smem_u32(&bar[par])), "r"(ph) : "memory");
        acc += rcv[par][(lane + i) % C][0];
    }
    const unsigned long long t1 = clock64();
    if (lane == 0 && g == 0) { out[0] = (t1 - t0) / iters; out[1] = acc; }
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__global__ void k_csync(unsigned long long* out, int iters) {
    const unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i)
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (t1 - t0) / iters;
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 64 * 8);
    unsigned long long h[64];
    for (int nt : {32, 160, 320, 512}) {
        k_lat<<<1, nt>>>(d, 1.25, 7u);
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        if (nt == 32)
            printf("cycles per dependent op: redux.max %llu, ballot %llu, shfl %llu, DFMA %llu, drcp %llu, ddiv %llu, LDS %llu, exact u64 argmax (2 redux + ballot) %llu\n",
                   h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7]);
        printf("bar.sync with %d threads: %llu cycles\n", nt, h[8]);
    }
    for (int C : {2, 4, 8, 16}) {
        cudaFuncSetAttribute(k_xchg, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaFuncSetAttribute(k_csync, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(C); cfg.blockDim = dim3(32);
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.attrs = at; cfg.numAttrs = 1;
        cudaError_t e = cudaLaunchKernelEx(&cfg, k_xchg, d, 2000);
        cudaError_t e2 = cudaDeviceSynchronize();
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        printf("cluster %2d: all-to-all st.async exchange round %llu cycles (%s/%s)", C, h[0], cudaGetErrorString(e), cudaGetErrorString(e2));
        cfg.blockDim = dim3(512);
        e = cudaLaunchKernelEx(&cfg, k_csync, d, 2000);
        e2 = cudaDeviceSynchronize();
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        printf(", barrier.cluster (512 threads) %llu cycles (%s/%s)\n", h[0], cudaGetErrorString(e), cudaGetErrorString(e2));
    }
    return 0;
}

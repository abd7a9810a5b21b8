// Cross-SM ping-pong latency through L2 (tagged 16-byte records, no fences) and
// through DSMEM inside a cluster.  Prints the one-way hop in cycles / ns.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ void st16(double2* p, double2 v) {
    asm volatile("st.global.cg.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}
__device__ __forceinline__ double2 ld16(const double2* p) {
    double2 v;
    asm volatile("ld.global.cg.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p) : "memory");
    return v;
}
__global__ void pp_global(double2* buf, int iters, long long* out, int far) {
    // CTA 0 and CTA 'far' (others idle)
    const int me = blockIdx.x == 0 ? 0 : (blockIdx.x == far ? 1 : -1);
    if (me < 0 || threadIdx.x) return;
    long long t0 = clock64();
    unsigned long long g0; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
    for (int i = 0; i < iters; ++i) {
        if (me == 0) {
            st16(buf + 0, make_double2(1.0 * i, __longlong_as_double(2 * i + 1)));
            while (__double_as_longlong(ld16(buf + 1).y) != 2 * i + 2) {}
        } else {
            while (__double_as_longlong(ld16(buf + 0).y) != 2 * i + 1) {}
            st16(buf + 1, make_double2(1.0 * i, __longlong_as_double(2 * i + 2)));
        }
    }
    unsigned long long g1; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
    if (me == 0) { out[0] = clock64() - t0; out[1] = (long long)(g1 - g0); }
}
__global__ void __cluster_dims__(2, 1, 1) pp_dsmem(int iters, long long* out) {
    __shared__ __align__(16) double2 box[2];
    unsigned rank; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    if (threadIdx.x == 0) { box[0] = make_double2(0, 0); box[1] = make_double2(0, 0); }
    asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (threadIdx.x == 0) {
        const unsigned other = rank ^ 1u;
        unsigned la = (unsigned)__cvta_generic_to_shared(&box[0]), ra;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(other));
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            if (rank == 0) {
                asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(ra), "d"(1.0), "d"(__longlong_as_double(2 * i + 1)) : "memory");
                double2 v;
                do { asm volatile("ld.volatile.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(la) : "memory"); }
                while (__double_as_longlong(v.y) != 2 * i + 2);
            } else {
                double2 v;
                do { asm volatile("ld.volatile.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(la) : "memory"); }
                while (__double_as_longlong(v.y) != 2 * i + 1);
                asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(ra), "d"(1.0), "d"(__longlong_as_double(2 * i + 2)) : "memory");
            }
        }
        if (rank == 0) out[0] = clock64() - t0;
    }
    asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
int main() {
    double2* buf; long long* out; cudaMalloc(&buf, 4096); cudaMalloc(&out, 64);
    const int iters = 2000;
    for (int far : {1, 2, 8, 37, 74, 100, 147}) {
        cudaMemset(buf, 0, 4096);
        pp_global<<<148, 32>>>(buf, iters, out, far);
        long long h[2]; cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
        printf("global CTA0<->CTA%-3d: one-way hop %.0f cycles, %.0f ns\n", far, h[0] / (2.0 * iters), h[1] / (2.0 * iters));
    }
    pp_dsmem<<<2, 32>>>(iters, out);
    long long h; cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
    printf("dsmem pair: one-way hop %.0f cycles (%s)\n", h / (2.0 * iters), cudaGetErrorString(cudaGetLastError()));
    return 0;
}

// Pair prep (shared by the standalone kernel in k2_blocked.cu and the second panel
// kernel of a pair in k2_panel.cu, which runs it in its CTA 0 right after its own
// descriptor is final): from the two panels' gather descriptors build the pair's
// composite descriptor, Wp[s][s'] = -W_k[s][P1[s']] and W_k's columns in the pair's
// final layout.
#pragma once
#include "mcnd_internal.h"

namespace mcnd {
namespace {

struct PairPrepSmem {
    K2Gather s0, s1;
    int cand[4 * kK2B];
    int nc, nm;
};

__device__ __forceinline__ int pi_of(const K2Gather* g, int x) {
    for (int k = 0; k < g->n_moved; ++k)
        if (g->moved_c[k] == x) return g->moved_src[k];
    return x;
}

// pi_of by one warp: the lanes scan the moved list together (entries are unique)
__device__ __forceinline__ int pi_of_warp(const K2Gather& g, int x, int lane) {
    const int n = g.n_moved;
    for (int k0 = 0; k0 < n; k0 += 32) {
        const int k = k0 + lane;
        const bool hit = k < n && g.moved_c[k] == x;
        const unsigned b = __ballot_sync(0xffffffffu, hit);
        if (b) return __shfl_sync(0xffffffffu, hit ? g.moved_src[k] : 0, __ffs(b) - 1);
    }
    return x;
}

// The pair's composite gather descriptor from the two panels' descriptors (staged in
// shared memory: g1 may have just been written by this CTA).  All NT threads call it;
// every lookup is done by a whole warp.
template <int NT>
__device__ void pair_prep_desc(const K2Gather* __restrict__ g0, const K2Gather* __restrict__ g1, int32_t m,
                               K2Gather* __restrict__ gpair, PairPrepSmem& sm, int tid) {
    constexpr int kWarps = NT / 32;
    const int lane = tid & 31, warp = tid >> 5;
    {
        constexpr int kWords = (int)(sizeof(K2Gather) / sizeof(int32_t));
        const int32_t* a0 = reinterpret_cast<const int32_t*>(g0);
        const int32_t* a1 = reinterpret_cast<const int32_t*>(g1);
        for (int i = tid; i < kWords; i += NT) {
            reinterpret_cast<int32_t*>(&sm.s0)[i] = __ldcg(a0 + i);
            reinterpret_cast<int32_t*>(&sm.s1)[i] = __ldcg(a1 + i);
        }
        if (tid == 0) { sm.nc = 0; sm.nm = 0; }
    }
    __syncthreads();
    const K2Gather& s0 = sm.s0;
    const K2Gather& s1 = sm.s1;
    for (int t = warp; t < kK2B; t += kWarps) {  // panel k's pivots, then panel k+1's mapped to width m
        const int src = pi_of_warp(s0, s1.P[t], lane);
        if (lane == 0) {
            gpair->P[t] = s0.P[t];
            gpair->P[kK2B + t] = src;
            gpair->l[t] = s1.l[t];
        }
    }
    const int wf = m - 2 * kK2B;  // candidate moved columns: targets of either panel inside the final width
    if (tid < s1.n_moved && s1.moved_c[tid] < wf) sm.cand[atomicAdd(&sm.nc, 1)] = s1.moved_c[tid];
    if (tid < s0.n_moved && s0.moved_c[tid] < wf) sm.cand[atomicAdd(&sm.nc, 1)] = s0.moved_c[tid];
    __syncthreads();
    const int nc = sm.nc;
    for (int i = warp; i < nc; i += kWarps) {
        const int c = sm.cand[i];
        bool dup = false;  // an earlier copy of the same column (deduplicated)
        for (int j0 = 0; j0 < i && !dup; j0 += 32)
            dup = __any_sync(0xffffffffu, j0 + lane < i && sm.cand[j0 + lane] == c);
        if (dup) continue;
        const int src = pi_of_warp(s0, pi_of_warp(s1, c, lane), lane);
        if (src != c && lane == 0) {
            const int k = atomicAdd(&sm.nm, 1);
            gpair->moved_c[k] = c;
            gpair->moved_src[k] = src;
        }
    }
    __syncthreads();
    if (tid == 0) gpair->n_moved = sm.nm;
}

// All NT threads of the CTA call it (contains __syncthreads).  g0: panel k (layout
// width m), g1: panel k+1 (width m-64); Wc rows 0..63 = W_k (width m-64 layout).
// The descriptors are staged in shared memory (L2 reads: g1 may have just been
// written by this CTA) so the column-map compositions walk shared memory.
template <int NT>
__device__ void pair_prep_body(const K2Gather* __restrict__ g0, const K2Gather* __restrict__ g1, int32_t m,
                               double* __restrict__ Wc, int64_t ldw, double* __restrict__ Wp,
                               K2Gather* __restrict__ gpair, PairPrepSmem& sm, int tid) {
    {
        constexpr int kWords = (int)(sizeof(K2Gather) / sizeof(int32_t));
        const int32_t* a0 = reinterpret_cast<const int32_t*>(g0);
        const int32_t* a1 = reinterpret_cast<const int32_t*>(g1);
        for (int i = tid; i < kWords; i += NT) {
            reinterpret_cast<int32_t*>(&sm.s0)[i] = __ldcg(a0 + i);
            reinterpret_cast<int32_t*>(&sm.s1)[i] = __ldcg(a1 + i);
        }
        if (tid == 0) { sm.nc = 0; sm.nm = 0; }
    }
    __syncthreads();
    const K2Gather& s0 = sm.s0;
    const K2Gather& s1 = sm.s1;
    // (a) Wp[s][s'] = W_k[s][P1[s']] (before W_k's columns are permuted)
#pragma unroll 4
    for (int e = tid; e < kK2B * kK2B; e += NT) {
        const int sr = e / kK2B, sp = e % kK2B;
        Wp[sr * kK2B + sp] = -Wc[(int64_t)sr * ldw + s1.P[sp]];  // negated: (-L1) = (-X) + (-L0)(-Wp)
    }
    // (b) composite gather columns: panel k's pivots, then panel k+1's pivots mapped to width m
    if (tid < kK2B) {
        gpair->P[tid] = s0.P[tid];
        gpair->P[kK2B + tid] = pi_of(&s0, s1.P[tid]);
        gpair->l[tid] = s1.l[tid];
    }
    // candidate moved columns of the pair: targets of either panel inside the final width
    const int wf = m - 2 * kK2B;
    if (tid < s1.n_moved && s1.moved_c[tid] < wf) sm.cand[atomicAdd(&sm.nc, 1)] = s1.moved_c[tid];
    if (tid < s0.n_moved && s0.moved_c[tid] < wf) sm.cand[atomicAdd(&sm.nc, 1)] = s0.moved_c[tid];
    __syncthreads();
    if (tid < sm.nc) {
        const int c = sm.cand[tid];
        bool first = true;
        for (int k = 0; k < tid && first; ++k) first = sm.cand[k] != c;
        if (first) {
            const int src = pi_of(&s0, pi_of(&s1, c));
            if (src != c) {
                const int k = atomicAdd(&sm.nm, 1);
                gpair->moved_c[k] = c;
                gpair->moved_src[k] = src;
            }
        }
    }
    __syncthreads();
    if (tid == 0) gpair->n_moved = sm.nm;
    // (c) W_k's columns into the pair's final layout: column c <- column pi_{k+1}(c)
    //     (sources lie in the tail [m-128, m-64), never written)
    const int nm1 = s1.n_moved;
    for (int e = tid; e < kK2B * nm1; e += NT) {
        const int sr = e / nm1, k = e % nm1;
        const int c = s1.moved_c[k];
        if (c < wf) Wc[(int64_t)sr * ldw + c] = Wc[(int64_t)sr * ldw + s1.moved_src[k]];
    }
}

}  // namespace
}  // namespace mcnd

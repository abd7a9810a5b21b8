// Standalone run of the K2 panel kernel on a random 64 x m panel, with per-step phase trace.
//   nvcc ... -DKP_SRC='"path/to/k2_panel.cu"' [-DKP_OLD] kp_bench.cu   (KP_OLD: the two-hop
//   protocol of commit 40a4218, separate CAND/WREC records) -- compare the printed checksums
//   of two builds: the protocols must produce bitwise the same W and pivots.
#ifndef KP_TRACE
#define KP_TRACE 1
#endif
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <vector>
#include <random>
#include <algorithm>
#ifndef KP_SRC
#define KP_SRC "../../paper_1811_08057_b200/csrc/k2_panel.cu"
#endif
#include KP_SRC
using namespace mcnd;
int main(int argc, char** argv) {
    const int m = argc > 1 ? atoi(argv[1]) : 8000;
    const int G = argc > 2 ? atoi(argv[2]) : 45;
    const int r1 = argc > 3 ? atoi(argv[3]) : 0;
    int cw = ((m + G - 1) / G + 1) / 2 * 2;
    const int64_t ld = (m + 15) / 16 * 16;
    std::vector<double> h((size_t)64 * ld);
    std::mt19937_64 rng(1);
    std::uniform_real_distribution<double> U(-1, 1);
    for (auto& x : h) x = U(rng);
    double *ws, *wit, *W; PivRec* rec; K2Gather* pan; unsigned* abort; ulonglong2 *cand, *wrec, *colb, *lastb; K1Err* err;
    cudaMalloc(&ws, h.size() * 8); cudaMemcpy(ws, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    cudaMalloc(&wit, 64 * 8); cudaMemset(wit, 0, 64 * 8);
    cudaMalloc(&W, (size_t)64 * ld * 8);
    cudaMalloc(&rec, 64 * sizeof(PivRec)); cudaMalloc(&pan, sizeof(K2Gather)); cudaMalloc(&abort, 4); cudaMemset(abort, 0, 4);
    cudaMalloc(&cand, 64 * kKPMaxG * 32); cudaMalloc(&wrec, 64 * kKPMaxG * 32); cudaMalloc(&colb, (size_t)64 * kKPMaxG * 64 * 16);
    cudaMalloc(&lastb, 64 * 64 * 16); cudaMalloc(&err, sizeof(K1Err)); cudaMemset(err, 0, sizeof(K1Err));
    cudaMemset(cand, 0, 64 * kKPMaxG * 32); cudaMemset(wrec, 0, 64 * kKPMaxG * 32);
    cudaMemset(colb, 0, (size_t)64 * kKPMaxG * 64 * 16); cudaMemset(lastb, 0, 64 * 64 * 16);
    KPParams p{};
    p.ws = ws; p.ld = ld; p.row0 = 0; p.m = m; p.G = G; p.cw = cw; p.wit = wit; p.rec = rec; p.epoch = 1;
    p.W = W; p.ldw = ld; p.pan = pan; p.abort = abort; p.cand = cand; p.colbuf = colb; p.lastbuf = lastb;
#ifdef KP_OLD
    p.wrec = wrec;
#else
    p.wrec = wrec;
#endif
    p.err = err; p.timeout_ns = 5000000000ull;
    if (r1) {  // second panel of a pair: the r1 prologue (rank-64 update of the rows)
        K2Gather hg{};
        for (int k = 0; k < 64; ++k) hg.P[k] = k;
        hg.n_moved = 0;
        K2Gather* dg; cudaMalloc(&dg, sizeof(K2Gather)); cudaMemcpy(dg, &hg, sizeof(hg), cudaMemcpyHostToDevice);
        double* W0; cudaMalloc(&W0, (size_t)64 * ld * 8);
        std::vector<double> hw((size_t)64 * ld);
        for (auto& x : hw) x = 1e-3 * U(rng);
        cudaMemcpy(W0, hw.data(), hw.size() * 8, cudaMemcpyHostToDevice);
        p.r1_g0 = dg; p.r1_W = W0; p.r1_ldw = ld;
        printf("with the r1 prologue\n");
    }
    float best = 1e30f;
    for (int it = 0; it < 5; ++it) {
        cudaMemcpy(ws, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
        p.tag0 = (unsigned)(1000 + it * 100);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        cudaError_t e = kp_launch(p, 0);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
        if (e != cudaSuccess) printf("launch: %s\n", cudaGetErrorString(e));
    }
    K1Err he{};
    cudaMemcpy(&he, err, sizeof(he), cudaMemcpyDeviceToHost);
    printf("m=%d G=%d cw=%d: best %.1f us (%.2f us/step), error %u torn %u\n", m, G, cw, best * 1e3, best * 1e3 / 64, he.error, he.torn);
    {
        std::vector<double> w1((size_t)64 * ld);
        std::vector<PivRec> rr(64);
        cudaMemcpy(w1.data(), W, w1.size() * 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(rr.data(), rec, 64 * sizeof(PivRec), cudaMemcpyDeviceToHost);
        unsigned long long hsum = 0, psum = 0;  // bit-pattern checksums (compare builds)
        for (int t = 0; t < 64; ++t) for (int c = 0; c < m - 64; ++c) {
            unsigned long long b; memcpy(&b, &w1[(size_t)t * ld + c], 8); hsum = hsum * 1099511628211ull ^ b; }
        for (int t = 0; t < 64; ++t) {
            unsigned long long b; memcpy(&b, &rr[t].v, 8); psum = (psum * 1099511628211ull ^ b) * 31 + (unsigned)rr[t].l; }
        printf("W checksum %016llx pivots %016llx piv0 %.17g l0 %d\n", hsum, psum, rr[0].v, rr[0].l);
    }
#if KP_TRACE
    unsigned long long tr[64][16];
    cudaMemcpyFromSymbol(tr, g_kp_trace, sizeof(tr));
    double p8 = 0, p9 = 0, p1 = 0, p3 = 0, p5 = 0, p6 = 0, p2 = 0, p4 = 0, tot = 0;
    for (int s = 1; s < 62; ++s) {
        p8 += (double)(tr[s][8] - tr[s][0]); p9 += (double)(tr[s][9] - tr[s][8]); p1 += (double)(tr[s][1] - tr[s][9]);
        p3 += (double)(tr[s][3] - tr[s][1]); p5 += (double)(tr[s][5] - tr[s][3]); p6 += (double)(tr[s][6] - tr[s][5]);
        p2 += (double)(tr[s][2] - tr[s][6]); p4 += (double)(tr[s][4] - tr[s][2]); tot += (double)(tr[s + 1][0] - tr[s][0]);
    }
    printf("per step (cycles, CTA 0): poll %.0f reduce %.0f ->sync %.0f D1loop %.0f D1red %.0f combine+put %.0f ->sync %.0f D2/E %.0f | total %.0f\n",
           p8 / 61, p9 / 61, p1 / 61, p3 / 61, p5 / 61, p6 / 61, p2 / 61, p4 / 61, tot / 61);
    {
        double e2 = 0, e15 = 0, d2w1 = 0, w0bar = 0;
        for (int s = 1; s < 62; ++s) {
            e2 += (double)(tr[s][12] - tr[s][2]); e15 += (double)(tr[s][13] - tr[s][2]); d2w1 += (double)(tr[s][14] - tr[s][2]);
            w0bar += (double)(tr[s + 1][10] - tr[s][2]);
        }
        printf("  from E start (cycles): E done warp 2 %.0f, warp 15 %.0f, D2 done warp 1 %.0f, warp 0 at the barrier %.0f\n",
               e2 / 61, e15 / 61, d2w1 / 61, w0bar / 61);
    }
    printf("  prologue %llu cycles, loop %llu, W %llu\n", tr[0][9] - tr[0][8], tr[0][10] - tr[0][9], tr[0][11] - tr[0][10]);
    {   // cross-CTA view (globaltimer ns): per step, the last publish -> each CTA's poll completion
        static unsigned long long gt[64][kKPMaxG][4];
        cudaMemcpyFromSymbol(gt, g_kp_gt, sizeof(gt));
        double a_hop = 0, a_spread = 0, a_fetch = 0, a_chain = 0, a_pubspread = 0; int cnt = 0;
        int slow[kKPMaxG] = {0};
        for (int s = 2; s < 62; ++s) {
            unsigned long long lastpub = 0, firstpub = ~0ull, pmin = ~0ull, pmax = 0; int who = 0;
            for (int g = 0; g < G; ++g) {
                if (gt[s][g][2] > lastpub) { lastpub = gt[s][g][2]; who = g; }
                firstpub = std::min(firstpub, gt[s][g][2]);
                pmin = std::min(pmin, gt[s][g][0]); pmax = std::max(pmax, gt[s][g][0]);
            }
            slow[who]++;
            double fetch = 0, chain = 0;
            for (int g = 0; g < G; ++g) { fetch += (double)(gt[s][g][1] - gt[s][g][0]); chain += (double)(gt[s + 1][g][2] - gt[s][g][1]); }
            a_hop += (double)(pmin - lastpub); a_spread += (double)(pmax - pmin); a_fetch += fetch / G; a_chain += chain / G;
            a_pubspread += (double)(lastpub - firstpub); ++cnt;
        }
        printf("  cross-CTA (ns/step): publish spread %.0f, last publish -> first poll done %.0f, poll-done spread %.0f, fetch %.0f, fetch done -> next publish %.0f\n",
               a_pubspread / cnt, a_hop / cnt, a_spread / cnt, a_fetch / cnt, a_chain / cnt);
        printf("  slowest publisher histogram:");
        for (int g = 0; g < G; ++g) if (slow[g]) printf(" %d:%d", g, slow[g]);
        printf("\n");
    }
#endif
    return 0;
}

// Standalone run of the K2 panel kernel on a random 64 x m panel, with per-step phase trace.
#ifndef KP_TRACE
#define KP_TRACE 1
#endif
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <vector>
#include <random>
#include "../../paper_1811_08057_b200/csrc/k2_panel.cu"
using namespace mcnd;
int main(int argc, char** argv) {
    const int m = argc > 1 ? atoi(argv[1]) : 16384;
    const int G = argc > 2 ? atoi(argv[2]) : 128;
    const int cl = argc > 3 ? atoi(argv[3]) : 0;
    int cw = ((m + G - 1) / G + 1) / 2 * 2;
    const int64_t ld = (m + 15) / 16 * 16;
    std::vector<double> h((size_t)64 * ld);
    std::mt19937_64 rng(1);
    std::uniform_real_distribution<double> U(-1, 1);
    for (auto& x : h) x = U(rng);
    double *ws, *wit, *W; PivRec* rec; K2Gather* pan; unsigned* abort; double2 *cand, *wrec, *colb, *lastb; K1Err* err;
    cudaMalloc(&ws, h.size() * 8); cudaMemcpy(ws, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    cudaMalloc(&wit, 64 * 8); cudaMemset(wit, 0, 64 * 8);
    cudaMalloc(&W, (size_t)64 * ld * 8);
    cudaMalloc(&rec, 64 * sizeof(PivRec)); cudaMalloc(&pan, sizeof(K2Gather)); cudaMalloc(&abort, 4); cudaMemset(abort, 0, 4);
    cudaMalloc(&cand, 64 * kKPMaxG * 16); cudaMalloc(&wrec, 64 * kKPMaxG * 16); cudaMalloc(&colb, (size_t)64 * kKPMaxG * 64 * 16);
    cudaMalloc(&lastb, 64 * 64 * 16); cudaMalloc(&err, sizeof(K1Err)); cudaMemset(err, 0, sizeof(K1Err));
    cudaMemset(cand, 0, 64 * kKPMaxG * 16); cudaMemset(wrec, 0, 64 * kKPMaxG * 16);
    cudaMemset(colb, 0, (size_t)64 * kKPMaxG * 64 * 16); cudaMemset(lastb, 0, 64 * 64 * 16);
    KPParams p{};
    p.ws = ws; p.ld = ld; p.row0 = 0; p.m = m; p.G = G; p.cw = cw; p.wit = wit; p.rec = rec; p.epoch = 1;
    p.W = W; p.ldw = ld; p.pan = pan; p.abort = abort; p.cand = cand; p.wrec = wrec; p.colbuf = colb; p.lastbuf = lastb;
    p.err = err; p.timeout_ns = 5000000000ull; p.cluster = cl;
    if (cl) printf("cluster fits: %d\n", kp_cluster_fits(G, cw));
    if (argc > 4 && atoi(argv[4])) {  // second panel of a pair: the r1 prologue (rank-64 update of the rows)
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
    for (int it = 0; it < 3; ++it) {
        cudaMemcpy(ws, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
        p.tag0 = (unsigned)(1000 + it * 100);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        cudaError_t e = kp_launch(p, 0);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("m=%d G=%d cl=%d cw=%d: %.1f us (%.2f us/step) %s\n", m, G, cl, cw, ms * 1e3, ms * 1e3 / 64, cudaGetErrorString(e));
    }
    {   // cross-check against the other transport on the same input (same G, cw: bitwise)
        std::vector<double> w1((size_t)64 * ld), w2((size_t)64 * ld);
        std::vector<PivRec> r1(64), r2(64);
        cudaMemcpy(w1.data(), W, w1.size() * 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(r1.data(), rec, 64 * sizeof(PivRec), cudaMemcpyDeviceToHost);
        cudaMemcpy(ws, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
        cudaMemset(W, 0, (size_t)64 * ld * 8);
        KPParams q = p; q.cluster = !cl; q.tag0 = 77777;
        cudaError_t e = kp_launch(q, 0);
        cudaDeviceSynchronize();
        cudaMemcpy(w2.data(), W, w2.size() * 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(r2.data(), rec, 64 * sizeof(PivRec), cudaMemcpyDeviceToHost);
        long dw = 0, dr = 0;
        for (int t = 0; t < 64; ++t) for (int c = 0; c < m - 64; ++c) dw += w1[(size_t)t * ld + c] != w2[(size_t)t * ld + c];
        for (int t = 0; t < 64; ++t) dr += (r1[t].v != r2[t].v) || (r1[t].l != r2[t].l);
        unsigned long long hsum = 0;  // bit-pattern checksum of W (compare builds)
        for (int t = 0; t < 64; ++t) for (int c = 0; c < m - 64; ++c) {
            unsigned long long b; memcpy(&b, &w1[(size_t)t * ld + c], 8); hsum = hsum * 1099511628211ull ^ b; }
        printf("W checksum %016llx\n", hsum);
        printf("cross-check vs cluster=%d (%s): W mismatches %ld, pivot mismatches %ld, piv0 %.17g l0 %d\n", !cl,
               cudaGetErrorString(e), dw, dr, r1[0].v, r1[0].l);
    }
#if KP_TRACE
    unsigned long long tr[64][12];
    cudaMemcpyFromSymbol(tr, g_kp_trace, sizeof(tr));
    const int idx[7] = {0, 1, 3, 5, 6, 2, 4};
    const char* nm[7] = {"A", "D1loop", "D1red", "combine+put", "sync", "D2", "tail"};
    double acc[7] = {0};
    for (int s = 1; s < 62; ++s) {
        for (int k = 0; k < 6; ++k) acc[k] += (double)(tr[s][idx[k + 1]] - tr[s][idx[k]]);
        acc[6] += (double)(tr[s + 1][0] - tr[s][0]);
    }
    printf("per step (cycles):");
    for (int k = 0; k < 7; ++k) printf(" %s %.0f", k == 6 ? "total" : nm[k], acc[k] / 61);
    printf("\n");
    {
        double p8 = 0, p9 = 0, p10 = 0, p1 = 0;
        for (int s = 1; s < 62; ++s) { p8 += (double)(tr[s][8] - tr[s][0]); p9 += (double)(tr[s][9] - tr[s][8]);
            p10 += (double)(tr[s][10] - tr[s][9]); p1 += (double)(tr[s][1] - tr[s][10]); }
        printf("  A detail: poll %.0f  reduce %.0f  fetch %.0f  sync %.0f\n", p8 / 61, p9 / 61, p10 / 61, p1 / 61);
    }
    printf("  prologue %llu cycles, loop %llu, W %llu (product %llu, descriptor %llu)\n", tr[0][9] - tr[0][8], tr[0][10] - tr[0][9],
           tr[0][11] - tr[0][10], tr[1][11] - tr[0][10], tr[0][11] - tr[1][11]);
#endif
    return 0;
}

// Standalone run of the K2 panel kernel on a random 64 x m panel, with per-step phase trace.
#define KP_TRACE 1
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <random>
#include "../../paper_1811_08057_b200/csrc/k2_panel.cu"
using namespace mcnd;
int main(int argc, char** argv) {
    const int m = argc > 1 ? atoi(argv[1]) : 16384;
    const int G = argc > 2 ? atoi(argv[2]) : 128;
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
    p.err = err; p.timeout_ns = 5000000000ull;
    for (int it = 0; it < 3; ++it) {
        cudaMemcpy(ws, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
        p.tag0 = (unsigned)(1000 + it * 100);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        cudaError_t e = kp_launch(p, 0);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("m=%d G=%d cw=%d: %.1f us (%.2f us/step) %s\n", m, G, cw, ms * 1e3, ms * 1e3 / 64, cudaGetErrorString(e));
    }
    unsigned long long tr[64][6];
    cudaMemcpyFromSymbol(tr, g_kp_trace, sizeof(tr));
    double acc[5] = {0};
    for (int s = 1; s < 63; ++s) {
        acc[0] += (tr[s][1] - tr[s][0]) * 1e-3;  // publish + exchange
        acc[1] += (tr[s][2] - tr[s][1]) * 1e-3;  // winner column fetch
        acc[2] += (tr[s][3] - tr[s][2]) * 1e-3;  // row s scale
        acc[3] += (tr[s][4] - tr[s][3]) * 1e-3;  // update
        acc[4] += (tr[s + 1][0] - tr[s][4]) * 1e-3;
    }
    printf("per step (us): exchange %.2f  fetch %.2f  scale %.2f  update %.2f  loop %.2f\n", acc[0] / 62, acc[1] / 62,
           acc[2] / 62, acc[3] / 62, acc[4] / 62);
    return 0;
}

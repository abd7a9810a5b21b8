// Cluster panel kernel (k2_cpanel.cu) against the column-distributed one (k2_panel.cu) on the same
// random 64 x m panel (or a pair: 128 rows, both panels in one launch): pivots, descriptors, W
// compared; best-of-5 times of both.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I ../../paper_1811_08057_b200/csrc \
//        kc_bench.cu ../../paper_1811_08057_b200/csrc/k2_panel.cu ../../paper_1811_08057_b200/csrc/k2_cpanel.cu -o kc_bench
//   ./kc_bench m [pair=0|1] [C] [cw]
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <random>
#include <algorithm>
#include "mcnd_internal.h"
using namespace mcnd;
#if KC_TRACE
namespace mcnd { void kc_debug_trace(unsigned long long*, unsigned long long*); void kc_debug_trace_halves(unsigned long long*); }
#endif

struct Out {
    std::vector<double> W, Wp;
    std::vector<PivRec> rec;
    K2Gather pan[2], gpair;
    float best_ms;
    K1Err err;
};

int main(int argc, char** argv) {
    const int m = argc > 1 ? atoi(argv[1]) : 5000;
    const int pair = argc > 2 ? atoi(argv[2]) : 0;
    int C = argc > 3 ? atoi(argv[3]) : 0;
    int cwc = argc > 4 ? atoi(argv[4]) : 0;
    const int rows = pair ? 128 : 64;
    const int64_t ld = (m + 15) / 16 * 16;
    std::vector<double> h((size_t)rows * ld);
    std::mt19937_64 rng(1);
    std::uniform_real_distribution<double> U(-1, 1);
    for (auto& x : h) x = U(rng);
    double *ws, *wit, *W, *Wp;
    PivRec* rec;
    K2Gather *pan, *gpair;
    unsigned *abort, *bars;
    ulonglong2 *cand, *wrec, *colb, *lastb;
    K1Err* err;
    cudaMalloc(&ws, h.size() * 8);
    cudaMalloc(&wit, rows * 8); cudaMemset(wit, 0, rows * 8);
    cudaMalloc(&W, (size_t)128 * ld * 8);
    cudaMalloc(&Wp, 64 * 64 * 8);
    cudaMalloc(&rec, 128 * sizeof(PivRec));
    cudaMalloc(&pan, 2 * sizeof(K2Gather)); cudaMalloc(&gpair, sizeof(K2Gather));
    cudaMalloc(&abort, 4); cudaMemset(abort, 0, 4);
    cudaMalloc(&bars, 64);
    cudaMalloc(&cand, 64 * kKPMaxG * 32); cudaMalloc(&wrec, 64 * kKPMaxG * 32);
    cudaMalloc(&colb, (size_t)64 * kKPMaxG * 64 * 16); cudaMalloc(&lastb, 64 * 64 * 16);
    cudaMalloc(&err, sizeof(K1Err));
    auto run = [&](bool cluster) -> Out {
        Out o;
        cudaMemset(err, 0, sizeof(K1Err));
        cudaMemset(cand, 0, 64 * kKPMaxG * 32); cudaMemset(wrec, 0, 64 * kKPMaxG * 32);
        cudaMemset(colb, 0, (size_t)64 * kKPMaxG * 64 * 16); cudaMemset(lastb, 0, 64 * 64 * 16);
        KPParams p{};
        p.ws = ws; p.ld = ld; p.row0 = 0; p.m = m; p.wit = wit; p.rec = rec; p.epoch = 1;
        p.W = W; p.ldw = ld; p.pan = pan; p.abort = abort; p.cand = cand; p.wrec = wrec; p.colbuf = colb; p.lastbuf = lastb;
        p.err = err; p.timeout_ns = 3000000000ull;
        if (cluster) {
            int cw = 0;
            int c = kc_plan(m, &cw);
            if (C) { c = C; cw = cwc ? cwc : ((m + C - 1) / C + 31) / 32 * 32; }
            if (!c) { printf("kc_plan: m=%d outside the cluster kernel's range\n", m); exit(1); }
            p.G = c; p.cw = cw;
        } else {
            int G = std::max(1, m / 176);
            int cw = ((m + G - 1) / G + 1) / 2 * 2;
            while (G > 1 && m - (G - 1) * cw < 64) { --G; cw = ((m + G - 1) / G + 1) / 2 * 2; }
            p.G = G; p.cw = cw;
        }
        KPParams q = p;
        if (pair) {
            q.row0 = 64; q.m = m - 64; q.rec = rec + 64; q.W = W + 64 * ld; q.pan = pan + 1;
            q.r1_g0 = pan; q.r1_W = W; q.r1_ldw = ld;
            q.pp_g0 = pan; q.pp_W = W; q.pp_ldw = ld; q.pp_Wp = Wp; q.pp_gpair = gpair; q.pp_m = m;
            q.pp_bar = bars; q.half_bar = bars + 1;
        }
        o.best_ms = 1e30f;
        for (int it = 0; it < 5; ++it) {
            cudaMemcpy(ws, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
            cudaMemset(bars, 0, 64);
            p.tag0 = (unsigned)(1000 + it * 200); q.tag0 = p.tag0 + 64;
            cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaEventRecord(e0);
            cudaError_t e = cluster ? kc_launch(p, 0, pair ? &q : nullptr) : kp_launch(p, 0, pair ? &q : nullptr);
            cudaEventRecord(e1);
            cudaError_t e2 = cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            if (ms < o.best_ms) o.best_ms = ms;
            if (e != cudaSuccess || e2 != cudaSuccess) { printf("launch: %s / %s\n", cudaGetErrorString(e), cudaGetErrorString(e2)); exit(2); }
        }
        printf("%s m=%d G=%d cw=%d: best %.1f us (%.3f us/pivot)\n", cluster ? "cluster" : "column ", m, p.G, p.cw,
               o.best_ms * 1e3, o.best_ms * 1e3 / rows);
        o.W.resize((size_t)128 * ld); o.Wp.resize(64 * 64); o.rec.resize(128);
        cudaMemcpy(o.W.data(), W, o.W.size() * 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(o.Wp.data(), Wp, 64 * 64 * 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(o.rec.data(), rec, 128 * sizeof(PivRec), cudaMemcpyDeviceToHost);
        cudaMemcpy(o.pan, pan, 2 * sizeof(K2Gather), cudaMemcpyDeviceToHost);
        cudaMemcpy(&o.gpair, gpair, sizeof(K2Gather), cudaMemcpyDeviceToHost);
        cudaMemcpy(&o.err, err, sizeof(K1Err), cudaMemcpyDeviceToHost);
        if (o.err.error) printf("  device error %u at step %u\n", o.err.error, o.err.err_step);
        return o;
    };
    Out a = run(false);
    Out b = run(true);
    int bad = 0;
    for (int s = 0; s < rows; ++s)
        if (a.rec[s].l != b.rec[s].l || fabs(a.rec[s].v - b.rec[s].v) > 1e-9 * fabs(a.rec[s].v)) {
            if (bad < 8) printf("  pivot %d: column %d vs %d, value %.17g vs %.17g\n", s, a.rec[s].l, b.rec[s].l, a.rec[s].v, b.rec[s].v);
            ++bad;
        }
    printf("pivots differing: %d of %d\n", bad, rows);
    auto cmp_desc = [&](const K2Gather& x, const K2Gather& y, int nP, const char* name) {
        int d = 0;
        for (int k = 0; k < nP; ++k) d += x.P[k] != y.P[k];
        for (int k = 0; k < 64; ++k) d += x.l[k] != y.l[k];
        std::vector<std::pair<int, int>> mx, my;
        for (int k = 0; k < x.n_moved; ++k) mx.push_back({x.moved_c[k], x.moved_src[k]});
        for (int k = 0; k < y.n_moved; ++k) my.push_back({y.moved_c[k], y.moved_src[k]});
        std::sort(mx.begin(), mx.end()); std::sort(my.begin(), my.end());
        printf("  %s: P/l mismatches %d, moved %d vs %d %s\n", name, d, x.n_moved, y.n_moved, mx == my ? "(same)" : "(DIFFERENT)");
    };
    cmp_desc(a.pan[0], b.pan[0], 64, "panel 0 descriptor");
    if (pair) { cmp_desc(a.pan[1], b.pan[1], 64, "panel 1 descriptor"); cmp_desc(a.gpair, b.gpair, 128, "pair descriptor"); }
    double wmax = 0, dmax = 0;
    for (int t = 0; t < rows; ++t) {
        const int wf = m - 64 * (t / 64 + 1) - (pair && t < 64 ? 64 : 0);  // first panel's W is permuted into the pair layout
        for (int c = 0; c < wf; ++c) {
            const double x = a.W[(size_t)t * ld + c], y = b.W[(size_t)t * ld + c];
            wmax = std::max(wmax, fabs(x));
            if (!(fabs(x - y) <= dmax)) dmax = fabs(x - y);
        }
    }
    printf("W: max |W| %.3e, max |diff| %.3e\n", wmax, dmax);
    if (pair) {
        double d = 0;
        for (int e = 0; e < 64 * 64; ++e) d = std::max(d, fabs(a.Wp[e] - b.Wp[e]));
        printf("Wp: max |diff| %.3e\n", d);
    }
#if KC_TRACE
    {
        static unsigned long long tr[64][16], tb[8][8];
        kc_debug_trace(&tr[0][0], &tb[0][0]);
        double d[5] = {0, 0, 0, 0, 0}, tot = 0; int cnt = 0;
        for (int s = 0; s < 64; ++s) {
            if ((s & 7) == 7) continue;
            for (int k = 0; k < 5; ++k) d[k] += (double)(tr[s][k + 1] - tr[s][k]);
            tot += (double)(tr[s + 1][0] - tr[s][0]); ++cnt;
        }
        printf("per pivot (cycles, CTA 0 thread 0): warp argmax+bar %.0f, CTA argmax+send %.0f, wait %.0f, cluster argmax %.0f, roles+update %.0f | step %.0f\n",
               d[0] / cnt, d[1] / cnt, d[2] / cnt, d[3] / cnt, d[4] / cnt, tot / cnt);
        {
            const int seq[] = {0, 13, 14, 15, 1, 8, 9, 10, 2, 3, 11, 12, 4, 5};
            const char* nm[] = {"local argmax", "redux+ballot", "winner STS", "bar.sync", "CTA compare (4 LDS.128)", "LDS wx", "st.async x3", "arrive", "wait",
                                "LDS rcv", "rcp+redux+ballot", "shfl x5", "roles+update"};
            double dd[13] = {0}; int cn = 0;
            for (int s = 0; s < 64; ++s) { if ((s & 7) == 7) continue; for (int k = 0; k < 13; ++k) dd[k] += (double)(tr[s][seq[k + 1]] - tr[s][seq[k]]); ++cn; }
            for (int k = 0; k < 13; ++k) printf("    %-28s %.0f\n", nm[k], dd[k] / cn);
        }
        {
            static unsigned long long th[2][16];
            kc_debug_trace_halves(&th[0][0]);
            const char* hn[] = {"load rows", "half barrier", "r1 gather", "r1 DMMA", "row maxima + micro-panels", "W out", "descriptor", "pair prep Wp",
                                "pair desc (CTA 0)", "cluster barrier", "W_k moved columns"};
            for (int h = 0; h < (pair ? 2 : 1); ++h) {
                printf("  half %d (cycles):", h);
                for (int k = 0; k < 10; ++k) if (th[h][k + 1] >= th[h][k] && th[h][k]) printf(" %s %llu,", hn[k], th[h][k + 1] - th[h][k]);
                printf(" total %llu\n", th[h][10] - th[h][0]);
            }
        }
        for (int j = 0; j < 8; ++j)
            printf("  micro-panel %d: chain %llu, W8+lists %llu, publish+cluster barrier %llu, read+write-back %llu, update %llu\n", j,
                   tb[j][1] - tb[j][0], 0ull, tb[j][2] - tb[j][1], tb[j][3] - tb[j][2], tb[j][4] - tb[j][3]);
    }
#endif
    return 0;
}

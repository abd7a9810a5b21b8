// Internal interfaces shared by the kernels (.cu) and the host runtime.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace mcnd {

constexpr double kSingularRtol = 1e-12;  // condense.py:29
constexpr int kK1Threads = 1024;         // one CTA per SM, 32 warps
constexpr int kK1MaxRowsPerCta = 512;    // per-CTA row table lives in shared memory
constexpr int kK1MaxChunk = 16384;       // pivot-row chunk staged in smem (doubles)
constexpr int32_t kNever = 0x7fffffff;   // pivot step of a row that is never a pivot

// Control block written by the persistent kernel (zeroed before each launch).
struct K1Ctrl {
    unsigned published;   // number of pivots published so far (pivot t visible iff published > t)
    unsigned error;       // nonzero: device-side timeout / protocol error
    unsigned err_step;
    unsigned pad;
};

// Persistent, barrier-free condensation kernel parameters (k1_condense.cu).
struct K1Params {
    const double* src;       // caller's matrix (device), read once in the prologue
    int64_t lds;
    double* ws;              // workspace: n rows x ld, condensed in place
    int64_t ld;
    int32_t n;
    int32_t n_steps;         // S condensation steps
    const int32_t* seq;      // pivot row of pivot t (t < S, plus t == S when a final 1x1 is published)
    const int32_t* row_pstep;    // pivot index of each row (kNever if never a pivot)
    const int32_t* cta_row_ptr;  // [G+1]
    const int32_t* cta_rows;     // rows dealt to each CTA, ascending pivot index
    double* piv_val;         // [S+1]
    int32_t* piv_col;        // [S+1] (-1: singular at that pivot)
    double* piv_wit;         // [S+1]
    double* row_wit;         // [n]  witnesses at exit
    K1Ctrl* ctrl;
    int32_t chunk;           // staged pivot-row chunk (even, <= kK1MaxChunk)
    unsigned long long timeout_ns;
};

cudaError_t k1_launch(const K1Params& p, int grid, bool fast, cudaStream_t s);
int k1_max_grid(int device);
size_t k1_smem_bytes(int chunk);

cudaError_t k3_launch(const double* a, int64_t batch, int64_t n, int64_t stride, bool fast,
                      int32_t* sign, double* log_abs, double* pivots, cudaStream_t s);

}  // namespace mcnd

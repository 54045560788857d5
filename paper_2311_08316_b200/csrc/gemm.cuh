// Arguments of the FP64 DMMA GEMM engine (gemm.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace cqg {

struct GemmArgs {
    int64_t M, N, K;
    const double *A;  // op(A) = A (M x K) or A^T (A is K x M); column-major
    int64_t lda;
    const double *B;  // K x N, column-major
    int64_t ldb;
    const double *Cin;  // read when beta != 0; optional column gather
    int64_t ldcin;
    const int64_t *cin_cols;
    double *Cout;
    int64_t ldc;
    double alpha, beta;
    int64_t k_per_split;      // split-K slice length (0 = K / splits)
    double *part;             // split-K partial tiles (BM*BN each) instead of C
    int64_t ntiles_part;      // tiles per slice in `part` / length of `tiles`
    const int2 *tiles;        // optional explicit (tile_m, tile_n) list
    const int64_t *skip_flag; // device flag: nonzero -> the launch is a no-op
    int upper_only;           // only entries i <= j (and tiles touching them)
    int64_t batch;            // > 1: grid.z indexes independent problems (no split-K)
    int64_t bs_a, bs_b, bs_cin, bs_c;  // per-problem element strides of A, B, Cin, Cout
    int vec16;                // set by gemm_ex: A/B tiles staged with 16-byte copies
    int tile_n64;             // tiles[]: column tile index in units of 64 columns (not BN)
};

// C_out = alpha op(A) B + beta C_in, optionally split over K into `splits`
// partial tiles (P.part non-null).
int gemm_ex(bool trans_a, GemmArgs P, int64_t splits, cudaStream_t st);

}  // namespace cqg

// Host-side internals shared by the .cu translation units: error state,
// launch accounting and the device workspace cache.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <string>
#include <vector>

#include "../../include/cqrrpt_gpu.h"

namespace cqg {

// ---- errors ---------------------------------------------------------------
void set_error(const std::string &msg);
int fail_cuda(const char *what);      // records cudaGetLastError + what
int fail_nomem(const char *what);
int fail_internal(const char *what);
int check_launch(const char *kernel);  // cudaGetLastError after a launch

#define CQ_TRY(expr)              \
    do {                          \
        int _rc = (expr);         \
        if (_rc) return _rc;      \
    } while (0)
#define CQ_CUDA(expr, what)                              \
    do {                                                 \
        if ((expr) != cudaSuccess) return fail_cuda(what); \
    } while (0)

// ---- launch accounting ----------------------------------------------------
void note_launch();
int num_sms();

// ---- workspace ------------------------------------------------------------
// Named device buffers that persist across calls on the calling host thread
// and device (grow-only). One CQRRPT call touches each name at most once
// concurrently, so reuse is safe within stream order.
class Workspace {
public:
    void *raw(const char *name, size_t bytes);
    template <class T>
    T *get(const char *name, size_t count) {
        return static_cast<T *>(raw(name, count * sizeof(T) + 256));
    }
};
Workspace &workspace();
void release_workspace();
size_t ws_bytes(const char *name);  // bytes currently held under `name` (this thread, current device)

// Streams / events cached per (host thread, current device) under a name
// (prio: 0 default, 1 highest, 2 second highest); cached_events returns an
// array of >= count events (valid until the same name grows again).
int current_device();
int cached_stream(const char *name, int prio, cudaStream_t *out);
int cached_events(const char *name, size_t count, cudaEvent_t **out);
// true exactly once per (device, key): one-time per-device function attributes
bool first_on_device(const void *key);

// ---- kernels' host entry points (implemented in the .cu files) -------------
int saso_plan(int64_t d, int64_t c0, int64_t count, int64_t nnz, uint64_t seed, uint32_t *plan, cudaStream_t st);
// Rows of A still arriving when the sketch is launched: chunk c (rows up to
// row_end[c], multiples of 256 except the last) is on the device once ev[c]
// has completed. The exact SASO sketch follows the chunks (its chains run in
// row order and are carried across launches); other paths wait for all.
struct InputChunks {
    int count;
    const cudaEvent_t *ev;
    const int64_t *row_end;
};
int saso_sketch(int64_t m, int64_t n, const double *a, int64_t lda, int64_t d, int64_t nnz, uint64_t seed,
                int64_t c0, double *msk, int64_t ldm, Workspace &ws, cudaStream_t st, bool allow_split = false,
                const InputChunks *chunks = nullptr);

// QRCP: fills Rsk (n x n, ldr; rows >= k_sk zero), Jdev (int64 n), k_sk (host).
int qrcp(int64_t d, int64_t n, double *b, int64_t ldb, double rank_tol, double *rsk, int64_t ldr, int64_t *jdev,
         int64_t *k_sk, Workspace &ws, cudaStream_t st);
int rank_stage1(int64_t k, int64_t n, const double *r, int64_t ldr, int64_t *k0, Workspace &ws, cudaStream_t st);

// Optional per-block sink of a TRSM's output: after each 64-column block the
// block is copied (D2H) on `copy` into host[:, c0:c0+64] (ld ldh), so the
// download of X overlaps the remaining blocks.
struct BlockSink {
    cudaStream_t copy;
    double *host;
    int64_t ldh;
};
// check_diag = false: U is a Cholesky factor from potrf (diagonal sqrt(d),
// d > 0), so the zero-diagonal check (a host synchronisation) is skipped
int trsm_right(int64_t m, int64_t k, const double *b, int64_t ldb, const int64_t *cols, const double *u,
               int64_t ldu, double *x, int64_t ldx, cudaStream_t st, const BlockSink *sink = nullptr,
               bool check_diag = true, const cudaEvent_t *block_ev = nullptr);
// INT8 tensor-core engine of trsm_right (oztrsm.cu): right-looking 128-column
// blocks, DMMA diagonal solves, tcgen05 kind::i8 emulated trailing updates.
// dinv: the 64 x 64 diagonal-block inverses (trtri_diag_blocks).
bool trsm_use_ozaki(int64_t m, int64_t k);
int trsm_right_oz(int64_t m, int64_t k, const double *b, int64_t ldb, const int64_t *cols, const double *u,
                  int64_t ldu, double *x, int64_t ldx, cudaStream_t st, const BlockSink *sink, const double *dinv,
                  const cudaEvent_t *block_ev);
// one 64-column block c0 of trsm_right (dinv_blk: inverse of U's diagonal block)
int trsm_block(int64_t m, int64_t k, int64_t c0, const double *b, int64_t ldb, const int64_t *cols, const double *u,
               int64_t ldu, const double *dinv_blk, double *x, int64_t ldx, cudaStream_t st, bool pdl = false);
int gram(int64_t m, int64_t k, const double *x, int64_t ldx, double *g, int64_t ldg, Workspace &ws,
         cudaStream_t st);
// the Gram on the INT8 tensor cores (Ozaki scheme II, ozaki.cu) and the DMMA one
int gram_ozaki(int64_t m, int64_t k, const double *x, int64_t ldx, double *g, int64_t ldg, Workspace &ws,
               cudaStream_t st);
bool gram_ozaki_available();
int gram_dmma(int64_t m, int64_t k, const double *x, int64_t ldx, double *g, int64_t ldg, Workspace &ws,
              cudaStream_t st);
// Column block [c0, c1) (rows 0..c1-1) of a Gram split over num_sms() slices
// of m (min(.., m/512)): the same entries for any blocking. gram_col_tiles
// appends the block's tile list; part holds gram_col_part_size(m, k, ntiles).
void gram_col_tiles(int64_t c0, int64_t c1, std::vector<int2> &tiles);
size_t gram_col_part_size(int64_t m, int64_t k, int64_t ntiles);
int gram_cols(int64_t m, int64_t k, int64_t c1, const int2 *tiles, int64_t ntiles, const double *x, int64_t ldx,
              double *g, int64_t ldg, double *part, cudaStream_t st);
// C (M x N, ldc) = alpha * op(A) * B + beta * C; op(A) = A (M x K) or A^T (A is K x M).
int gemm(bool trans_a, int64_t M, int64_t N, int64_t K, double alpha, const double *a, int64_t lda,
         const double *b, int64_t ldb, double beta, double *c, int64_t ldc, cudaStream_t st);
int potrf(int64_t n, double *g, int64_t ldg, int64_t *failure_index, Workspace &ws, cudaStream_t st);
// Column block [c0, c1) of potrf's right-looking factor (64-aligned c0): every
// update and panel solve of steps j < c0 that reaches these columns, in block
// order, then the diagonal block -- bitwise potrf's entries once all blocks
// left of c0 are done. fail: device flag (1-based index, 0 = none).
int potrf_cols(int64_t n, double *g, int64_t ldg, int64_t c0, int64_t c1, int64_t *fail, cudaStream_t st);
// C = alpha op(A) B + beta C with K split into `splits` slices summed in order
int gemm_fill(bool trans_a, int64_t M, int64_t N, int64_t K, double alpha, const double *a, int64_t lda,
              const double *b, int64_t ldb, double beta, double *c, int64_t ldc, Workspace &ws, cudaStream_t st);
int gemm_splitk(bool trans_a, int64_t M, int64_t N, int64_t K, double alpha, const double *a, int64_t lda,
                const double *b, int64_t ldb, double beta, double *c, int64_t ldc, int64_t splits, Workspace &ws,
                cudaStream_t st);
// SRFT sketch (sketch.cc:100-119, 147-166), bit-identical, single rank
int srft_sketch(int64_t m, int64_t n, const double *a, int64_t lda, int64_t d, uint64_t seed, double *msk,
                int64_t ldm, Workspace &ws, cudaStream_t st);
// Gaussian sketch (sketch.cc:62-72, apply = matmul): msk = S A, S generated on device
int gaussian_sketch(int64_t m, int64_t n, const double *a, int64_t lda, int64_t d, uint64_t seed, int64_t c0,
                    double *msk, int64_t ldm, Workspace &ws, cudaStream_t st);
int trmm_upper(int64_t k, int64_t n, const double *a, int64_t lda, const double *b, int64_t ldb, double *c,
               int64_t ldc, Workspace &ws, cudaStream_t st);

// small utilities (util.cu)
int fill_identity(int64_t n, double *a, int64_t lda, cudaStream_t st);
int trtri_upper(int64_t k, const double *r, int64_t ldr, double *x, int64_t ldx, Workspace &ws, cudaStream_t st);
// inverses of the 64 x 64 diagonal blocks of triu(r), block b at dinv + b*4096
// (column-major, ld 64; a ragged last block is padded with the identity)
int trtri_diag_blocks(int64_t k, const double *r, int64_t ldr, double *dinv, cudaStream_t st);
int zero_strict_lower(int64_t n, double *a, int64_t lda, cudaStream_t st);
int frob_norm_upper(int64_t n, const double *a, int64_t lda, double *out_host, Workspace &ws, cudaStream_t st);
int copy_matrix(int64_t m, int64_t n, const double *src, int64_t lds, double *dst, int64_t ldd, cudaStream_t st);

// stage-2 estimators (cond.cu)
// first power iterate of ||(R_ell - I) v0|| for each ell in ells (host list) -> host values
int identity_deviation_first(const double *r, int64_t ldr, const int64_t *ells, int nells, double *out_host,
                             Workspace &ws, cudaStream_t st);
// full reference cond_estimate on the leading ell block; rinv = explicit inverse (ld ldr) for krylov
int cond_estimate(int64_t ell, const double *r, int64_t ldr, const double *rinv, int64_t ldi, int method,
                  double *value_host, Workspace &ws, cudaStream_t st);
// several leading blocks at once (one CTA group per probe; same values as cond_estimate)
int cond_estimate_batch(int nells, const int64_t *ells_host, const double *r, int64_t ldr, const double *rinv,
                        int64_t ldi, int method, double *values_host, Workspace &ws, cudaStream_t st);
int spectral_norm_estimate(int64_t m, int64_t n, const double *a, int64_t lda, double *value_host, Workspace &ws,
                           cudaStream_t st);

}  // namespace cqg

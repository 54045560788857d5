/* cqrrpt_gpu.h — C ABI of the B200-native CQRRPT (sm_100a).
 *
 * This is the drop-in boundary for the reference's hot path
 *
 *   CqrrptOutput cqrrpt(const DenseMatrix &m, const CqrrptConfig &cfg = {});
 *       /root/reference/proj/include/cqrrpt/cqrrpt.hh:140, body cqrrpt.cc:317-328
 *   CqrrptOutput cqrrpt_core(const DenseMatrix &m, const SketchOperator &s,
 *                            const CqrrptConfig &cfg);
 *       cqrrpt.hh:136, body cqrrpt.cc:233-315
 *
 * re-expressed in the (m, n, A, lda, d_factor) -> (R, J, k, Q in place)
 * convention of BASELINE.json:north_star, with plain pointers and sizes, no
 * C++ types and no exceptions. A C++ adapter with the reference's own
 * signature lives in include/cqrrpt_b200.hh.
 *
 * Conventions
 *   - Matrices are column-major FP64 with an explicit leading dimension
 *     (DenseMatrix is column-major, dense_matrix.hh:36-41).
 *   - Pivots J are 0-based int64 (qrcp.hh:21-23).
 *   - Return 0 on success; -i when argument i is invalid (LAPACK style; these
 *     are exactly the reference's std::invalid_argument conditions,
 *     cqrrpt.cc:38-42, sketch.cc:54,74-75); a positive value for a CUDA/NCCL
 *     failure (CQRRPT_GPU_ERR_*). A zero diagonal in a triangular solve (the
 *     reference's std::domain_error, linalg.cc:250-252) is
 *     CQRRPT_GPU_ERR_SINGULAR.
 *   - All device work is ordered on ctx->stream; the call returns after the
 *     outputs are complete (k is needed on the host to size later phases).
 *   - Multi-GPU: one process (or host thread) per GPU. Each rank passes its
 *     local rows (m_local, A_local, lda) and ctx->global_row_offset, because
 *     SASO column c of S is a function of the GLOBAL row index (sketch.cc:81).
 *     The d x n sketch and the k0 x k0 Gram are sum-allreduced (NCCL or a
 *     caller-supplied callback); R, J, k, k0 come out identical on all ranks.
 */
#ifndef CQRRPT_GPU_H
#define CQRRPT_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CQRRPT_GPU_ABI_VERSION 1

/* error codes (positive) */
#define CQRRPT_GPU_ERR_CUDA 1
#define CQRRPT_GPU_ERR_NCCL 2
#define CQRRPT_GPU_ERR_SINGULAR 3 /* trsm_right zero diagonal: linalg.cc:250-252 */
#define CQRRPT_GPU_ERR_NOMEM 4
#define CQRRPT_GPU_ERR_INTERNAL 5

/* cond estimators (cqrrpt.hh:61) */
#define CQRRPT_COND_DIAG_RATIO 0
#define CQRRPT_COND_KRYLOV_BOUNDS 1
#define CQRRPT_COND_IDENTITY_DEVIATION 2
/* identity_deviation with NestedCondEstimator's krylov_bounds fallback when it
 * returns +inf (cqrrpt.cc:57-58): what rank_stage2 evaluates per probe */
#define CQRRPT_COND_NESTED_IDENTITY_DEVIATION 3

/* ctx->flags */
#define CQRRPT_GPU_OUTPUTS_ON_HOST 0x1 /* R and J are host pointers (default: device) */
#define CQRRPT_GPU_EXACT_STAGE2 0x2    /* always run the reference's binary search with
                                          power-iteration estimates (also fills cond_m_pre) */
#define CQRRPT_GPU_NO_STAGE1 0x4       /* CqrrptConfig::stage1_enabled = false */
#define CQRRPT_GPU_DIAGNOSTICS 0x8     /* truncation_ratio (spectral norm of R_sk) */
#define CQRRPT_GPU_TIMINGS 0x10        /* per-phase CUDA-event timings into ctx->timings_ms */
/* sketch families (SketchFamily, sketch.hh) */
#define CQRRPT_SKETCH_SASO 0
#define CQRRPT_SKETCH_GAUSSIAN 1
#define CQRRPT_SKETCH_SRFT 2     /* single rank: the transform mixes every row */

#define CQRRPT_GPU_FAST_SKETCH 0x20    /* allow a c-split sketch (partials summed in a fixed order):
                                          deterministic, not bit-identical to the reference's
                                          single FMA chain; fills the GPU when n is small */
#define CQRRPT_GPU_NO_WAVEFRONT 0x40   /* cqrrpt_gpu_dgeqpt_host (one rank): run precondition,
                                          Gram, Cholesky and Q as whole passes instead of the
                                          128-column wavefront that streams Q out during them;
                                          the wavefront's Gram sums m in different fixed slices,
                                          so Q and R differ in the last bits */
#define CQRRPT_GPU_WAVEFRONT 0x80      /* cqrrpt_gpu_dgeqpt (one rank): use the wavefront too
                                          (same bits as dgeqpt_host's default; slower on the
                                          device alone) */

/* Sum-allreduce of `count` doubles in place on device memory, ordered on
 * `stream`. Return 0 on success. */
typedef int (*cqrrpt_gpu_allreduce_fn)(double *buf, size_t count, void *stream, void *user);

typedef struct cqrrpt_gpu_comm cqrrpt_gpu_comm; /* opaque NCCL communicator wrapper */

typedef struct cqrrpt_gpu_ctx {
    /* in */
    void *stream;                /* cudaStream_t; NULL = legacy default stream */
    int32_t rank, nranks;        /* row-shard identity; nranks <= 1 means single GPU */
    int64_t global_row_offset;   /* global index of local row 0 */
    cqrrpt_gpu_comm *comm;       /* NCCL communicator (cqrrpt_gpu_comm_init), or NULL */
    cqrrpt_gpu_allreduce_fn allreduce; /* used when comm == NULL and nranks > 1 */
    void *allreduce_user;
    int32_t cond_method;         /* CQRRPT_COND_* (default identity_deviation = 2) */
    int32_t flags;               /* CQRRPT_GPU_* */
    int32_t sketch_family;       /* CQRRPT_SKETCH_SASO (default), _GAUSSIAN or _SRFT */
    int32_t reserved0;
    /* out: diagnostics (cqrrpt.hh:104-122) */
    int64_t d;                   /* sketch rows ceil(d_factor * n) */
    int64_t k_sk;                /* QRCP steps on the sketch */
    int64_t k0_final;            /* k0 after Cholesky-failure shrink */
    int32_t retries;             /* Cholesky-failure retries (rank_stage2) */
    int32_t stage2_exact;        /* 1 if the binary search ran, 0 if fast-accepted */
    double cond_m_pre;           /* est.at(k) (cqrrpt.cc:205): filled when the stage-2 search
                                    ran, or with CQRRPT_GPU_DIAGNOSTICS (evaluated after the
                                    timed phases on the fast-accept path); NaN otherwise */
    double cond_upper_bound;     /* ||R_pre||_F ||R_pre^-1||_F (fast path) */
    double truncation_ratio;     /* ||C_k||_F / ||R_sk||_2 (CQRRPT_GPU_DIAGNOSTICS) */
    double flop_estimate;        /* flop_model (cqrrpt.cc:330-338) */
    /* phase timings (CQRRPT_GPU_TIMINGS), milliseconds, PhaseTimings order:
     * sketch, qrcp, rank_select, precondition, cholesky_qr, undo, total,
     * + [7] communication (allreduce) */
    double timings_ms[8];
    /* in (appended in ABI 1.1): > 0 sets the sketch row count d directly
     * instead of ceil(d_factor * n) -- cqrrpt_core with an explicit operator
     * of d rows (cqrrpt.hh:136); d_factor is then only validated (>= 1), as
     * the reference's check_config does */
    int64_t sketch_rows;
} cqrrpt_gpu_ctx;

/* Fill a context with defaults (single GPU, default stream). */
void cqrrpt_gpu_ctx_init(cqrrpt_gpu_ctx *ctx);

/* CQRRPT of a tall FP64 matrix (north_star entry point).
 *   m, n      local rows, columns (m_local on a shard; n identical on all ranks)
 *   A, lda    device, column-major. On return A[:, :k] holds Q (in place);
 *             with CQRRPT_GPU_WAVEFRONT and k < k0, A[:, k:k0] holds
 *             speculative columns.
 *             Columns k..n-1 of A are left unspecified.
 *   d_factor  sketch oversampling gamma >= 1 (CqrrptConfig::gamma, cqrrpt.hh:93)
 *   nnz       SASO nonzeros per column of S, 1 <= nnz <= d (cqrrpt.hh:95)
 *   seed      sketch seed (CqrrptConfig::seed)
 *   eps_tol   stage-2 tolerance > u (CqrrptConfig::eps_tol, default 1e-4)
 *   R, ldr    out: k x n upper-trapezoidal (ldr >= n), device unless
 *             CQRRPT_GPU_OUTPUTS_ON_HOST. Rows >= k untouched.
 *   J         out: n pivots, 0-based (device unless OUTPUTS_ON_HOST)
 *   k, k0     out (host): final rank and stage-1 rank
 */
int cqrrpt_gpu_dgeqpt(int64_t m, int64_t n, double *A, int64_t lda, double d_factor, int64_t nnz,
                      uint64_t seed, double eps_tol, double *R, int64_t ldr, int64_t *J, int64_t *k,
                      int64_t *k0, cqrrpt_gpu_ctx *ctx);

/* Host-buffer variant (the reference's data in/out convention, cqrrpt.hh:140):
 * A_host (m x n, lda) is uploaded, Q (m x k) is downloaded into Q_host
 * (ldq >= m, room for k0 columns) block by block while the device is still
 * computing, R (k x n, ldr) and J (0-based) land on the host. One rank: Q's
 * blocks are formed and sent as soon as their Gram/Cholesky columns exist
 * (speculating k = k0); if stage 2 truncates to k < k0, columns k..k0-1 of
 * Q_host hold the speculative blocks (unspecified). Pinned host memory gives
 * full PCIe bandwidth and real overlap. */
int cqrrpt_gpu_dgeqpt_host(int64_t m, int64_t n, const double *A_host, int64_t lda, double d_factor, int64_t nnz,
                           uint64_t seed, double eps_tol, double *Q_host, int64_t ldq, double *R_host, int64_t ldr,
                           int64_t *J_host, int64_t *k, int64_t *k0, cqrrpt_gpu_ctx *ctx);

/* ---------------------------------------------------------------------------
 * Phase-level entry points (the same kernels the driver composes; exposed for
 * parity tests and for callers that run their own collectives).
 * All pointers are device pointers unless stated; `stream` is a cudaStream_t.
 * ------------------------------------------------------------------------- */

/* sketch_rows_for (cqrrpt.cc:211-213) */
int64_t cqrrpt_gpu_sketch_rows(double d_factor, int64_t n);

/* SASO plan for global S columns [c0, c0+count): plan[c*nnz+t] =
 * row | (sign << 31), sign 1 = +1/sqrt(d). sample_sketch (sketch.cc:73-99). */
int cqrrpt_gpu_saso_plan(int64_t d, int64_t c0, int64_t count, int64_t nnz, uint64_t seed,
                         uint32_t *plan, void *stream);

/* M_sk (d x n, ldm) = S[:, c0:c0+m] * A (m x n, lda); apply (sketch.cc:131-146).
 * Deterministic (fixed-order partial sums). */
int cqrrpt_gpu_saso_sketch(int64_t m, int64_t n, const double *A, int64_t lda, int64_t d,
                           int64_t nnz, uint64_t seed, int64_t c0, double *Msk, int64_t ldm,
                           void *stream);
/* Gaussian family (sketch.cc:62-72, apply = matmul): Msk (d x n, ldm) =
 * S[:, c0:c0+m] A with S(i, c) = normal(c*d + i)/sqrt(d) from the reference's
 * counter stream (c = global row), generated on device chunk by chunk and
 * multiplied by a split-K DMMA GEMM (fixed-order slice sum). */
int cqrrpt_gpu_gaussian_sketch(int64_t m, int64_t n, const double *A, int64_t lda, int64_t d, uint64_t seed,
                               int64_t c0, double *Msk, int64_t ldm, void *stream);

/* SRFT family (sketch.cc:100-119 sample, 147-166 apply): Msk (d x n, ldm) =
 * sqrt(P/d)/sqrt(P) * (FWHT(signs .* A zero-padded to P = next_pow2(m)))[rows],
 * bit-identical to the reference (the butterflies run stage by stage in its
 * order). Needs 1 <= d <= m and the whole matrix on one device. */
int cqrrpt_gpu_srft_sketch(int64_t m, int64_t n, const double *A, int64_t lda, int64_t d, uint64_t seed,
                           double *Msk, int64_t ldm, void *stream);

/* As cqrrpt_gpu_saso_sketch; flags & CQRRPT_GPU_FAST_SKETCH allows the
 * c-split decomposition (deterministic, not bit-identical). */
int cqrrpt_gpu_saso_sketch_ex(int64_t m, int64_t n, const double *A, int64_t lda, int64_t d, int64_t nnz,
                              uint64_t seed, int64_t c0, double *Msk, int64_t ldm, uint32_t flags, void *stream);

/* Max-norm Householder QRCP of the d x n sketch (qrcp.cc:35-97, want_q=false).
 * Msk is overwritten. R_sk (n x n buffer, ldr >= n; first k_sk rows valid,
 * exactly upper-trapezoidal), J (n, 0-based), k_sk (host). rank_tol < 0
 * selects the default n*u. */
int cqrrpt_gpu_qrcp(int64_t d, int64_t n, double *Msk, int64_t ldm, double rank_tol, double *Rsk,
                    int64_t ldr, int64_t *J, int64_t *k_sk, void *stream);

/* rank_stage1 (cqrrpt.cc:92-112) on a k x n upper-trapezoidal R (device). */
int cqrrpt_gpu_rank_stage1(int64_t k, int64_t n, const double *R, int64_t ldr, int64_t *k0,
                           void *stream);

/* rank_stage2 (cqrrpt.cc:149-209), the routine cqrrpt_gpu_dgeqpt runs after
 * stage 1 (one rank): M_pre = M_k0 A_sk^{-1} (m x k0, A_sk upper k0 x k0),
 * upper Cholesky of M_pre^T M_pre into R_pre (k0 x k0 buffer, ldr >= k0, on
 * device) with the failure-shrink retry, then the NestedCondEstimator binary
 * search for the largest leading block with cond <= sqrt(eps_tol/u).
 * Outputs: M_pre columns [0, k0_final) and R_pre's leading rank x rank block
 * (device), rank, k0_final, retries and cond_at_rank (= est.at(rank), 1.0 for
 * rank 0) on the host. flags: CQRRPT_GPU_EXACT_STAGE2 forces the search (the
 * result is the same; the fast accept is exact). A zero diagonal in A_sk
 * returns CQRRPT_GPU_ERR_SINGULAR (the reference's std::domain_error). */
int cqrrpt_gpu_rank_stage2(int64_t m, int64_t k0, const double *M_k0, int64_t ldm, const double *A_sk, int64_t ldas,
                           double eps_tol, int32_t cond_method, int32_t flags, double *M_pre, int64_t ldp, double *R_pre,
                           int64_t ldr, int64_t *rank, int64_t *k0_final, int32_t *retries, double *cond_at_rank,
                           void *stream);

/* X (m x k, ldx) = B[:, cols] * U^{-1}, U upper-triangular k x k (ldu);
 * cols = NULL means identity. trsm_right (linalg.cc:244-277) fused with the
 * pivoted column gather (dense_matrix.hh:70-80). X must not alias B. */
int cqrrpt_gpu_trsm_right(int64_t m, int64_t k, const double *B, int64_t ldb, const int64_t *cols,
                          const double *U, int64_t ldu, double *X, int64_t ldx, void *stream);

/* Which engine cqrrpt_gpu_trsm_right (and the driver's two solves) uses for an
 * m x k solve with even m, 16-byte aligned operands and even leading
 * dimensions (else always DMMA): 0 =
 * DMMA (FP64 tensor cores), 1 = the exact INT8 tensor-core emulation
 * (tcgen05 kind::i8; from m >= 131072 and k >= 768, or CQRRPT_GPU_TRSM=oz |
 * dmma). Diagnostic; no device work. */
int cqrrpt_gpu_trsm_engine(int64_t m, int64_t k);

/* G (k x k, ldg) = X^T X, bitwise symmetric; gram (linalg.cc:298-307). */
int cqrrpt_gpu_gram(int64_t m, int64_t k, const double *X, int64_t ldx, double *G, int64_t ldg,
                    void *stream);

/* Upper Cholesky G = R^T R in place on the upper triangle of G (ldg);
 * strict lower triangle is zeroed. failure_index (host): 0 on success, else
 * the 1-based first non-positive pivot and the leading (j-1) block is valid
 * (cholesky, linalg.cc:223-242). */
int cqrrpt_gpu_potrf(int64_t n, double *G, int64_t ldg, int64_t *failure_index, void *stream);

/* cond_estimate (cqrrpt.cc:114-147) of the leading ell x ell block of an
 * upper-triangular R (ldr), reference semantics (power iterations capped at
 * 200, 1e-6 inflation). value on host. */
int cqrrpt_gpu_cond_estimate(int64_t ell, const double *R, int64_t ldr, int32_t method, double *value,
                             void *stream);

/* CholeskyQR (twice = 0) / CholeskyQR2 (twice = 1) of the m x n (m >= n)
 * device matrix A: Q overwrites A, R (n x n, ldr) is upper triangular.
 * cholesky_qr / cholesky_qr2 (cqrrpt.cc:75-90). A non-positive-definite Gram
 * returns 0 with *failure_index = the 1-based first failing minor (A and R
 * then hold partial results); m < n returns -2 (the reference throws
 * std::invalid_argument). The comparator of the reference's stability check. */
int cqrrpt_gpu_cholesky_qr(int64_t m, int64_t n, double *A, int64_t lda, double *R, int64_t ldr, int32_t twice,
                           int64_t *failure_index, void *stream);

/* X (k x k, ldx) = triu(R)^{-1}: recursive blocked inverse (64 x 64 diagonal
 * blocks, then log2(k/64) levels of batched DMMA GEMMs). Stage 2 uses it in
 * place of the reference's per-iteration triangular solves
 * (inverse_norm_estimate, linalg.cc:486-500). R must have a nonzero diagonal. */
int cqrrpt_gpu_trtri_upper(int64_t k, const double *R, int64_t ldr, double *X, int64_t ldx, void *stream);

/* C (k x n, ldc) = triu(A) (k x k, lda) * triu(B) (k x n, ldb): exactly
 * upper-trapezoidal; multiply_upper_triangular (cqrrpt.cc:23-36). */
int cqrrpt_gpu_trmm_upper(int64_t k, int64_t n, const double *A, int64_t lda, const double *B,
                          int64_t ldb, double *C, int64_t ldc, void *stream);

/* Device evaluator of validate() (qrcp.cc:150-196) plus the BASELINE
 * Frobenius metric. A is the ORIGINAL matrix (m x n), Q (m x k), R (k x n),
 * J (device). Outputs on host: orth_fro = ||Q^T Q - I||_F,
 * orth_2 = ||Q^T Q - I||_2 (power iteration), recon = ||A[:,J] - QR||_F/||A||_F. */
int cqrrpt_gpu_validate(int64_t m, int64_t n, int64_t k, const double *A, int64_t lda, const double *Q,
                        int64_t ldq, const double *R, int64_t ldr, const int64_t *J, double *orth_fro,
                        double *orth_2, double *recon, void *stream);

/* flop_model (cqrrpt.cc:330-338) with C_sk = 2 nnz m n (sketch.cc:216-217). */
double cqrrpt_gpu_flop_model(int64_t m, int64_t n, int64_t k, int64_t d, double c_sk);

/* ---------------------------------------------------------------------------
 * NCCL (dlopen'ed libnccl.so.2; no link-time dependency)
 * ------------------------------------------------------------------------- */
/* 128-byte ncclUniqueId, created on rank 0 and broadcast by the caller. */
int cqrrpt_gpu_comm_unique_id(unsigned char id[128]);
int cqrrpt_gpu_comm_init(int32_t nranks, int32_t rank, const unsigned char id[128],
                         cqrrpt_gpu_comm **comm);
int cqrrpt_gpu_comm_allreduce(cqrrpt_gpu_comm *comm, double *buf, size_t count, void *stream);
void cqrrpt_gpu_comm_destroy(cqrrpt_gpu_comm *comm);

/* Helpers for caller-supplied collectives (cqrrpt_gpu_allreduce_fn):
 * y += x on device (ordered on stream); synchronous copy of any direction;
 * stream synchronisation. */
int cqrrpt_gpu_add(double *y, const double *x, size_t n, void *stream);
int cqrrpt_gpu_copy(void *dst, const void *src, size_t bytes, void *stream);
int cqrrpt_gpu_stream_sync(void *stream);

/* Free the library's cached device workspaces (calling thread). */
void cqrrpt_gpu_release_workspace(void);

/* Last error message of this thread (never NULL). */
const char *cqrrpt_gpu_last_error(void);

/* Number of kernel launches issued by this library on the calling thread
 * since the last reset (evidence for bench.py's gpu_launches). */
int64_t cqrrpt_gpu_launch_count(int32_t reset);

#ifdef __cplusplus
}
#endif
#endif

/* TEST INFRASTRUCTURE ONLY — the CPU oracle for the CQRRPT hot path.
 *
 * A plain-C restatement of the reference algorithm (/root/reference/proj,
 * arXiv 2311.08316's artifact). Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load it, and only as the checker. The
 * product (paper_2311_08316_b200/) never links or calls it.
 *
 * Pinned against the compiled reference (oracle/_ref) bit-for-bit by
 * tests/test_oracle_pin.py and against the reference's own known answers by
 * tests/test_oracle_known_answers.py.
 *
 * Matrices are column-major FP64 with an explicit leading dimension unless a
 * function says "packed" (ld = rows). Error returns mirror the reference's
 * exceptions: -1 invalid_argument, -2 domain_error.
 */
#ifndef CQRRPT_ORACLE_H
#define CQRRPT_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_UNIT_ROUNDOFF 1.1102230246251565e-16 /* 2^-53, cqrrpt.hh:14 */

/* rng.hh:18-53 */
uint64_t orc_rng_bits(uint64_t seed, uint64_t counter);
double orc_rng_normal(uint64_t seed, uint64_t counter);
uint64_t orc_rng_below(uint64_t seed, uint64_t counter, uint64_t bound);
uint64_t orc_mix_seed(uint64_t seed, uint64_t salt);

/* testmat.cc generators (harness inputs, not hot path) */
int orc_gen_gaussian(int64_t m, int64_t n, uint64_t seed, double *out);
/* gaussian_block (testmat.cc:17-25) on an already mixed stream seed */
int orc_gaussian_block(int64_t m, int64_t n, uint64_t stream_seed, double *out);
int orc_gen_exact_rank(int64_t m, int64_t n, int64_t r, uint64_t seed, double *out);
int orc_gen_spectral_list(int64_t m, int64_t n, const double *sigma, uint64_t seed, double *out);
int orc_gen_kahan(int64_t n, double theta, double *out);
/* SURVEY 8(d) C5 generator: seeded Fisher-Yates permutation (verify.cc:45-55
 * with seed mix_seed(0, 0x7065726d)), column j scaled by 10^(-span*pi[j]/(n-1)). */
int orc_c5_scale_columns(int64_t m, int64_t n, int64_t ld, double span_decades, uint64_t seed,
                         double *a, int64_t *perm_out);
/* Memory-lean (streaming) forms of the same generators for the full-size
 * parity tests: rows [r0, r1) of gen_gaussian(m, n, seed) into out (ld), and
 * the C5 column factors f[j] = 10^(-span*pi[j]/(n-1)) (a row block scaled by
 * a[j*ld+i] *= f[j] is bitwise the same block of orc_c5_scale_columns). */
int orc_gen_gaussian_rows(int64_t m, int64_t n, uint64_t seed, int64_t r0, int64_t r1, double *out, int64_t ld);
int orc_c5_column_factors(int64_t n, double span_decades, uint64_t seed, double *f);

/* sketch.cc:52-99 SASO sampling for global columns [c0, c0+count) of S.
 * rows/vals: count*nnz entries, column-major per S column. */
int orc_saso_sample(int64_t d, int64_t c0, int64_t count, int64_t nnz, uint64_t seed,
                    int64_t *rows, double *vals);
/* sketch.cc:100-119 / 147-166: SRFT sample and apply (out d x n, ld_out). */
int orc_srft_sample(int64_t d, int64_t m, uint64_t seed, double *signs, int64_t *rows);
int orc_srft_apply(int64_t d, int64_t m, int64_t n, uint64_t seed, const double *a, int64_t lda, double *out,
                   int64_t ld_out);
/* sketch.cc:62-72: Gaussian operator columns c0..c0+m-1 -> s (d x m, ld d). */
int orc_gaussian_sample(int64_t d, int64_t m, uint64_t seed, int64_t c0, double *s);
/* sketch.cc:131-146: out (d x n, ld_out) += S[:, c0:c0+m] * A (m x n, lda). */
int orc_saso_apply(int64_t d, int64_t m, int64_t n, int64_t nnz, uint64_t seed, int64_t c0,
                   const double *a, int64_t lda, double *out, int64_t ld_out);
double orc_sketch_flops_saso(int64_t nnz, int64_t m, int64_t n_cols);

/* linalg.cc:36-50 */
double orc_dot(const double *a, const double *b, int64_t n);

/* qrcp.cc:35-97. r_out: k x n packed (caller sizes min(rows,n)*n);
 * pivots: n. gaps (optional, length min(rows,n)): relative gap between the
 * best and second-best squared trailing norm at each step (tie margin). */
int orc_qrcp_maxnorm(int64_t rows, int64_t n, const double *a, int64_t lda, double rank_tol,
                     double *r_out, int64_t *pivots, int64_t *rank, double *gaps);

/* cqrrpt.cc:92-112 */
int64_t orc_rank_stage1(int64_t k, int64_t n, const double *r, int64_t ldr, double u);

/* linalg.cc:223-242: r_out packed n x n (leading j x j valid on failure). */
int orc_cholesky(int64_t n, const double *g, int64_t ldg, double *r_out, int64_t *failure_index);
/* linalg.cc:244-277: x (m x k, ldx) = b * r^{-1}; b may alias x. */
int orc_trsm_right(int64_t m, int64_t k, const double *b, int64_t ldb, const double *r,
                   int64_t ldr, double *x, int64_t ldx);
/* linalg.cc:298-307: g (k x k packed) = a^T a, bitwise symmetric. */
int orc_gram(int64_t m, int64_t k, const double *a, int64_t lda, double *g);

/* linalg.cc:446-501 */
double orc_spectral_norm_estimate(int64_t m, int64_t n, const double *a, int64_t lda, int *converged);
double orc_inverse_norm_estimate(int64_t n, const double *r, int64_t ldr, int *converged);
/* cqrrpt.cc:114-147. method: 0 diag_ratio, 1 krylov_bounds, 2 identity_deviation */
double orc_cond_estimate(int64_t n, const double *x, int64_t ldx, int method, int *is_upper,
                         int *converged);

/* cqrrpt.cc:149-209. m_k0: m x k0 (ldm). a_sk: k0 x k0 (lda).
 * m_pre (m x k0 packed, optional) receives the preconditioned columns;
 * r_pre (rank x rank packed, optional). */
typedef struct {
    int64_t rank;
    int64_t k0_final;
    int32_t retries;
    double cond_at_rank;
    int32_t n_probes;       /* binary-search probes evaluated */
    int64_t probes[64];     /* the ell values probed, in order */
    double probe_raw[64];   /* raw estimator value at each probe */
} orc_stage2_info;
int orc_rank_stage2(int64_t m, int64_t k0, const double *m_k0, int64_t ldm, const double *a_sk,
                    int64_t lda, double eps_tol, double u, int method, double *m_pre, double *r_pre,
                    orc_stage2_info *info);

/* cqrrpt.cc:23-36: c (k x n packed) = a (k x k, lda) * b (k x n, ldb), upper only */
void orc_multiply_upper_triangular(int64_t k, int64_t n, const double *a, int64_t lda,
                                   const double *b, int64_t ldb, double *c);

/* cqrrpt.cc:330-338 (exact __int128 polynomial) */
double orc_flop_model(int64_t m, int64_t n, int64_t k, int64_t d, double c_sk);
int64_t orc_sketch_rows_for(double gamma, int64_t n);

/* Full SASO driver cqrrpt.cc:317-328 + core 233-315 (validation off).
 * q_out: m x k packed (caller sizes m*n), r_out: k x n packed (caller n*n),
 * pivots: n. m_sk_out (optional): d x n sketch. r_sk_out (optional): k_sk x n.
 * diag: [cond_m_pre, truncation_ratio, flop_estimate, k_sk, d, retries, k0_final] */
int orc_cqrrpt(int64_t m, int64_t n, const double *a, int64_t lda, double gamma, int64_t nnz,
               double eps_tol, uint64_t seed, int method, int stage1, double *q_out,
               double *r_out, int64_t *pivots, int64_t *k0_out, int64_t *k_out, double *diag,
               double *m_sk_out, double *r_sk_out);

/* qrcp.cc:150-196 validate(): orth (spectral, power iteration), orth_fro
 * (||Q^T Q - I||_F, BASELINE metric), recon_rel, max_below_diag. */
int orc_validate(int64_t m, int64_t n, int64_t k, const double *a, int64_t lda, const double *q,
                 int64_t ldq, const double *r, int64_t ldr, const int64_t *pivots, double *orth,
                 double *orth_fro, double *recon, double *below);

#ifdef __cplusplus
}
#endif
#endif

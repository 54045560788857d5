/* TEST INFRASTRUCTURE ONLY — CPU oracle for the CQRRPT hot path.
 *
 * A plain-C restatement of the reference algorithm. Every function cites the
 * reference file:line (relative to /root/reference/proj) it follows.
 *
 * Floating-point contraction is written out explicitly. The reference is
 * compiled (oracle/Makefile: GCC 13, -O3, x86-64-v3, GCC's default
 * -ffp-contract=fast) and GCC fuses some `acc += a*b` statements into FMAs
 * but not others: element-wise updates (axpy, the SASO scatter, the QRCP
 * norm downdate) are fused; in-order reductions that GCC vectorises as
 * fold-left reductions (dot's 4-lane body, solve_upper, the triangular
 * product) keep product and add separate except for an odd count's last
 * term, which the scalar epilogue fuses. This file is compiled with
 * -ffp-contract=off and spells each of those choices out with fma(), so the
 * operation sequence — and every bit — is the built reference's.
 * tests/test_oracle_pin.py asserts bit-equality against oracle/_ref on
 * seeded inputs.
 *
 * Never used by the product path: paper_2311_08316_b200/ does not link it.
 */
#include "cqrrpt_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define U ORC_UNIT_ROUNDOFF
#define POWER_CAP 200        /* linalg.cc:19 */
#define POWER_TOL 1e-10      /* linalg.cc:20 */
#define SASO_SALT 0x7361736fULL /* sketch.cc:19 */

/* ------------------------------------------------------------------------ */
/* RNG: rng.hh:18-53                                                        */
/* ------------------------------------------------------------------------ */
uint64_t orc_rng_bits(uint64_t seed, uint64_t counter) {
    uint64_t z = seed + (counter + 1) * 0x9e3779b97f4a7c15ULL; /* rng.hh:20 */
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

static double uniform01(uint64_t seed, uint64_t c) { /* rng.hh:27-29 */
    return (double)((orc_rng_bits(seed, c) >> 11) + 1) * 0x1.0p-53;
}

double orc_rng_normal(uint64_t seed, uint64_t counter) { /* rng.hh:32-36 */
    double u1 = uniform01(seed, 2 * counter);
    double u2 = (double)(orc_rng_bits(seed, 2 * counter + 1) >> 11) * 0x1.0p-53;
    return sqrt(-2.0 * log(u1)) * cos(6.283185307179586476925287 * u2);
}

uint64_t orc_rng_below(uint64_t seed, uint64_t counter, uint64_t bound) { /* rng.hh:39-41 */
    return (uint64_t)(((unsigned __int128)orc_rng_bits(seed, counter) * bound) >> 64);
}

uint64_t orc_mix_seed(uint64_t seed, uint64_t salt) { /* rng.hh:50-53 */
    return orc_rng_bits(seed, 0x5eedULL + salt);
}

/* sketch.cc:100-119: SRFT sample. signs (m), rows (d) in [0, padded). */
int64_t orc_next_pow2(int64_t m) { /* sketch.cc:23-27 */
    int64_t p = 1;
    while (p < m) p <<= 1;
    return p;
}

int orc_srft_sample(int64_t d, int64_t m, uint64_t seed, double *signs, int64_t *rows) {
    if (d < 1 || m < 1 || d > m) return -1;
    const int64_t padded = orc_next_pow2(m);
    const uint64_t sign_seed = orc_mix_seed(seed, 0x7369676eULL), sel_seed = orc_mix_seed(seed, 0x73656c65ULL);
    for (int64_t i = 0; i < m; ++i) signs[i] = (orc_rng_bits(sign_seed, (uint64_t)i) & 1) ? 1.0 : -1.0;
    int64_t *perm = (int64_t *)malloc(sizeof(int64_t) * (size_t)padded);
    if (!perm) return -2;
    for (int64_t i = 0; i < padded; ++i) perm[i] = i;
    for (int64_t i = 0; i < d; ++i) {
        const int64_t j = i + (int64_t)orc_rng_below(sel_seed, (uint64_t)i, (uint64_t)(padded - i));
        const int64_t t = perm[i];
        perm[i] = perm[j];
        perm[j] = t;
    }
    for (int64_t i = 0; i < d; ++i) rows[i] = perm[i];
    free(perm);
    return 0;
}

/* sketch.cc:31-39: unnormalised in-place Walsh-Hadamard butterflies */
static void orc_fwht(double *x, int64_t len) {
    for (int64_t half = 1; half < len; half <<= 1)
        for (int64_t base = 0; base < len; base += 2 * half)
            for (int64_t j = base; j < base + half; ++j) {
                const double a = x[j], b = x[j + half];
                x[j] = a + b;
                x[j + half] = a - b;
            }
}

/* sketch.cc:147-166: out (d x n, ld_out) = SRFT(A) for A (m x n, lda) */
int orc_srft_apply(int64_t d, int64_t m, int64_t n, uint64_t seed, const double *a, int64_t lda, double *out,
                   int64_t ld_out) {
    if (d < 1 || m < 1 || d > m) return -1;
    const int64_t padded = orc_next_pow2(m);
    double *signs = (double *)malloc(sizeof(double) * (size_t)m);
    int64_t *rows = (int64_t *)malloc(sizeof(int64_t) * (size_t)d);
    double *buf = (double *)malloc(sizeof(double) * (size_t)padded);
    if (!signs || !rows || !buf) return -2;
    int rc = orc_srft_sample(d, m, seed, signs, rows);
    if (rc) return rc;
    const double scale = sqrt((double)padded / (double)d);
    const double factor = scale / sqrt((double)padded);
    for (int64_t j = 0; j < n; ++j) {
        for (int64_t i = 0; i < padded; ++i) buf[i] = 0.0;
        for (int64_t i = 0; i < m; ++i) buf[i] = signs[i] * a[j * lda + i];
        orc_fwht(buf, padded);
        for (int64_t r = 0; r < d; ++r) out[j * ld_out + r] = factor * buf[rows[r]];
    }
    free(signs);
    free(rows);
    free(buf);
    return 0;
}

/* sketch.cc:62-72: Gaussian S columns c0 .. c0+m-1 (global rows of M), d x m
   column-major: S(i, c) = normal(c * d + i) / sqrt(d) from mix_seed(seed, 0x6761757373). */
int orc_gaussian_sample(int64_t d, int64_t m, uint64_t seed, int64_t c0, double *s) {
    if (d < 1 || m < 0) return -1;
    const uint64_t stream = orc_mix_seed(seed, 0x6761757373ULL);
    const double scale = 1.0 / sqrt((double)d);
    for (int64_t c = 0; c < m; ++c)
        for (int64_t i = 0; i < d; ++i) s[c * d + i] = orc_rng_normal(stream, (uint64_t)((c0 + c) * d + i)) * scale;
    return 0;
}


/* ------------------------------------------------------------------------ */
/* dense kernels: linalg.cc                                                 */
/* ------------------------------------------------------------------------ */
double orc_dot(const double *a, const double *b, int64_t n) { /* linalg.cc:36-50 */
    /* Fixed 4-way reassociation as written in the reference. As compiled
     * (GCC 13, -O3, x86-64-v3) the 4-lane main loop keeps the product and the
     * add separate, while the scalar epilogue fuses its LAST product into an
     * FMA; restated literally here so the bits match the built reference. */
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int64_t i = 0;
    for (; i + 4 <= n; i += 4) {
        s0 = s0 + a[i] * b[i];
        s1 = s1 + a[i + 1] * b[i + 1];
        s2 = s2 + a[i + 2] * b[i + 2];
        s3 = s3 + a[i + 3] * b[i + 3];
    }
    double s = (i > 0) ? (s0 + s1) + (s2 + s3) : 0.0;
    int64_t rem = n - i;
    if (rem >= 2) {
        s = s + a[i] * b[i];
        s = s + a[i + 1] * b[i + 1];
        i += 2;
        rem -= 2;
    }
    if (rem == 1) s = fma(a[i], b[i], s);
    return s;
}

/* y += alpha * x  (linalg.cc:26-28, contracted) */
static void axpy(double alpha, const double *x, double *y, int64_t n) {
    for (int64_t i = 0; i < n; ++i) y[i] = fma(alpha, x[i], y[i]);
}

static double max_abs_block(int64_t m, int64_t n, const double *a, int64_t lda) { /* linalg.cc:92-97 */
    double mx = 0.0;
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < m; ++i) {
            double v = fabs(a[j * lda + i]);
            mx = (mx < v) ? v : mx; /* std::max(m, v) */
        }
    return mx;
}

/* linalg.cc:110-124 (make_reflector) on column j of b (rows x ?, ld) */
static double make_reflector(double *b, int64_t rows, int64_t ld, int64_t j) {
    double *colj = b + j * ld;
    double x0 = colj[j];
    double tail_sq = orc_dot(colj + j + 1, colj + j + 1, rows - j - 1);
    double norm_x = sqrt(fma(x0, x0, tail_sq));
    if (norm_x == 0.0) return 0.0;
    double sign = (x0 >= 0.0) ? 1.0 : -1.0;
    double alpha = -sign * norm_x;
    double v0 = x0 - alpha;
    for (int64_t i = j + 1; i < rows; ++i) colj[i] /= v0;
    colj[j] = alpha;
    return (norm_x + fabs(x0)) / norm_x;
}

/* linalg.cc:126-136 (apply_reflector): reflector in column jv of house,
 * applied to column c of target, rows j..rows-1 */
static void apply_reflector(const double *house, int64_t ldh, int64_t jv, double beta, int64_t j,
                            double *target, int64_t ldt, int64_t c, int64_t rows) {
    const double *w = house + jv * ldh;
    double *t = target + c * ldt;
    double tau = t[j];
    tau += orc_dot(w + j + 1, t + j + 1, rows - j - 1);
    tau *= beta;
    t[j] -= tau;
    axpy(-tau, w + j + 1, t + j + 1, rows - j - 1);
}

/* linalg.cc:139-149 */
static void householder_reduce(double *b, int64_t m, int64_t n, double *betas) {
    for (int64_t j = 0; j < n; ++j) {
        double beta = make_reflector(b, m, m, j);
        betas[j] = beta;
        if (beta == 0.0) continue;
#pragma omp parallel for schedule(static) if ((m - j) * (n - j) > (1 << 16))
        for (int64_t c = j + 1; c < n; ++c) apply_reflector(b, m, j, beta, j, b, m, c, m);
    }
}

/* linalg.cc:186-197: thin Q (m x k) */
static void accumulate_q(const double *b, int64_t m, const double *betas, int64_t k, double *q) {
    memset(q, 0, sizeof(double) * (size_t)(m * k));
    for (int64_t j = 0; j < k; ++j) q[j * m + j] = 1.0;
    for (int64_t j = k - 1; j >= 0; --j) {
        double beta = betas[j];
        if (beta == 0.0) continue;
#pragma omp parallel for schedule(static) if ((m - j) * (k - j) > (1 << 16))
        for (int64_t c = j; c < k; ++c) apply_reflector(b, m, j, beta, j, q, m, c, m);
    }
}

/* linalg.cc:151-161 */
static void apply_q_left(const double *b, int64_t m, int64_t nb, const double *betas, double *target,
                         int64_t nt) {
    for (int64_t j = nb - 1; j >= 0; --j) {
        double beta = betas[j];
        if (beta == 0.0) continue;
#pragma omp parallel for schedule(static) if ((m - j) * nt > (1 << 16))
        for (int64_t c = 0; c < nt; ++c) apply_reflector(b, m, j, beta, j, target, m, c, m);
    }
}

/* linalg.cc:52-66: c (m x n packed) = a (m x k, lda) * b (k x n, ldb) */
static void matmul(int64_t m, int64_t k, int64_t n, const double *a, int64_t lda, const double *b,
                   int64_t ldb, double *c) {
    memset(c, 0, sizeof(double) * (size_t)(m * n));
#pragma omp parallel for schedule(static) if (m * k * n > (1 << 16))
    for (int64_t j = 0; j < n; ++j) {
        double *cj = c + j * m;
        for (int64_t t = 0; t < k; ++t) {
            double btj = b[j * ldb + t];
            if (btj != 0.0) axpy(btj, a + t * lda, cj, m);
        }
    }
}

/* linalg.cc:223-242 */
int orc_cholesky(int64_t n, const double *g, int64_t ldg, double *r_out, int64_t *failure_index) {
    double *r = (double *)calloc((size_t)(n * n) + 1, sizeof(double));
    if (!r) return -5;
    *failure_index = 0;
    for (int64_t j = 0; j < n; ++j) {
        double *rj = r + j * n;
        for (int64_t i = 0; i < j; ++i) {
            double s = g[j * ldg + i] - orc_dot(r + i * n, rj, i);
            rj[i] = s / r[i * n + i];
        }
        double d = g[j * ldg + j] - orc_dot(rj, rj, j);
        if (d <= 0.0 || !isfinite(d)) {
            /* leading j x j block is a valid factor (linalg.cc:236-237) */
            for (int64_t c = 0; c < j; ++c)
                for (int64_t i = 0; i < j; ++i) r_out[c * j + i] = r[c * n + i];
            *failure_index = j + 1;
            free(r);
            return 0;
        }
        rj[j] = sqrt(d);
    }
    memcpy(r_out, r, sizeof(double) * (size_t)(n * n));
    free(r);
    return 0;
}

/* linalg.cc:244-277 */
int orc_trsm_right(int64_t m, int64_t k, const double *b, int64_t ldb, const double *r, int64_t ldr,
                   double *x, int64_t ldx) {
    for (int64_t j = 0; j < k; ++j)
        if (r[j * ldr + j] == 0.0) return -2; /* domain_error, linalg.cc:250-252 */
    if (x != b)
        for (int64_t j = 0; j < k; ++j) memcpy(x + j * ldx, b + j * ldb, sizeof(double) * (size_t)m);
    /* row-block parallel; the per-element operation sequence is chunk-independent */
    const int64_t chunk = 4096;
#pragma omp parallel for schedule(static) if (m * k * k > (1 << 16))
    for (int64_t i0 = 0; i0 < m; i0 += chunk) {
        int64_t len = (i0 + chunk < m) ? chunk : m - i0;
        for (int64_t j = 0; j < k; ++j) {
            double *xj = x + j * ldx + i0;
            for (int64_t t = 0; t < j; ++t) {
                double rtj = r[j * ldr + t];
                if (rtj != 0.0) axpy(-rtj, x + t * ldx + i0, xj, len);
            }
            double inv = 1.0 / r[j * ldr + j];
            for (int64_t i = 0; i < len; ++i) xj[i] *= inv;
        }
    }
    return 0;
}

/* linalg.cc:279-286 */
static void solve_upper(int64_t n, const double *r, int64_t ldr, double *x) {
    for (int64_t i = n - 1; i >= 0; --i) {
        double s = x[i];
        /* in-order reduction; as built only an odd count's last term is fused */
        for (int64_t j = i + 1; j < n; ++j)
            s = (j == n - 1 && ((n - i - 1) & 1)) ? fma(-r[j * ldr + i], x[j], s) : s - r[j * ldr + i] * x[j];
        x[i] = s / r[i * ldr + i];
    }
}

/* linalg.cc:288-296 */
static void solve_upper_transposed(int64_t n, const double *r, int64_t ldr, double *x) {
    for (int64_t i = 0; i < n; ++i) {
        double s = x[i];
        const double *ri = r + i * ldr;
        for (int64_t j = 0; j < i; ++j) s = (j == i - 1 && (i & 1)) ? fma(-ri[j], x[j], s) : s - ri[j] * x[j];
        x[i] = s / ri[i];
    }
}

/* linalg.cc:298-307 */
int orc_gram(int64_t m, int64_t k, const double *a, int64_t lda, double *g) {
#pragma omp parallel for schedule(dynamic, 4) if (m * k * k > (1 << 16))
    for (int64_t j = 0; j < k; ++j)
        for (int64_t i = 0; i <= j; ++i) g[j * k + i] = orc_dot(a + i * lda, a + j * lda, m);
    for (int64_t j = 0; j < k; ++j)
        for (int64_t i = 0; i < j; ++i) g[i * k + j] = g[j * k + i];
    return 0;
}

/* ------------------------------------------------------------------------ */
/* power iteration: linalg.cc:434-501                                       */
/* ------------------------------------------------------------------------ */
static void deterministic_unit_vector(int64_t n, double *v) { /* linalg.cc:434-442 */
    for (int64_t i = 0; i < n; ++i) v[i] = orc_rng_normal(0x5eedcafe01234567ULL, (uint64_t)i);
    double nrm = sqrt(orc_dot(v, v, n));
    if (nrm == 0.0) {
        v[0] = 1.0;
        return;
    }
    for (int64_t i = 0; i < n; ++i) v[i] /= nrm;
}

typedef struct {
    int kind; /* 0: y = A x, z = A^T y (dense m x n); 1: inverse of upper-tri n x n */
    int64_t m, n, ld;
    const double *a;
} op_t;

static void op_forward(const op_t *op, const double *x, double *y) {
    if (op->kind == 0) { /* linalg.cc:473-476 */
        for (int64_t i = 0; i < op->m; ++i) y[i] = 0.0;
        for (int64_t j = 0; j < op->n; ++j) axpy(x[j], op->a + j * op->ld, y, op->m);
    } else { /* linalg.cc:493-496 */
        memcpy(y, x, sizeof(double) * (size_t)op->n);
        solve_upper(op->n, op->a, op->ld, y);
    }
}

static void op_adjoint(const op_t *op, const double *y, double *z) {
    if (op->kind == 0) { /* linalg.cc:477-480 */
        for (int64_t j = 0; j < op->n; ++j) z[j] = orc_dot(op->a + j * op->ld, y, op->m);
    } else { /* linalg.cc:497-500 */
        memcpy(z, y, sizeof(double) * (size_t)op->n);
        solve_upper_transposed(op->n, op->a, op->ld, z);
    }
}

/* linalg.cc:446-465 */
static double power_iterate(const op_t *op, int *converged) {
    int64_t n = op->n, mrows = (op->kind == 0) ? op->m : op->n;
    double *v = (double *)malloc(sizeof(double) * (size_t)(n + 1));
    double *w = (double *)malloc(sizeof(double) * (size_t)(mrows + 1));
    double *z = (double *)malloc(sizeof(double) * (size_t)(n + 1));
    deterministic_unit_vector(n, v);
    double est = 0.0, prev = -1.0;
    int conv = 0;
    for (int it = 0; it < POWER_CAP; ++it) {
        op_forward(op, v, w);
        double nw = sqrt(orc_dot(w, w, mrows));
        if (nw == 0.0) {
            est = 0.0;
            conv = 1;
            goto done;
        }
        est = (est < nw) ? nw : est; /* std::max(est, nw) */
        if (prev >= 0.0 && fabs(est - prev) <= POWER_TOL * est) {
            conv = 1;
            goto done;
        }
        prev = est;
        op_adjoint(op, w, z);
        double nz = sqrt(orc_dot(z, z, n));
        if (nz == 0.0) {
            conv = 1;
            goto done;
        }
        for (int64_t i = 0; i < n; ++i) v[i] = z[i] / nz;
    }
done:
    free(v);
    free(w);
    free(z);
    if (converged) *converged = conv;
    return est;
}

double orc_spectral_norm_estimate(int64_t m, int64_t n, const double *a, int64_t lda, int *converged) {
    if (m == 0 || n == 0) { /* linalg.cc:470 */
        if (converged) *converged = 1;
        return 0.0;
    }
    op_t op = {0, m, n, lda, a};
    return power_iterate(&op, converged);
}

double orc_inverse_norm_estimate(int64_t n, const double *r, int64_t ldr, int *converged) {
    if (converged) *converged = 1;
    if (n == 0) return 0.0;
    for (int64_t j = 0; j < n; ++j)
        if (r[j * ldr + j] == 0.0) return INFINITY; /* linalg.cc:489-490 */
    op_t op = {1, n, n, ldr, r};
    return power_iterate(&op, converged);
}

/* cqrrpt.cc:114-147 */
double orc_cond_estimate(int64_t n, const double *x, int64_t ldx, int method, int *is_upper,
                         int *converged) {
    int up = 1, conv = 1;
    double value = 1.0;
    if (n == 0) goto out;
    if (method == 0) { /* diag_ratio */
        double hi = 0.0, lo = INFINITY;
        for (int64_t i = 0; i < n; ++i) {
            double d = fabs(x[i * ldx + i]);
            hi = (hi < d) ? d : hi;
            lo = (d < lo) ? d : lo;
        }
        double v = (lo == 0.0) ? INFINITY : hi / lo;
        value = (v < 1.0) ? 1.0 : v;
        up = 0;
    } else if (method == 1) { /* krylov_bounds */
        int c1 = 1, c2 = 1;
        double hi = orc_spectral_norm_estimate(n, n, x, ldx, &c1);
        double inv = orc_inverse_norm_estimate(n, x, ldx, &c2);
        double v = hi * (1.0 + 1e-6) * inv * (1.0 + 1e-6);
        value = (v < 1.0) ? 1.0 : v;
        conv = c1 && c2;
    } else { /* identity_deviation */
        double *dev = (double *)malloc(sizeof(double) * (size_t)(n * n));
        for (int64_t j = 0; j < n; ++j) memcpy(dev + j * n, x + j * ldx, sizeof(double) * (size_t)n);
        for (int64_t i = 0; i < n; ++i) dev[i * n + i] -= 1.0;
        int c1 = 1;
        double tau = orc_spectral_norm_estimate(n, n, dev, n, &c1) * (1.0 + 1e-6);
        free(dev);
        conv = c1;
        if (tau >= 1.0) {
            value = INFINITY;
        } else {
            double v = (1.0 + tau) / (1.0 - tau);
            value = (v < 1.0) ? 1.0 : v;
        }
    }
out:
    if (is_upper) *is_upper = up;
    if (converged) *converged = conv;
    return value;
}

/* ------------------------------------------------------------------------ */
/* generators: testmat.cc                                                   */
/* ------------------------------------------------------------------------ */
static void gaussian_block(int64_t m, int64_t n, uint64_t stream_seed, double *g) { /* testmat.cc:17-25 */
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < m; ++i) g[j * m + i] = orc_rng_normal(stream_seed, (uint64_t)(j * m + i));
}

int orc_gaussian_block(int64_t m, int64_t n, uint64_t stream_seed, double *out) { /* testmat.cc:17-25 */
    gaussian_block(m, n, stream_seed, out);
    return 0;
}

int orc_gen_gaussian(int64_t m, int64_t n, uint64_t seed, double *out) { /* testmat.cc:141-143 */
    gaussian_block(m, n, orc_mix_seed(seed, 0x676175ULL), out);
    return 0;
}

int orc_gen_exact_rank(int64_t m, int64_t n, int64_t r, uint64_t seed, double *out) { /* 145-151 */
    if (r < 1 || r > (m < n ? m : n)) return -1;
    double *a = (double *)malloc(sizeof(double) * (size_t)(m * r));
    double *b = (double *)malloc(sizeof(double) * (size_t)(r * n));
    gaussian_block(m, r, orc_mix_seed(seed, 0xaaaaULL), a);
    gaussian_block(r, n, orc_mix_seed(seed, 0xbbbbULL), b);
    matmul(m, r, n, a, m, b, r, out);
    free(a);
    free(b);
    return 0;
}

int orc_gen_spectral_list(int64_t m, int64_t n, const double *sigma, uint64_t seed, double *out) {
    /* testmat.cc:79-93 */
    if (m < n) return -1;
    for (int64_t i = 0; i < n; ++i)
        if (sigma[i] <= 0.0 || (i > 0 && sigma[i] > sigma[i - 1])) return -1; /* testmat.cc:72-75 */
    double *left = (double *)malloc(sizeof(double) * (size_t)(m * n));
    double *betas = (double *)malloc(sizeof(double) * (size_t)n);
    gaussian_block(m, n, orc_mix_seed(seed, 0x6c656674ULL), left);
    householder_reduce(left, m, n, betas);
    double *vb = (double *)malloc(sizeof(double) * (size_t)(n * n));
    double *vbet = (double *)malloc(sizeof(double) * (size_t)n);
    double *v = (double *)malloc(sizeof(double) * (size_t)(n * n));
    gaussian_block(n, n, orc_mix_seed(seed, 0x72696768ULL), vb);
    householder_reduce(vb, n, n, vbet); /* householder_qr(...).q, linalg.cc:201-208 */
    accumulate_q(vb, n, vbet, n, v);
    memset(out, 0, sizeof(double) * (size_t)(m * n));
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < n; ++i) out[j * m + i] = sigma[i] * v[i * n + j];
    apply_q_left(left, m, n, betas, out, n);
    free(left);
    free(betas);
    free(vb);
    free(vbet);
    free(v);
    return 0;
}

int orc_gen_kahan(int64_t n, double theta, double *out) { /* testmat.cc:126-139 */
    if (n < 1 || !(theta > 0.0) || !(theta < 1.5707963267948966)) return -1;
    double s = sin(theta), c = cos(theta);
    memset(out, 0, sizeof(double) * (size_t)(n * n));
    double row_scale = 1.0;
    for (int64_t i = 0; i < n; ++i) {
        out[i * n + i] = row_scale;
        for (int64_t j = i + 1; j < n; ++j) out[j * n + i] = -c * row_scale;
        row_scale *= s;
    }
    return 0;
}

static void c5_permutation(int64_t n, uint64_t seed, int64_t *p) {
    /* pi = Fisher-Yates as verify.cc:45-55, stream mix_seed(seed, "perm") */
    for (int64_t i = 0; i < n; ++i) p[i] = i;
    uint64_t s = orc_mix_seed(seed, 0x7065726dULL);
    for (int64_t i = 0; i < n - 1; ++i) {
        int64_t j = i + (int64_t)orc_rng_below(s, (uint64_t)i, (uint64_t)(n - i));
        int64_t t = p[i];
        p[i] = p[j];
        p[j] = t;
    }
}

int orc_c5_column_factors(int64_t n, double span_decades, uint64_t seed, double *f) {
    int64_t *p = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + 1));
    c5_permutation(n, seed, p);
    for (int64_t j = 0; j < n; ++j) f[j] = pow(10.0, -span_decades * (double)p[j] / (double)(n - 1));
    free(p);
    return 0;
}

int orc_gen_gaussian_rows(int64_t m, int64_t n, uint64_t seed, int64_t r0, int64_t r1, double *out, int64_t ld) {
    /* rows [r0, r1) of gaussian_block(m, n, mix_seed(seed, "gau")): element (i, j) is draw j*m + i */
    if (r0 < 0 || r1 > m || r0 > r1 || ld < r1 - r0) return -1;
    const uint64_t s = orc_mix_seed(seed, 0x676175ULL);
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = r0; i < r1; ++i) out[j * ld + (i - r0)] = orc_rng_normal(s, (uint64_t)(j * m + i));
    return 0;
}

int orc_c5_scale_columns(int64_t m, int64_t n, int64_t ld, double span_decades, uint64_t seed,
                         double *a, int64_t *perm_out) {
    int64_t *p = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + 1));
    c5_permutation(n, seed, p);
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < n; ++j) {
        double f = pow(10.0, -span_decades * (double)p[j] / (double)(n - 1));
        for (int64_t i = 0; i < m; ++i) a[j * ld + i] *= f;
    }
    if (perm_out) memcpy(perm_out, p, sizeof(int64_t) * (size_t)n);
    free(p);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* SASO sketch: sketch.cc                                                   */
/* ------------------------------------------------------------------------ */
int orc_saso_sample(int64_t d, int64_t c0, int64_t count, int64_t nnz, uint64_t seed, int64_t *rows,
                    double *vals) {
    if (d < 1) return -1;                 /* sketch.cc:54 */
    if (nnz < 1 || nnz > d) return -1;    /* sketch.cc:74-75 */
    const double val = 1.0 / sqrt((double)d); /* sketch.cc:79 */
#pragma omp parallel for schedule(static) if (count > 4096)
    for (int64_t cc = 0; cc < count; ++cc) {
        uint64_t cs = orc_mix_seed(seed, SASO_SALT + (uint64_t)(c0 + cc)); /* sketch.cc:81 */
        uint64_t ctr = 0;
        int64_t *r = rows + cc * nnz;
        double *v = vals + cc * nnz;
        for (int64_t t = 0; t < nnz; ++t) {
            int64_t cand;
            int fresh;
            do { /* rejection until distinct: sketch.cc:88-93 */
                cand = (int64_t)orc_rng_below(cs, ctr++, (uint64_t)d);
                fresh = 1;
                for (int64_t u = 0; u < t; ++u)
                    if (r[u] == cand) {
                        fresh = 0;
                        break;
                    }
            } while (!fresh);
            r[t] = cand;
            v[t] = (orc_rng_bits(cs, ctr++) & 1) ? val : -val; /* sketch.cc:95 */
        }
    }
    return 0;
}

int orc_saso_apply(int64_t d, int64_t m, int64_t n, int64_t nnz, uint64_t seed, int64_t c0,
                   const double *a, int64_t lda, double *out, int64_t ld_out) {
    int64_t *rows = (int64_t *)malloc(sizeof(int64_t) * (size_t)(m * nnz + 1));
    double *vals = (double *)malloc(sizeof(double) * (size_t)(m * nnz + 1));
    int rc = orc_saso_sample(d, c0, m, nnz, seed, rows, vals);
    if (rc == 0) {
#pragma omp parallel for schedule(static) if (m * n * nnz > (1 << 16))
        for (int64_t j = 0; j < n; ++j) { /* sketch.cc:134-144 */
            const double *mj = a + j * lda;
            double *oj = out + j * ld_out;
            for (int64_t c = 0; c < m; ++c) {
                double x = mj[c];
                if (x == 0.0) continue;
                const int64_t *r = rows + c * nnz;
                const double *v = vals + c * nnz;
                for (int64_t t = 0; t < nnz; ++t) oj[r[t]] = fma(v[t], x, oj[r[t]]);
            }
        }
    }
    free(rows);
    free(vals);
    return rc;
}

double orc_sketch_flops_saso(int64_t nnz, int64_t m, int64_t n_cols) { /* sketch.cc:216-217 */
    return 2.0 * (double)nnz * (double)m * (double)n_cols;
}

/* ------------------------------------------------------------------------ */
/* QRCP: qrcp.cc:35-97                                                      */
/* ------------------------------------------------------------------------ */
int orc_qrcp_maxnorm(int64_t rows, int64_t n, const double *a, int64_t lda, double rank_tol,
                     double *r_out, int64_t *pivots, int64_t *rank, double *gaps) {
    if (rows < 1) return -1; /* qrcp.cc:37 */
    if (rank_tol < 0.0) rank_tol = (double)n * U; /* qrcp.cc:17,38 */
    double *b = (double *)malloc(sizeof(double) * (size_t)(rows * n + 1));
    double *w = (double *)malloc(sizeof(double) * (size_t)(n + 1));
    double *w_ref = (double *)malloc(sizeof(double) * (size_t)(n + 1));
    for (int64_t j = 0; j < n; ++j) memcpy(b + j * rows, a + j * lda, sizeof(double) * (size_t)rows);
    for (int64_t j = 0; j < n; ++j) pivots[j] = j;
    for (int64_t j = 0; j < n; ++j) { /* qrcp.cc:48-51 */
        w[j] = orc_dot(b + j * rows, b + j * rows, rows);
        w_ref[j] = w[j];
    }
    double max_norm0 = 0.0;
    for (int64_t j = 0; j < n; ++j) max_norm0 = (max_norm0 < w[j]) ? w[j] : max_norm0;
    max_norm0 = sqrt(max_norm0);
    const double stop = rank_tol * max_norm0;
    const double sqrt_u = sqrt(U);

    int64_t k = 0;
    const int64_t steps = (rows < n) ? rows : n;
    for (int64_t i = 0; i < steps; ++i) {
        int64_t p = i; /* argmax_from: lowest index attaining the max, qrcp.cc:26-31 */
        for (int64_t j = i + 1; j < n; ++j)
            if (w[j] > w[p]) p = j;
        if (gaps) { /* tie-margin instrumentation (not in the reference) */
            double second = -INFINITY;
            for (int64_t j = i; j < n; ++j)
                if (j != p && w[j] > second) second = w[j];
            gaps[i] = (w[p] > 0.0 && second > -INFINITY) ? (w[p] - second) / w[p] : INFINITY;
        }
        if (sqrt(w[p] > 0.0 ? w[p] : 0.0) <= stop) break; /* qrcp.cc:62 */
        if (p != i) { /* qrcp.cc:63-66 */
            double *ci = b + i * rows, *cp = b + p * rows;
            for (int64_t r = 0; r < rows; ++r) {
                double t = ci[r];
                ci[r] = cp[r];
                cp[r] = t;
            }
        }
        int64_t tp = pivots[i];
        pivots[i] = pivots[p];
        pivots[p] = tp;
        double tw = w[i];
        w[i] = w[p];
        w[p] = tw;
        tw = w_ref[i];
        w_ref[i] = w_ref[p];
        w_ref[p] = tw;

        double beta = make_reflector(b, rows, rows, i);
        if (beta != 0.0) {
#pragma omp parallel for schedule(static) if ((rows - i) * (n - i) > (1 << 16))
            for (int64_t c = i + 1; c < n; ++c) apply_reflector(b, rows, i, beta, i, b, rows, c, rows);
        }
        k = i + 1;
        for (int64_t j = i + 1; j < n; ++j) { /* qrcp.cc:76-88 */
            double t = b[j * rows + i];
            double updated = fma(-t, t, w[j]);
            if (updated <= sqrt_u * w_ref[j]) {
                const double *cj = b + j * rows + i + 1;
                updated = orc_dot(cj, cj, rows - i - 1);
                w_ref[j] = updated;
            }
            w[j] = updated;
        }
    }
    /* extract_upper: linalg.cc:177-183, k x n packed */
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < k; ++i) r_out[j * k + i] = (i <= j) ? b[j * rows + i] : 0.0;
    *rank = k;
    free(b);
    free(w);
    free(w_ref);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* CQRRPT pieces: cqrrpt.cc                                                 */
/* ------------------------------------------------------------------------ */
int64_t orc_rank_stage1(int64_t k, int64_t n, const double *r, int64_t ldr, double u) {
    /* cqrrpt.cc:92-112 */
    double s = max_abs_block(k, n, r, ldr);
    if (s == 0.0) return 0;
    double *row_mass = (double *)malloc(sizeof(double) * (size_t)(k + 1));
    for (int64_t i = 0; i < k; ++i) {
        double acc = 0.0;
        for (int64_t j = i; j < n; ++j) acc = acc + r[j * ldr + i] * r[j * ldr + i]; /* not contracted as built */
        row_mass[i] = acc;
    }
    const double target = (u * s) * (u * s);
    double tail = 0.0;
    int64_t k0 = k;
    for (int64_t ell = k - 1; ell >= 0; --ell) {
        tail += row_mass[ell];
        if (tail <= target) k0 = ell;
    }
    free(row_mass);
    return k0;
}

void orc_multiply_upper_triangular(int64_t k, int64_t n, const double *a, int64_t lda,
                                   const double *b, int64_t ldb, double *c) {
    /* cqrrpt.cc:23-36 */
    memset(c, 0, sizeof(double) * (size_t)(k * n));
    for (int64_t j = 0; j < n; ++j) {
        int64_t top = (j < k - 1) ? j : k - 1;
        for (int64_t i = 0; i <= top; ++i) {
            double s = 0.0;
            int64_t cnt = top - i + 1; /* odd count: last term fused (as built) */
            for (int64_t t = i; t <= top; ++t)
                s = (t == top && (cnt & 1)) ? fma(a[t * lda + i], b[j * ldb + t], s) : s + a[t * lda + i] * b[j * ldb + t];
            c[j * k + i] = s;
        }
    }
}

double orc_flop_model(int64_t m, int64_t n, int64_t k, int64_t d, double c_sk) { /* cqrrpt.cc:330-338 */
    if (k < 0 || k > ((d < n) ? d : n)) return -1.0;
    __int128 mm = m, kk = k, nn = n, dd = d;
    __int128 num = 12 * mm * kk * kk + 6 * mm * kk * (kk + 1) + 24 * dd * nn * kk -
                   12 * kk * kk * (dd + nn) + 10 * kk * kk * kk + 3 * kk * kk + kk;
    return (double)num / 6.0 + c_sk;
}

int64_t orc_sketch_rows_for(double gamma, int64_t n) { /* cqrrpt.cc:211-213 */
    return (int64_t)ceil(gamma * (double)n);
}

/* NestedCondEstimator (cqrrpt.cc:47-71) state */
typedef struct {
    const double *r;
    int64_t ldr;
    int method;
    int64_t n_memo;
    int64_t ell[64];
    double raw[64];
    orc_stage2_info *info;
} nested_est;

static double nested_at(nested_est *e, int64_t ell) {
    if (ell <= 0) return 1.0;
    int found = 0;
    for (int64_t i = 0; i < e->n_memo; ++i)
        if (e->ell[i] == ell) found = 1;
    if (!found) {
        double v = orc_cond_estimate(ell, e->r, e->ldr, e->method, NULL, NULL);
        if (e->method == 2 && isinf(v)) v = orc_cond_estimate(ell, e->r, e->ldr, 1, NULL, NULL);
        if (e->n_memo < 64) {
            e->ell[e->n_memo] = ell;
            e->raw[e->n_memo] = v;
            e->n_memo++;
        }
        if (e->info && e->info->n_probes < 64) {
            e->info->probes[e->info->n_probes] = ell;
            e->info->probe_raw[e->info->n_probes] = v;
            e->info->n_probes++;
        }
    }
    double v = 1.0;
    for (int64_t i = 0; i < e->n_memo; ++i)
        if (e->ell[i] <= ell) v = (v < e->raw[i]) ? e->raw[i] : v;
    return v;
}

int orc_rank_stage2(int64_t m, int64_t k0, const double *m_k0, int64_t ldm, const double *a_sk,
                    int64_t lda, double eps_tol, double u, int method, double *m_pre_out,
                    double *r_pre_out, orc_stage2_info *info) {
    /* cqrrpt.cc:149-209 */
    if (k0 < 1) return -1;
    orc_stage2_info local;
    if (!info) info = &local;
    memset(info, 0, sizeof(*info));
    double *m_pre = (double *)malloc(sizeof(double) * (size_t)(m * k0 + 1));
    double *g = (double *)malloc(sizeof(double) * (size_t)(k0 * k0 + 1));
    double *r_full = (double *)malloc(sizeof(double) * (size_t)(k0 * k0 + 1));
    int64_t ldr_full = k0;
    int rc = 0;
    for (int attempt = 0;; ++attempt) {
        rc = orc_trsm_right(m, k0, m_k0, ldm, a_sk, lda, m_pre, m);
        if (rc) goto out;
        orc_gram(m, k0, m_pre, m, g);
        int64_t fi = 0;
        orc_cholesky(k0, g, k0, r_full, &fi);
        if (fi == 0) {
            ldr_full = k0;
            break;
        }
        int64_t shrunk = fi - 1;
        info->retries = attempt + 1;
        if (shrunk <= 0) {
            info->rank = 0;
            info->k0_final = 0;
            goto out;
        }
        if (attempt + 1 >= 3) { /* accept the last well-formed leading block */
            k0 = shrunk;
            ldr_full = shrunk; /* cholesky wrote the j x j factor packed */
            break;
        }
        k0 = shrunk;
    }
    info->k0_final = k0;
    {
        const double threshold = sqrt(eps_tol / u);
        nested_est est;
        memset(&est, 0, sizeof(est));
        est.r = r_full;
        est.ldr = ldr_full;
        est.method = method;
        est.info = info;
        int64_t lo = 0, hi = k0;
        while (lo < hi) {
            int64_t mid = lo + (hi - lo + 1) / 2;
            if (nested_at(&est, mid) <= threshold)
                lo = mid;
            else
                hi = mid - 1;
        }
        info->rank = lo;
        info->cond_at_rank = (lo > 0) ? nested_at(&est, lo) : 1.0;
        if (r_pre_out)
            for (int64_t j = 0; j < lo; ++j)
                for (int64_t i = 0; i < lo; ++i) r_pre_out[j * lo + i] = r_full[j * ldr_full + i];
        if (m_pre_out) memcpy(m_pre_out, m_pre, sizeof(double) * (size_t)(m * k0));
    }
out:
    free(m_pre);
    free(g);
    free(r_full);
    return rc;
}

int orc_cqrrpt(int64_t m, int64_t n, const double *a, int64_t lda, double gamma, int64_t nnz,
               double eps_tol, uint64_t seed, int method, int stage1, double *q_out, double *r_out,
               int64_t *pivots, int64_t *k0_out, int64_t *k_out, double *diag, double *m_sk_out,
               double *r_sk_out) {
    /* cqrrpt.cc:317-328 */
    if (gamma < 1.0) return -1;       /* cqrrpt.cc:39 */
    if (!(eps_tol > U)) return -1;    /* cqrrpt.cc:40-41 */
    *k0_out = 0;
    *k_out = 0;
    if (n == 0) return 0;
    int64_t d = orc_sketch_rows_for(gamma, n);
    if (d < 1 || m < 1) return -1;
    if (nnz < 1 || nnz > d) return -1;
    const double u = U;
    int rc = 0;
    double *m_sk = (double *)calloc((size_t)(d * n) + 1, sizeof(double));
    int64_t ksteps = (d < n) ? d : n;
    double *r_sk = (double *)calloc((size_t)(ksteps * n) + 1, sizeof(double));
    double *m_pre = NULL, *r_pre = NULL, *m_k0 = NULL;
    /* cqrrpt_core: cqrrpt.cc:233-315 */
    rc = orc_saso_apply(d, m, n, nnz, seed, 0, a, lda, m_sk, d);
    if (rc) goto out;
    if (m_sk_out) memcpy(m_sk_out, m_sk, sizeof(double) * (size_t)(d * n));
    int64_t k_sk = 0;
    rc = orc_qrcp_maxnorm(d, n, m_sk, d, -1.0, r_sk, pivots, &k_sk, NULL);
    if (rc) goto out;
    if (r_sk_out) memcpy(r_sk_out, r_sk, sizeof(double) * (size_t)(k_sk * n));
    int64_t k0 = stage1 ? orc_rank_stage1(k_sk, n, r_sk, k_sk, u) : k_sk;
    *k0_out = k0;
    if (diag) {
        diag[3] = (double)k_sk;
        diag[4] = (double)d;
    }
    if (k0 == 0) {
        if (diag) {
            diag[0] = 1.0;
            diag[1] = 0.0;
            diag[2] = orc_flop_model(m, n, 0, d, orc_sketch_flops_saso(nnz, m, n));
            diag[5] = 0;
            diag[6] = 0;
        }
        goto out;
    }
    m_k0 = (double *)malloc(sizeof(double) * (size_t)(m * k0)); /* select_columns */
    for (int64_t j = 0; j < k0; ++j) memcpy(m_k0 + j * m, a + pivots[j] * lda, sizeof(double) * (size_t)m);
    m_pre = (double *)malloc(sizeof(double) * (size_t)(m * k0));
    r_pre = (double *)malloc(sizeof(double) * (size_t)(k0 * k0));
    orc_stage2_info info;
    rc = orc_rank_stage2(m, k0, m_k0, m, r_sk, k_sk, eps_tol, u, method, m_pre, r_pre, &info);
    if (rc) goto out;
    int64_t k = info.rank;
    if (diag) {
        diag[5] = info.retries;
        diag[6] = (double)info.k0_final;
    }
    if (k == 0) {
        if (diag) {
            diag[0] = 1.0;
            diag[1] = 0.0;
            diag[2] = orc_flop_model(m, n, 0, d, orc_sketch_flops_saso(nnz, m, n));
        }
        goto out;
    }
    *k_out = k;
    rc = orc_trsm_right(m, k, m_pre, m, r_pre, k, q_out, m); /* cqrrpt.cc:280 */
    if (rc) goto out;
    orc_multiply_upper_triangular(k, n, r_pre, k, r_sk, k_sk, r_out); /* cqrrpt.cc:284 */
    if (diag) { /* cqrrpt.cc:298-303 */
        diag[0] = info.cond_at_rank;
        int64_t cr = k_sk - k, cc = n - k;
        double *cblk = (double *)malloc(sizeof(double) * (size_t)(cr * cc + 1));
        for (int64_t j = 0; j < cc; ++j)
            for (int64_t i = 0; i < cr; ++i) cblk[j * cr + i] = r_sk[(k + j) * k_sk + k + i];
        double c_k = sqrt(orc_dot(cblk, cblk, cr * cc));
        free(cblk);
        double r_norm = orc_spectral_norm_estimate(k_sk, n, r_sk, k_sk, NULL);
        diag[1] = (r_norm > 0.0) ? c_k / r_norm : 0.0;
        diag[2] = orc_flop_model(m, n, k, d, orc_sketch_flops_saso(nnz, m, n));
    }
out:
    free(m_sk);
    free(r_sk);
    free(m_k0);
    free(m_pre);
    free(r_pre);
    return rc;
}

/* qrcp.cc:150-196 */
int orc_validate(int64_t m, int64_t n, int64_t k, const double *a, int64_t lda, const double *q,
                 int64_t ldq, const double *r, int64_t ldr, const int64_t *pivots, double *orth,
                 double *orth_fro, double *recon, double *below) {
    char *seen = (char *)calloc((size_t)n + 1, 1);
    int valid = 1;
    for (int64_t j = 0; j < n; ++j) {
        int64_t p = pivots[j];
        if (p < 0 || p >= n || seen[p]) {
            valid = 0;
            break;
        }
        seen[p] = 1;
    }
    free(seen);
    *orth = 0.0;
    if (orth_fro) *orth_fro = 0.0;
    if (k > 0 && m > 0) {
        double *qtq = (double *)malloc(sizeof(double) * (size_t)(k * k));
#pragma omp parallel for schedule(static)
        for (int64_t j = 0; j < k; ++j) /* matmul_at_b, linalg.cc:68-78 */
            for (int64_t i = 0; i < k; ++i) qtq[j * k + i] = orc_dot(q + i * ldq, q + j * ldq, m);
        for (int64_t i = 0; i < k; ++i) qtq[i * k + i] -= 1.0;
        *orth = orc_spectral_norm_estimate(k, k, qtq, k, NULL);
        if (orth_fro) *orth_fro = sqrt(orc_dot(qtq, qtq, k * k));
        free(qtq);
    }
    double *mm = (double *)malloc(sizeof(double) * (size_t)(m * n + 1));
    for (int64_t j = 0; j < n; ++j) memcpy(mm + j * m, a + j * lda, sizeof(double) * (size_t)m);
    double m_norm = sqrt(orc_dot(mm, mm, m * n));
    *recon = INFINITY;
    if (valid) {
        double *qr = (double *)malloc(sizeof(double) * (size_t)(m * n + 1));
        if (k > 0)
            matmul(m, k, n, q, ldq, r, ldr, qr);
        else
            memset(qr, 0, sizeof(double) * (size_t)(m * n));
        double diff = 0.0;
        const int64_t tot = m * n;
        for (int64_t j = 0; j < n; ++j)
            for (int64_t i = 0; i < m; ++i) {
                double dd = a[pivots[j] * lda + i] - qr[j * m + i];
                diff = (j * m + i == tot - 1 && (tot & 1)) ? fma(dd, dd, diff) : diff + dd * dd;
            }
        diff = sqrt(diff);
        *recon = (m_norm > 0.0) ? diff / m_norm : (diff > 0.0 ? INFINITY : 0.0);
        free(qr);
    }
    free(mm);
    double mb = 0.0;
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = j + 1; i < k; ++i) {
            double v = fabs(r[j * ldr + i]);
            mb = (mb < v) ? v : mb;
        }
    *below = mb;
    return valid ? 0 : 1;
}

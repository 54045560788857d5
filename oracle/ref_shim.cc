// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// C-ABI shim over the UNMODIFIED reference library (/root/reference/proj/src,
// compiled from where it lies by oracle/Makefile into oracle/_ref/). It lets
// the Python test-suite and bench.py's CPU-baseline / `--impl reference` arm
// call the reference's own `cqrrpt()` and its building blocks through plain
// pointers, and lets us pin oracle/cqrrpt_oracle.c against the reference
// bit-for-bit in this container.
//
// Every entry point returns 0 on success and a negative code when the
// reference threw:  -1 invalid_argument, -2 domain_error, -3 logic_error,
// -4 runtime_error, -5 anything else.
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

#include "cqrrpt/cqrrpt.hh"
#include "cqrrpt/matrix_market.hh"
#include "cqrrpt/linalg.hh"
#include "cqrrpt/qrcp.hh"
#include "cqrrpt/rng.hh"
#include "cqrrpt/sketch.hh"
#include "cqrrpt/testmat.hh"

namespace cq = cqrrpt;

namespace {

template <class F>
int guarded(F &&f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument &) {
        return -1;
    } catch (const std::domain_error &) {
        return -2;
    } catch (const std::logic_error &) {
        return -3;
    } catch (const std::runtime_error &) {
        return -4;
    } catch (...) {
        return -5;
    }
}

cq::DenseMatrix from_ptr(int64_t m, int64_t n, const double *a) {
    cq::DenseMatrix out(m, n);
    if (m * n > 0) std::memcpy(out.data(), a, sizeof(double) * static_cast<size_t>(m * n));
    return out;
}

void to_ptr(const cq::DenseMatrix &a, double *out) {
    if (a.size() > 0) std::memcpy(out, a.data(), sizeof(double) * a.size());
}

cq::CondMethod method_of(int32_t m) {
    switch (m) {
        case 0: return cq::CondMethod::diag_ratio;
        case 1: return cq::CondMethod::krylov_bounds;
        case 2: return cq::CondMethod::identity_deviation;
    }
    throw std::logic_error("bad cond method");
}

}  // namespace

extern "C" {

int ref_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void ref_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

// ---- generators (testmat.cc) ------------------------------------------------
int ref_gen_gaussian(int64_t m, int64_t n, uint64_t seed, double *out) {
    return guarded([&] { to_ptr(cq::gen_gaussian(m, n, seed), out); });
}

int ref_gen_exact_rank(int64_t m, int64_t n, int64_t r, uint64_t seed, double *out) {
    return guarded([&] { to_ptr(cq::gen_exact_rank(m, n, r, seed), out); });
}

int ref_gen_spectral_list(int64_t m, int64_t n, const double *sigma, uint64_t seed, double *out) {
    return guarded([&] {
        std::vector<double> s(sigma, sigma + n);
        to_ptr(cq::gen_spectral(m, n, cq::SpectrumSpec::explicit_list(s), seed), out);
    });
}

int ref_gen_spectral_poly(int64_t m, int64_t n, double cond, uint64_t seed, double *out) {
    return guarded([&] {
        to_ptr(cq::gen_spectral(m, n, cq::SpectrumSpec::polynomial_decay(cond), seed), out);
    });
}

int ref_gen_kahan(int64_t n, double theta, double *out) {
    return guarded([&] { to_ptr(cq::gen_kahan(n, theta), out); });
}

// ---- RNG (rng.hh) -----------------------------------------------------------
uint64_t ref_rng_bits(uint64_t seed, uint64_t counter) { return cq::CounterRng(seed).bits(counter); }
uint64_t ref_mix_seed(uint64_t seed, uint64_t salt) { return cq::mix_seed(seed, salt); }
double ref_rng_normal(uint64_t seed, uint64_t counter) { return cq::CounterRng(seed).normal(counter); }

// ---- SASO sketch (sketch.cc) ------------------------------------------------
int ref_saso_sample(int64_t d, int64_t m, int64_t nnz, uint64_t seed, int64_t *rows, double *vals) {
    return guarded([&] {
        cq::SketchOperator s = cq::sample_sketch(cq::SketchFamily::saso, d, m, nnz, seed);
        std::memcpy(rows, s.saso_rows.data(), sizeof(int64_t) * s.saso_rows.size());
        std::memcpy(vals, s.saso_vals.data(), sizeof(double) * s.saso_vals.size());
    });
}

int ref_saso_apply(int64_t d, int64_t m, int64_t n, int64_t nnz, uint64_t seed, const double *a,
                   double *out) {
    return guarded([&] {
        cq::SketchOperator s = cq::sample_sketch(cq::SketchFamily::saso, d, m, nnz, seed);
        to_ptr(cq::apply(s, from_ptr(m, n, a)), out);
    });
}

// SRFT family (sketch.cc:100-119 sample, 147-166 apply): out (d x n)
int ref_srft_sketch_apply(int64_t d, int64_t m, int64_t n, uint64_t seed, const double *a, double *out) {
    return guarded([&] {
        cq::SketchOperator s = cq::sample_sketch(cq::SketchFamily::srft, d, m, 0, seed);
        to_ptr(cq::apply(s, from_ptr(m, n, a)), out);
    });
}

int ref_gaussian_sketch_apply(int64_t d, int64_t m, int64_t n, uint64_t seed, const double *a,
                              double *out) {
    return guarded([&] {
        cq::SketchOperator s = cq::sample_sketch(cq::SketchFamily::gaussian, d, m, 0, seed);
        to_ptr(cq::apply(s, from_ptr(m, n, a)), out);
    });
}

double ref_sketch_flops_saso(int64_t d, int64_t m, int64_t nnz, int64_t n_cols) {
    cq::SketchOperator s;
    s.family = cq::SketchFamily::saso;
    s.d = d;
    s.m = m;
    s.nnz_per_col = nnz;
    return cq::sketch_flops(s, n_cols);
}

// ---- QRCP (qrcp.cc) ---------------------------------------------------------
// r_out: k x n column-major (caller sizes it min(rows,n) x n), pivots: n.
int ref_qrcp_maxnorm(int64_t rows, int64_t n, const double *a, double rank_tol, double *r_out,
                     int64_t *pivots, int64_t *rank) {
    return guarded([&] {
        cq::PivotedQR dec = cq::qrcp_maxnorm(from_ptr(rows, n, a), rank_tol, false);
        to_ptr(dec.r, r_out);
        std::memcpy(pivots, dec.pivots.data(), sizeof(int64_t) * dec.pivots.size());
        *rank = dec.rank;
    });
}

// ---- dense kernels (linalg.cc) ---------------------------------------------
int ref_cholesky(int64_t n, const double *g, double *r_out, int64_t *failure_index) {
    return guarded([&] {
        cq::CholeskyResult ch = cq::cholesky(from_ptr(n, n, g));
        // the factor is (j x j) on failure; write it packed with ld = its rows
        to_ptr(ch.factor, r_out);
        *failure_index = ch.failure_index;
    });
}

int ref_trsm_right(int64_t m, int64_t k, const double *b, const double *r, double *x) {
    return guarded([&] { to_ptr(cq::trsm_right(from_ptr(m, k, b), from_ptr(k, k, r)), x); });
}

int ref_gram(int64_t m, int64_t k, const double *a, double *g) {
    return guarded([&] { to_ptr(cq::gram(from_ptr(m, k, a)), g); });
}

// Matrix Market (matrix_market.cc:12-93)
int ref_mm_write(const char *path, int64_t m, int64_t n, const double *a, int32_t coordinate) {
    return guarded([&] {
        cq::write_matrix_market(std::string(path), from_ptr(m, n, a),
                                coordinate ? cq::MatrixMarketFormat::coordinate : cq::MatrixMarketFormat::array);
    });
}

// out == NULL: only the shape
int ref_mm_read(const char *path, int64_t *m, int64_t *n, double *out) {
    return guarded([&] {
        cq::DenseMatrix a = cq::read_matrix_market(std::string(path));
        *m = a.rows();
        *n = a.cols();
        if (out) to_ptr(a, out);
    });
}

// cholesky_qr / cholesky_qr2 (cqrrpt.cc:75-90): q (m x n), r (n x n) on success
int ref_cholesky_qr(int64_t m, int64_t n, const double *a, int32_t twice, double *q_out, double *r_out,
                    int64_t *failure_index) {
    return guarded([&] {
        cq::CholeskyQrResult res = twice ? cq::cholesky_qr2(from_ptr(m, n, a)) : cq::cholesky_qr(from_ptr(m, n, a));
        *failure_index = res.failure_index;
        if (res.ok()) {
            to_ptr(res.q, q_out);
            to_ptr(res.r, r_out);
        }
    });
}

int ref_spectral_norm_estimate(int64_t m, int64_t n, const double *a, double *value, int32_t *conv) {
    return guarded([&] {
        cq::NormEstimate e = cq::spectral_norm_estimate(from_ptr(m, n, a));
        *value = e.value;
        *conv = e.converged ? 1 : 0;
    });
}

int ref_inverse_norm_estimate(int64_t n, const double *r, double *value, int32_t *conv) {
    return guarded([&] {
        cq::NormEstimate e = cq::inverse_norm_estimate(from_ptr(n, n, r));
        *value = e.value;
        *conv = e.converged ? 1 : 0;
    });
}

// ---- CQRRPT pieces (cqrrpt.cc) ---------------------------------------------
int ref_rank_stage1(int64_t k, int64_t n, const double *r, int64_t *k0) {
    return guarded([&] { *k0 = cq::rank_stage1(from_ptr(k, n, r)); });
}

int ref_cond_estimate(int64_t n, const double *x, int32_t method, double *value, int32_t *upper,
                      int32_t *conv) {
    return guarded([&] {
        cq::CondBound b = cq::cond_estimate(from_ptr(n, n, x), method_of(method));
        *value = b.value;
        *upper = b.is_upper_bound ? 1 : 0;
        *conv = b.converged ? 1 : 0;
    });
}

// m_pre_out: m x k0_final (caller sizes m x k0), r_pre_out: rank x rank.
int ref_rank_stage2(int64_t m, int64_t k0, const double *m_k0, const double *a_sk, double eps_tol,
                    int32_t method, int64_t *rank, int64_t *k0_final, int32_t *retries,
                    double *cond_at_rank, double *r_pre_out, double *m_pre_out) {
    return guarded([&] {
        cq::Stage2Result s = cq::rank_stage2(from_ptr(m, k0, m_k0), from_ptr(k0, k0, a_sk), eps_tol,
                                             cq::unit_roundoff, method_of(method));
        *rank = s.rank;
        *k0_final = s.k0_final;
        *retries = s.retries;
        *cond_at_rank = s.cond_at_rank;
        if (r_pre_out) to_ptr(s.r_pre, r_pre_out);
        if (m_pre_out) to_ptr(s.m_pre, m_pre_out);
    });
}

double ref_flop_model(int64_t m, int64_t n, int64_t k, int64_t d, double c_sk) {
    try {
        return cq::flop_model(m, n, k, d, c_sk);
    } catch (...) {
        return -1.0;
    }
}

int64_t ref_sketch_rows_for(double gamma, int64_t n) { return cq::sketch_rows_for(gamma, n); }

// Full driver. q_out: m x n (first k columns written), r_out: n x n max
// (k x n written, ld = k), pivots: n. diag[0..3] = cond_m_pre, truncation
// ratio, flop estimate, validation pass; timings[0..6] = PhaseTimings.
// valid[0..2] = orth_loss (spectral), recon_rel, max_below_diag (only when
// validate != 0).
int ref_cqrrpt(int64_t m, int64_t n, const double *a, double gamma, int64_t nnz, double eps_tol,
               uint64_t seed, int32_t method, int32_t stage1, int32_t validate, double *q_out,
               double *r_out, int64_t *pivots, int64_t *k0, int64_t *k, double *diag,
               double *timings, double *valid) {
    return guarded([&] {
        cq::CqrrptConfig cfg;
        cfg.gamma = gamma;
        cfg.family = cq::SketchFamily::saso;
        cfg.nnz_per_col = nnz;
        cfg.eps_tol = eps_tol;
        cfg.cond_method = method_of(method);
        cfg.stage1_enabled = stage1 != 0;
        cfg.seed = seed;
        cfg.validate_output = validate != 0;
        cq::CqrrptOutput out = cq::cqrrpt(from_ptr(m, n, a), cfg);
        *k0 = out.k0;
        *k = out.k;
        if (q_out) to_ptr(out.factorization.q, q_out);
        if (r_out) to_ptr(out.factorization.r, r_out);
        if (pivots && !out.factorization.pivots.empty())
            std::memcpy(pivots, out.factorization.pivots.data(),
                        sizeof(int64_t) * out.factorization.pivots.size());
        if (diag) {
            diag[0] = out.diagnostics.cond_m_pre;
            diag[1] = out.diagnostics.truncation_ratio;
            diag[2] = out.diagnostics.flop_estimate;
            diag[3] = out.diagnostics.validation ? (out.diagnostics.validation->pass ? 1.0 : 0.0) : -1.0;
        }
        if (timings) {
            const cq::PhaseTimings &t = out.diagnostics.timings;
            timings[0] = t.sketch;
            timings[1] = t.qrcp;
            timings[2] = t.rank_select;
            timings[3] = t.precondition;
            timings[4] = t.cholesky_qr;
            timings[5] = t.undo;
            timings[6] = t.total;
        }
        if (valid && out.diagnostics.validation) {
            valid[0] = out.diagnostics.validation->orth_loss;
            valid[1] = out.diagnostics.validation->recon_rel;
            valid[2] = out.diagnostics.validation->max_below_diag;
        }
    });
}

// validate() on caller-supplied factors (qrcp.cc:150-196).
int ref_validate(int64_t m, int64_t n, int64_t k, const double *a, const double *q, const double *r,
                 const int64_t *pivots, double tol, double *orth, double *recon, double *below,
                 int32_t *pass) {
    return guarded([&] {
        cq::PivotedQR dec;
        dec.q = from_ptr(m, k, q);
        dec.r = from_ptr(k, n, r);
        dec.pivots.assign(pivots, pivots + n);
        dec.rank = k;
        cq::ValidationReport rep = cq::validate(dec, from_ptr(m, n, a), tol);
        *orth = rep.orth_loss;
        *recon = rep.recon_rel;
        *below = rep.max_below_diag;
        *pass = rep.pass ? 1 : 0;
    });
}

}  // extern "C"

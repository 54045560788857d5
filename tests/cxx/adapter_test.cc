// Reference-signature adapter test (C++): restates assertions of the
// reference's own test_cqrrpt.cc through cqrrpt_b200::cqrrpt on the GPU, with
// inputs and expected pivots from the CPU oracle (test infrastructure).
#include <cmath>
#include <cstdio>
#include <stdexcept>

#include "cqrrpt_b200.hh"
#include "../../oracle/cqrrpt_oracle.h"

namespace cq = cqrrpt_b200;
static int failures = 0;
#define CHECK(c)                                                   \
    do {                                                           \
        if (!(c)) {                                                \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); \
            ++failures;                                            \
        }                                                          \
    } while (0)

static cq::DenseMatrix gaussian(int64_t m, int64_t n, uint64_t seed) {
    cq::DenseMatrix a(m, n);
    orc_gen_gaussian(m, n, seed, a.data());
    return a;
}

int main() {
    // full rank tall matrix: k = n, validation passes, pivots equal the reference's
    {
        cq::DenseMatrix m = gaussian(2000, 64, 21);
        cq::CqrrptConfig cfg;
        cfg.nnz_per_col = 8;
        cq::CqrrptOutput out = cq::cqrrpt(m, cfg);
        CHECK(out.k0 == 64 && out.k == 64);
        CHECK(out.diagnostics.validation.has_value() && out.diagnostics.validation->pass);
        std::vector<double> q(2000 * 64), r(64 * 64);
        std::vector<int64_t> piv(64);
        int64_t k0 = 0, k = 0;
        double diag[8];
        orc_cqrrpt(2000, 64, m.data(), 2000, 1.25, 8, 1e-4, 0, 2, 1, q.data(), r.data(), piv.data(), &k0, &k, diag,
                   nullptr, nullptr);
        CHECK(k == out.k);
        for (int i = 0; i < 64; ++i) CHECK(piv[i] == out.factorization.pivots[i]);
    }
    // test_cqrrpt.cc:243-251: exact rank 10 detected
    {
        cq::DenseMatrix m(200, 40);
        orc_gen_exact_rank(200, 40, 10, 24, m.data());
        cq::CqrrptConfig cfg;
        cfg.seed = 25;
        cq::CqrrptOutput out = cq::cqrrpt(m, cfg);
        CHECK(out.k == 10);
    }
    // test_cqrrpt.cc:262-268: zero matrix -> rank 0
    {
        cq::CqrrptOutput out = cq::cqrrpt(cq::DenseMatrix(30, 5));
        CHECK(out.k == 0 && out.k0 == 0 && out.factorization.q.cols() == 0 && out.factorization.r.rows() == 0);
    }
    // test_cqrrpt.cc:348-356: config invariants throw std::invalid_argument
    {
        cq::DenseMatrix m = gaussian(20, 4, 29);
        bool t1 = false, t2 = false;
        cq::CqrrptConfig bad;
        bad.gamma = 0.5;
        try { cq::cqrrpt(m, bad); } catch (const std::invalid_argument &) { t1 = true; }
        cq::CqrrptConfig bad2;
        bad2.eps_tol = cq::unit_roundoff / 2;
        try { cq::cqrrpt(m, bad2); } catch (const std::invalid_argument &) { t2 = true; }
        CHECK(t1 && t2);
    }
    // test_cqrrpt.cc:270-283: bitwise deterministic, seed-sensitive
    {
        cq::DenseMatrix m = gaussian(150, 20, 26);
        cq::CqrrptConfig cfg;
        cfg.seed = 27;
        cq::CqrrptOutput a = cq::cqrrpt(m, cfg), b = cq::cqrrpt(m, cfg);
        CHECK(a.factorization.q == b.factorization.q && a.factorization.r == b.factorization.r);
        CHECK(a.factorization.pivots == b.factorization.pivots && a.k == b.k);
        cfg.seed = 28;
        cq::CqrrptOutput c = cq::cqrrpt(m, cfg);
        CHECK(!(a.factorization.r == c.factorization.r));
    }
    // test_cqrrpt.cc:253-260 defaults
    CHECK(cq::sketch_rows_for(1.25, 50) == 63 && cq::sketch_rows_for(3.0, 500) == 1500);
    CHECK(cq::CqrrptConfig{}.nnz_per_col == 4 && cq::CqrrptConfig{}.gamma == 1.25);
    std::printf("%s (%d failures)\n", failures ? "FAILED" : "OK", failures);
    return failures ? 1 : 0;
}

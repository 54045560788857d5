// What a reference caller gets: the reference's own cqrrpt::cqrrpt() call
// site (cqrrpt.hh:140) linked against the GPU drop-in
// (paper_2311_08316_b200/dropin/cqrrpt_dropin.cc) -- host DenseMatrix in,
// host factors out, exactly the reference's API -- timed wall-clock per call,
// best of R after a warm-up, on a BASELINE-shaped input built with the
// reference's own generator (gen_gaussian, C5-style column scaling optional).
// Built by oracle/Makefile (target acceptance) next to acceptance_gpu.
//   usage: dropin_bench m n [reps] [gamma] [nnz]
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "cqrrpt/cqrrpt.hh"
#include "cqrrpt/testmat.hh"

int main(int argc, char **argv) {
    if (argc < 3) {
        std::fprintf(stderr, "usage: %s m n [reps] [gamma] [nnz]\n", argv[0]);
        return 2;
    }
    const int64_t m = std::atoll(argv[1]), n = std::atoll(argv[2]);
    const int reps = argc > 3 ? std::atoi(argv[3]) : 5;
    cqrrpt::CqrrptConfig cfg;
    cfg.gamma = argc > 4 ? std::atof(argv[4]) : 1.25;
    cfg.nnz_per_col = argc > 5 ? std::atoll(argv[5]) : 8;
    cfg.validate_output = false;
    cqrrpt::DenseMatrix a = cqrrpt::gen_gaussian(m, n, 0);
    double best = 1e300, dev_total = 0.0;
    int64_t k = 0;
    for (int r = 0; r <= reps; ++r) {
        auto t0 = std::chrono::steady_clock::now();
        cqrrpt::CqrrptOutput out = cqrrpt::cqrrpt(a, cfg);
        const double t = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (r > 0 && t < best) {
            best = t;
            dev_total = out.diagnostics.timings.total;
        }
        k = out.k;
    }
    const double canon = 2.0 * double(m) * double(n) * double(n) - 2.0 * std::pow(double(n), 3) / 3.0;
    std::printf("{\"call\": \"cqrrpt::cqrrpt (reference API, GPU drop-in)\", \"m\": %lld, \"n\": %lld, \"k\": %lld, "
                "\"best_wall_s\": %.6f, \"device_total_s\": %.6f, \"canonical_gflops_wall\": %.1f, \"reps\": %d}\n",
                (long long)m, (long long)n, (long long)k, best, dev_total, canon / best / 1e9, reps);
    return 0;
}

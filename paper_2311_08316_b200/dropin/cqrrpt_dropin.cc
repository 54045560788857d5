// cqrrpt_dropin.cc -- the reference's own entry points, defined over the
// B200 C ABI.
//
//   cqrrpt::CqrrptOutput cqrrpt::cqrrpt(const DenseMatrix &, const CqrrptConfig &)
//       /root/reference/proj/include/cqrrpt/cqrrpt.hh:140 (body cqrrpt.cc:317-328)
//   cqrrpt::CqrrptOutput cqrrpt::cqrrpt_core(const DenseMatrix &, const SketchOperator &,
//                                            const CqrrptConfig &)
//       cqrrpt.hh:136 (body cqrrpt.cc:233-315)
//
// Compiled against the reference's public headers (-I <reference>/include),
// this translation unit replaces cqrrpt.cc's two definitions: a caller of the
// reference library links it (and libcqrrpt_gpu.so) ahead of the reference's
// cqrrpt.o -- or, as oracle/Makefile does for the reference's acceptance
// suite, links the reference objects with those two symbols weakened -- and
// every existing call site runs on the GPU with the reference's types,
// argument meaning and exceptions:
//   std::invalid_argument  gamma < 1, eps_tol <= u, operator/matrix mismatch,
//                          SASO nnz outside [1, d], SRFT d > m (C ABI -i)
//   std::domain_error      zero diagonal in a triangular solve (CQRRPT_GPU_ERR_SINGULAR)
//   std::runtime_error     CUDA / NCCL failures (positive C ABI codes)
// M is read through the host entry point cqrrpt_gpu_dgeqpt_host (its pages
// are registered with CUDA for full-bandwidth DMA when large), Q (m x k),
// R (k x n) and the 0-based pivots come back into the reference's
// DenseMatrix / std::vector. The operator of cqrrpt_core is regenerated on
// the device from (family, d, m, nnz, seed) -- bit-identical for SASO and
// SRFT -- after checking that the caller's materialisation is that seeded
// draw (all of it for SASO; spot entries for Gaussian / SRFT).
// validate_output runs the validate() contract (qrcp.cc:150-196) on the
// device with the reference's tolerance (cqrrpt.cc:309-312).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <thread>
#include <string>
#include <vector>

#include "cqrrpt/cqrrpt.hh"
#include "cqrrpt/rng.hh"
#include "cqrrpt/sketch.hh"
#include "cqrrpt_gpu.h"

namespace cqrrpt {
namespace {

constexpr double kU = 1.1102230246251565e-16;  // unit_roundoff, cqrrpt.hh:14

[[noreturn]] void raise(int rc, const char *what) {
    std::string msg = std::string(what) + ": " + cqrrpt_gpu_last_error();
    if (rc < 0) throw std::invalid_argument(msg);
    if (rc == CQRRPT_GPU_ERR_SINGULAR) throw std::domain_error(msg);
    throw std::runtime_error(msg);
}

void check_config_(const CqrrptConfig &cfg) {  // cqrrpt.cc:38-42
    if (cfg.gamma < 1.0) throw std::invalid_argument("cqrrpt: gamma must be >= 1");
    if (!(cfg.eps_tol > kU)) throw std::invalid_argument("cqrrpt: eps_tol must exceed the unit roundoff");
}

int32_t family_code(SketchFamily f) {
    switch (f) {
        case SketchFamily::gaussian: return CQRRPT_SKETCH_GAUSSIAN;
        case SketchFamily::saso: return CQRRPT_SKETCH_SASO;
        case SketchFamily::srft: return CQRRPT_SKETCH_SRFT;
    }
    throw std::logic_error("cqrrpt: unknown sketch family");
}

// Page-lock a host range for the duration of a call (large buffers only:
// registration costs ~ms, pageable copies cost ~3x the PCIe time).
struct Pinned {
    void *p = nullptr;
    Pinned(const void *ptr, size_t bytes, bool read_only) {
        if (!ptr || bytes < (size_t(64) << 20)) return;
        unsigned flags = cudaHostRegisterPortable | (read_only ? cudaHostRegisterReadOnly : 0u);
        if (cudaHostRegister(const_cast<void *>(ptr), bytes, flags) == cudaSuccess) p = const_cast<void *>(ptr);
        else cudaGetLastError();  // already registered / not supported: pageable copies
    }
    ~Pinned() {
        if (p) cudaHostUnregister(p);
    }
};

// Host transfer staging for the drop-in (CQRRPT_DROPIN_HOST = staged |
// register | pageable; default staged): the caller's M and the returned Q
// are ordinary pageable std::vector storage. "staged" keeps a grow-only
// pinned buffer per process and copies M into it / Q out of it with all host
// threads (page-locking the caller's buffers on every call costs more than
// the copies); "register" page-locks the caller's buffers for the call;
// "pageable" hands them to the copy engine as they are.
struct Staging {
    std::mutex mu;
    void *p = nullptr;
    size_t bytes = 0;
    void *get(size_t want) {
        if (want <= bytes) return p;
        if (p) cudaFreeHost(p);
        p = nullptr;
        bytes = 0;
        if (cudaHostAlloc(&p, want, cudaHostAllocPortable) != cudaSuccess) {
            cudaGetLastError();
            p = nullptr;
            return nullptr;
        }
        bytes = want;
        return p;
    }
};
Staging &staging() {
    static Staging s;
    return s;
}
void par_copy(void *dst, const void *src, size_t bytes) {
    const size_t nt = std::max<size_t>(1, std::min<size_t>(std::thread::hardware_concurrency(), bytes >> 24));
    std::vector<std::thread> th;
    const size_t per = (bytes + nt - 1) / nt;
    for (size_t t = 0; t < nt; ++t) {
        const size_t b0 = t * per, b1 = std::min(bytes, b0 + per);
        if (b0 < b1)
            th.emplace_back([=] { std::memcpy(static_cast<char *>(dst) + b0, static_cast<const char *>(src) + b0, b1 - b0); });
    }
    for (auto &x : th) x.join();
}
int host_mode() {
    const char *e = std::getenv("CQRRPT_DROPIN_HOST");
    if (e && std::string(e) == "register") return 1;
    if (e && std::string(e) == "pageable") return 2;
    return 0;
}

struct DevBuf {
    void *p = nullptr;
    explicit DevBuf(size_t bytes) {
        if (bytes && cudaMalloc(&p, bytes) != cudaSuccess) {
            cudaGetLastError();
            throw std::runtime_error("cqrrpt: cudaMalloc failed");
        }
    }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
};

// The caller's operator must be the seeded draw the device regenerates.
void check_operator(const SketchOperator &s) {
    if (s.family == SketchFamily::saso) {
        if (s.nnz_per_col < 1 || s.nnz_per_col > s.d)
            throw std::invalid_argument("sample_sketch: SASO needs 1 <= nnz_per_col <= d");
        const size_t cnt = size_t(s.m * s.nnz_per_col);
        if (s.saso_rows.size() != cnt || s.saso_vals.size() != cnt)
            throw std::invalid_argument("cqrrpt_core: SASO operator without its materialisation");
        DevBuf plan(sizeof(uint32_t) * cnt);
        int rc = cqrrpt_gpu_saso_plan(s.d, 0, s.m, s.nnz_per_col, s.seed, static_cast<uint32_t *>(plan.p), nullptr);
        if (rc) raise(rc, "cqrrpt_core: saso_plan");
        std::vector<uint32_t> h(cnt);
        if (cudaMemcpy(h.data(), plan.p, sizeof(uint32_t) * cnt, cudaMemcpyDeviceToHost) != cudaSuccess)
            throw std::runtime_error("cqrrpt_core: plan copy failed");
        const double val = 1.0 / std::sqrt(static_cast<double>(s.d));  // sketch.cc:79
        for (size_t e = 0; e < cnt; ++e) {
            const bool pos = (h[e] >> 31) != 0;
            if (int64_t(h[e] & 0x7fffffffu) != s.saso_rows[e] || s.saso_vals[e] != (pos ? val : -val))
                throw std::invalid_argument("cqrrpt_core: SASO operator is not sample_sketch(saso, d, m, nnz, seed)");
        }
    } else if (s.family == SketchFamily::gaussian) {
        // sketch.cc:62-72: S(i, j) = normal(j d + i) / sqrt(d) on mix_seed(seed, "gauss")
        if (s.dense.rows() != s.d || s.dense.cols() != s.m)
            throw std::invalid_argument("cqrrpt_core: Gaussian operator without its materialisation");
        CounterRng rng(mix_seed(s.seed, 0x6761757373ULL));  // kGaussianSalt (sketch.cc:18)
        const double scale = 1.0 / std::sqrt(static_cast<double>(s.d));
        const int64_t cols[3] = {0, s.m / 2, s.m - 1};
        for (int64_t j : cols)
            for (int64_t i : {int64_t(0), s.d - 1})
                if (s.dense(i, j) != rng.normal(static_cast<uint64_t>(j * s.d + i)) * scale)
                    throw std::invalid_argument("cqrrpt_core: Gaussian operator is not sample_sketch(gaussian, d, m, seed)");
    } else {
        int64_t padded = 1;
        while (padded < s.m) padded <<= 1;
        if (s.srft_padded != padded || int64_t(s.srft_rows.size()) != s.d || int64_t(s.srft_signs.size()) != s.m)
            throw std::invalid_argument("cqrrpt_core: SRFT operator without its materialisation");
        CounterRng sign_rng(mix_seed(s.seed, 0x7369676eULL));  // kSrftSignSalt (sketch.cc:20)
        CounterRng sel_rng(mix_seed(s.seed, 0x73656c65ULL));   // kSrftSelectSalt (sketch.cc:21)
        for (int64_t i : {int64_t(0), s.m / 2, s.m - 1})
            if (s.srft_signs[size_t(i)] != ((sign_rng.bits(static_cast<uint64_t>(i)) & 1) ? 1.0 : -1.0))
                throw std::invalid_argument("cqrrpt_core: SRFT operator is not sample_sketch(srft, d, m, seed)");
        if (s.srft_rows[0] != static_cast<int64_t>(sel_rng.below(0, static_cast<uint64_t>(padded))))
            throw std::invalid_argument("cqrrpt_core: SRFT operator is not sample_sketch(srft, d, m, seed)");
    }
}

// validate() (qrcp.cc:150-196) of the result against m on the device
ValidationReport validate_on_device(const PivotedQR &dec, const DenseMatrix &m, double tol) {
    ValidationReport v;
    const int64_t rows = m.rows(), n = m.cols(), k = dec.rank;
    std::vector<char> seen(size_t(n), 0);
    v.pivots_valid = int64_t(dec.pivots.size()) == n;
    for (int64_t p : dec.pivots) {
        if (!v.pivots_valid) break;
        if (p < 0 || p >= n || seen[size_t(p)]) v.pivots_valid = false;
        else seen[size_t(p)] = 1;
    }
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = j + 1; i < k; ++i) v.max_below_diag = std::max(v.max_below_diag, std::abs(dec.r(i, j)));
    v.diag_nonincreasing = true;
    for (int64_t i = 1; i < std::min(k, n); ++i)
        if (std::abs(dec.r(i, i)) > std::abs(dec.r(i - 1, i - 1))) v.diag_nonincreasing = false;
    if (v.pivots_valid) {
        DevBuf a(sizeof(double) * size_t(rows * n)), q(sizeof(double) * size_t(rows * std::max<int64_t>(k, 1))),
            r(sizeof(double) * size_t(std::max<int64_t>(k, 1) * n)), j(sizeof(int64_t) * size_t(n));
        cudaMemcpy(a.p, m.data(), sizeof(double) * size_t(rows * n), cudaMemcpyHostToDevice);
        if (k > 0) {
            cudaMemcpy(q.p, dec.q.data(), sizeof(double) * size_t(rows * k), cudaMemcpyHostToDevice);
            cudaMemcpy(r.p, dec.r.data(), sizeof(double) * size_t(k * n), cudaMemcpyHostToDevice);
        }
        cudaMemcpy(j.p, dec.pivots.data(), sizeof(int64_t) * size_t(n), cudaMemcpyHostToDevice);
        double orth_fro = 0.0;
        int rc = cqrrpt_gpu_validate(rows, n, k, static_cast<double *>(a.p), rows, static_cast<double *>(q.p), rows,
                                     static_cast<double *>(r.p), std::max<int64_t>(k, 1), static_cast<int64_t *>(j.p),
                                     &orth_fro, &v.orth_loss, &v.recon_rel, nullptr);
        if (rc) raise(rc, "validate");
    } else {
        v.recon_rel = INFINITY;
    }
    v.pass = v.pivots_valid && v.max_below_diag == 0.0 && v.orth_loss <= tol && v.recon_rel <= tol;
    return v;
}

CqrrptOutput run(const DenseMatrix &m, const CqrrptConfig &cfg, int32_t family, int64_t d, int64_t nnz,
                 uint64_t seed) {
    if (cfg.measure_distortion)
        throw std::invalid_argument("cqrrpt: measure_distortion (a desk-scale SVD diagnostic) is not offered "
                                    "by the GPU drop-in");
    const int64_t rows = m.rows(), n = m.cols();
    CqrrptOutput out;
    cqrrpt_gpu_ctx ctx;
    cqrrpt_gpu_ctx_init(&ctx);
    ctx.cond_method = int32_t(cfg.cond_method);
    ctx.sketch_family = family;
    ctx.sketch_rows = d;
    // cond_m_pre and truncation_ratio as the reference reports them; the
    // default fast-accept stage 2 is exact, so no forced search
    ctx.flags = CQRRPT_GPU_TIMINGS | CQRRPT_GPU_DIAGNOSTICS | (cfg.stage1_enabled ? 0 : CQRRPT_GPU_NO_STAGE1);
    std::vector<double> r(size_t(n * n), 0.0);
    std::vector<int64_t> piv(size_t(n), 0);
    int64_t k = 0, k0 = 0;
    PivotedQR &f = out.factorization;
    const size_t abytes = sizeof(double) * m.size();
    const int mode = host_mode();
    Staging &stg = staging();
    std::unique_lock<std::mutex> lock(stg.mu, std::defer_lock);
    double *pin = nullptr;
    if (mode == 0) {
        lock.lock();
        pin = static_cast<double *>(stg.get(2 * abytes));  // [A | Q]
    }
    if (pin) {
        par_copy(pin, m.data(), abytes);
        double *qpin = pin + m.size();
        int rc = cqrrpt_gpu_dgeqpt_host(rows, n, pin, std::max<int64_t>(rows, 1), cfg.gamma, nnz, seed, cfg.eps_tol,
                                        qpin, std::max<int64_t>(rows, 1), r.data(), n, piv.data(), &k, &k0, &ctx);
        if (rc) raise(rc, "cqrrpt");
        f.q = DenseMatrix(rows, k);
        par_copy(f.q.data(), qpin, sizeof(double) * size_t(rows * k));
    } else {
        DenseMatrix q(rows, n);  // room for k0 columns; trimmed to k below
        {
            Pinned pa(mode == 1 ? m.data() : nullptr, mode == 1 ? abytes : 0, true),
                pq(mode == 1 ? q.data() : nullptr, mode == 1 ? sizeof(double) * q.size() : 0, false);
            int rc = cqrrpt_gpu_dgeqpt_host(rows, n, m.data(), std::max<int64_t>(rows, 1), cfg.gamma, nnz, seed,
                                            cfg.eps_tol, q.data(), std::max<int64_t>(rows, 1), r.data(), n,
                                            piv.data(), &k, &k0, &ctx);
            if (rc) raise(rc, "cqrrpt");
        }
        f.q = (k == n) ? std::move(q) : q.leading_columns(k);
    }
    out.k0 = k0;
    out.k = k;
    f.rank = k;
    f.pivots = std::move(piv);
    f.r = DenseMatrix(k, n);
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < k; ++i) f.r(i, j) = r[size_t(j * n + i)];
    CqrrptDiagnostics &dg = out.diagnostics;
    dg.cond_m_pre = ctx.cond_m_pre;
    dg.truncation_ratio = ctx.truncation_ratio;
    dg.flop_estimate = ctx.flop_estimate;
    dg.timings = PhaseTimings{ctx.timings_ms[0] * 1e-3, ctx.timings_ms[1] * 1e-3, ctx.timings_ms[2] * 1e-3,
                              ctx.timings_ms[3] * 1e-3, ctx.timings_ms[4] * 1e-3, ctx.timings_ms[5] * 1e-3,
                              ctx.timings_ms[6] * 1e-3};
    if (cfg.validate_output) {  // cqrrpt.cc:309-312
        const double tol = std::max(100.0 * static_cast<double>(n) * kU, 10.0 * cfg.eps_tol);
        dg.validation = validate_on_device(f, m, tol);
    }
    return out;
}

}  // namespace

CqrrptOutput cqrrpt_core(const DenseMatrix &m, const SketchOperator &s, const CqrrptConfig &cfg) {
    check_config_(cfg);
    if (s.m != m.rows()) throw std::invalid_argument("cqrrpt_core: operator domain does not match matrix rows");
    if (m.cols() == 0) {
        CqrrptOutput out;
        out.factorization.q = DenseMatrix(m.rows(), 0);
        out.factorization.r = DenseMatrix(0, 0);
        return out;
    }
    check_operator(s);
    return run(m, cfg, family_code(s.family), s.d, s.family == SketchFamily::saso ? s.nnz_per_col : 1, s.seed);
}

CqrrptOutput cqrrpt(const DenseMatrix &m, const CqrrptConfig &cfg) {
    check_config_(cfg);
    if (m.cols() == 0) {  // cqrrpt.cc:319-324
        CqrrptOutput out;
        out.factorization.q = DenseMatrix(m.rows(), 0);
        out.factorization.r = DenseMatrix(0, 0);
        return out;
    }
    if (cfg.family == SketchFamily::saso && cfg.nnz_per_col < 1)
        throw std::invalid_argument("sample_sketch: SASO needs 1 <= nnz_per_col <= d");
    return run(m, cfg, family_code(cfg.family), 0, cfg.family == SketchFamily::saso ? cfg.nnz_per_col : 1, cfg.seed);
}

}  // namespace cqrrpt

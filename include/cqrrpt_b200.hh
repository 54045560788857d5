// cqrrpt_b200.hh — C++ adapter with the reference's own signature.
//
//   namespace cqrrpt_b200 {
//     CqrrptOutput cqrrpt(const DenseMatrix &m, const CqrrptConfig &cfg = {});
//   }
//
// mirrors cqrrpt::cqrrpt (/root/reference/proj/include/cqrrpt/cqrrpt.hh:140)
// and its types (dense_matrix.hh:15-89, qrcp.hh:19-60, cqrrpt.hh:61-129): same
// member names, same meaning, same exceptions (std::invalid_argument for bad
// configurations, std::domain_error for a singular preconditioner). A
// reference caller switches with `namespace cqrrpt = cqrrpt_b200;`.
//
// Host data in, host data out (like the reference): the adapter runs the host
// entry point cqrrpt_gpu_dgeqpt_host (include/cqrrpt_gpu.h) on sm_100a, which
// uploads M, factors it and streams Q (m x k), R (k x n) and the pivots back.
// Header-only; link libcqrrpt_gpu.so and the CUDA runtime.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "cqrrpt_gpu.h"

namespace cqrrpt_b200 {

inline constexpr double unit_roundoff = 1.1102230246251565e-16;  // cqrrpt.hh:14

// Column-major dense matrix (dense_matrix.hh:15-89, the subset callers use).
class DenseMatrix {
public:
    DenseMatrix() : rows_(0), cols_(0) {}
    DenseMatrix(int64_t rows, int64_t cols) : rows_(rows), cols_(cols), data_(size_t(rows * cols), 0.0) {
        if (rows < 0 || cols < 0) throw std::invalid_argument("DenseMatrix: negative dimension");
    }
    static DenseMatrix identity(int64_t n) {
        DenseMatrix m(n, n);
        for (int64_t i = 0; i < n; ++i) m(i, i) = 1.0;
        return m;
    }
    int64_t rows() const { return rows_; }
    int64_t cols() const { return cols_; }
    bool empty() const { return rows_ == 0 || cols_ == 0; }
    double &operator()(int64_t i, int64_t j) { return data_[size_t(j * rows_ + i)]; }
    double operator()(int64_t i, int64_t j) const { return data_[size_t(j * rows_ + i)]; }
    std::span<double> col(int64_t j) { return {data_.data() + j * rows_, size_t(rows_)}; }
    std::span<const double> col(int64_t j) const { return {data_.data() + j * rows_, size_t(rows_)}; }
    double *data() { return data_.data(); }
    const double *data() const { return data_.data(); }
    size_t size() const { return data_.size(); }
    bool operator==(const DenseMatrix &o) const { return rows_ == o.rows_ && cols_ == o.cols_ && data_ == o.data_; }

private:
    int64_t rows_, cols_;
    std::vector<double> data_;
};

enum class SketchFamily { gaussian, saso, srft };                         // sketch.hh:24
enum class CondMethod { diag_ratio, krylov_bounds, identity_deviation };  // cqrrpt.hh:61

struct CqrrptConfig {  // cqrrpt.hh:92-102
    double gamma = 1.25;
    SketchFamily family = SketchFamily::saso;
    int64_t nnz_per_col = 4;
    double eps_tol = 1e-4;
    CondMethod cond_method = CondMethod::identity_deviation;
    bool stage1_enabled = true;
    uint64_t seed = 0;
    bool measure_distortion = false;
    bool validate_output = true;
};

struct PhaseTimings {  // cqrrpt.hh:104-112 (seconds; CUDA events on the stream)
    double sketch = 0.0, qrcp = 0.0, rank_select = 0.0, precondition = 0.0, cholesky_qr = 0.0, undo = 0.0,
           total = 0.0;
};

struct ValidationReport {  // qrcp.hh:53-60 (+ Frobenius orthogonality)
    double orth_loss = 0.0, orth_loss_fro = 0.0, recon_rel = 0.0, max_below_diag = 0.0;
    bool pivots_valid = false, diag_nonincreasing = false, pass = false;
};

struct CqrrptDiagnostics {  // cqrrpt.hh:114-122
    std::optional<double> distortion, effective_distortion;
    double cond_m_pre = 1.0;
    double truncation_ratio = 0.0;
    double flop_estimate = 0.0;
    PhaseTimings timings;
    std::optional<ValidationReport> validation;
};

struct PivotedQR {  // qrcp.hh:19-24
    DenseMatrix q, r;
    std::vector<int64_t> pivots;
    int64_t rank = 0;
};

struct CqrrptOutput {  // cqrrpt.hh:124-129
    PivotedQR factorization;
    int64_t k0 = 0;
    int64_t k = 0;
    CqrrptDiagnostics diagnostics;
};

inline int64_t sketch_rows_for(double gamma, int64_t n) { return cqrrpt_gpu_sketch_rows(gamma, n); }

inline double flop_model(int64_t m, int64_t n, int64_t k, int64_t d, double c_sk) {
    double v = cqrrpt_gpu_flop_model(m, n, k, d, c_sk);
    if (v < 0) throw std::invalid_argument("flop_model: requires 0 <= k <= min(d, n)");
    return v;
}

namespace detail {
inline void throw_for(int rc, const char *what) {
    std::string msg = std::string(what) + ": " + cqrrpt_gpu_last_error();
    if (rc < 0) throw std::invalid_argument(msg);
    if (rc == CQRRPT_GPU_ERR_SINGULAR) throw std::domain_error(msg);
    throw std::runtime_error(msg);
}
struct DevBuf {
    void *p = nullptr;
    explicit DevBuf(size_t bytes) {
        if (bytes && cudaMalloc(&p, bytes) != cudaSuccess) throw std::runtime_error("cudaMalloc failed");
    }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
};
// page-lock a large host range for the duration of a call
struct Pinned {
    void *p = nullptr;
    Pinned(const void *ptr, size_t bytes, bool read_only) {
        if (bytes < (size_t(64) << 20)) return;
        unsigned flags = cudaHostRegisterPortable | (read_only ? cudaHostRegisterReadOnly : 0u);
        if (cudaHostRegister(const_cast<void *>(ptr), bytes, flags) == cudaSuccess) p = const_cast<void *>(ptr);
        else cudaGetLastError();
    }
    ~Pinned() {
        if (p) cudaHostUnregister(p);
    }
};
}  // namespace detail

// Drop-in for cqrrpt::cqrrpt (cqrrpt.cc:317-328) through the host entry point
// cqrrpt_gpu_dgeqpt_host: M's pages are registered for full-bandwidth DMA
// when large, A arrives in row chunks the exact sketch follows, Q streams back
// block by block while the device still computes. validate_output is
// evaluated on the device (cqrrpt_gpu_validate) with the reference's
// tolerance. (The reference's own headers + types: paper_2311_08316_b200/
// dropin/cqrrpt_dropin.cc defines cqrrpt::cqrrpt / cqrrpt_core themselves.)
inline CqrrptOutput cqrrpt(const DenseMatrix &m, const CqrrptConfig &cfg = {}) {
    if (cfg.gamma < 1.0) throw std::invalid_argument("cqrrpt: gamma must be >= 1");
    if (!(cfg.eps_tol > unit_roundoff)) throw std::invalid_argument("cqrrpt: eps_tol must exceed the unit roundoff");
    CqrrptOutput out;
    const int64_t rows = m.rows(), n = m.cols();
    if (n == 0) {
        out.factorization.q = DenseMatrix(rows, 0);
        out.factorization.r = DenseMatrix(0, 0);
        return out;
    }
    cqrrpt_gpu_ctx ctx;
    cqrrpt_gpu_ctx_init(&ctx);
    ctx.cond_method = int32_t(cfg.cond_method);
    ctx.sketch_family = cfg.family == SketchFamily::gaussian ? CQRRPT_SKETCH_GAUSSIAN
                        : cfg.family == SketchFamily::srft  ? CQRRPT_SKETCH_SRFT
                                                            : CQRRPT_SKETCH_SASO;
    // the default fast-accept stage 2 is exact; DIAGNOSTICS fills cond_m_pre
    ctx.flags = CQRRPT_GPU_TIMINGS | CQRRPT_GPU_DIAGNOSTICS | (cfg.stage1_enabled ? 0 : CQRRPT_GPU_NO_STAGE1);
    DenseMatrix q(rows, n);  // room for k0 columns
    std::vector<double> r(size_t(n * n), 0.0);
    std::vector<int64_t> piv(size_t(n), 0);
    int64_t k = 0, k0 = 0;
    {
        detail::Pinned pa(m.data(), sizeof(double) * m.size(), true), pq(q.data(), sizeof(double) * q.size(), false);
        int rc = cqrrpt_gpu_dgeqpt_host(rows, n, m.data(), std::max<int64_t>(rows, 1), cfg.gamma, cfg.nnz_per_col,
                                        cfg.seed, cfg.eps_tol, q.data(), std::max<int64_t>(rows, 1), r.data(), n,
                                        piv.data(), &k, &k0, &ctx);
        if (rc) detail::throw_for(rc, "cqrrpt");
    }
    out.k = k;
    out.k0 = k0;
    PivotedQR &f = out.factorization;
    f.rank = k;
    f.pivots = std::move(piv);
    if (k == n) {
        f.q = std::move(q);
    } else {
        f.q = DenseMatrix(rows, k);
        std::memcpy(f.q.data(), q.data(), sizeof(double) * size_t(rows * k));
    }
    f.r = DenseMatrix(k, n);
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < k; ++i) f.r(i, j) = r[size_t(j * n + i)];
    auto &d = out.diagnostics;
    d.cond_m_pre = ctx.cond_m_pre;
    d.truncation_ratio = ctx.truncation_ratio;
    d.flop_estimate = ctx.flop_estimate;
    d.timings = PhaseTimings{ctx.timings_ms[0] * 1e-3, ctx.timings_ms[1] * 1e-3, ctx.timings_ms[2] * 1e-3,
                             ctx.timings_ms[3] * 1e-3, ctx.timings_ms[4] * 1e-3, ctx.timings_ms[5] * 1e-3,
                             ctx.timings_ms[6] * 1e-3};
    if (cfg.validate_output) {  // qrcp.cc:150-196 with tol = max(100 n u, 10 eps_tol) (cqrrpt.cc:310)
        ValidationReport v;
        const double tol = std::max(100.0 * double(n) * unit_roundoff, 10.0 * cfg.eps_tol);
        std::vector<char> seen(size_t(n), 0);
        v.pivots_valid = true;
        for (int64_t p : f.pivots) {
            if (p < 0 || p >= n || seen[size_t(p)]) {
                v.pivots_valid = false;
                break;
            }
            seen[size_t(p)] = 1;
        }
        for (int64_t jj = 0; jj < n; ++jj)
            for (int64_t ii = jj + 1; ii < k; ++ii) v.max_below_diag = std::max(v.max_below_diag, std::abs(f.r(ii, jj)));
        v.diag_nonincreasing = true;
        for (int64_t ii = 1; ii < std::min(k, n); ++ii)
            if (std::abs(f.r(ii, ii)) > std::abs(f.r(ii - 1, ii - 1))) v.diag_nonincreasing = false;
        if (v.pivots_valid) {
            const size_t abytes = sizeof(double) * size_t(rows * n);
            detail::DevBuf a(abytes), qd(sizeof(double) * size_t(rows * std::max<int64_t>(k, 1))),
                rd(sizeof(double) * size_t(std::max<int64_t>(k, 1) * n)), jd(sizeof(int64_t) * size_t(n));
            cudaMemcpy(a.p, m.data(), abytes, cudaMemcpyHostToDevice);
            if (k > 0) {
                cudaMemcpy(qd.p, f.q.data(), sizeof(double) * size_t(rows * k), cudaMemcpyHostToDevice);
                cudaMemcpy(rd.p, f.r.data(), sizeof(double) * size_t(k * n), cudaMemcpyHostToDevice);
            }
            cudaMemcpy(jd.p, f.pivots.data(), sizeof(int64_t) * size_t(n), cudaMemcpyHostToDevice);
            int rc = cqrrpt_gpu_validate(rows, n, k, static_cast<double *>(a.p), rows, static_cast<double *>(qd.p), rows,
                                         static_cast<double *>(rd.p), std::max<int64_t>(k, 1),
                                         static_cast<int64_t *>(jd.p), &v.orth_loss_fro, &v.orth_loss, &v.recon_rel,
                                         nullptr);
            if (rc) detail::throw_for(rc, "validate");
        } else {
            v.recon_rel = INFINITY;
        }
        v.pass = v.pivots_valid && v.max_below_diag == 0.0 && v.orth_loss <= tol && v.recon_rel <= tol;
        d.validation = v;
    }
    return out;
}

}  // namespace cqrrpt_b200

// K7: stage-2 condition estimators on device.
//
// Reference: cond_estimate (cqrrpt.cc:114-147), NestedCondEstimator
// (cqrrpt.cc:47-71), power_iterate (linalg.cc:446-465) with the deterministic
// start vector CounterRng(0x5eedcafe01234567).normal(i) normalised
// (linalg.cc:434-442), cap 200 iterations, stop at |est-prev| <= 1e-10 est.
//
// The full estimator runs as ONE single-CTA kernel per estimate (all 200
// iterations inside the kernel; a launch per matvec would cost more than the
// matvec). The inverse-norm estimate uses the explicit inverse of R (the
// leading block of R^{-1} is the inverse of the leading block of R), so both
// matvecs are GEMVs instead of triangular solves.
#include <vector>

#include "common.cuh"
#include "internal.hh"

namespace cqg {

constexpr int kPowThreads = 1024;

struct PowOp {
    const double *a;
    int64_t ld, rows, cols;
    int kind;  // 0 dense, 1 upper triangular, 2 upper triangular minus identity
};

CQ_DEVI double op_entry(const PowOp &op, int64_t i, int64_t j) {
    double v = op.a[j * op.ld + i];
    if (op.kind == 2 && i == j) v -= 1.0;
    return v;
}

// deterministic_unit_vector(n) (linalg.cc:434-442) uses normal_dev (common.cuh)
__device__ void start_vector(int64_t n, double *v, double *scratch) {
    double s = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        double x = normal_dev(0x5eedcafe01234567ULL, (uint64_t)i);
        v[i] = x;
        s = fma(x, x, s);
    }
    double nrm = sqrt(block_sum(s, scratch));
    __syncthreads();
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) v[i] = (nrm == 0.0) ? (i == 0 ? 1.0 : 0.0) : v[i] / nrm;
    __syncthreads();
}

// y = op x (rows), threads over rows, j ascending (the reference's axpy order)
__device__ void op_forward(const PowOp &op, const double *x, double *y) {
    for (int64_t i = threadIdx.x; i < op.rows; i += blockDim.x) {
        double s = 0.0;
        const int64_t jb = (op.kind == 0) ? 0 : i;
        for (int64_t j = jb; j < op.cols; ++j) s = fma(x[j], op_entry(op, i, j), s);
        y[i] = s;
    }
    __syncthreads();
}

// z = op^T y (cols), warp per column
__device__ void op_adjoint(const PowOp &op, const double *y, double *z) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int64_t j = wid; j < op.cols; j += nw) {
        const int64_t ie = (op.kind == 0) ? op.rows : j + 1;
        double s = 0.0;
        for (int64_t i = lane; i < ie; i += 32) s = fma(op_entry(op, i, j), y[i], s);
        s = warp_sum(s);
        if (lane == 0) z[j] = s;
    }
    __syncthreads();
}

// returns est (and converged flag) of sigma_max(op) by the reference's power iteration
__device__ double power_iterate_dev(const PowOp &op, double *v, double *w, double *z, double *scratch, int *conv) {
    start_vector(op.cols, v, scratch);
    double est = 0.0, prev = -1.0;
    for (int it = 0; it < 200; ++it) {
        op_forward(op, v, w);
        double s = 0.0;
        for (int64_t i = threadIdx.x; i < op.rows; i += blockDim.x) s = fma(w[i], w[i], s);
        double nw = sqrt(block_sum(s, scratch));
        if (nw == 0.0) {
            *conv = 1;
            return 0.0;
        }
        est = (est < nw) ? nw : est;
        if (prev >= 0.0 && fabs(est - prev) <= 1e-10 * est) {
            *conv = 1;
            return est;
        }
        prev = est;
        op_adjoint(op, w, z);
        s = 0.0;
        for (int64_t i = threadIdx.x; i < op.cols; i += blockDim.x) s = fma(z[i], z[i], s);
        double nz = sqrt(block_sum(s, scratch));
        if (nz == 0.0) {
            *conv = 1;
            return est;
        }
        __syncthreads();
        for (int64_t i = threadIdx.x; i < op.cols; i += blockDim.x) v[i] = z[i] / nz;
        __syncthreads();
    }
    *conv = 0;
    return est;
}

// method: 0 diag_ratio, 1 krylov_bounds, 2 identity_deviation (+inf when
// tau >= 1), 3 identity_deviation with NestedCondEstimator's fallback to
// krylov_bounds when it is +inf (cqrrpt.cc:57-58).
__global__ void __launch_bounds__(kPowThreads) cond_estimate_kernel(int64_t ell, const double *__restrict__ r,
                                                                    int64_t ldr, const double *__restrict__ rinv,
                                                                    int64_t ldi, int method, double *work,
                                                                    double *out) {
    __shared__ double scratch[32];
    double *v = work, *w = work + ell, *z = work + 2 * ell;
    int conv = 1;
    double value = 1.0;
    if (ell <= 0) {
        if (threadIdx.x == 0) out[0] = 1.0;
        return;
    }
    if (method == 0) {
        double hi = 0.0, lo = INFINITY;
        for (int64_t i = threadIdx.x; i < ell; i += blockDim.x) {
            double d = fabs(r[i * ldr + i]);
            hi = fmax(hi, d);
            lo = fmin(lo, d);
        }
        hi = warp_max(hi);
        lo = -warp_max(-lo);
        __shared__ double sh[32], sl[32];
        if ((threadIdx.x & 31) == 0) {
            sh[threadIdx.x >> 5] = hi;
            sl[threadIdx.x >> 5] = lo;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int q = 0; q < (int)(blockDim.x >> 5); ++q) {
                hi = fmax(hi, sh[q]);
                lo = fmin(lo, sl[q]);
            }
            double vv = (lo == 0.0) ? INFINITY : hi / lo;
            out[0] = vv < 1.0 ? 1.0 : vv;
            out[1] = 1.0;
        }
        return;
    }
    bool need_krylov = (method == 1);
    if (method == 2 || method == 3) {
        PowOp dev{r, ldr, ell, ell, 2};
        double tau = power_iterate_dev(dev, v, w, z, scratch, &conv) * (1.0 + 1e-6);
        if (tau >= 1.0) {
            if (method == 3) need_krylov = true;  // NestedCondEstimator fallback (cqrrpt.cc:57-58)
            else value = INFINITY;                // cond_estimate itself returns +inf (cqrrpt.cc:141-142)
        } else {
            double vv = (1.0 + tau) / (1.0 - tau);
            value = vv < 1.0 ? 1.0 : vv;
        }
    }
    if (need_krylov) {
        int c1 = 1, c2 = 1;
        PowOp fwd{r, ldr, ell, ell, 1};
        double hi = power_iterate_dev(fwd, v, w, z, scratch, &c1);
        double inv;
        bool zero_diag = false;
        for (int64_t i = 0; i < ell; ++i)
            if (r[i * ldr + i] == 0.0) zero_diag = true;
        if (zero_diag) {
            inv = INFINITY;  // linalg.cc:489-490
        } else {
            PowOp ri{rinv, ldi, ell, ell, 1};
            inv = power_iterate_dev(ri, v, w, z, scratch, &c2);
        }
        double vv = hi * (1.0 + 1e-6) * inv * (1.0 + 1e-6);
        value = vv < 1.0 ? 1.0 : vv;
        conv = c1 && c2;
    }
    if (threadIdx.x == 0) {
        out[0] = value;
        out[1] = conv;
    }
}

// First power iterate of identity_deviation for every binary-search probe:
// ||(R_ell - I) v0_ell|| with v0_ell = g[:ell] / ||g[:ell]|| (g the fixed
// normal sequence, linalg.cc:434-442). All probes share g, so one pass over R
// serves them all: row i walks j ascending and records its running sum
// S_i(ell) = sum_{i<=j<ell} R(i,j) g_j at each probe boundary.
// CTA = 32 rows x 8 column chunks; per-CTA partial sums, fixed-order final.
constexpr int kIdRows = 32, kIdChunks = 8, kIdMaxProbes = 64;

__global__ void idev_gvec_kernel(int64_t n, double *__restrict__ g) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        g[i] = normal_dev(0x5eedcafe01234567ULL, (uint64_t)i);
}

__global__ void __launch_bounds__(kIdRows *kIdChunks) idev_rows_kernel(const double *__restrict__ r, int64_t ldr,
                                                                        const int64_t *__restrict__ ells, int np,
                                                                        int64_t maxl, const double *__restrict__ g,
                                                                        double *__restrict__ part) {
    extern __shared__ double sp[];  // [np][kIdChunks][kIdRows]
    const int lane = threadIdx.x & 31, ch = threadIdx.x >> 5;
    const int64_t i = (int64_t)blockIdx.x * kIdRows + lane;
    const int64_t L = (maxl + kIdChunks - 1) / kIdChunks;
    const int64_t jb = cmax<int64_t>(i, ch * L), je = cmin<int64_t>(maxl, (ch + 1) * L);
    double s = 0.0;
    int p = 0;
    // probes ending at or before this chunk's first column get nothing from it
    while (p < np && ells[p] <= jb) sp[(p++ * kIdChunks + ch) * kIdRows + lane] = 0.0;
    int64_t next = p < np ? ells[p] : INT64_MAX;  // next probe boundary
    auto record = [&](int64_t jend) {
        while (next == jend) {
            sp[(p++ * kIdChunks + ch) * kIdRows + lane] = s;
            next = p < np ? ells[p] : INT64_MAX;
        }
    };
    if (i < maxl) {
        int64_t j = jb;
        for (; j + 8 <= je; j += 8) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = r[(j + u) * ldr + i];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                s = fma(v[u], g[j + u], s);
                record(j + u + 1);
            }
        }
        for (; j < je; ++j) {
            s = fma(r[j * ldr + i], g[j], s);
            record(j + 1);
        }
    }
    for (; p < np; ++p) sp[(p * kIdChunks + ch) * kIdRows + lane] = s;  // probes beyond the chunk
    __syncthreads();
    // (row, probe): S = sum of chunks in order, w = S - g_i for i < ell
    for (int q = ch; q < np; q += kIdChunks) {
        double w2 = 0.0;
        if (i < ells[q]) {
            double S = 0.0;
            for (int c = 0; c < kIdChunks; ++c) S += sp[(q * kIdChunks + c) * kIdRows + lane];
            const double w = S - g[i];
            w2 = w * w;
        }
        w2 = warp_sum(w2);
        if (lane == 0) part[(int64_t)q * gridDim.x + blockIdx.x] = w2;
    }
}

__global__ void __launch_bounds__(256) idev_final_kernel(const int64_t *__restrict__ ells, int np,
                                                         const double *__restrict__ g,
                                                         const double *__restrict__ part, int64_t nblk,
                                                         double *__restrict__ out) {
    __shared__ double scratch[32];
    for (int q = 0; q < np; ++q) {
        double s = 0.0;
        for (int64_t i = threadIdx.x; i < ells[q]; i += blockDim.x) s = fma(g[i], g[i], s);
        const double nrm2 = block_sum(s, scratch);
        __syncthreads();
        double t = 0.0;
        for (int64_t b = threadIdx.x; b < nblk; b += blockDim.x) t += part[q * nblk + b];
        const double w2 = block_sum(t, scratch);
        __syncthreads();
        if (threadIdx.x == 0) out[q] = (nrm2 == 0.0) ? 0.0 : sqrt(w2 / nrm2);
    }
}

__global__ void __launch_bounds__(kPowThreads) spectral_kernel(const double *__restrict__ a, int64_t lda, int64_t m,
                                                               int64_t n, double *work, double *out) {
    __shared__ double scratch[32];
    int conv = 1;
    PowOp op{a, lda, m, n, 0};
    double est = (m == 0 || n == 0) ? 0.0 : power_iterate_dev(op, work, work + n, work + n + m, scratch, &conv);
    if (threadIdx.x == 0) out[0] = est;
}

int identity_deviation_first(const double *r, int64_t ldr, const int64_t *ells, int nells, double *out_host,
                             Workspace &ws, cudaStream_t st) {
    if (nells <= 0) return 0;
    if (nells > kIdMaxProbes) return fail_internal("identity_deviation_first: too many probes");
    std::vector<int64_t> sorted(ells, ells + nells);
    for (int i = 1; i < nells; ++i)
        if (sorted[i] < sorted[i - 1]) return fail_internal("identity_deviation_first: probes must ascend");
    const int64_t maxl = sorted.back();
    const int64_t nblk = (maxl + kIdRows - 1) / kIdRows;
    int64_t *dl = ws.get<int64_t>("idev.ells", nells);
    double *g = ws.get<double>("idev.g", (size_t)maxl + 1);
    double *part = ws.get<double>("idev.part", (size_t)nells * nblk);
    double *dout = ws.get<double>("idev.out", nells);
    if (!dl || !g || !part || !dout) return fail_nomem("idev workspace");
    CQ_CUDA(cudaMemcpyAsync(dl, sorted.data(), sizeof(int64_t) * nells, cudaMemcpyHostToDevice, st), "ells h2d");
    idev_gvec_kernel<<<(unsigned)std::min<int64_t>((maxl + 255) / 256, 1024), 256, 0, st>>>(maxl, g);
    note_launch();
    const size_t smem = sizeof(double) * (size_t)nells * kIdChunks * kIdRows;
    if (first_on_device((const void *)idev_rows_kernel))
        CQ_CUDA(cudaFuncSetAttribute(idev_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)(sizeof(double) * kIdMaxProbes * kIdChunks * kIdRows)),
                "idev smem attr");
    idev_rows_kernel<<<(unsigned)nblk, kIdRows * kIdChunks, smem, st>>>(r, ldr, dl, nells, maxl, g, part);
    note_launch();
    idev_final_kernel<<<1, 256, 0, st>>>(dl, nells, g, part, nblk, dout);
    note_launch();
    CQ_TRY(check_launch("idev kernels"));
    CQ_CUDA(cudaMemcpyAsync(out_host, dout, sizeof(double) * nells, cudaMemcpyDeviceToHost, st), "idev d2h");
    CQ_CUDA(cudaStreamSynchronize(st), "idev sync");
    return 0;
}

// ---------------------------------------------------------------------------
// Grid-wide estimator (the exact stage-2 path): the same power iterations and
// control flow as cond_estimate_kernel, with each matvec spread over the grid
// (cooperative launch). y = op x: CTA rows in 32-row chunks (lane = row,
// warp = column residue mod 8, coalesced column segments); z = op^T y: warp
// per column. Vectors live in global memory and are staged in shared memory
// per half-iteration; norms are per-CTA partials summed in CTA order by every
// CTA, so all CTAs take the same branches and the result is deterministic.
// Three grid barriers per iteration.
// ---------------------------------------------------------------------------
constexpr int kGridPowThreads = 256;

struct GridPow {
    double *v, *w, *z;   // global vectors (length >= max(rows, cols))
    double *part;        // per-CTA partial sums [gridDim.x]
    unsigned long long *bar;
    unsigned long long nbar;
    double *s_vec;       // shared staging (>= max(rows, cols))
    double *s_red;       // shared [8][32] + 32
};

CQ_DEVI void gp_sync(GridPow &g) { grid_barrier_mono(g.bar, (++g.nbar) * (unsigned long long)gridDim.x); }

// sum over CTAs of the partials, in CTA order (identical in every CTA)
CQ_DEVI double gp_total(GridPow &g, double mine) {
    double *sr = g.s_red + 256;
    const double blk = block_sum(mine, sr);
    if (threadIdx.x == 0) g.part[blockIdx.x] = blk;
    gp_sync(g);
    double t = 0.0;
    if (threadIdx.x == 0) {
        for (int b = 0; b < (int)gridDim.x; ++b) t += ld_cg(g.part + b);
        sr[0] = t;
    }
    __syncthreads();
    t = sr[0];
    __syncthreads();
    return t;
}

// y[rows of this CTA] = op x (x = src, global), returns this thread's share of sum y^2
CQ_DEVI double gp_forward(const PowOp &op, const double *src, double *dst, GridPow &g) {
    for (int64_t j = threadIdx.x; j < op.cols; j += blockDim.x) g.s_vec[j] = ld_cg(src + j);
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t chunks = (op.rows + 31) / 32;
    double sq = 0.0;
    for (int64_t ch = blockIdx.x; ch < chunks; ch += gridDim.x) {
        const int64_t i = ch * 32 + lane;
        const int64_t jb = (op.kind == 0) ? 0 : ch * 32;  // upper: columns before the chunk are zero
        double acc = 0.0;
        if (i < op.rows)
            for (int64_t j = jb + wid; j < op.cols; j += 8)
                if (op.kind == 0 || j >= i) acc = fma(g.s_vec[j], op_entry(op, i, j), acc);
        g.s_red[wid * 32 + lane] = acc;
        __syncthreads();
        if (wid == 0) {
            double y = 0.0;
            for (int q = 0; q < 8; ++q) y += g.s_red[q * 32 + lane];
            if (i < op.rows) {
                dst[i] = y;
                sq = fma(y, y, sq);
            }
        }
        __syncthreads();
    }
    return sq;
}

// z[cols of this CTA] = op^T y (y = src, global), returns this thread's share of sum z^2
CQ_DEVI double gp_adjoint(const PowOp &op, const double *src, double *dst, GridPow &g) {
    for (int64_t i = threadIdx.x; i < op.rows; i += blockDim.x) g.s_vec[i] = ld_cg(src + i);
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    double sq = 0.0;
    for (int64_t j = blockIdx.x * (int64_t)nw + wid; j < op.cols; j += (int64_t)gridDim.x * nw) {
        const int64_t ie = (op.kind == 0) ? op.rows : j + 1;
        double s = 0.0;
        for (int64_t i = lane; i < ie; i += 32) s = fma(op_entry(op, i, j), g.s_vec[i], s);
        s = warp_sum(s);
        if (lane == 0) {
            dst[j] = s;
            sq = fma(s, s, sq);
        }
    }
    return sq;
}

// power_iterate (linalg.cc:446-465) over the grid; same control flow as power_iterate_dev
CQ_DEVI double gp_power(const PowOp &op, GridPow &g, int *conv) {
    const int64_t n = op.cols;
    // deterministic_unit_vector (linalg.cc:434-442)
    double sq = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double x = normal_dev(0x5eedcafe01234567ULL, (uint64_t)i);
        g.v[i] = x;
        sq = fma(x, x, sq);
    }
    const double nrm = sqrt(gp_total(g, sq));
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        g.v[i] = (nrm == 0.0) ? (i == 0 ? 1.0 : 0.0) : g.v[i] / nrm;
    gp_sync(g);
    double est = 0.0, prev = -1.0;
    for (int it = 0; it < 200; ++it) {
        const double nw = sqrt(gp_total(g, gp_forward(op, g.v, g.w, g)));
        if (nw == 0.0) {
            *conv = 1;
            return 0.0;
        }
        est = (est < nw) ? nw : est;
        if (prev >= 0.0 && fabs(est - prev) <= 1e-10 * est) {
            *conv = 1;
            return est;
        }
        prev = est;
        const double nz = sqrt(gp_total(g, gp_adjoint(op, g.w, g.z, g)));
        if (nz == 0.0) {
            *conv = 1;
            return est;
        }
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
             i += (int64_t)gridDim.x * blockDim.x)
            g.v[i] = ld_cg(g.z + i) / nz;
        gp_sync(g);
    }
    *conv = 0;
    return est;
}

struct CondGridArgs {
    int64_t ell, ldr, ldi;
    const double *r, *rinv;
    int method;
    double *v, *w, *z, *part;
    unsigned long long *bar;
    double *out;
};

// methods 1..3 of cond_estimate_kernel, grid-wide (method 0 stays single-CTA)
__global__ void __launch_bounds__(kGridPowThreads) cond_grid_kernel(CondGridArgs A) {
    extern __shared__ double gsm[];
    GridPow g{A.v, A.w, A.z, A.part, A.bar, 0, gsm + 8 * 32 + 64, gsm};
    const int64_t ell = A.ell;
    int conv = 1;
    double value = 1.0;
    bool need_krylov = (A.method == 1);
    if (A.method == 2 || A.method == 3) {
        PowOp dev{A.r, A.ldr, ell, ell, 2};
        const double tau = gp_power(dev, g, &conv) * (1.0 + 1e-6);
        if (tau >= 1.0) {
            if (A.method == 3) need_krylov = true;  // NestedCondEstimator fallback (cqrrpt.cc:57-58)
            else value = INFINITY;                  // cond_estimate returns +inf (cqrrpt.cc:141-142)
        } else {
            const double vv = (1.0 + tau) / (1.0 - tau);
            value = vv < 1.0 ? 1.0 : vv;
        }
    }
    if (need_krylov) {
        int c1 = 1, c2 = 1;
        PowOp fwd{A.r, A.ldr, ell, ell, 1};
        const double hi = gp_power(fwd, g, &c1);
        bool zero_diag = false;
        for (int64_t i = 0; i < ell; ++i)
            if (A.r[i * A.ldr + i] == 0.0) zero_diag = true;
        double inv;
        if (zero_diag) {
            inv = INFINITY;  // linalg.cc:489-490
        } else {
            PowOp ri{A.rinv, A.ldi, ell, ell, 1};
            inv = gp_power(ri, g, &c2);
        }
        const double vv = hi * (1.0 + 1e-6) * inv * (1.0 + 1e-6);
        value = vv < 1.0 ? 1.0 : vv;
        conv = c1 && c2;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        A.out[0] = value;
        A.out[1] = conv;
    }
}

int cond_estimate(int64_t ell, const double *r, int64_t ldr, const double *rinv, int64_t ldi, int method,
                  double *value_host, Workspace &ws, cudaStream_t st) {
    double *dout = ws.get<double>("cond.out", 2);
    if (method == 0 || ell < 256) {  // small blocks: one CTA runs every iteration
        double *work = ws.get<double>("cond.work", (size_t)(3 * std::max<int64_t>(ell, 1)));
        cond_estimate_kernel<<<1, kPowThreads, 0, st>>>(ell, r, ldr, rinv, ldi, method, work, dout);
        note_launch();
        CQ_TRY(check_launch("cond_estimate_kernel"));
    } else {
        const int sms = num_sms();
        const int G = (int)std::max<int64_t>(1, std::min<int64_t>(sms, (ell + 31) / 32));
        CondGridArgs a;
        a.ell = ell;
        a.ldr = ldr;
        a.ldi = ldi;
        a.r = r;
        a.rinv = rinv;
        a.method = method;
        a.v = ws.get<double>("condg.v", (size_t)ell);
        a.w = ws.get<double>("condg.w", (size_t)ell);
        a.z = ws.get<double>("condg.z", (size_t)ell);
        a.part = ws.get<double>("condg.part", (size_t)G);
        a.bar = ws.get<unsigned long long>("condg.bar", 1);
        a.out = dout;
        if (!a.v || !a.w || !a.z || !a.part || !a.bar) return fail_nomem("cond estimator");
        const size_t smem = sizeof(double) * (size_t)(8 * 32 + 64 + ell);
        if (first_on_device((const void *)cond_grid_kernel))
            CQ_CUDA(cudaFuncSetAttribute(cond_grid_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024),
                    "cond grid smem");
        if (smem > 200 * 1024) return fail_internal("cond estimator: block too large for shared memory");
        CQ_CUDA(cudaMemsetAsync(a.bar, 0, sizeof(unsigned long long), st), "cond bar");
        void *args[] = {&a};
        CQ_CUDA(cudaLaunchCooperativeKernel((void *)cond_grid_kernel, dim3(G), dim3(kGridPowThreads), args, smem, st),
                "cond grid launch");
        note_launch();
    }
    CQ_CUDA(cudaMemcpyAsync(value_host, dout, sizeof(double), cudaMemcpyDeviceToHost, st), "cond d2h");
    CQ_CUDA(cudaStreamSynchronize(st), "cond sync");
    return 0;
}

int spectral_norm_estimate(int64_t m, int64_t n, const double *a, int64_t lda, double *value_host, Workspace &ws,
                           cudaStream_t st) {
    double *work = ws.get<double>("spec.work", (size_t)(2 * n + m + 1));
    double *dout = ws.get<double>("spec.out", 1);
    spectral_kernel<<<1, kPowThreads, 0, st>>>(a, lda, m, n, work, dout);
    note_launch();
    CQ_TRY(check_launch("spectral_kernel"));
    CQ_CUDA(cudaMemcpyAsync(value_host, dout, sizeof(double), cudaMemcpyDeviceToHost, st), "spec d2h");
    CQ_CUDA(cudaStreamSynchronize(st), "spec sync");
    return 0;
}

}  // namespace cqg

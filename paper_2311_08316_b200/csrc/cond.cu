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
// Grouped estimator: several probes (leading blocks ell) at once, each on its
// own group of CTAs (cooperative launch of sum of group sizes). The same
// power iterations and control flow as cond_estimate_kernel, with each matvec
// spread over the group: y = op x over 32-row chunks (lane = row, warp =
// column residue mod 8, coalesced column segments), z = op^T y warp per
// column. Vectors live in global memory and are staged in shared memory per
// half-iteration; norms are per-CTA partials summed in CTA order by every
// CTA of the group, so the group's CTAs take the same branches and the result
// is deterministic. A probe's group size depends only on ell (group_size), so
// an estimate does not depend on which other probes share the launch: the
// binary search (one probe per launch) and the fast-accept diagnostics (all
// probes in one launch) report bitwise the same values.
// ---------------------------------------------------------------------------
constexpr int kGridPowThreads = 256;
constexpr int kMaxGroup = 16;

static int group_size(int64_t ell) { return (int)std::max<int64_t>(1, std::min<int64_t>(kMaxGroup, (ell + 127) / 128)); }

struct GridPow {
    double *v, *w, *z;   // group vectors (length >= max(rows, cols))
    double *part;        // per-CTA partial sums [group size]
    unsigned long long *bar;
    unsigned long long nbar;
    int gb, gn;          // this CTA's rank in its group, group size
    double *s_vec;       // shared staging (>= max(rows, cols))
    double *s_red;       // shared [8][32] + 32
};

CQ_DEVI void gp_sync(GridPow &g) { grid_barrier_mono(g.bar, (++g.nbar) * (unsigned long long)g.gn); }

// sum over the group's CTAs of the partials, in CTA order (identical in every CTA)
CQ_DEVI double gp_total(GridPow &g, double mine) {
    double *sr = g.s_red + 256;
    const double blk = block_sum(mine, sr);
    if (threadIdx.x == 0) g.part[g.gb] = blk;
    gp_sync(g);
    double t = 0.0;
    if (threadIdx.x == 0) {
        for (int b = 0; b < g.gn; ++b) t += ld_cg(g.part + b);
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
    for (int64_t ch = g.gb; ch < chunks; ch += g.gn) {
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
    for (int64_t j = g.gb * (int64_t)nw + wid; j < op.cols; j += (int64_t)g.gn * nw) {
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

// power_iterate (linalg.cc:446-465) over the group; same control flow as power_iterate_dev
CQ_DEVI double gp_power(const PowOp &op, GridPow &g, int *conv) {
    const int64_t n = op.cols;
    // deterministic_unit_vector (linalg.cc:434-442)
    double sq = 0.0;
    for (int64_t i = g.gb * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)g.gn * blockDim.x) {
        const double x = normal_dev(0x5eedcafe01234567ULL, (uint64_t)i);
        g.v[i] = x;
        sq = fma(x, x, sq);
    }
    const double nrm = sqrt(gp_total(g, sq));
    for (int64_t i = g.gb * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)g.gn * blockDim.x)
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
        for (int64_t i = g.gb * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)g.gn * blockDim.x)
            g.v[i] = ld_cg(g.z + i) / nz;
        gp_sync(g);
    }
    *conv = 0;
    return est;
}

struct CondGroupArgs {
    int nprobes;
    const int64_t *ells;      // [nprobes]
    const int *first_cta;     // [nprobes + 1]: CTAs [first_cta[p], first_cta[p+1]) run probe p
    int64_t ldr, ldi, vlen;   // vector stride per probe
    const double *r, *rinv;
    int method;
    double *vec;              // [nprobes][3][vlen]
    double *part;             // [total CTAs]
    unsigned long long *bar;  // [nprobes] (zeroed)
    double *out;              // [nprobes][2]
};

// methods 1..3 of cond_estimate_kernel, one probe per CTA group
__global__ void __launch_bounds__(kGridPowThreads) cond_group_kernel(CondGroupArgs A) {
    extern __shared__ double gsm[];
    int p = 0;
    while (p + 1 < A.nprobes && (int)blockIdx.x >= A.first_cta[p + 1]) ++p;
    const int gb = (int)blockIdx.x - A.first_cta[p], gn = A.first_cta[p + 1] - A.first_cta[p];
    double *vec = A.vec + (int64_t)p * 3 * A.vlen;
    GridPow g{vec, vec + A.vlen, vec + 2 * A.vlen, A.part + A.first_cta[p], A.bar + p, 0, gb, gn,
              gsm + 8 * 32 + 64, gsm};
    const int64_t ell = A.ells[p];
    int conv = 1;
    double value = 1.0;
    bool need_krylov = (A.method == 1);
    if (ell > 0 && (A.method == 2 || A.method == 3)) {
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
    if (ell > 0 && need_krylov) {
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
    if (gb == 0 && threadIdx.x == 0) {
        A.out[2 * p] = value;
        A.out[2 * p + 1] = conv;
    }
}

int cond_estimate_batch(int nells, const int64_t *ells_host, const double *r, int64_t ldr, const double *rinv,
                        int64_t ldi, int method, double *values_host, Workspace &ws, cudaStream_t st) {
    if (nells <= 0) return 0;
    if (method == 0) {  // diag ratio: a single pass each
        for (int q = 0; q < nells; ++q) CQ_TRY(cond_estimate(ells_host[q], r, ldr, rinv, ldi, 0, values_host + q, ws, st));
        return 0;
    }
    const int sms = num_sms();
    if (first_on_device((const void *)cond_group_kernel))
        CQ_CUDA(cudaFuncSetAttribute(cond_group_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024),
                "cond group smem");
    int64_t maxl = 1;
    for (int q = 0; q < nells; ++q) maxl = std::max<int64_t>(maxl, ells_host[q]);
    const size_t smem = sizeof(double) * (size_t)(8 * 32 + 64 + maxl);
    if (smem > 200 * 1024) return fail_internal("cond estimator: block too large for shared memory");
    int per_sm = 0;
    CQ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cond_group_kernel, kGridPowThreads, smem),
            "cond occupancy");
    const int slots = std::max(1, per_sm) * sms;  // co-resident CTAs (cooperative launch)
    double *vec = ws.get<double>("condg.vec", (size_t)(3 * maxl * nells));
    double *outd = ws.get<double>("condg.out", (size_t)(2 * nells));
    unsigned long long *bar = ws.get<unsigned long long>("condg.bar", (size_t)nells);
    int64_t *dells = ws.get<int64_t>("condg.ells", (size_t)nells);
    int *dfirst = ws.get<int>("condg.first", (size_t)nells + 1);
    double *part = ws.get<double>("condg.part", (size_t)nells * kMaxGroup);
    if (!vec || !outd || !bar || !dells || !dfirst || !part) return fail_nomem("cond estimator");
    std::vector<int> first((size_t)nells + 1, 0);
    std::vector<double> hout((size_t)(2 * nells));
    // launches of as many whole probe groups as fit co-resident
    for (int q0 = 0; q0 < nells;) {
        int q1 = q0, ctas = 0;
        while (q1 < nells && ctas + group_size(ells_host[q1]) <= slots) ctas += group_size(ells_host[q1++]);
        if (q1 == q0) return fail_internal("cond estimator: group larger than the GPU");
        const int np = q1 - q0;
        first[0] = 0;
        for (int q = 0; q < np; ++q) first[(size_t)q + 1] = first[(size_t)q] + group_size(ells_host[q0 + q]);
        CQ_CUDA(cudaMemcpyAsync(dells, ells_host + q0, sizeof(int64_t) * np, cudaMemcpyHostToDevice, st), "ells");
        CQ_CUDA(cudaMemcpyAsync(dfirst, first.data(), sizeof(int) * (np + 1), cudaMemcpyHostToDevice, st), "groups");
        CQ_CUDA(cudaMemsetAsync(bar, 0, sizeof(unsigned long long) * np, st), "cond bars");
        CondGroupArgs a;
        a.nprobes = np;
        a.ells = dells;
        a.first_cta = dfirst;
        a.ldr = ldr;
        a.ldi = ldi;
        a.vlen = maxl;
        a.r = r;
        a.rinv = rinv;
        a.method = method;
        a.vec = vec;
        a.part = part;
        a.bar = bar;
        a.out = outd;
        void *args[] = {&a};
        CQ_CUDA(cudaLaunchCooperativeKernel((void *)cond_group_kernel, dim3(first[(size_t)np]),
                                            dim3(kGridPowThreads), args, smem, st),
                "cond group launch");
        note_launch();
        CQ_CUDA(cudaMemcpyAsync(hout.data() + 2 * q0, outd, sizeof(double) * 2 * np, cudaMemcpyDeviceToHost, st),
                "cond d2h");
        CQ_CUDA(cudaStreamSynchronize(st), "cond sync");  // host arrays reused by the next launch
        q0 = q1;
    }
    for (int q = 0; q < nells; ++q) values_host[q] = hout[(size_t)(2 * q)];
    return 0;
}

int cond_estimate(int64_t ell, const double *r, int64_t ldr, const double *rinv, int64_t ldi, int method,
                  double *value_host, Workspace &ws, cudaStream_t st) {
    if (method != 0 && ell > 0) return cond_estimate_batch(1, &ell, r, ldr, rinv, ldi, method, value_host, ws, st);
    double *dout = ws.get<double>("cond.out", 2);
    double *work = ws.get<double>("cond.work", (size_t)(3 * std::max<int64_t>(ell, 1)));
    cond_estimate_kernel<<<1, kPowThreads, 0, st>>>(ell, r, ldr, rinv, ldi, method, work, dout);
    note_launch();
    CQ_TRY(check_launch("cond_estimate_kernel"));
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

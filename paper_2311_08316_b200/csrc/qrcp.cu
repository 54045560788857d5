// K3: max-norm Householder QRCP of the d x n sketch, K4: stage-1 rank.
//
// Reference: qrcp_maxnorm (qrcp.cc:35-97) with make_reflector /
// apply_reflector (linalg.cc:110-136), extract_upper (linalg.cc:177-183);
// rank_stage1 (cqrrpt.cc:92-112).
//
// One cooperative persistent kernel runs all n steps (the QRCP is a chain of
// n dependent steps; launching per step would cost more than the step).
// Columns never move in memory: a logical->physical column map (ping-pong per
// step) implements the reference's column swaps, and the physical index of
// the column finally at logical position j is exactly J[j] (the pivots are
// the original column indices). Logical position j is owned by CTA j % G;
// a warp applies the step's reflector to one column and downdates its
// squared norm with the reference's cancellation safeguard
// (updated <= sqrt(u) * w_ref -> recompute from the updated column,
// qrcp.cc:76-88). The pivot search uses the reference's rule: largest
// downdated squared norm, lowest logical index on ties (qrcp.cc:26-31), and
// the stop test sqrt(max(w_p,0)) <= n*u*max_j ||col_j|| (qrcp.cc:52-62).
// Every CTA recomputes the pivot column's reflector redundantly (same code,
// same order -> identical bits), so one grid barrier per step suffices.
#include "common.cuh"
#include "internal.hh"

namespace cqg {

constexpr int kQrcpThreads = 256;  // 64 quads of 4 lanes

// The reference's dot (linalg.cc:36-50) as compiled (oracle/cqrrpt_oracle.c
// orc_dot): four interleaved accumulators s_q over the 4-aligned body with
// separately rounded products, (s0 + s1) + (s2 + s3), then the <4-element
// tail with the last term of an odd count fused. Lane q of a 4-lane quad
// owns s_q; the result is returned in all 4 lanes. This file is compiled
// with --fmad=false: every FMA below is an explicit fma().
template <class FA, class FB>
CQ_DEVI double quad_dot(unsigned qmask, int q, int64_t c, FA fa, FB fb) {
    const int64_t body = c & ~(int64_t)3;
    double s = 0.0;
    for (int64_t e = q; e < body; e += 4) s = s + fa(e) * fb(e);
    double pair = s + __shfl_xor_sync(qmask, s, 1);
    double tot = pair + __shfl_xor_sync(qmask, pair, 2);
    int64_t e = body, rem = c - body;
    if (rem >= 2) {
        tot = tot + fa(e) * fb(e);
        tot = tot + fa(e + 1) * fb(e + 1);
        e += 2;
        rem -= 2;
    }
    if (rem == 1) tot = fma(fa(e), fb(e), tot);
    return tot;
}

struct QrcpArgs {
    int64_t d, n, ld;
    double *b;
    double *w[2];
    double *wref;
    int32_t *cmap[2];
    int32_t *piv;     // physical pivot chosen at each step
    double *alpha;    // R(i,i)
    double *pv[2];    // per-CTA argmax partials
    int32_t *pi[2];
    unsigned int *bar;
    int64_t *k_out;
    int32_t *final_buf;  // which cmap buffer holds positions >= k
    double rank_tol;
    int64_t steps;
};

__global__ void __launch_bounds__(kQrcpThreads, 1) qrcp_kernel(QrcpArgs A) {
    extern __shared__ double s_v[];  // pivot column rows i..d-1, then scaled reflector
    __shared__ double s_av[kQrcpThreads / 32];
    __shared__ int32_t s_ai[kQrcpThreads / 32];
    __shared__ double s_bc[4];
    const int G = gridDim.x, cta = blockIdx.x;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = kQrcpThreads / 32;
    const int q = lane & 3;
    const int quad = threadIdx.x >> 2;  // 0..63
    const unsigned qmask = 0xfu << (lane & ~3);
    const int64_t d = A.d, n = A.n, ld = A.ld;
    const double sqrt_u = sqrt(kUnitRoundoff);

    auto block_argmax = [&](ArgMax a) -> ArgMax {
        a = warp_argmax(a);
        __syncthreads();
        if (lane == 0) {
            s_av[wid] = a.v;
            s_ai[wid] = a.i;
        }
        __syncthreads();
        ArgMax r{-INFINITY, 0x7fffffff};
        if (lane < nw) r = ArgMax{s_av[lane], s_ai[lane]};
        return warp_argmax(r);
    };

    // ---- initial squared norms w_j = dot(col_j, col_j) (qrcp.cc:48-51) ----
    ArgMax loc{-INFINITY, 0x7fffffff};
    {
        const int64_t nper = (n + G - 1) / G;  // positions cta, cta+G, ...
        for (int64_t t0 = 0; t0 < nper; t0 += kQrcpThreads / 4) {
            const int64_t j = cta + (t0 + quad) * G;
            const bool act = (t0 + quad) < nper && j < n;
            const double *col = A.b + (act ? j : 0) * ld;
            double s = quad_dot(qmask, q, act ? d : 0, [&](int64_t e) { return col[e]; },
                                [&](int64_t e) { return col[e]; });
            if (act && q == 0) {
                A.w[0][j] = s;
                A.wref[j] = s;
                A.cmap[0][j] = (int32_t)j;
                loc = argmax_combine(loc, ArgMax{s, (int32_t)j});
            }
        }
    }
    loc = block_argmax(loc);
    if (threadIdx.x == 0) {
        A.pv[0][cta] = loc.v;
        A.pi[0][cta] = loc.i;
    }
    grid_barrier(A.bar, G);

    double stop = 0.0;
    int64_t k = 0;
    int64_t i = 0;
    for (; i < A.steps; ++i) {
        const int cur = (int)(i & 1), nxt = cur ^ 1;
        // ---- pivot: lowest index attaining the max (qrcp.cc:26-31) -------
        ArgMax g{-INFINITY, 0x7fffffff};
        if (threadIdx.x < G) g = ArgMax{ld_cg(A.pv[cur] + threadIdx.x), ld_cg(A.pi[cur] + threadIdx.x)};
        g = block_argmax(g);
        if (i == 0) stop = A.rank_tol * sqrt(fmax(g.v, 0.0));  // max_norm0 (qrcp.cc:52-55)
        const double wp = g.v;
        const int64_t p = g.i;
        if (sqrt(wp > 0.0 ? wp : 0.0) <= stop) break;  // qrcp.cc:62
        const int32_t phys_p = ld_cg(A.cmap[cur] + p);
        const int32_t phys_i = ld_cg(A.cmap[cur] + i);
        const double *x = A.b + (int64_t)phys_p * ld;
        const int64_t c = d - i - 1;  // rows below the diagonal

        // ---- make_reflector (linalg.cc:110-124) ---------------------------
        for (int64_t r = threadIdx.x; r < d - i; r += kQrcpThreads) s_v[r] = ld_cg(x + i + r);
        __syncthreads();
        if (wid == 0 && lane < 4) {
            double tail_sq = quad_dot(0xfu, q, c, [&](int64_t e) { return s_v[1 + e]; },
                                      [&](int64_t e) { return s_v[1 + e]; });
            if (q == 0) {
                double x0 = s_v[0];
                double norm_x = sqrt(fma(x0, x0, tail_sq));
                double alpha = x0, v0 = 1.0, beta = 0.0;
                if (norm_x != 0.0) {
                    double sign = (x0 >= 0.0) ? 1.0 : -1.0;
                    alpha = -sign * norm_x;
                    v0 = x0 - alpha;
                    beta = (norm_x + fabs(x0)) / norm_x;
                }
                s_bc[0] = alpha;
                s_bc[1] = v0;
                s_bc[2] = beta;
            }
        }
        __syncthreads();
        const double alpha = s_bc[0], v0 = s_bc[1], beta = s_bc[2];
        if (beta != 0.0)
            for (int64_t r = threadIdx.x; r < c; r += kQrcpThreads) s_v[1 + r] = s_v[1 + r] / v0;  // colj[i] /= v0
        __syncthreads();
        const double *sv = s_v + 1;

        // ---- apply_reflector + norm downdate on owned positions j > i ----
        ArgMax mine{-INFINITY, 0x7fffffff};
        const int64_t jfirst = i + 1 + ((cta - (i + 1)) % G + G) % G;
        const int64_t nown = (jfirst < n) ? (n - jfirst + G - 1) / G : 0;
        for (int64_t t0 = 0; t0 < nown; t0 += kQrcpThreads / 4) {
            const bool act = (t0 + quad) < nown;
            const int64_t j = jfirst + (t0 + quad) * G;
            const bool isp = act && (j == p);
            const int32_t pj = !act ? 0 : (isp ? phys_i : ld_cg(A.cmap[cur] + j));
            const double wj = !act ? 0.0 : (isp ? ld_cg(A.w[cur] + i) : ld_cg(A.w[cur] + j));
            const double wrefj = !act ? 0.0 : (isp ? ld_cg(A.wref + i) : ld_cg(A.wref + j));
            double *col = A.b + (int64_t)pj * ld;
            const int64_t cc = act ? c : 0;
            double t = act ? ld_cg(col + i) : 0.0;
            if (beta != 0.0) {
                double dot = quad_dot(qmask, q, cc, [&](int64_t e) { return sv[e]; },
                                      [&](int64_t e) { return ld_cg(col + i + 1 + e); });
                double tau = t;  // linalg.cc:131-135
                tau += dot;
                tau *= beta;
                t = t - tau;
                for (int64_t e = q; e < cc; e += 4) __stcg(col + i + 1 + e, fma(-tau, sv[e], ld_cg(col + i + 1 + e)));
                __syncwarp(qmask);
            }
            double updated = fma(-t, t, wj);  // qrcp.cc:77-78
            double newref = wrefj;
            if (updated <= sqrt_u * wrefj) {   // qrcp.cc:82-86 (uniform within the quad)
                updated = quad_dot(qmask, q, cc, [&](int64_t e) { return ld_cg(col + i + 1 + e); },
                                   [&](int64_t e) { return ld_cg(col + i + 1 + e); });
                newref = updated;
            }
            if (act && q == 0) {
                __stcg(col + i, t);
                __stcg(A.w[nxt] + j, updated);
                __stcg(A.wref + j, newref);
                __stcg(A.cmap[nxt] + j, pj);
                mine = argmax_combine(mine, ArgMax{updated, (int32_t)j});
            }
        }
        mine = block_argmax(mine);
        if (threadIdx.x == 0) {
            __stcg(A.pv[nxt] + cta, mine.v);
            __stcg(A.pi[nxt] + cta, mine.i);
            if (cta == 0) {
                __stcg(A.piv + i, phys_p);
                __stcg(A.alpha + i, alpha);
            }
        }
        k = i + 1;
        grid_barrier(A.bar, G);
    }
    if (cta == 0 && threadIdx.x == 0) {
        *A.k_out = k;
        *A.final_buf = (int32_t)(k & 1);
    }
}

// J[j] = pivot at step j (j < k) or the column map (j >= k);
// R[r][j] (r < k) = alpha on the diagonal, B[r][J[j]] above it, 0 below.
__global__ void qrcp_extract_kernel(int64_t d, int64_t n, const double *__restrict__ b, int64_t ldb,
                                    const int64_t *__restrict__ kdev, const int32_t *__restrict__ piv,
                                    const int32_t *__restrict__ cmap0, const int32_t *__restrict__ cmap1,
                                    const int32_t *__restrict__ fbuf, const double *__restrict__ alpha,
                                    double *__restrict__ r_out, int64_t ldr, int64_t *__restrict__ jout) {
    const int64_t j = blockIdx.x;
    const int64_t k = *kdev;
    const int32_t *cm = (*fbuf) ? cmap1 : cmap0;
    const int64_t pj = (j < k) ? piv[j] : cm[j];
    if (threadIdx.x == 0) jout[j] = pj;
    const double *col = b + pj * ldb;
    for (int64_t r = threadIdx.x; r < n; r += blockDim.x) {
        double v = 0.0;
        if (r < k) {
            if (r < j) v = col[r];
            else if (r == j) v = alpha[j];
        }
        r_out[j * ldr + r] = v;
    }
}

// rank_stage1 (cqrrpt.cc:92-112) in the reference's arithmetic order.
// Row masses: thread per row, acc = acc + R(i,j)^2 over j ascending (not
// contracted as built); row max |R(i,:)| for max_abs (order-free).
__global__ void row_stats_kernel(int64_t k, int64_t n, const double *__restrict__ r, int64_t ldr,
                                 double *__restrict__ mass, double *__restrict__ rmax) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const bool act = i < k;
    double acc = 0.0, mx = 0.0;
    for (int64_t j = 0; j < n; ++j) {  // all lanes walk j together: coalesced over rows
        double v = act ? r[j * ldr + i] : 0.0;
        mx = fmax(mx, fabs(v));
        if (j >= i) acc = acc + v * v;
    }
    if (act) {
        mass[i] = acc;
        rmax[i] = mx;
    }
}

// Tail accumulation from the bottom, sequential as in the reference.
__global__ void stage1_kernel(int64_t k, const double *__restrict__ mass, const double *__restrict__ rmax, double u,
                              int64_t *__restrict__ k0_out) {
    __shared__ double s_red[32];
    double mx = 0.0;
    for (int64_t i = threadIdx.x; i < k; i += blockDim.x) mx = fmax(mx, rmax[i]);
    mx = warp_max(mx);
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x != 0) return;
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s = fmax(s, s_red[w]);
    if (s == 0.0) {
        *k0_out = 0;
        return;
    }
    const double target = (u * s) * (u * s);
    double tail = 0.0;
    int64_t k0 = k;
    for (int64_t ell = k - 1; ell >= 0; --ell) {
        tail += mass[ell];
        if (tail <= target) k0 = ell;
    }
    *k0_out = k0;
}

int qrcp(int64_t d, int64_t n, double *b, int64_t ldb, double rank_tol, double *rsk, int64_t ldr, int64_t *jdev,
         int64_t *k_sk, Workspace &ws, cudaStream_t st) {
    if (d < 1) return fail_internal("qrcp: need at least one row");
    if (rank_tol < 0.0) rank_tol = (double)n * kUnitRoundoff;  // qrcp.cc:17,38
    const int sms = num_sms();
    int G = (int)std::min<int64_t>(std::min<int64_t>(sms, kQrcpThreads), std::max<int64_t>(1, (n + 7) / 8));
    int maxb = 0;
    CQ_CUDA(cudaFuncSetAttribute(qrcp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024), "qrcp smem");
    CQ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&maxb, qrcp_kernel, kQrcpThreads, sizeof(double) * (d + 1)),
            "occupancy");
    G = std::min(G, std::max(1, maxb) * sms);
    QrcpArgs a;
    a.d = d;
    a.n = n;
    a.ld = ldb;
    a.b = b;
    a.w[0] = ws.get<double>("qrcp.w0", n);
    a.w[1] = ws.get<double>("qrcp.w1", n);
    a.wref = ws.get<double>("qrcp.wref", n);
    a.cmap[0] = ws.get<int32_t>("qrcp.c0", n);
    a.cmap[1] = ws.get<int32_t>("qrcp.c1", n);
    a.piv = ws.get<int32_t>("qrcp.piv", n);
    a.alpha = ws.get<double>("qrcp.alpha", n);
    a.pv[0] = ws.get<double>("qrcp.pv0", 256);
    a.pv[1] = ws.get<double>("qrcp.pv1", 256);
    a.pi[0] = ws.get<int32_t>("qrcp.pi0", 256);
    a.pi[1] = ws.get<int32_t>("qrcp.pi1", 256);
    a.bar = ws.get<unsigned int>("qrcp.bar", 4);
    a.k_out = ws.get<int64_t>("qrcp.k", 2);
    a.final_buf = ws.get<int32_t>("qrcp.fb", 2);
    a.rank_tol = rank_tol;
    a.steps = std::min(d, n);
    if (!a.w[0] || !a.bar || !a.k_out) return fail_nomem("qrcp workspace");
    CQ_CUDA(cudaMemsetAsync(a.bar, 0, 4 * sizeof(unsigned int), st), "memset bar");
    const size_t smem = sizeof(double) * (size_t)(d + 1);
    if (smem > 200 * 1024) return fail_internal("qrcp: d too large for the shared-memory reflector (d <= 25600)");
    CQ_CUDA(cudaFuncSetAttribute(qrcp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "qrcp smem");
    void *args[] = {&a};
    CQ_CUDA(cudaLaunchCooperativeKernel((void *)qrcp_kernel, dim3(G), dim3(kQrcpThreads), args, smem, st),
            "qrcp cooperative launch");
    note_launch();
    qrcp_extract_kernel<<<(unsigned)n, 128, 0, st>>>(d, n, b, ldb, a.k_out, a.piv, a.cmap[0], a.cmap[1],
                                                      a.final_buf, a.alpha, rsk, ldr, jdev);
    note_launch();
    CQ_TRY(check_launch("qrcp_extract_kernel"));
    CQ_CUDA(cudaMemcpyAsync(k_sk, a.k_out, sizeof(int64_t), cudaMemcpyDeviceToHost, st), "k_sk d2h");
    CQ_CUDA(cudaStreamSynchronize(st), "qrcp sync");
    return 0;
}

int rank_stage1(int64_t k, int64_t n, const double *r, int64_t ldr, int64_t *k0, Workspace &ws, cudaStream_t st) {
    if (k <= 0) {
        *k0 = 0;
        return 0;
    }
    double *mass = ws.get<double>("s1.mass", k);
    double *rmax = ws.get<double>("s1.rmax", k);
    int64_t *kd = ws.get<int64_t>("s1.k0", 1);
    row_stats_kernel<<<(unsigned)((k + 127) / 128), 128, 0, st>>>(k, n, r, ldr, mass, rmax);
    note_launch();
    stage1_kernel<<<1, 1024, 0, st>>>(k, mass, rmax, kUnitRoundoff, kd);
    note_launch();
    CQ_TRY(check_launch("stage1_kernel"));
    CQ_CUDA(cudaMemcpyAsync(k0, kd, sizeof(int64_t), cudaMemcpyDeviceToHost, st), "k0 d2h");
    CQ_CUDA(cudaStreamSynchronize(st), "stage1 sync");
    return 0;
}

}  // namespace cqg

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
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "internal.hh"

namespace cqg {

constexpr int kQrcpThreads = 256;  // 8 warps; a warp owns one column at a time

// ---------------------------------------------------------------------------
// The reference's dot (linalg.cc:36-50) as compiled (see oracle/cqrrpt_oracle.c
// orc_dot): four interleaved accumulators s_q over the 4-aligned body with
// separately rounded products, (s0 + s1) + (s2 + s3), then the <4-element
// tail with the last term of an odd count fused. Lanes 0..3 of a warp own
// s_0..s_3 (the ordered chains); the other lanes stage operands. This file is
// compiled with --fmad=false: every FMA below is an explicit fma().
// ---------------------------------------------------------------------------

// lanes 0..3: accumulate body elements [b0, b0+len) of a.b into s (e = lane mod 4)
CQ_DEVI double chain_chunk(double s, const double *a, const double *b, int64_t len, int lane) {
    int64_t e = lane;
    for (; e + 28 < len; e += 32) {
        double av[8], bv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            av[u] = a[e + 4 * u];
            bv[u] = b[e + 4 * u];
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) s = s + av[u] * bv[u];
    }
    for (; e < len; e += 4) s = s + a[e] * b[e];
    return s;
}

// lanes 0..3: (s0+s1)+(s2+s3), then the tail (elements body..c-1 via fa/fb)
template <class FA, class FB>
CQ_DEVI double chain_finish(double s, int64_t c, FA fa, FB fb) {
    const int64_t body = c & ~(int64_t)3;
    double pair = s + __shfl_xor_sync(0xfu, s, 1);
    double tot = pair + __shfl_xor_sync(0xfu, pair, 2);
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

// Warp-cooperative reference dot of sa[0..c) (shared, or nullptr = the column
// itself) with the global column g[0..c): the column is staged through the
// warp's shared buffer wb (WB doubles) with coalesced loads; lanes 0..3 run
// the ordered chains from shared memory. Result broadcast to all lanes.
CQ_DEVI double warp_ref_dot(const double *sa, const double *g, int64_t c, double *wb, int WB, int lane) {
    const int64_t body = c & ~(int64_t)3;
    double s = 0.0;
    for (int64_t b0 = 0; b0 < body; b0 += WB) {
        const int len = (int)cmin<int64_t>(WB, body - b0);
#pragma unroll 4
        for (int e = lane; e < len; e += 32) wb[e] = ld_cg(g + b0 + e);
        __syncwarp();
        if (lane < 4) s = chain_chunk(s, sa ? sa + b0 : wb, wb, len, lane);
        __syncwarp();
    }
    double tot = 0.0;
    if (lane < 4) {
        tot = chain_finish(s, c, [&](int64_t x) { return sa ? sa[x] : ld_cg(g + x); },
                           [&](int64_t x) { return ld_cg(g + x); });
    }
    return __shfl_sync(0xffffffffu, tot, 0);
}

struct QrcpArgs {
    int64_t d, n, ld;
    double *b;
    double *w[2];
    double *wref;
    int32_t *cmap[2];
    int32_t *piv;     // physical pivot chosen at each step
    double *alpha;    // R(i,i)
    double *pv[2];    // per-CTA argmax partials: value, logical index, physical column
    int32_t *pi[2];
    int32_t *pp[2];
    unsigned int *bar;
    int64_t *k_out;
    int32_t *final_buf;  // which cmap buffer holds positions >= k
    double rank_tol;
    int64_t steps;
    int wb;              // per-warp staging buffer (doubles, multiple of 32)
    unsigned long long *trace;  // optional per-step phase timestamps (CTA 0)
};

CQ_DEVI void trace_mark(unsigned long long *tr, int64_t i, int slot) {
    if (tr && blockIdx.x == 0 && threadIdx.x == 0 && i < 512) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        tr[i * 6 + slot] = t;
    }
}

// Lanes of a warp stage g[0..len) into wb (coalesced).
CQ_DEVI void warp_stage(double *wb, const double *g, int64_t len, int lane) {
#pragma unroll 4
    for (int64_t e = lane; e < len; e += 32) wb[e] = ld_cg(g + e);
}

__global__ void __launch_bounds__(kQrcpThreads, 1) qrcp_kernel(QrcpArgs A) {
    extern __shared__ double smem[];
    __shared__ double s_av[kQrcpThreads / 32];
    __shared__ int32_t s_ai[kQrcpThreads / 32], s_ap[kQrcpThreads / 32];
    __shared__ double s_bc[4];
    const int G = gridDim.x, cta = blockIdx.x;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = kQrcpThreads / 32;
    const int64_t d = A.d, n = A.n, ld = A.ld;
    const int WB = A.wb;
    double *wb = smem + wid * WB;   // warp staging buffer: the warp's column tail
    double *s_v = smem + nw * WB;   // pivot column / scaled reflector (d+1)
    const double sqrt_u = sqrt(kUnitRoundoff);

    // block argmax carrying the physical column of the winner
    auto block_argmax = [&](ArgMax a, int32_t phys, int32_t *phys_out) -> ArgMax {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            ArgMax b;
            b.v = __shfl_xor_sync(0xffffffffu, a.v, o);
            b.i = __shfl_xor_sync(0xffffffffu, a.i, o);
            int32_t bp = __shfl_xor_sync(0xffffffffu, phys, o);
            ArgMax c = argmax_combine(a, b);
            if (c.i != a.i || c.v != a.v) phys = bp;
            a = c;
        }
        __syncthreads();
        if (lane == 0) {
            s_av[wid] = a.v;
            s_ai[wid] = a.i;
            s_ap[wid] = phys;
        }
        __syncthreads();
        ArgMax r{-INFINITY, 0x7fffffff};
        int32_t rp = 0;
        if (lane < nw) {
            r = ArgMax{s_av[lane], s_ai[lane]};
            rp = s_ap[lane];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            ArgMax b;
            b.v = __shfl_xor_sync(0xffffffffu, r.v, o);
            b.i = __shfl_xor_sync(0xffffffffu, r.i, o);
            int32_t bp = __shfl_xor_sync(0xffffffffu, rp, o);
            ArgMax c = argmax_combine(r, b);
            if (c.i != r.i || c.v != r.v) rp = bp;
            r = c;
        }
        *phys_out = rp;
        return r;
    };

    // ---- initial squared norms w_j = dot(col_j, col_j) (qrcp.cc:48-51) ----
    ArgMax loc{-INFINITY, 0x7fffffff};
    int32_t locp = 0;
    for (int64_t j = cta + (int64_t)wid * G; j < n; j += (int64_t)nw * G) {
        double s = warp_ref_dot(nullptr, A.b + j * ld, d, wb, WB, lane);
        if (lane == 0) {
            A.w[0][j] = s;
            A.wref[j] = s;
            A.cmap[0][j] = (int32_t)j;
        }
        ArgMax c = argmax_combine(loc, ArgMax{s, (int32_t)j});
        if (c.i != loc.i) locp = (int32_t)j;
        loc = c;
    }
    {
        int32_t bp;
        loc = block_argmax(loc, locp, &bp);
        if (threadIdx.x == 0) {
            A.pv[0][cta] = loc.v;
            A.pi[0][cta] = loc.i;
            A.pp[0][cta] = bp;
        }
    }
    grid_barrier(A.bar, G);

    double stop = 0.0;
    int64_t k = 0;
    int64_t i = 0;
    for (; i < A.steps; ++i) {
        const int cur = (int)(i & 1), nxt = cur ^ 1;
        const int64_t c = d - i - 1;  // rows below the diagonal
        const bool fits = c <= WB;
        trace_mark(A.trace, i, 0);

        // ---- prefetch this warp's first owned column (independent of the pivot)
        const int64_t jfirst = i + 1 + ((cta - (i + 1)) % G + G) % G;
        const int64_t j_w = jfirst + (int64_t)wid * G;
        int32_t pj0 = 0;
        double wj0 = 0.0, wrefj0 = 0.0, t0 = 0.0;
        if (j_w < n) {
            pj0 = ld_cg(A.cmap[cur] + j_w);
            wj0 = ld_cg(A.w[cur] + j_w);
            wrefj0 = ld_cg(A.wref + j_w);
            const double *col = A.b + (int64_t)pj0 * ld;
            t0 = ld_cg(col + i);
            if (fits) warp_stage(wb, col + i + 1, c, lane);
        }
        const int32_t phys_i = ld_cg(A.cmap[cur] + i);
        const double w_i = ld_cg(A.w[cur] + i), wref_i = ld_cg(A.wref + i);

        // ---- pivot: lowest index attaining the max (qrcp.cc:26-31) -------
        ArgMax g{-INFINITY, 0x7fffffff};
        int32_t gp = 0;
        if (threadIdx.x < G) {
            g = ArgMax{ld_cg(A.pv[cur] + threadIdx.x), ld_cg(A.pi[cur] + threadIdx.x)};
            gp = ld_cg(A.pp[cur] + threadIdx.x);
        }
        int32_t phys_p;
        g = block_argmax(g, gp, &phys_p);
        if (i == 0) stop = A.rank_tol * sqrt(fmax(g.v, 0.0));  // max_norm0 (qrcp.cc:52-55)
        const double wp = g.v;
        const int64_t p = g.i;
        if (sqrt(wp > 0.0 ? wp : 0.0) <= stop) break;  // qrcp.cc:62
        const double *x = A.b + (int64_t)phys_p * ld;
        trace_mark(A.trace, i, 1);

        // ---- make_reflector (linalg.cc:110-124), redundantly per CTA ------
        for (int64_t r = threadIdx.x; r < d - i; r += kQrcpThreads) s_v[r] = ld_cg(x + i + r);
        __syncthreads();
        if (wid == 0 && lane < 4) {
            double s = chain_chunk(0.0, s_v + 1, s_v + 1, c & ~(int64_t)3, lane);
            double tail_sq = chain_finish(s, c, [&](int64_t e) { return s_v[1 + e]; },
                                          [&](int64_t e) { return s_v[1 + e]; });
            if (lane == 0) {
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
        trace_mark(A.trace, i, 2);

        // ---- apply_reflector + norm downdate, one owned column per warp --
        ArgMax mine{-INFINITY, 0x7fffffff};
        int32_t minep = 0;
        bool first = true;
        for (int64_t j = j_w; j < n; j += (int64_t)nw * G, first = false) {
            const bool isp = (j == p);
            int32_t pj;
            double wj, wrefj, t;
            bool staged = false;
            if (first && !isp) {
                pj = pj0;
                wj = wj0;
                wrefj = wrefj0;
                t = t0;
                staged = fits;
            } else {
                pj = isp ? phys_i : ld_cg(A.cmap[cur] + j);
                wj = isp ? w_i : ld_cg(A.w[cur] + j);
                wrefj = isp ? wref_i : ld_cg(A.wref + j);
                t = ld_cg(A.b + (int64_t)pj * ld + i);
                if (fits) {
                    __syncwarp();
                    warp_stage(wb, A.b + (int64_t)pj * ld + i + 1, c, lane);
                    staged = true;
                }
            }
            double *col = A.b + (int64_t)pj * ld;
            double *tail = col + i + 1;
            if (staged) __syncwarp();
            if (beta != 0.0) {  // apply_reflector (linalg.cc:126-136)
                double dot;
                if (staged) {
                    double s = 0.0;
                    if (lane < 4) {
                        s = chain_chunk(0.0, sv, wb, c & ~(int64_t)3, lane);
                        s = chain_finish(s, c, [&](int64_t e) { return sv[e]; }, [&](int64_t e) { return wb[e]; });
                    }
                    dot = __shfl_sync(0xffffffffu, s, 0);
                } else {
                    dot = warp_ref_dot(sv, tail, c, wb, WB, lane);
                }
                double tau = t;
                tau += dot;
                tau *= beta;
                t = t - tau;
                if (staged) {
#pragma unroll 4
                    for (int64_t e = lane; e < c; e += 32) {
                        double nv = fma(-tau, sv[e], wb[e]);
                        wb[e] = nv;
                        __stcg(tail + e, nv);
                    }
                } else {
#pragma unroll 4
                    for (int64_t e = lane; e < c; e += 32) __stcg(tail + e, fma(-tau, sv[e], ld_cg(tail + e)));
                }
                __syncwarp();
            }
            double updated = fma(-t, t, wj);  // qrcp.cc:77-78
            double newref = wrefj;
            if (updated <= sqrt_u * wrefj) {  // qrcp.cc:82-86 (warp-uniform)
                if (staged) {
                    double s = 0.0;
                    if (lane < 4) {
                        s = chain_chunk(0.0, wb, wb, c & ~(int64_t)3, lane);
                        s = chain_finish(s, c, [&](int64_t e) { return wb[e]; }, [&](int64_t e) { return wb[e]; });
                    }
                    updated = __shfl_sync(0xffffffffu, s, 0);
                } else {
                    updated = warp_ref_dot(nullptr, tail, c, wb, WB, lane);
                }
                newref = updated;
            }
            if (lane == 0) {
                __stcg(col + i, t);
                __stcg(A.w[nxt] + j, updated);
                __stcg(A.wref + j, newref);
                __stcg(A.cmap[nxt] + j, pj);
            }
            ArgMax cnd = argmax_combine(mine, ArgMax{updated, (int32_t)j});
            if (cnd.i != mine.i) minep = pj;
            mine = cnd;
            __syncwarp();
        }
        trace_mark(A.trace, i, 3);
        {
            int32_t bp;
            mine = block_argmax(mine, minep, &bp);
            if (threadIdx.x == 0) {
                __stcg(A.pv[nxt] + cta, mine.v);
                __stcg(A.pi[nxt] + cta, mine.i);
                __stcg(A.pp[nxt] + cta, bp);
                if (cta == 0) {
                    __stcg(A.piv + i, phys_p);
                    __stcg(A.alpha + i, alpha);
                }
            }
        }
        k = i + 1;
        trace_mark(A.trace, i, 4);
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
    // shared memory: 8 warp staging buffers + the pivot column (d+1 doubles)
    const int64_t budget = (200 * 1024) / (int64_t)sizeof(double);
    if (d + 1 + 8 * 128 > budget) return fail_internal("qrcp: d too large for the shared-memory reflector");
    const int WB = (int)std::min<int64_t>(4096, ((budget - (d + 1)) / 8) & ~(int64_t)31);
    const size_t smem = sizeof(double) * (size_t)(8 * WB + d + 1);
    CQ_CUDA(cudaFuncSetAttribute(qrcp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "qrcp smem");
    // one owned column per warp per step at the start (8 warps per CTA)
    int G = (int)std::min<int64_t>(std::min<int64_t>(sms, kQrcpThreads), std::max<int64_t>(1, (n + 7) / 8));
    int maxb = 0;
    CQ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&maxb, qrcp_kernel, kQrcpThreads, smem), "occupancy");
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
    a.pp[0] = ws.get<int32_t>("qrcp.pp0", 256);
    a.pp[1] = ws.get<int32_t>("qrcp.pp1", 256);
    a.bar = ws.get<unsigned int>("qrcp.bar", 4);
    a.k_out = ws.get<int64_t>("qrcp.k", 2);
    a.final_buf = ws.get<int32_t>("qrcp.fb", 2);
    a.rank_tol = rank_tol;
    a.steps = std::min(d, n);
    if (!a.w[0] || !a.bar || !a.k_out) return fail_nomem("qrcp workspace");
    CQ_CUDA(cudaMemsetAsync(a.bar, 0, 4 * sizeof(unsigned int), st), "memset bar");
    a.wb = WB;
    static const bool tracing = getenv("CQRRPT_QRCP_TRACE") != nullptr;
    a.trace = tracing ? ws.get<unsigned long long>("qrcp.trace", 512 * 6) : nullptr;
    if (a.trace) CQ_CUDA(cudaMemsetAsync(a.trace, 0, 512 * 6 * sizeof(unsigned long long), st), "trace memset");
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
    if (a.trace) {  // debug: mean per-phase ns over the first steps
        std::vector<unsigned long long> h(512 * 6);
        cudaMemcpy(h.data(), a.trace, h.size() * 8, cudaMemcpyDeviceToHost);
        double acc[5] = {0, 0, 0, 0, 0};
        int cnt = 0;
        for (int s2 = 0; s2 + 1 < 512 && s2 + 1 < *k_sk; ++s2) {
            for (int q = 0; q < 4; ++q) acc[q] += (double)(h[s2 * 6 + q + 1] - h[s2 * 6 + q]);
            acc[4] += (double)(h[(s2 + 1) * 6] - h[s2 * 6 + 4]);
            ++cnt;
        }
        if (cnt)
            fprintf(stderr, "qrcp trace (G=%d, d=%lld, n=%lld, %d steps): argmax %.0f ns, reflector %.0f ns, "
                    "columns %.0f ns, partials %.0f ns, barrier %.0f ns\n", G, (long long)d, (long long)n, cnt,
                    acc[0] / cnt, acc[1] / cnt, acc[2] / cnt, acc[3] / cnt, acc[4] / cnt);
    }
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

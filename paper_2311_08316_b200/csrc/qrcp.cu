// K3: max-norm Householder QRCP of the d x n sketch, K4: stage-1 rank.
//
// Reference: qrcp_maxnorm (qrcp.cc:35-97) with make_reflector /
// apply_reflector (linalg.cc:110-136), extract_upper (linalg.cc:177-183);
// rank_stage1 (cqrrpt.cc:92-112).
//
// Bit-exact restatement: every floating-point operation of the reference is
// performed in the reference's order (dot products with its fixed 4-way
// reassociation, its FMA contractions as built), so R_sk, J and k_sk are
// bit-identical to the reference's on the same sketch.
//
// One cooperative persistent kernel runs all n steps (the QRCP is a chain of
// n dependent steps). Columns never move in memory: a logical->physical
// column map (ping-pong per step) implements the reference's swaps, and the
// physical index of the column finally at logical position j is J[j].
// Logical position j is owned by CTA j % G and, inside it, by one warp. Per
// step:
//   * every CTA reduces the per-CTA argmax partials (largest downdated squared
//     norm, lowest index on ties, qrcp.cc:26-31) and tests the stop rule
//     sqrt(max(w_p,0)) <= n*u*max_j||col_j|| (qrcp.cc:52-62);
//   * every CTA builds the pivot column's reflector redundantly (same code,
//     same order -> identical bits), so one grid barrier per step suffices;
//   * each warp applies it to its column and downdates the squared norm with
//     the cancellation safeguard (qrcp.cc:76-88).
// Columns are staged into shared memory with L2-coherent cp.async while the
// pivot is decided; the products of each dot are formed by all 32 lanes in
// parallel and only the ordered additions (lanes 0..3, one per reference
// accumulator) stay serial. Grid barrier: the flagged argmax records
// (rec_publish / rec_wait), one L2 round trip per step.
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "internal.hh"

namespace cqg {

constexpr int kQrcpThreads = 256;  // 8 warps; a warp owns one column at a time
constexpr int kQrcpWarps = kQrcpThreads / 32;

// ---------------------------------------------------------------------------
// The reference's dot (linalg.cc:36-50) as compiled (see oracle/cqrrpt_oracle.c
// orc_dot): accumulators s_q (q = e mod 4) over the 4-aligned body with
// separately rounded products, (s0 + s1) + (s2 + s3), then the <4-element
// tail: products added in order, the last term of an odd count fused.
// This file is compiled with --fmad=false: every FMA below is an explicit fma().
// ---------------------------------------------------------------------------

// lanes 0..3: add the precomputed products p[e] (e = lane mod 4, e < body) to s
// The loads of group g+1 are issued before the adds of group g, so only the
// dependent DADD latency stays on the chain (body < 2^31: shared memory).
CQ_DEVI double chain_sum(double s, const double *p, int64_t body64, int lane) {
    const int body = (int)body64;
    int e = lane;
    if (e + 28 < body) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = p[e + 4 * u];
        for (e += 32; e + 28 < body; e += 32) {
            double nx[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) nx[u] = p[e + 4 * u];
#pragma unroll
            for (int u = 0; u < 8; ++u) s = s + v[u];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = nx[u];
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) s = s + v[u];
    }
    for (; e < body; e += 4) s = s + p[e];
    return s;
}

// lanes 0..3: (s0+s1)+(s2+s3), then the tail elements body..c-1 of a.b
template <class FA, class FB>
CQ_DEVI double chain_finish(double s, int64_t c, FA fa, FB fb, unsigned quad = 0xfu) {
    const int64_t body = c & ~(int64_t)3;
    double pair = s + __shfl_xor_sync(quad, s, 1);
    double tot = pair + __shfl_xor_sync(quad, pair, 2);
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

// lanes 0..3: s += a[e] * b[e] (product rounded, then added) for e = q, q+4,
// ... < body, in order -- the same bits as adding precomputed products
// (chain_sum); the loads of group g+1 are issued before the adds of group g
CQ_DEVI double chain_dot(double s, const double *a, const double *bb, int body, int q) {
    int e = q;
    if (e + 28 < body) {
        double xa[8], xb[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            xa[u] = a[e + 4 * u];
            xb[u] = bb[e + 4 * u];
        }
        for (e += 32; e + 28 < body; e += 32) {
            double na[8], nb[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                na[u] = a[e + 4 * u];
                nb[u] = bb[e + 4 * u];
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) s = s + xa[u] * xb[u];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                xa[u] = na[u];
                xb[u] = nb[u];
            }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) s = s + xa[u] * xb[u];
    }
    for (; e < body; e += 4) s = s + a[e] * bb[e];
    return s;
}

// lanes 0..3: s += a[e] * a[e] for e = q, q+4, ... < body, in order (the
// squares of chain_dot(a, a) with one load per element)
CQ_DEVI double chain_sq(double s, const double *a, int body, int q) {
    int e = q;
    if (e + 28 < body) {
        double xa[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) xa[u] = a[e + 4 * u];
        for (e += 32; e + 28 < body; e += 32) {
            double na[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) na[u] = a[e + 4 * u];
#pragma unroll
            for (int u = 0; u < 8; ++u) s = s + xa[u] * xa[u];
#pragma unroll
            for (int u = 0; u < 8; ++u) xa[u] = na[u];
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) s = s + xa[u] * xa[u];
    }
    for (; e < body; e += 4) s = s + a[e] * a[e];
    return s;
}

// Async L2-coherent copy of g[0..len) into shared memory. The copy starts at
// the 16-byte aligned address at or below g; returns the element offset of
// g[0] inside dst (0 or 1). Only bytes inside [g-1, g+len) are read.
CQ_DEVI int stage_async(double *dst, const double *g, int64_t len, int tid, int nthreads) {
    const int off = (int)((reinterpret_cast<uintptr_t>(g) >> 3) & 1);
    const double *base = g - off;
    const int64_t total = len + off;
    for (int64_t q = tid; 2 * q < total; q += nthreads) {
        const int64_t rem = total - 2 * q;
        cp_async16_zfill(dst + 2 * q, base + 2 * q, rem >= 2 ? 16 : 8);
    }
    return off;
}

CQ_DEVI void trace_mark(unsigned long long *tr, int64_t i, int slot) {
    if (tr && threadIdx.x == 0 && i < 4096) tr[((int64_t)blockIdx.x * 4096 + i) * 16 + slot] = (unsigned long long)clock64();
}

// Warp-level reference dot of sa[0..c) (shared memory; nullptr = the column
// with itself) and the global column g[0..c). g streams through the warp's two
// half-buffers b0/b1 (CHD data doubles each, a multiple of 4) with
// double-buffered L2-coherent cp.async; all lanes form the products, lanes
// 0..3 add them in the reference's order. `pre0`: chunk 0 is already in flight
// into b0 (prefetched). When the whole column fits in one chunk the products
// go to b1, so b0 keeps the column (*kept = true) for the update pass.
CQ_DEVI double stream_dot(const double *sa, const double *g, int64_t c, double *b0, double *b1, int CHD, bool pre0,
                          bool *kept, int lane, unsigned long long *tr = nullptr, int64_t step = 0) {
    const int off = (int)((reinterpret_cast<uintptr_t>(g) >> 3) & 1);  // same for every chunk
    const int64_t body = c & ~(int64_t)3;
    const int64_t nch = (c + CHD - 1) / CHD;
    *kept = (nch == 1);
    double s = 0.0;
    if (nch > 0 && !pre0) {
        stage_async(b0, g, cmin<int64_t>(CHD, c), lane, 32);
        cp_async_commit();
    }
    for (int64_t k = 0; k < nch; ++k) {
        if (k + 1 < nch) {
            stage_async(((k + 1) & 1) ? b1 : b0, g + (k + 1) * CHD, cmin<int64_t>(CHD, c - (k + 1) * CHD), lane, 32);
            cp_async_commit();
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncwarp();
        double *buf = ((k & 1) ? b1 : b0) + off;
        const int64_t base = k * CHD;
        const int64_t bl = cmax<int64_t>(0, cmin<int64_t>(CHD, body - base));
        double *prod = (nch == 1) ? b1 : buf;
        // loads of 8 elements are issued before their products are stored
        // (prod may alias buf, so the compiler would otherwise serialise)
        const int blen = (int)bl;
        for (int e0 = lane; e0 < blen; e0 += 256) {
            double xa[8], xb[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int e = e0 + 32 * u;
                xb[u] = e < blen ? buf[e] : 0.0;
                xa[u] = e < blen ? (sa ? sa[base + e] : xb[u]) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int e = e0 + 32 * u;
                if (e < blen) prod[e] = xa[u] * xb[u];
            }
        }
        __syncwarp();
        if (k == 0) trace_mark(tr, step, 5);
        if (lane < 4) s = chain_sum(s, prod, bl, lane);
        __syncwarp();
    }
    // the <4 tail elements are still in the last chunk's buffer (products
    // only overwrote its first bl entries)
    const int64_t lastbase = (nch - 1) * CHD;
    const double *lastbuf = (((nch - 1) & 1) ? b1 : b0) + off - lastbase;
    double tot = 0.0;
    if (lane < 4)
        tot = chain_finish(s, c, [&](int64_t x) { return sa ? sa[x] : lastbuf[x]; },
                           [&](int64_t x) { return lastbuf[x]; });
    return __shfl_sync(0xffffffffu, tot, 0);
}

// Two reference dots at once, sa.ga[0..c) and sa.gb[0..c): both columns
// stream through quarter buffers (chunk CQ, double-buffered: even chunks in
// b0, odd ones in b1, A in the first half of each, B in the second), all
// lanes form the products in place, lanes 0..3 run A's ordered chain and
// lanes 4..7 B's in the same instructions. With one chunk the products go to
// the other half-buffer so the columns stay staged (*kept) for the update.
// Returns the dots in lanes 0 (A) and 4 (B), broadcast.
CQ_DEVI void stream_dot2(const double *sa, const double *ga, const double *gb, int64_t c, double *b0, double *b1,
                         int CQ, bool *kept, int lane, double *dota, double *dotb) {
    const int QS = CQ + 4;  // quarter stride (alignment slack)
    const int offa = (int)((reinterpret_cast<uintptr_t>(ga) >> 3) & 1);
    const int offb = (int)((reinterpret_cast<uintptr_t>(gb) >> 3) & 1);
    const int64_t body = c & ~(int64_t)3;
    const int64_t nch = (c + CQ - 1) / CQ;
    *kept = (nch == 1);
    auto qa = [&](int64_t k) { return ((k & 1) ? b1 : b0); };
    auto qb = [&](int64_t k) { return ((k & 1) ? b1 : b0) + QS; };
    if (nch > 0) {
        stage_async(qa(0), ga, cmin<int64_t>(CQ, c), lane, 32);
        stage_async(qb(0), gb, cmin<int64_t>(CQ, c), lane, 32);
        cp_async_commit();
    }
    const bool mine = lane < 8;
    const int q = lane & 3;
    double s = 0.0;
    for (int64_t k = 0; k < nch; ++k) {
        if (k + 1 < nch) {
            const int64_t nb = (k + 1) * CQ, nl = cmin<int64_t>(CQ, c - nb);
            stage_async(qa(k + 1), ga + nb, nl, lane, 32);
            stage_async(qb(k + 1), gb + nb, nl, lane, 32);
            cp_async_commit();
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncwarp();
        double *bufa = qa(k) + offa, *bufb = qb(k) + offb;
        const int64_t base = k * CQ;
        const int bl = (int)cmax<int64_t>(0, cmin<int64_t>(CQ, body - base));
        double *pa = (nch == 1) ? b1 + 2 : bufa;  // products (past the data when kept)
        double *pb = (nch == 1) ? b1 + 2 + QS : bufb;
        for (int e0 = lane; e0 < bl; e0 += 128) {
            double xa[4], xb[4], xs[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int e = e0 + 32 * u;
                xs[u] = e < bl ? sa[base + e] : 0.0;
                xa[u] = e < bl ? bufa[e] : 0.0;
                xb[u] = e < bl ? bufb[e] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int e = e0 + 32 * u;
                if (e < bl) {
                    pa[e] = xs[u] * xa[u];
                    pb[e] = xs[u] * xb[u];
                }
            }
        }
        __syncwarp();
        if (mine) s = chain_sum(s, lane < 4 ? pa : pb, bl, q);
        __syncwarp();
    }
    // the <4 tail elements are still in the last chunk's buffers
    const int64_t lastbase = (nch - 1) * CQ;
    const double *la = qa(nch - 1) + offa - lastbase, *lb = qb(nch - 1) + offb - lastbase;
    double tot = 0.0;
    if (lane < 4)
        tot = chain_finish(s, c, [&](int64_t x) { return sa[x]; }, [&](int64_t x) { return la[x]; }, 0xfu);
    else if (lane < 8)
        tot = chain_finish(s, c, [&](int64_t x) { return sa[x]; }, [&](int64_t x) { return lb[x]; }, 0xf0u);
    *dota = __shfl_sync(0xffffffffu, tot, 0);
    *dotb = __shfl_sync(0xffffffffu, tot, 4);
}

// Per-CTA argmax records double as the grid barrier. A record is four 8-byte
// words, each carrying the step flag in its high half, so a reader that sees
// the flag in all four words holds the whole record (8-byte accesses are
// single-copy atomic) -- the LL-protocol idea. The writer fences after the
// CTA barrier (its columns become visible first); readers fence after
// polling. One L2 round trip per step replaces barrier + partials read.
CQ_DEVI void rec_publish(unsigned long long *slot, uint32_t flag, double v, int32_t idx, int32_t phys) {
    const unsigned long long f = (unsigned long long)flag << 32;
    const unsigned long long w0 = f | (uint32_t)__double2hiint(v), w1 = f | (uint32_t)__double2loint(v);
    const unsigned long long w2 = f | (uint32_t)idx, w3 = f | (uint32_t)phys;
    asm volatile("fence.acq_rel.gpu;" ::: "memory");  // release: the CTA's writes (ordered by bar.sync) first
    asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(slot), "l"(w0), "l"(w1) : "memory");
    asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(slot + 2), "l"(w2), "l"(w3) : "memory");
}

CQ_DEVI void rec_wait(const unsigned long long *slot, uint32_t flag, double *v, int32_t *idx, int32_t *phys) {
    unsigned long long w0, w1, w2, w3;
    for (;;) {
        asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(slot) : "memory");
        asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(w2), "=l"(w3) : "l"(slot + 2) : "memory");
        if ((uint32_t)(w0 >> 32) == flag && (uint32_t)(w1 >> 32) == flag && (uint32_t)(w2 >> 32) == flag &&
            (uint32_t)(w3 >> 32) == flag)
            break;
    }
    *v = __hiloint2double((int)(uint32_t)w0, (int)(uint32_t)w1);
    *idx = (int32_t)(uint32_t)w2;
    *phys = (int32_t)(uint32_t)w3;
}

// A flagged double (two 8-byte words: flag | hi, flag | lo), same protocol.
CQ_DEVI void dbl_publish(unsigned long long *slot, uint32_t flag, double v) {
    const unsigned long long f = (unsigned long long)flag << 32;
    asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(slot),
                 "l"(f | (uint32_t)__double2hiint(v)), "l"(f | (uint32_t)__double2loint(v))
                 : "memory");
}
CQ_DEVI double dbl_wait(const unsigned long long *slot, uint32_t flag) {
    unsigned long long w0, w1;
    do {
        asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(slot) : "memory");
    } while ((uint32_t)(w0 >> 32) != flag || (uint32_t)(w1 >> 32) != flag);
    return __hiloint2double((int)(uint32_t)w0, (int)(uint32_t)w1);
}

// argmax carrying the winner's physical column
struct ArgMax3 {
    double v;
    int32_t i, p;
};
CQ_DEVI ArgMax3 argmax3_combine(ArgMax3 a, ArgMax3 b) {
    if (b.v > a.v || (b.v == a.v && b.i < a.i)) return b;
    return a;
}
CQ_DEVI ArgMax3 warp_argmax3(ArgMax3 a) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        ArgMax3 b;
        b.v = __shfl_xor_sync(0xffffffffu, a.v, o);
        b.i = __shfl_xor_sync(0xffffffffu, a.i, o);
        b.p = __shfl_xor_sync(0xffffffffu, a.p, o);
        a = argmax3_combine(a, b);
    }
    return a;
}

// One warp waits for the G records of a step (lane l: records l, l+32, ...,
// all loads of a pass in flight together) and returns their argmax.
CQ_DEVI ArgMax3 poll_records(const unsigned long long *recs, int G, uint32_t flag, int lane) {
    ArgMax3 best{-INFINITY, 0x7fffffff, 0};
    unsigned pending = 0;
    for (int r = 0; r < 8; ++r)
        if (lane + 32 * r < G) pending |= 1u << r;
    while (pending) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            if (!(pending & (1u << r))) continue;
            const unsigned long long *slot = recs + (size_t)(lane + 32 * r) * 4;
            unsigned long long w0, w1, w2, w3;
            asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(slot) : "memory");
            asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(w2), "=l"(w3) : "l"(slot + 2) : "memory");
            if ((uint32_t)(w0 >> 32) == flag && (uint32_t)(w1 >> 32) == flag && (uint32_t)(w2 >> 32) == flag &&
                (uint32_t)(w3 >> 32) == flag) {
                pending &= ~(1u << r);
                best = argmax3_combine(best, ArgMax3{__hiloint2double((int)(uint32_t)w0, (int)(uint32_t)w1),
                                                     (int32_t)(uint32_t)w2, (int32_t)(uint32_t)w3});
            }
        }
    }
    return warp_argmax3(best);
}

struct QrcpArgs {
    int64_t d, n, ld;
    double *b;
    double *w[2];
    double *wref;
    int32_t *cmap[2];
    int32_t *piv;     // physical pivot chosen at each step
    double *alpha;    // R(i,i)
    unsigned long long *rec;  // [2][256][4] flagged argmax records (value hi/lo, index, physical column)
    unsigned long long *tsq;  // [n][2] flagged next-step reflector tails sum of squares, by physical column
    int64_t *k_out;
    int32_t *final_buf;  // which cmap buffer holds positions >= k
    double rank_tol;
    int64_t steps;
    int64_t steps_grid;  // steps run by this kernel; the cluster kernel takes [steps_grid, steps)
    double *stop_out;    // rank_tol * max_norm0, for the cluster kernel
    int wb;                     // per-warp buffer (doubles, multiple of 32)
    int general;                // 1: never take the fast column phase (tests)
    int xlen;                   // pivot buffer length (doubles, >= d + 2, even)
    unsigned long long *trace;  // optional per-step phase timestamps (CTA 0)
};


__global__ void __launch_bounds__(kQrcpThreads, 1) qrcp_kernel(QrcpArgs A) {
    extern __shared__ __align__(16) double smem[];
    __shared__ double s_av[kQrcpWarps];
    __shared__ int32_t s_ai[kQrcpWarps], s_ap[kQrcpWarps];
    __shared__ double s_bc[4];
    __shared__ int s_poff;
    __shared__ double s_ct[kQrcpWarps], s_tau[kQrcpWarps];  // fast column phase: R(i,j), tau per warp
    __shared__ int s_coff[kQrcpWarps];                        // column offset in its warp buffer (-1: none)
    __shared__ int32_t s_cpj[kQrcpWarps];                     // its physical column
    __shared__ double s_tsq;                                  // the pivot's speculative tail_sq
    __shared__ double s_pv;                                   // this step's pivot: value, position, column
    __shared__ int32_t s_pi, s_pp;
    __shared__ double s_cv[2][kQrcpWarps];                    // warp candidates, by step parity
    __shared__ int32_t s_ci[2][kQrcpWarps], s_cp[2][kQrcpWarps];
    const int G = gridDim.x, cta = blockIdx.x;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t d = A.d, n = A.n, ld = A.ld;
    const int WB = A.wb;
    double *wb = smem + wid * WB;                // warp buffer: two halves b0/b1
    double *b0 = wb, *b1 = wb + WB / 2;
    const int CHD = ((WB / 2) - 2) & ~3;         // data doubles per chunk (alignment slack 2)
    // all-resident phase: a column's rows i..d-1 may use the whole warp buffer
    // (its norm recompute and next-step tail form their squares on the fly)
    const int CAPF = (WB - 8) & ~3;
    // general phase, two columns per warp at once: quarter-buffer chunks
    const int CQ = ((WB / 2 - 12) / 2) & ~3;
    double *s_x = smem + kQrcpWarps * WB;        // pivot column rows i..d-1 (+ alignment slack)
    double *s_sv = s_x + A.xlen;                 // products, then the scaled reflector (d doubles)
    const double sqrt_u = sqrt(kUnitRoundoff);
    // Speculative reflector tails: when every CTA is in the fast column phase
    // at step i (all columns resident), each warp finishes step i by forming
    // dot(col[i+2:], col[i+2:]) of its updated column in the reference order
    // (the tail_sq of make_reflector, linalg.cc:113-114, should that column be
    // the pivot of step i+1) while the grid barrier is in flight; step i+1
    // then reads the pivot's value instead of running that ordered chain.
    auto spec_at = [&](int64_t i) {
        return !A.general && i >= 0 && (n - i - 1) <= (int64_t)kQrcpWarps * G && (d - i - 1) <= (int64_t)CAPF;
    };

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
        if (lane < kQrcpWarps) {
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
    for (int64_t j = cta + (int64_t)wid * G; j < n; j += (int64_t)kQrcpWarps * G) {
        bool kept;
        double s = stream_dot(nullptr, A.b + j * ld, d, b0, b1, CHD, false, &kept, lane);
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
        if (threadIdx.x == 0) rec_publish(A.rec + (size_t)cta * 4, 1u, loc.v, loc.i, bp);  // consumed at step 0
    }

    double stop = 0.0;
    int64_t k = 0;
    int64_t i = 0;
    // Fast column phase (<= 8 remaining positions per CTA, tails fit a half
    // buffer): warp w owns the CTA's position k = w (mod 8) for good and keeps
    // its column resident in b0 across steps (rb[r] = row r), with its physical
    // index and norms in registers; only the warp that receives the column
    // swapped out of position i restages from global memory.
    bool resident = false;
    double *rb = b0;
    int32_t r_pj = 0;
    double r_w = 0.0, r_wref = 0.0;
    for (; i < A.steps_grid; ++i) {
        const int cur = (int)(i & 1), nxt = cur ^ 1;
        const int64_t c = d - i - 1;  // rows below the diagonal
        const int64_t body = c & ~(int64_t)3;
        trace_mark(A.trace, i, 0);

        const int64_t jfirst = i + 1 + ((cta - (i + 1)) % G + G) % G;
        const int64_t ncol_cta = (jfirst < n) ? (n - jfirst + G - 1) / G : 0;
        const bool fast = ncol_cta <= kQrcpWarps && c <= CAPF && !A.general;
        int64_t j_w;
        if (fast) {
            const int64_t kf = (jfirst - cta) / G;
            j_w = cta + (kf + (((int64_t)wid - kf) % kQrcpWarps + kQrcpWarps) % kQrcpWarps) * G;
        } else {
            j_w = jfirst + (int64_t)wid * G;
        }
        // ---- general path: prefetch chunk 0 of this warp's first owned column
        // (async, independent of the pivot decision; own columns were written
        // by this CTA at the previous step)
        int32_t pj0 = 0;
        double wj0 = 0.0, wrefj0 = 0.0, t0 = 0.0;
        const bool pair_first = !fast && j_w + (int64_t)kQrcpWarps * G < n;  // first iteration takes two columns
        if (!fast && j_w < n && !pair_first) {
            pj0 = ld_cg(A.cmap[cur] + j_w);
            wj0 = ld_cg(A.w[cur] + j_w);
            wrefj0 = ld_cg(A.wref + j_w);
            const double *col = A.b + (int64_t)pj0 * ld;
            stage_async(b0, col + i + 1, cmin<int64_t>(CHD, c), lane, 32);
            cp_async_commit();
            t0 = ld_cg(col + i);
        }
        // ---- grid barrier + pivot: warp 0 polls every CTA's record of the
        // previous step (lane l: records l, l+32, ...) and reduces them --
        // lowest index attaining the max (qrcp.cc:26-31; the rule is order
        // independent); its acquire fence + one CTA barrier publish the pivot
        if (wid == 0) {
            const ArgMax3 gw = poll_records(A.rec + (size_t)cur * 256 * 4, G, (uint32_t)(i + 1), lane);
            asm volatile("fence.acq_rel.gpu;" ::: "memory");  // acquire: the records' writers' data
            if (lane == 0) {
                s_pv = gw.v;
                s_pi = gw.i;
                s_pp = gw.p;
            }
        }
        __syncthreads();
        trace_mark(A.trace, i, 11);
        ArgMax g{s_pv, s_pi};
        const int32_t phys_p = s_pp;
        trace_mark(A.trace, i, 12);
        if (i == 0) {
            stop = A.rank_tol * sqrt(fmax(g.v, 0.0));  // max_norm0 (qrcp.cc:52-55)
            if (cta == 0 && threadIdx.x == 0) *A.stop_out = stop;
        }
        const double wp = g.v;
        const int64_t p = g.i;
        if (sqrt(wp > 0.0 ? wp : 0.0) <= stop) {
            cp_async_wait<0>();
            break;  // qrcp.cc:62
        }
        const double *x = A.b + (int64_t)phys_p * ld;
        trace_mark(A.trace, i, 1);

        // ---- make_reflector (linalg.cc:110-124), redundantly per CTA ------
        bool restage = false;
        {
            const int off = stage_async(s_x, x + i, d - i, threadIdx.x, kQrcpThreads);
            if (threadIdx.x == 0) s_poff = off;
            cp_async_commit();
            // the pivot's speculative tail (another L2 round trip) overlaps the copy
            if (threadIdx.x == 32 && spec_at(i - 1)) s_tsq = dbl_wait(A.tsq + 2 * (size_t)phys_p, (uint32_t)(i + 1));
            // fast path: a warp whose column is not resident yet (first fast
            // step), or that receives the column swapped out of position i,
            // stages rows i..d-1 of it after its share of the pivot column; the
            // reflector does not wait for that copy, the column phase does.
            if (fast && j_w < n && (!resident || j_w == p)) {
                if (j_w == p) {  // the column from position i (written last step)
                    r_pj = ld_cg(A.cmap[cur] + i);
                    r_w = ld_cg(A.w[cur] + i);
                    r_wref = ld_cg(A.wref + i);
                } else {
                    r_pj = ld_cg(A.cmap[cur] + j_w);
                    r_w = ld_cg(A.w[cur] + j_w);
                    r_wref = ld_cg(A.wref + j_w);
                }
                const double *colr = A.b + (int64_t)r_pj * ld;
                const int64_t base = (i - (d - CAPF - 1)) & ~(int64_t)1;  // even slot for row i (>= 0)
                const int offr = stage_async(b0 + base, colr + i, d - i, lane, 32);
                rb = b0 + base + offr - i;
                cp_async_commit();
                restage = true;
            }
            if (restage)
                cp_async_wait<1>();
            else
                cp_async_wait<0>();  // also completes the general path's column prefetch
            __syncthreads();
        }
        trace_mark(A.trace, i, 8);
        const double *xs = s_x + s_poff;  // xs[0] = x_i, xs[1 + e] = tail element e
        auto reflector_scalars = [&](double tail_sq) {
            double x0 = xs[0];
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
        };
        if (spec_at(i - 1)) {  // the pivot's owner formed tail_sq at step i-1
            if (threadIdx.x == 0) reflector_scalars(s_tsq);
            trace_mark(A.trace, i, 9);
        } else {
            for (int e0 = threadIdx.x; e0 < (int)body; e0 += 4 * kQrcpThreads) {
                double xv[4];
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    xv[u] = e0 + u * kQrcpThreads < (int)body ? xs[1 + e0 + u * kQrcpThreads] : 0.0;
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (e0 + u * kQrcpThreads < (int)body) s_sv[e0 + u * kQrcpThreads] = xv[u] * xv[u];
            }
            __syncthreads();
            trace_mark(A.trace, i, 9);
            if (wid == 0 && lane < 4) {
                double s = chain_sum(0.0, s_sv, body, lane);
                double tail_sq = chain_finish(s, c, [&](int64_t e) { return xs[1 + e]; },
                                              [&](int64_t e) { return xs[1 + e]; });
                if (lane == 0) reflector_scalars(tail_sq);
            }
        }
        __syncthreads();
        trace_mark(A.trace, i, 10);
        const double alpha = s_bc[0], v0 = s_bc[1], beta = s_bc[2];
        for (int r0 = threadIdx.x; r0 < (int)c; r0 += 4 * kQrcpThreads) {  // colj[i] /= v0
            double xv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) xv[u] = r0 + u * kQrcpThreads < (int)c ? xs[1 + r0 + u * kQrcpThreads] : 0.0;
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (r0 + u * kQrcpThreads < (int)c) s_sv[r0 + u * kQrcpThreads] = (beta != 0.0) ? xv[u] / v0 : xv[u];
        }
        __syncthreads();
        const double *sv = s_sv;
        trace_mark(A.trace, i, 2);

        // ---- apply_reflector + norm downdate --------------------------------
        ArgMax mine{-INFINITY, 0x7fffffff};
        int32_t minep = 0;
        bool spec_has = false;  // this warp holds a resident column to form the next tail for
        if (fast) {
            // Every warp's column is resident in its b0 (rb[r] = row r). Warp 0
            // runs the CTA's <= 8 dots at once: lanes 4g..4g+3 are the
            // reference's four accumulators for the column of warp g, products
            // formed on the fly; warp buffers are 4 doubles apart modulo 16
            // (+-1 for alignment), so one load feeds all 8 columns in about two
            // wavefronts. Then each warp updates its own column.
            if (restage) {
                cp_async_wait<0>();
                __syncwarp();
            }
            const bool has = j_w < n;
            const int32_t pj = r_pj;
            const double wj = r_w, wrefj = r_wref;
            double t = has ? rb[i] : 0.0;
            double *col = A.b + (int64_t)pj * ld;
            double *tail = col + i + 1;
            if (lane == 0) {
                s_ct[wid] = t;
                s_coff[wid] = has ? (int)(rb + i + 1 - smem) : -1;
                s_cpj[wid] = pj;
            }
            __syncthreads();
            trace_mark(A.trace, i, 5);
            if (wid == 0 && beta != 0.0) {  // apply_reflector's dot (linalg.cc:126-136)
                const int gq = lane >> 2, q = lane & 3;
                const int go = s_coff[gq];
                const double *cg = smem + (go > 0 ? go : 0);
                double sacc = 0.0;
                if (go >= 0) {
                    // the next group's loads are issued before this group's
                    // adds: only the dependent DADDs remain on the chain
                    const int bd = (int)body;
                    int e = q;
                    if (e + 28 < bd) {
                        double xa[8], xb[8];
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            xa[u] = sv[e + 4 * u];
                            xb[u] = cg[e + 4 * u];
                        }
                        for (e += 32; e + 28 < bd; e += 32) {
                            double na[8], nb[8];
#pragma unroll
                            for (int u = 0; u < 8; ++u) {
                                na[u] = sv[e + 4 * u];
                                nb[u] = cg[e + 4 * u];
                            }
#pragma unroll
                            for (int u = 0; u < 8; ++u) sacc = sacc + xa[u] * xb[u];
#pragma unroll
                            for (int u = 0; u < 8; ++u) {
                                xa[u] = na[u];
                                xb[u] = nb[u];
                            }
                        }
#pragma unroll
                        for (int u = 0; u < 8; ++u) sacc = sacc + xa[u] * xb[u];
                    }
                    for (; e < bd; e += 4) sacc = sacc + sv[e] * cg[e];
                }
                const double pair = sacc + __shfl_xor_sync(0xffffffffu, sacc, 1);
                double tot = pair + __shfl_xor_sync(0xffffffffu, pair, 2);
                if (q == 0 && go >= 0) {
                    int64_t e = body, rem = c - body;
                    if (rem >= 2) {
                        tot = tot + sv[e] * cg[e];
                        tot = tot + sv[e + 1] * cg[e + 1];
                        e += 2;
                        rem -= 2;
                    }
                    if (rem == 1) tot = fma(sv[e], cg[e], tot);
                    double tau = s_ct[gq];
                    tau += tot;
                    tau *= beta;
                    s_tau[gq] = tau;
                }
            }
            __syncthreads();
            trace_mark(A.trace, i, 6);
            if (has) {
                const double tau = (beta != 0.0) ? s_tau[wid] : 0.0;
                if (beta != 0.0) t = t - tau;
                double updated = fma(-t, t, wj);  // qrcp.cc:77-78
                double newref = wrefj;
                const bool recompute = updated <= sqrt_u * wrefj;  // qrcp.cc:82-86 (warp-uniform)
                if (recompute && A.trace && lane == 0 && i < 4096)
                    atomicAdd(&A.trace[((int64_t)blockIdx.x * 4096 + i) * 16 + 14], 1ULL);  // recompute count
                double *cb = rb + i + 1;
                if (beta != 0.0) {
                    const int ci = (int)c;
                    for (int e0 = lane; e0 < ci; e0 += 256) {
                        double xv[8], xc[8];
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            const int e = e0 + 32 * u;
                            xv[u] = e < ci ? sv[e] : 0.0;
                            xc[u] = e < ci ? cb[e] : 0.0;
                        }
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            const int e = e0 + 32 * u;
                            if (e < ci) {
                                const double nv = fma(-tau, xv[u], xc[u]);
                                cb[e] = nv;  // stays resident for the next step
                                __stcg(tail + e, nv);
                            }
                        }
                    }
                    __syncwarp();
                }
                if (recompute) {  // squares formed on the fly (same rounded products)
                    double s2 = 0.0;
                    if (lane < 4) {
                        s2 = chain_sq(0.0, cb, (int)body, lane);
                        s2 = chain_finish(s2, c, [&](int64_t e) { return cb[e]; }, [&](int64_t e) { return cb[e]; });
                    }
                    updated = __shfl_sync(0xffffffffu, s2, 0);
                    newref = updated;
                    __syncwarp();
                }
                if (lane == 0) {
                    __stcg(col + i, t);
                    __stcg(A.w[nxt] + j_w, updated);
                    __stcg(A.wref + j_w, newref);
                    __stcg(A.cmap[nxt] + j_w, pj);
                }
                r_w = updated;
                r_wref = newref;
                const ArgMax cnd = argmax_combine(mine, ArgMax{updated, (int32_t)j_w});
                if (cnd.i != mine.i) minep = pj;
                mine = cnd;
            }
            resident = true;
            spec_has = has;
            trace_mark(A.trace, i, 7);
        }
        bool first = true;
        for (int64_t j = fast ? n : j_w; j < n; j += (int64_t)kQrcpWarps * G, first = false) {
            if (j + (int64_t)kQrcpWarps * G < n) {
                // ---- two columns at once (the second is this warp's next) ----
                const int64_t jB = j + (int64_t)kQrcpWarps * G;
                int32_t pjA, pjB;
                double wA, wB, wrA, wrB, tA, tB;
                {
                    const int64_t jsA = (j == p) ? i : j, jsB = (jB == p) ? i : jB;
                    pjA = ld_cg(A.cmap[cur] + jsA);
                    pjB = ld_cg(A.cmap[cur] + jsB);
                    wA = ld_cg(A.w[cur] + jsA);
                    wB = ld_cg(A.w[cur] + jsB);
                    wrA = ld_cg(A.wref + jsA);
                    wrB = ld_cg(A.wref + jsB);
                    tA = ld_cg(A.b + (int64_t)pjA * ld + i);
                    tB = ld_cg(A.b + (int64_t)pjB * ld + i);
                }
                double *colA = A.b + (int64_t)pjA * ld, *colB = A.b + (int64_t)pjB * ld;
                double *tailA = colA + i + 1, *tailB = colB + i + 1;
                const int QS = CQ + 4;
                const int offA = (int)((reinterpret_cast<uintptr_t>(tailA) >> 3) & 1);
                const int offB = (int)((reinterpret_cast<uintptr_t>(tailB) >> 3) & 1);
                __syncwarp();
                if (beta != 0.0) {  // apply_reflector (linalg.cc:126-136) to both
                    bool kept2 = false;
                    double dA, dB;
                    stream_dot2(sv, tailA, tailB, c, b0, b1, CQ, &kept2, lane, &dA, &dB);
                    double tauA = tA, tauB = tB;
                    tauA += dA;
                    tauB += dB;
                    tauA *= beta;
                    tauB *= beta;
                    tA = tA - tauA;
                    tB = tB - tauB;
                    if (kept2) {  // both columns still staged in b0
                        const double *cbA = b0 + offA, *cbB = b0 + QS + offB;
                        for (int64_t e = lane; e < c; e += 32) {
                            const double sve = sv[e];
                            __stcg(tailA + e, fma(-tauA, sve, cbA[e]));
                            __stcg(tailB + e, fma(-tauB, sve, cbB[e]));
                        }
                    } else {  // restream both (double-buffered quarter chunks)
                        const int64_t nch = (c + CQ - 1) / CQ;
                        stage_async(b0, tailA, cmin<int64_t>(CQ, c), lane, 32);
                        stage_async(b0 + QS, tailB, cmin<int64_t>(CQ, c), lane, 32);
                        cp_async_commit();
                        for (int64_t kk = 0; kk < nch; ++kk) {
                            if (kk + 1 < nch) {
                                const int64_t nb = (kk + 1) * CQ, nl = cmin<int64_t>(CQ, c - nb);
                                double *h = ((kk + 1) & 1) ? b1 : b0;
                                stage_async(h, tailA + nb, nl, lane, 32);
                                stage_async(h + QS, tailB + nb, nl, lane, 32);
                                cp_async_commit();
                                cp_async_wait<1>();
                            } else {
                                cp_async_wait<0>();
                            }
                            __syncwarp();
                            const double *h = (kk & 1) ? b1 : b0;
                            const double *bufA = h + offA, *bufB = h + QS + offB;
                            const int64_t base = kk * CQ, len = cmin<int64_t>(CQ, c - base);
#pragma unroll 4
                            for (int64_t e = lane; e < len; e += 32) {
                                const double sve = sv[base + e];
                                __stcg(tailA + base + e, fma(-tauA, sve, bufA[e]));
                                __stcg(tailB + base + e, fma(-tauB, sve, bufB[e]));
                            }
                            __syncwarp();
                        }
                    }
                    __syncwarp();
                }
                // downdates (qrcp.cc:77-88); a recompute re-reads the updated column
                double updA = fma(-tA, tA, wA), updB = fma(-tB, tB, wB);
                double refA = wrA, refB = wrB;
                if (updA <= sqrt_u * wrA) {
                    bool k2;
                    updA = stream_dot(nullptr, tailA, c, b0, b1, CHD, false, &k2, lane);
                    refA = updA;
                }
                if (updB <= sqrt_u * wrB) {
                    bool k2;
                    updB = stream_dot(nullptr, tailB, c, b0, b1, CHD, false, &k2, lane);
                    refB = updB;
                }
                if (lane == 0) {
                    __stcg(colA + i, tA);
                    __stcg(A.w[nxt] + j, updA);
                    __stcg(A.wref + j, refA);
                    __stcg(A.cmap[nxt] + j, pjA);
                    __stcg(colB + i, tB);
                    __stcg(A.w[nxt] + jB, updB);
                    __stcg(A.wref + jB, refB);
                    __stcg(A.cmap[nxt] + jB, pjB);
                }
                ArgMax cnd = argmax_combine(mine, ArgMax{updA, (int32_t)j});
                if (cnd.i != mine.i) minep = pjA;
                mine = cnd;
                cnd = argmax_combine(mine, ArgMax{updB, (int32_t)jB});
                if (cnd.i != mine.i) minep = pjB;
                mine = cnd;
                __syncwarp();
                j = jB;  // the loop step moves past the pair
                continue;
            }
            const bool isp = (j == p);
            int32_t pj;
            double wj, wrefj, t;
            bool pre = false;
            if (first && !isp) {
                pj = pj0;
                wj = wj0;
                wrefj = wrefj0;
                t = t0;
                pre = true;  // chunk 0 of this column is already in flight into b0
            } else {
                if (first) {  // the prefetched column was the swapped one: drain it
                    cp_async_wait<0>();
                    __syncwarp();
                }
                // the pivot's position receives the column from position i
                // (written last step by CTA i % G, visible after the barrier)
                const int64_t js = isp ? i : j;
                pj = ld_cg(A.cmap[cur] + js);
                wj = ld_cg(A.w[cur] + js);
                wrefj = ld_cg(A.wref + js);
                t = ld_cg(A.b + (int64_t)pj * ld + i);
            }
            double *col = A.b + (int64_t)pj * ld;
            double *tail = col + i + 1;
            const int off = (int)((reinterpret_cast<uintptr_t>(tail) >> 3) & 1);
            bool kept = false;
            __syncwarp();
            if (beta != 0.0) {  // apply_reflector (linalg.cc:126-136)
                const double dot = stream_dot(sv, tail, c, b0, b1, CHD, pre, &kept, lane,
                                              (first && wid == 0) ? A.trace : nullptr, i);
                if (first && wid == 0) trace_mark(A.trace, i, 6);
                double tau = t;
                tau += dot;
                tau *= beta;
                t = t - tau;
                if (kept) {  // column still in b0: update from shared memory
                    double *cb = b0 + off;
                    const int ci = (int)c;
                    for (int e0 = lane; e0 < ci; e0 += 256) {
                        double xv[8], xc[8];
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            const int e = e0 + 32 * u;
                            xv[u] = e < ci ? sv[e] : 0.0;
                            xc[u] = e < ci ? cb[e] : 0.0;
                        }
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            const int e = e0 + 32 * u;
                            if (e < ci) {
                                const double nv = fma(-tau, xv[u], xc[u]);
                                cb[e] = nv;
                                __stcg(tail + e, nv);
                            }
                        }
                    }
                } else {  // restream the column (double-buffered)
                    const int64_t nch = (c + CHD - 1) / CHD;
                    stage_async(b0, tail, cmin<int64_t>(CHD, c), lane, 32);
                    cp_async_commit();
                    for (int64_t kk = 0; kk < nch; ++kk) {
                        if (kk + 1 < nch) {
                            stage_async(((kk + 1) & 1) ? b1 : b0, tail + (kk + 1) * CHD,
                                        cmin<int64_t>(CHD, c - (kk + 1) * CHD), lane, 32);
                            cp_async_commit();
                            cp_async_wait<1>();
                        } else {
                            cp_async_wait<0>();
                        }
                        __syncwarp();
                        const double *buf = ((kk & 1) ? b1 : b0) + off;
                        const int64_t base = kk * CHD, len = cmin<int64_t>(CHD, c - base);
#pragma unroll 8
                        for (int64_t e = lane; e < len; e += 32)
                            __stcg(tail + base + e, fma(-tau, sv[base + e], buf[e]));
                        __syncwarp();
                    }
                }
                __syncwarp();
            } else if (pre) {
                cp_async_wait<0>();  // drain the prefetch before b0 is reused
                __syncwarp();
            }
            if (first && wid == 0) trace_mark(A.trace, i, 7);
            double updated = fma(-t, t, wj);  // qrcp.cc:77-78
            double newref = wrefj;
            if (updated <= sqrt_u * wrefj) {  // qrcp.cc:82-86 (warp-uniform)
                if (kept) {                   // updated column is in b0
                    const double *cb = b0 + off;
                    for (int64_t e = lane; e < body; e += 32) b1[e] = cb[e] * cb[e];
                    __syncwarp();
                    double s = 0.0;
                    if (lane < 4) {
                        s = chain_sum(0.0, b1, body, lane);
                        s = chain_finish(s, c, [&](int64_t e) { return cb[e]; }, [&](int64_t e) { return cb[e]; });
                    }
                    updated = __shfl_sync(0xffffffffu, s, 0);
                    __syncwarp();
                } else {
                    bool k2;
                    updated = stream_dot(nullptr, tail, c, b0, b1, CHD, false, &k2, lane);
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
            // warp candidates (warp-uniform) -> slot [step parity][warp]; after
            // one barrier warp 0 reduces them and publishes the CTA's record
            // named barrier 1: only warp 0 (the publisher) waits; warps 1..7
            // arrive and go on to their speculative tails. Barrier 2 hands
            // warp 0's updated column to warp 1, which forms its tail.
            const bool spec_next = spec_at(i) && i + 1 < A.steps;
            if (lane == 0) {
                s_cv[cur][wid] = mine.v;
                s_ci[cur][wid] = mine.i;
                s_cp[cur][wid] = minep;
            }
            // (only in the all-resident phase: in the streaming phase the warp
            // -> position map shifts every step, so every warp must see its
            // siblings' map and tracker writes before the next step)
            if (!spec_next) {
                __syncthreads();
            } else if (wid == 0) {
                asm volatile("bar.arrive 2, 64;" ::: "memory");
                asm volatile("bar.sync 1, %0;" ::"r"(kQrcpThreads) : "memory");
            } else {
                asm volatile("bar.arrive 1, %0;" ::"r"(kQrcpThreads) : "memory");
            }
            if (wid == 0) {
                ArgMax3 r{-INFINITY, 0x7fffffff, 0};
                if (lane < kQrcpWarps) r = ArgMax3{s_cv[cur][lane], s_ci[cur][lane], s_cp[cur][lane]};
                r = warp_argmax3(r);
                trace_mark(A.trace, i, 13);
                if (lane == 0) {
                    if (cta == 0) {
                        __stcg(A.piv + i, phys_p);
                        __stcg(A.alpha + i, alpha);
                    }
                    rec_publish(A.rec + ((size_t)nxt * 256 + cta) * 4, (uint32_t)(i + 2), r.v, r.i, r.p);
                }
            }
        }
        k = i + 1;
        trace_mark(A.trace, i, 4);
        if (spec_at(i) && i + 1 < A.steps && wid >= 1) {
            // next step's tail of the resident columns: rows i+2..d-1, squares
            // then the reference's ordered chain, as in make_reflector. Warp 0
            // goes straight to the next grid poll; warp 1 runs warp 0's chain
            // (lanes 4..7) next to its own (lanes 0..3), so the chains overlap
            // the barrier instead of preceding it.
            const int64_t c2 = d - i - 2, body2 = c2 & ~(int64_t)3;
            if (wid == 1) asm volatile("bar.sync 2, 64;" ::: "memory");  // warp 0's column is updated
            const bool two = (wid == 1) && s_coff[0] >= 0;  // set this step
            const double *cbo = two ? smem + s_coff[0] + 1 : nullptr;  // warp 0's rows i+2..
            const bool mine_q = lane < 4 && spec_has, other_q = lane >= 4 && lane < 8 && two;
            double s2 = 0.0;
            if (mine_q || other_q) {  // squares formed on the fly (same rounded products)
                const double *cq = mine_q ? rb + i + 2 : cbo;
                s2 = chain_sq(0.0, cq, (int)body2, lane & 3);
                s2 = chain_finish(s2, c2, [&](int64_t e) { return cq[e]; }, [&](int64_t e) { return cq[e]; },
                                  mine_q ? 0xfu : 0xf0u);
            }
            if (lane == 0 && spec_has) dbl_publish(A.tsq + 2 * (size_t)r_pj, (uint32_t)(i + 2), s2);
            if (lane == 4 && two) dbl_publish(A.tsq + 2 * (size_t)s_cpj[0], (uint32_t)(i + 2), s2);
            __syncwarp();
        }
    }
    if (cta == 0 && threadIdx.x == 0) {
        *A.k_out = k;
        *A.final_buf = (int32_t)(k & 1);
    }
}

// ---------------------------------------------------------------------------
// K3b: the QRCP tail inside one thread-block cluster.
//
// Once the trailing matrix (rows i_s..d-1 of positions i_s..n-1) fits in the
// shared memory of a cluster (one column per warp, 16 warps per CTA, up to 16
// CTAs), the remaining steps run with every column resident: the per-CTA
// argmax records are exchanged through distributed shared memory after a
// hardware cluster barrier (instead of flagged records through L2 across the
// whole GPU), and every CTA reads the pivot column straight out of its owner's
// shared memory. Ownership follows the column, not the position: a swap only
// exchanges the two columns' position labels, no data moves. Arithmetic is
// the grid kernel's, operation for operation (make_reflector, apply_reflector,
// the downdate and its recompute in the reference's order), so R, J and k stay
// bit-identical.
// ---------------------------------------------------------------------------
constexpr int kClWarps = 16;
constexpr int kClThreads = kClWarps * 32;

struct QrcpClusterArgs {
    int64_t d, n, ld;
    double *b;
    const double *w_in, *wref_in;  // trackers at step i_s (by position)
    const int32_t *cmap_in;        // position -> column at step i_s (nullptr: identity)
    int32_t *cmap_out;             // final map for positions >= k (the buffer *final_buf names)
    int32_t *piv;
    double *alpha;
    int64_t *k_out;
    int32_t *final_buf;
    int fb_value;
    double rank_tol;
    const double *stop_in;  // nullptr: i_s == 0, computed here
    int64_t i_s, steps;
    int rows;  // buffer rows per warp (>= d - i_s)
    unsigned long long *trace;  // optional per-step phase clocks (CTA 0, thread 0)
};

CQ_DEVI uint32_t cl_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
CQ_DEVI uint32_t cl_map(uint32_t laddr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(laddr), "r"(rank));
    return r;
}
CQ_DEVI double cl_ld_f64(uint32_t a) {
    double v;
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
    return v;
}
CQ_DEVI int32_t cl_ld_s32(uint32_t a) {
    int32_t v;
    asm volatile("ld.shared::cluster.s32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
// cluster barrier with cluster-scope ordering only: the data exchanged inside
// the cluster phase is shared memory (the R entries written to global are read
// by the next kernel), so a .release arrive (a GPU-scope MEMBAR) is not needed
CQ_DEVI void cl_sync() {
    asm volatile(
        "fence.acq_rel.cluster;\nbarrier.cluster.arrive.relaxed.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::
            : "memory");
}

// the reference's dot (linalg.cc:36-50) of two shared arrays, one warp
CQ_DEVI double warp_ref_dot(const double *a, const double *bb, int64_t c, int lane) {
    double s = 0.0;
    if (lane < 4) {
        s = chain_dot(0.0, a, bb, (int)(c & ~(int64_t)3), lane);
        s = chain_finish(s, c, [&](int64_t e) { return a[e]; }, [&](int64_t e) { return bb[e]; });
    }
    return __shfl_sync(0xffffffffu, s, 0);
}

__global__ void __launch_bounds__(kClThreads, 1) qrcp_cluster_kernel(QrcpClusterArgs A) {
    extern __shared__ __align__(16) double smem[];
    __shared__ double s_cv[kClWarps];
    __shared__ int32_t s_cpos[kClWarps], s_cphys[kClWarps];
    // every CTA's record of the step (by parity), pushed here by its owner:
    // value, position, column, owner warp
    __shared__ double s_rv[2][16];
    __shared__ int32_t s_rpos[2][16], s_rphys[2][16], s_rown[2][16];
    __shared__ double s_pv, s_bc[3];
    __shared__ int32_t s_ppos, s_pphys, s_pown;
    __shared__ int s_stop;
    const int64_t d = A.d, n = A.n, ld = A.ld, i_s = A.i_s;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const uint32_t rank = cl_rank(), CS = gridDim.x;  // one cluster
    if (tid == 0) s_stop = 0;
    if (A.stop_in && __ldcg(A.k_out) < i_s) return;  // the grid phase already stopped (rank < i_s)
    const int R = A.rows;
    double *colbuf = smem + (size_t)wid * R;     // rows i_s..d-1 of this warp's column
    double *s_x = smem + (size_t)kClWarps * R;   // pivot rows i..d-1
    double *s_sv = s_x + R;                      // scaled reflector
    const double sqrt_u = sqrt(kUnitRoundoff);

    // ---- this warp's column: the one at position i_s + rank + CS * wid ----
    const int64_t pos0 = i_s + rank + (int64_t)CS * wid;
    const bool active = pos0 < n;
    int64_t pos = pos0;
    int32_t phys = 0;
    double w = 0.0, wref = 0.0;
    if (active) {
        phys = A.cmap_in ? __ldcg(A.cmap_in + pos0) : (int32_t)pos0;
        const double *g = A.b + (int64_t)phys * ld + i_s;
        // L2-only loads: nothing of this kernel lives in L1, so the L1
        // invalidation of every cluster barrier's acquire has nothing to drop
        for (int64_t r = lane; r < d - i_s; r += 32) colbuf[r] = __ldcg(g + r);
        __syncwarp();
        if (A.stop_in) {
            w = __ldcg(A.w_in + pos0);
            wref = __ldcg(A.wref_in + pos0);
        } else {  // initial squared norms (qrcp.cc:48-51)
            w = warp_ref_dot(colbuf, colbuf, d, lane);
            wref = w;
        }
    }
    double stop = A.stop_in ? __ldcg(A.stop_in) : 0.0;
    int64_t k = i_s;
    for (int64_t i = i_s; i < A.steps; ++i) {
        const int par = (int)(i & 1);
        if (A.trace && tid == 0 && rank == 0 && i - i_s < 4096) A.trace[(i - i_s) * 16 + 0] = clock64();
        // ---- argmax over positions >= i (qrcp.cc:26-31) -------------------
        if (lane == 0) {
            const bool cand = active && pos >= i;
            s_cv[wid] = cand ? w : -INFINITY;
            s_cpos[wid] = cand ? (int32_t)pos : 0x7fffffff;
            s_cphys[wid] = phys;
        }
        __syncthreads();
        if (wid == 0) {
            ArgMax3 r{-INFINITY, 0x7fffffff, 0};
            int32_t own = 0;
            if (lane < kClWarps) {
                r = ArgMax3{s_cv[lane], s_cpos[lane], s_cphys[lane]};
                own = lane;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                ArgMax3 b2{__shfl_xor_sync(0xffffffffu, r.v, o), __shfl_xor_sync(0xffffffffu, r.i, o),
                           __shfl_xor_sync(0xffffffffu, r.p, o)};
                const int32_t ob = __shfl_xor_sync(0xffffffffu, own, o);
                const ArgMax3 c2 = argmax3_combine(r, b2);
                if (c2.i != r.i || c2.v != r.v) own = ob;
                r = c2;
            }
            // lane q < CS pushes the record into CTA q's slot [par][rank]
            r.v = __shfl_sync(0xffffffffu, r.v, 0);
            r.i = __shfl_sync(0xffffffffu, r.i, 0);
            r.p = __shfl_sync(0xffffffffu, r.p, 0);
            own = __shfl_sync(0xffffffffu, own, 0);
            if (lane < (int)CS) {
                const int32_t ow2 = (int32_t)(rank * kClWarps) + own;
                asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(cl_map(smem_u32(&s_rv[par][rank]), lane)), "d"(r.v)
                             : "memory");
                asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(cl_map(smem_u32(&s_rpos[par][rank]), lane)),
                             "r"(r.i)
                             : "memory");
                asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(cl_map(smem_u32(&s_rphys[par][rank]), lane)),
                             "r"(r.p)
                             : "memory");
                asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(cl_map(smem_u32(&s_rown[par][rank]), lane)),
                             "r"(ow2)
                             : "memory");
            }
        }
        if (A.trace && tid == 0 && rank == 0 && i - i_s < 4096) A.trace[(i - i_s) * 16 + 1] = clock64();
        cl_sync();  // every CTA's record of this step has landed in every CTA
        if (A.trace && tid == 0 && rank == 0 && i - i_s < 4096) A.trace[(i - i_s) * 16 + 2] = clock64();
        if (wid == 0) {
            ArgMax3 r{-INFINITY, 0x7fffffff, 0};
            int32_t own = 0;
            if (lane < (int)CS) {
                r.v = s_rv[par][lane];
                r.i = s_rpos[par][lane];
                r.p = s_rphys[par][lane];
                own = s_rown[par][lane];
            }
            __syncwarp();
            if (A.trace && lane == 0 && rank == 0 && i - i_s < 4096) A.trace[(i - i_s) * 16 + 9] = clock64() + (unsigned long long)(r.v > 1e300 ? 1 : 0);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                ArgMax3 b2{__shfl_xor_sync(0xffffffffu, r.v, o), __shfl_xor_sync(0xffffffffu, r.i, o),
                           __shfl_xor_sync(0xffffffffu, r.p, o)};
                const int32_t ob = __shfl_xor_sync(0xffffffffu, own, o);
                const ArgMax3 c2 = argmax3_combine(r, b2);
                if (c2.i != r.i || c2.v != r.v) own = ob;
                r = c2;
            }
            if (A.trace && lane == 0 && rank == 0 && i - i_s < 4096) A.trace[(i - i_s) * 16 + 10] = clock64() + (unsigned long long)(r.v > 1e300 ? 1 : 0);
            if (lane == 0) {
                s_pv = r.v;
                s_ppos = r.i;
                s_pphys = r.p;
                s_pown = own;
                if (i == 0) stop = A.rank_tol * sqrt(fmax(r.v, 0.0));  // max_norm0 (qrcp.cc:52-55)
                s_stop = sqrt(r.v > 0.0 ? r.v : 0.0) <= stop ? 1 : 0;  // qrcp.cc:62
                if (A.trace && rank == 0 && i - i_s < 4096) A.trace[(i - i_s) * 16 + 8] = clock64();
            }
        }
        __syncthreads();
        if (A.trace && tid == 0 && rank == 0 && i - i_s < 4096) A.trace[(i - i_s) * 16 + 3] = clock64();
        if (s_stop) break;
        const int64_t p = s_ppos;
        const int32_t phys_p = s_pphys;
        const uint32_t oc = (uint32_t)s_pown / kClWarps, ow = (uint32_t)s_pown % kClWarps;
        // ---- pivot rows i..d-1 from its owner's shared memory -------------
        {
            const uint32_t src = cl_map(smem_u32(smem + (size_t)ow * R + (i - i_s)), oc);
            for (int64_t e = tid; e < d - i; e += kClThreads) s_x[e] = cl_ld_f64(src + 8u * (uint32_t)e);
        }
        __syncthreads();
        if (A.trace && tid == 0 && rank == 0 && i - i_s < 4096) A.trace[(i - i_s) * 16 + 4] = clock64();

        const int64_t c = d - i - 1;
        // ---- make_reflector (linalg.cc:110-124) -----------------------------
        const int64_t body = c & ~(int64_t)3;
        for (int64_t e = tid; e < body; e += kClThreads) s_sv[e] = s_x[1 + e] * s_x[1 + e];
        __syncthreads();
        if (wid == 0 && lane < 4) {
            double tail_sq = chain_sum(0.0, s_sv, body, lane);
            tail_sq = chain_finish(tail_sq, c, [&](int64_t e) { return s_x[1 + e]; },
                                   [&](int64_t e) { return s_x[1 + e]; });
            if (lane == 0) {
                const double x0 = s_x[0];
                const double norm_x = sqrt(fma(x0, x0, tail_sq));
                double alpha = x0, v0 = 1.0, beta = 0.0;
                if (norm_x != 0.0) {
                    const double sign = (x0 >= 0.0) ? 1.0 : -1.0;
                    alpha = -sign * norm_x;
                    v0 = x0 - alpha;
                    beta = (norm_x + fabs(x0)) / norm_x;
                }
                s_bc[0] = alpha;
                s_bc[1] = v0;
                s_bc[2] = beta;
                if (rank == 0) {
                    A.piv[i] = phys_p;
                    A.alpha[i] = alpha;
                }
            }
        }
        __syncthreads();
        const double v0 = s_bc[1], beta = s_bc[2];
        if (A.trace && tid == 0 && rank == 0 && i - i_s < 4096) A.trace[(i - i_s) * 16 + 5] = clock64();
        for (int64_t e = tid; e < c; e += kClThreads) s_sv[e] = (beta != 0.0) ? s_x[1 + e] / v0 : s_x[1 + e];
        __syncthreads();
        if (A.trace && tid == 0 && rank == 0 && i - i_s < 4096) A.trace[(i - i_s) * 16 + 6] = clock64();

        // ---- swap = relabel positions p <-> i ------------------------------
        if (pos == p) pos = i;
        else if (pos == i) pos = p;
        // ---- apply_reflector + downdate (linalg.cc:126-136, qrcp.cc:72-88) --
        if (active && pos > i) {
            double *col = colbuf + (i - i_s);  // col[0] = row i
            double t = col[0];
            if (beta != 0.0) {
                const double dot = warp_ref_dot(s_sv, col + 1, c, lane);
                double tau = t;
                tau += dot;
                tau *= beta;
                t = t - tau;
                for (int64_t e = lane; e < c; e += 32) col[1 + e] = fma(-tau, s_sv[e], col[1 + e]);
                __syncwarp();
            }
            double updated = fma(-t, t, w);  // qrcp.cc:77-78
            double newref = wref;
            if (updated <= sqrt_u * wref) {  // qrcp.cc:82-86
                updated = warp_ref_dot(col + 1, col + 1, c, lane);
                newref = updated;
            }
            w = updated;
            wref = newref;
            if (lane == 0) A.b[(int64_t)phys * ld + i] = t;  // R(i, j)
        }
        if (A.trace && tid == 0 && rank == 0 && i - i_s < 4096) A.trace[(i - i_s) * 16 + 7] = clock64();
        k = i + 1;
    }
    // positions >= k keep their columns (J tail); rank 0 reports k
    if (active && lane == 0 && pos >= k) A.cmap_out[pos] = phys;
    if (rank == 0 && tid == 0) {
        *A.k_out = k;
        *A.final_buf = A.fb_value;
    }
    cl_sync();  // no CTA exits while another may still read its shared memory
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
// Row masses: acc = acc + R(i,j)^2 over j ascending (not contracted as built);
// row max |R(i,:)| for max_abs (order-free). CTA = 32 rows: all 8 warps stage
// 32 x 64 column tiles (cp.async, coalesced, double-buffered, [c][33]) and
// warp 0 (lane = row) runs the rows' ordered chains from shared memory.
constexpr int kRsCols = 64, kRsLd = 33;

__global__ void __launch_bounds__(256) row_stats_kernel(int64_t k, int64_t n, const double *__restrict__ r,
                                                        int64_t ldr, double *__restrict__ mass,
                                                        double *__restrict__ rmax) {
    __shared__ __align__(16) double tile[2][kRsCols * kRsLd];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t i0 = (int64_t)blockIdx.x * 32;
    const int64_t ntile = (n + kRsCols - 1) / kRsCols;
    auto issue = [&](int64_t t, int buf) {
        const int64_t row = i0 + lane;
        for (int c = wid; c < kRsCols; c += 8) {
            const int64_t col = t * kRsCols + c;
            const bool ok = row < k && col < n;
            cp_async8_zfill(&tile[buf][c * kRsLd + lane], r + (ok ? col * ldr + row : 0), ok ? 8 : 0);
        }
        cp_async_commit();
    };
    issue(0, 0);
    const int64_t i = i0 + lane;
    double acc = 0.0, mx = 0.0;
    for (int64_t t = 0; t < ntile; ++t) {
        if (t + 1 < ntile) {
            issue(t + 1, (int)((t + 1) & 1));
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        if (wid == 0) {
            const double *tb = tile[t & 1];
            const int64_t jb = t * kRsCols;
            const int cols = (int)cmin<int64_t>(kRsCols, n - jb);
            for (int c = 0; c < cols; ++c) {
                const double v = tb[c * kRsLd + lane];
                mx = fmax(mx, fabs(v));
                if (jb + c >= i) acc = acc + v * v;
            }
        }
        __syncthreads();  // the buffer is refilled next iteration
    }
    if (wid == 0 && i < k) {
        mass[i] = acc;
        rmax[i] = mx;
    }
}

// Tail accumulation from the bottom, sequential as in the reference; the
// masses are staged in shared memory first (the scan is one thread).
constexpr int kStage1Smem = 6016;

__global__ void __launch_bounds__(1024) stage1_kernel(int64_t k, const double *__restrict__ mass,
                                                      const double *__restrict__ rmax, double u,
                                                      int64_t *__restrict__ k0_out) {
    __shared__ double s_red[32];
    __shared__ double s_mass[kStage1Smem];
    double mx = 0.0;
    for (int64_t i = threadIdx.x; i < k; i += blockDim.x) {
        mx = fmax(mx, rmax[i]);
        if (i < kStage1Smem) s_mass[i] = mass[i];
    }
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
        tail += (ell < kStage1Smem) ? s_mass[ell] : mass[ell];
        if (tail <= target) k0 = ell;
    }
    *k0_out = k0;
}

int qrcp(int64_t d, int64_t n, double *b, int64_t ldb, double rank_tol, double *rsk, int64_t ldr, int64_t *jdev,
         int64_t *k_sk, Workspace &ws, cudaStream_t st) {
    if (d < 1) return fail_internal("qrcp: need at least one row");
    if (rank_tol < 0.0) rank_tol = (double)n * kUnitRoundoff;  // qrcp.cc:17,38
    // One cooperative (grid-synchronising) QRCP per device at a time: host
    // threads sharing a GPU never have two co-residency-dependent grids live.
    static std::mutex mu;
    std::lock_guard<std::mutex> lock(mu);
    const int sms = num_sms();
    // shared memory: pivot buffer (d+2, even) + reflector (d) + 8 warp buffers
    const int64_t budget = (212 * 1024) / (int64_t)sizeof(double);
    const int xlen = (int)(((d + 2) + 1) & ~(int64_t)1);
    const int64_t room = budget - xlen - d;
    if (room < 8 * 128) return fail_internal("qrcp: d too large for the shared-memory reflector");
    // per warp: two halves; one half holds a whole column when it fits
    // +4: warp buffers 4 doubles apart modulo 16 (bank-staggered for the
    // fast path's 8-column chain loads); stays 16-byte aligned
    const int WB = (int)std::min<int64_t>(2 * (((d + 2 + 31) / 32) * 32), (room / 8) & ~(int64_t)63) + 4;
    const size_t smem = sizeof(double) * (size_t)(8 * (int64_t)WB + xlen + d);
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
    a.rec = ws.get<unsigned long long>("qrcp.rec", 2 * 256 * 4);
    a.tsq = ws.get<unsigned long long>("qrcp.tsq", 2 * (size_t)n);
    a.k_out = ws.get<int64_t>("qrcp.k", 2);
    a.final_buf = ws.get<int32_t>("qrcp.fb", 2);
    a.rank_tol = rank_tol;
    a.steps = std::min(d, n);
    a.stop_out = ws.get<double>("qrcp.stop", 1);
    // ---- cluster QRCP: positions i_s..n-1 (one column per warp, 16 warps per
    // CTA) with rows i_s..d-1 fit in one cluster's shared memory. 16 CTAs
    // (non-portable) when the GPU can co-schedule them, else 8.
    int cs = 0;
    int64_t i_s = a.steps;
    size_t cl_smem = 0;
    const bool cluster_ok = getenv("CQRRPT_QRCP_GENERAL") == nullptr && getenv("CQRRPT_QRCP_NOCLUSTER") == nullptr;
    if (cluster_ok) {
        static int cs_ok16_dev[64] = {0}, cs_ok8_dev[64] = {0};  // per device (attributes are per device)
        const int dev = current_device() & 63;
        int &cs_ok16 = cs_ok16_dev[dev], &cs_ok8 = cs_ok8_dev[dev];
        const int64_t rows_max = 1600;
        if (first_on_device((const void *)qrcp_cluster_kernel)) {
            const size_t smem_max = sizeof(double) * (size_t)(kClWarps + 2) * rows_max;
            cudaFuncSetAttribute(qrcp_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_max);
            cudaFuncSetAttribute(qrcp_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            for (int c2 : {16, 8}) {
                cudaLaunchConfig_t cfg = {};
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeClusterDimension;
                at[0].val.clusterDim.x = c2;
                at[0].val.clusterDim.y = 1;
                at[0].val.clusterDim.z = 1;
                cfg.gridDim = dim3(c2);
                cfg.blockDim = dim3(kClThreads);
                cfg.dynamicSmemBytes = smem_max;
                cfg.attrs = at;
                cfg.numAttrs = 1;
                int ncl = 0;
                if (cudaOccupancyMaxActiveClusters(&ncl, qrcp_cluster_kernel, &cfg) == cudaSuccess && ncl >= 1)
                    (c2 == 16 ? cs_ok16 : cs_ok8) = 1;
            }
            cudaGetLastError();
        }
        for (int c2 : {16, 8}) {
            if (!(c2 == 16 ? cs_ok16 : cs_ok8)) continue;
            const int64_t cand = std::max<int64_t>({0, n - (int64_t)c2 * kClWarps, d - rows_max});
            // measured (B200): ~10% faster per step than the grid kernel when
            // the whole factorization fits (C1, C5-256); for a tail after a
            // grid phase (C2: last 256 steps) it is no faster, so only then
            if (cand == 0 && a.steps >= 16) {
                cs = c2;
                i_s = cand;
                break;
            }
        }
        if (cs) {
            const int64_t rows = ((d - i_s) + 1) & ~(int64_t)1;
            cl_smem = sizeof(double) * (size_t)(kClWarps + 2) * (size_t)rows;
        }
    }
    a.steps_grid = i_s;
    a.wb = WB;
    a.xlen = xlen;
    // CQRRPT_QRCP_GENERAL=1 forces the general column phase (tests cover both)
    a.general = getenv("CQRRPT_QRCP_GENERAL") != nullptr ? 1 : 0;
    if (!a.w[0] || !a.rec || !a.tsq || !a.k_out) return fail_nomem("qrcp workspace");
    // flags restart at 1 every call: clear the previous call's records
    CQ_CUDA(cudaMemsetAsync(a.rec, 0, 2 * 256 * 4 * sizeof(unsigned long long), st), "memset records");
    CQ_CUDA(cudaMemsetAsync(a.tsq, 0, 2 * (size_t)n * sizeof(unsigned long long), st), "memset tails");
    static const bool tracing = getenv("CQRRPT_QRCP_TRACE") != nullptr;
    a.trace = tracing ? ws.get<unsigned long long>("qrcp.trace", 256 * 4096 * 16) : nullptr;
    if (a.trace)
        CQ_CUDA(cudaMemsetAsync(a.trace, 0, 256 * 4096 * 16 * sizeof(unsigned long long), st), "trace memset");
    if (i_s > 0) {
        void *args[] = {&a};
        CQ_CUDA(cudaLaunchCooperativeKernel((void *)qrcp_kernel, dim3(G), dim3(kQrcpThreads), args, smem, st),
                "qrcp cooperative launch");
        note_launch();
    }
    if (cs) {
        QrcpClusterArgs c{};
        c.d = d;
        c.n = n;
        c.ld = ldb;
        c.b = b;
        c.w_in = a.w[i_s & 1];
        c.wref_in = a.wref;
        c.cmap_in = i_s > 0 ? a.cmap[i_s & 1] : nullptr;
        c.cmap_out = a.cmap[0];
        c.piv = a.piv;
        c.alpha = a.alpha;
        c.k_out = a.k_out;
        c.final_buf = a.final_buf;
        c.fb_value = 0;
        c.rank_tol = rank_tol;
        c.stop_in = i_s > 0 ? a.stop_out : nullptr;
        c.i_s = i_s;
        c.steps = a.steps;
        c.rows = (int)(((d - i_s) + 1) & ~(int64_t)1);
        static const bool cl_tracing = getenv("CQRRPT_QRCP_TRACE") != nullptr;
        c.trace = cl_tracing ? ws.get<unsigned long long>("qrcp.cltrace", 4096 * 16) : nullptr;
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(cs);
        cfg.blockDim = dim3(kClThreads);
        cfg.dynamicSmemBytes = cl_smem;
        cfg.stream = st;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        CQ_CUDA(cudaLaunchKernelEx(&cfg, qrcp_cluster_kernel, c), "qrcp cluster launch");
        note_launch();
        if (c.trace) {
            std::vector<unsigned long long> h(4096 * 16);
            cudaStreamSynchronize(st);
            cudaMemcpy(h.data(), c.trace, h.size() * 8, cudaMemcpyDeviceToHost);
            const int64_t ns = std::min<int64_t>(a.steps - i_s - 1, 4095);
            double acc[8] = {0}, red = 0.0, ph[3] = {0, 0, 0};
            for (int64_t s2 = 0; s2 < ns; ++s2) {
                for (int q = 0; q < 7; ++q) acc[q] += (double)(h[s2 * 16 + q + 1] - h[s2 * 16 + q]);
                acc[7] += (double)(h[(s2 + 1) * 16] - h[s2 * 16 + 7]);
                red += (double)(h[s2 * 16 + 8] - h[s2 * 16 + 2]);
                ph[0] += (double)(h[s2 * 16 + 9] - h[s2 * 16 + 2]);
                ph[1] += (double)(h[s2 * 16 + 10] - h[s2 * 16 + 9]);
                ph[2] += (double)(h[s2 * 16 + 8] - h[s2 * 16 + 10]);
            }
            fprintf(stderr,
                    "qrcp cluster trace (CS=%d, i_s=%lld, %lld steps; SM cycles/step): cand %.0f, cl_sync %.0f, "
                    "pivot %.0f (warp-0 reduce %.0f), xfetch %.0f, reflector %.0f, divide %.0f, columns %.0f, loop %.0f\n",
                    cs, (long long)i_s, (long long)ns, acc[0] / ns, acc[1] / ns, acc[2] / ns, red / ns, acc[3] / ns,
                    acc[4] / ns, acc[5] / ns, acc[6] / ns, acc[7] / ns);
            fprintf(stderr, "   reduce split: loads %.0f, shuffles %.0f, stop test %.0f\n", ph[0] / ns, ph[1] / ns, ph[2] / ns);
        }
    }
    qrcp_extract_kernel<<<(unsigned)n, 128, 0, st>>>(d, n, b, ldb, a.k_out, a.piv, a.cmap[0], a.cmap[1],
                                                      a.final_buf, a.alpha, rsk, ldr, jdev);
    note_launch();
    CQ_TRY(check_launch("qrcp_extract_kernel"));
    CQ_CUDA(cudaMemcpyAsync(k_sk, a.k_out, sizeof(int64_t), cudaMemcpyDeviceToHost, st), "k_sk d2h");
    CQ_CUDA(cudaStreamSynchronize(st), "qrcp sync");
    if (a.trace) {  // debug: mean per-phase SM cycles per quarter of the steps
        std::vector<unsigned long long> h((size_t)G * 4096 * 16);
        cudaMemcpy(h.data(), a.trace, h.size() * 8, cudaMemcpyDeviceToHost);
        const int steps = (int)std::min<int64_t>(std::min<int64_t>(*k_sk, i_s), 4096) - 1;  // grid-kernel steps
        for (int qt = 0; qt < 4 && steps > 4; ++qt) {
            double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            int cnt = 0, cnt5 = 0;
            for (int s2 = qt * steps / 4; s2 < (qt + 1) * steps / 4; ++s2) {
                const unsigned long long *t = &h[s2 * 16];
                for (int q = 0; q < 4; ++q) acc[q] += (double)(t[q + 1] - t[q]);
                acc[4] += (double)(h[(s2 + 1) * 16] - t[4]);
                if (t[5] && t[6] && t[7]) {  // warp 0's first column: products, dot, update
                    acc[5] += (double)(t[5] - t[2]);
                    acc[6] += (double)(t[6] - t[5]);
                    acc[7] += (double)(t[7] - t[6]);
                    ++cnt5;
                }
                ++cnt;
            }
            cnt5 = cnt5 ? cnt5 : 1;
            double wmax = 0, wmean = 0, rmax = 0, cmax = 0, pmax = 0;  // own work (slot 1 -> 4) over CTAs
            int nst = 0;
            for (int s2 = qt * steps / 4; s2 < (qt + 1) * steps / 4; ++s2) {
                double mx = 0, mr = 0, mc = 0, mp = 0, sm = 0;
                for (int q2 = 0; q2 < G; ++q2) {
                    const unsigned long long *t = &h[((size_t)q2 * 4096 + s2) * 16];
                    const double w = (double)(t[4] - t[1]);
                    sm += w;
                    mx = std::max(mx, w);
                    mr = std::max(mr, (double)(t[2] - t[1]));
                    mc = std::max(mc, (double)(t[3] - t[2]));
                    mp = std::max(mp, (double)(t[4] - t[3]));
                }
                wmax += mx;
                wmean += sm / G;
                rmax += mr;
                cmax += mc;
                pmax += mp;
                ++nst;
            }
            {
                static const int seq[] = {0, 11, 12, 1, 8, 9, 10, 2, 3, 13, 4};
                static const char *nm[] = {"pre+poll", "pivot-argmax", "stop", "x-fetch", "squares", "norm-chain",
                                           "divide", "columns", "block-argmax", "publish"};
                double seg[10] = {0};
                long cntc = 0;
                for (int s2 = qt * steps / 4; s2 < (qt + 1) * steps / 4; ++s2)
                    for (int q2 = 0; q2 < G; ++q2, ++cntc) {
                        const unsigned long long *t = &h[((size_t)q2 * 4096 + s2) * 16];
                        for (int z = 0; z < 10; ++z) seg[z] += (double)(t[seq[z + 1]] - t[seq[z]]);
                    }
                fprintf(stderr, "   mean over CTAs:");
                for (int z = 0; z < 10; ++z) fprintf(stderr, " %s %.0f", nm[z], seg[z] / cntc);
                fprintf(stderr, "\n");
            }
            fprintf(stderr, "   own work over CTAs: mean %.0f, max %.0f (max reflector %.0f, columns %.0f, partials %.0f)\n",
                    wmean / nst, wmax / nst, rmax / nst, cmax / nst, pmax / nst);
            {
                long nrec = 0, steps_with = 0;
                for (int s2 = qt * steps / 4; s2 < (qt + 1) * steps / 4; ++s2) {
                    long ns = 0;
                    for (int q2 = 0; q2 < G; ++q2) ns += (long)h[((size_t)q2 * 4096 + s2) * 16 + 14];
                    nrec += ns;
                    steps_with += ns > 0;
                }
                fprintf(stderr, "   recomputes (fast phase): %ld, steps with >= 1: %ld of %d\n", nrec, steps_with, cnt);
            }
            fprintf(stderr,
                    "qrcp trace q%d (G=%d, d=%lld, n=%lld, WB=%d, %d steps; SM cycles): argmax %.0f, reflector %.0f, "
                    "columns %.0f (pre %.0f, chain %.0f, update %.0f), partials %.0f, barrier %.0f\n",
                    qt, G, (long long)d, (long long)n, WB, cnt, acc[0] / cnt, acc[1] / cnt, acc[2] / cnt,
                    acc[5] / cnt5, acc[6] / cnt5, acc[7] / cnt5, acc[3] / cnt, acc[4] / cnt);
        }
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
    row_stats_kernel<<<(unsigned)((k + 31) / 32), 256, 0, st>>>(k, n, r, ldr, mass, rmax);
    note_launch();
    stage1_kernel<<<1, 1024, 0, st>>>(k, mass, rmax, kUnitRoundoff, kd);
    note_launch();
    CQ_TRY(check_launch("stage1_kernel"));
    CQ_CUDA(cudaMemcpyAsync(k0, kd, sizeof(int64_t), cudaMemcpyDeviceToHost, st), "k0 d2h");
    CQ_CUDA(cudaStreamSynchronize(st), "stage1 sync");
    return 0;
}

}  // namespace cqg

// Host orchestration of the B200 CQRRPT pipeline and the C ABI
// (include/cqrrpt_gpu.h).
//
// Reference control flow: cqrrpt (cqrrpt.cc:317-328) -> cqrrpt_core
// (cqrrpt.cc:233-315) -> rank_stage2 (cqrrpt.cc:149-209). The phases, their
// kernels and where the two cross-GPU sums sit:
//
//   sketch      K1 plan + K2 apply            -> allreduce(d*n)       [rank-local rows]
//   qrcp        K3 cooperative QRCP           (replicated, deterministic)
//   rank_select K4 stage-1 + stage-2 search   (replicated)
//   precondition K5a gather+TRSM (DMMA)       [rank-local rows]
//   cholesky_qr K5b Gram (DMMA) -> allreduce(k0*k0) -> K6 potrf -> K8 Q TRSM
//   undo        K9 R = R_pre R_sk[:k,:]       (replicated)
#include <dlfcn.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <vector>

#include "common.cuh"
#include "internal.hh"

namespace cqg {
int64_t launch_count(bool reset);
const char *last_error();
}  // namespace cqg

using namespace cqg;

// ---------------------------------------------------------------------------
// NCCL via dlopen
// ---------------------------------------------------------------------------
namespace {
typedef int (*nccl_get_id_t)(void *);
struct NcclId {
    char internal[128];
};
typedef int (*nccl_init_rank2_t)(void **, int, NcclId, int);
typedef int (*nccl_allreduce_t)(const void *, void *, size_t, int, int, void *, cudaStream_t);
typedef int (*nccl_destroy_t)(void *);
typedef const char *(*nccl_errstr_t)(int);
struct NcclApi {
    bool loaded = false;
    nccl_get_id_t get_id = nullptr;
    nccl_init_rank2_t init_rank = nullptr;
    nccl_allreduce_t allreduce = nullptr;
    nccl_destroy_t destroy = nullptr;
    nccl_errstr_t errstr = nullptr;
};
NcclApi &nccl() {
    static NcclApi api;
    if (!api.loaded) {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (h) {
            api.get_id = (nccl_get_id_t)dlsym(h, "ncclGetUniqueId");
            api.init_rank = (nccl_init_rank2_t)dlsym(h, "ncclCommInitRank");
            api.allreduce = (nccl_allreduce_t)dlsym(h, "ncclAllReduce");
            api.destroy = (nccl_destroy_t)dlsym(h, "ncclCommDestroy");
            api.errstr = (nccl_errstr_t)dlsym(h, "ncclGetErrorString");
        }
        api.loaded = true;
    }
    return api;
}
}  // namespace

struct cqrrpt_gpu_comm {
    void *comm = nullptr;
    int nranks = 1, rank = 0;
};

// ---------------------------------------------------------------------------
// timing helper
// ---------------------------------------------------------------------------
namespace {
struct PhaseClock {
    bool on = false;
    cudaStream_t st = nullptr;
    cudaEvent_t ev[16];
    int n = 0;
    int tag[16];
    void start(bool enable, cudaStream_t s) {
        on = enable;
        st = s;
        n = 0;
        if (on) mark(-1);
    }
    void mark(int phase) {
        if (!on || n >= 16) return;
        cudaEventCreate(&ev[n]);
        cudaEventRecord(ev[n], st);
        tag[n++] = phase;
    }
    ~PhaseClock() {  // early (error) returns: events not consumed by finish()
        for (int i = 0; i < n; ++i) cudaEventDestroy(ev[i]);
    }
    void finish(double *out) {
        if (!on) return;
        cudaEventSynchronize(ev[n - 1]);
        for (int i = 0; i < 8; ++i) out[i] = 0.0;
        for (int i = 1; i < n; ++i) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, ev[i - 1], ev[i]);
            if (tag[i] >= 0 && tag[i] < 8) out[tag[i]] += ms;
        }
        float tot = 0.f;
        cudaEventElapsedTime(&tot, ev[0], ev[n - 1]);
        out[6] = tot;
        for (int i = 0; i < n; ++i) cudaEventDestroy(ev[i]);
        n = 0;
    }
};
enum { PH_SKETCH = 0, PH_QRCP = 1, PH_RANK = 2, PH_PRE = 3, PH_CHOL = 4, PH_UNDO = 5, PH_COMM = 7 };

int do_allreduce(cqrrpt_gpu_ctx *ctx, double *buf, size_t count, cudaStream_t st) {
    if (ctx->nranks <= 1) return 0;
    if (ctx->comm) return cqrrpt_gpu_comm_allreduce(ctx->comm, buf, count, st);
    if (ctx->allreduce) {
        int rc = ctx->allreduce(buf, count, st, ctx->allreduce_user);
        if (rc) {
            set_error("user allreduce failed");
            return CQRRPT_GPU_ERR_NCCL;
        }
        return 0;
    }
    set_error("nranks > 1 but neither comm nor allreduce callback given");
    return CQRRPT_GPU_ERR_NCCL;
}
}  // namespace

extern "C" {

void cqrrpt_gpu_ctx_init(cqrrpt_gpu_ctx *ctx) {
    std::memset(ctx, 0, sizeof(*ctx));
    ctx->nranks = 1;
    ctx->cond_method = CQRRPT_COND_IDENTITY_DEVIATION;
    ctx->cond_m_pre = NAN;
}

const char *cqrrpt_gpu_last_error(void) { return cqg::last_error(); }
int64_t cqrrpt_gpu_launch_count(int32_t reset) { return cqg::launch_count(reset != 0); }

int64_t cqrrpt_gpu_sketch_rows(double d_factor, int64_t n) {
    return (int64_t)std::ceil(d_factor * (double)n);  // cqrrpt.cc:211-213
}

double cqrrpt_gpu_flop_model(int64_t m, int64_t n, int64_t k, int64_t d, double c_sk) {
    if (k < 0 || k > std::min(d, n)) return -1.0;  // cqrrpt.cc:331-332
    __int128 mm = m, kk = k, nn = n, dd = d;
    __int128 num = 12 * mm * kk * kk + 6 * mm * kk * (kk + 1) + 24 * dd * nn * kk - 12 * kk * kk * (dd + nn) +
                   10 * kk * kk * kk + 3 * kk * kk + kk;
    return (double)num / 6.0 + c_sk;
}

}  // extern "C"

namespace {
// One rank: precondition, Gram, Cholesky and Q as a wavefront of 128-column
// blocks, so the latency-bound Cholesky columns overlap the DMMA passes and,
// on the host entry point, Q's download starts right after the QRCP instead
// of after the whole Gram + Cholesky. Block b needs M_pre's columns
// < 128(b+1) (precondition TRSM on `st`, an event per 64 columns), then on
// `s2`: its Gram columns (gram_cols: split over m finely enough that the
// first, small blocks fill the GPU; a fixed order, but not gram()'s), the
// Cholesky steps that reach it (potrf_cols: bitwise potrf's factor of that
// Gram), the inverses of its diagonal blocks and its Q blocks, which the copy
// stream downloads. Q is speculated on k = k0 (stage 2 runs after the last
// block, on this R); the caller redoes the final solve when stage 2 truncates
// or the Cholesky fails. Q goes to a separate buffer (the precondition still
// gathers A's columns while Q blocks are written).
// Returns 0 with *done = false when the buffers do not fit (whole passes).
int wavefront_q(int64_t m, int64_t k0, double *A, int64_t lda, const int64_t *jd, const double *rsk, int64_t ldk,
                double *mpre, int64_t ldp, double *gmat, const BlockSink *sink, int64_t *fi, bool *done,
                PhaseClock &clk, Workspace &ws, cudaStream_t st) {
    *done = false;
    *fi = 0;
    constexpr int64_t NB = 64, WB = 128;  // solve block, wavefront block
    const int64_t nsub = (k0 + NB - 1) / NB, nw = (k0 + WB - 1) / WB;
    static thread_local std::vector<int2> tiles_h;
    static thread_local std::vector<int64_t> toff;
    tiles_h.clear();
    toff.assign((size_t)nw + 1, 0);
    int64_t max_t = 0;
    for (int64_t b = 0; b < nw; ++b) {
        gram_col_tiles(b * WB, std::min(k0, (b + 1) * WB), tiles_h);
        toff[(size_t)b + 1] = (int64_t)tiles_h.size();
        max_t = std::max(max_t, toff[(size_t)b + 1] - toff[(size_t)b]);
    }
    const size_t part_n = gram_col_part_size(m, k0, max_t);
    // Q: in place into A (device entry point; its blocks wait until the
    // precondition has gathered all of A's columns) or, with a host sink, into
    // a separate buffer so Q's first blocks are formed while A is still read
    // With a host sink Q goes to its own buffer so its first blocks can be
    // formed while the precondition still gathers A's columns. When that
    // buffer does not fit next to A and M_pre (C5-2048: 3 x 64 GiB) the whole
    // passes run instead: Q written in place into A after the precondition,
    // with its blocks streamed during the wavefront's DMMA Gram columns, was
    // measured slower there (C5-2048 e2e 3.39 -> 3.61 s: the INT8 Gram of the
    // whole passes is 2x faster than the column-block Gram).
    // CQRRPT_WF_INPLACE=1 forces that in-place variant (tests).
    int64_t ldq = sink ? ldp : lda;
    const bool force_inplace = sink && getenv("CQRRPT_WF_INPLACE") != nullptr;
    double *qws = (sink && !force_inplace) ? ws.get<double>("wf.q", (size_t)(ldq * k0)) : A;
    if (!qws) return 0;  // does not fit: whole passes
    const bool inplace = !sink || force_inplace;
    if (inplace) {
        qws = A;
        ldq = lda;
    }
    double *part = ws.get<double>("wf.part", part_n);
    if (!part) return 0;  // does not fit: whole passes
    int2 *tiles = ws.get<int2>("wf.tiles", tiles_h.size());
    double *dinv = ws.get<double>("wf.dinv", (size_t)(nsub * NB * NB));
    int64_t *fail = ws.get<int64_t>("wf.fail", 1);
    if (!tiles || !dinv || !fail || part_n == 0) return fail_nomem("wavefront workspace");
    // Streams by priority: s2 (Cholesky columns, Q blocks: what the download
    // waits for) > s3 (Gram columns, which only need M_pre and so run ahead)
    // > st (the precondition). Gram block b writes G's columns of block b and
    // the mirrored entries below the diagonal in rows of block b; s2 reads only
    // upper-triangle entries of blocks < b, so the two overlap safely.
    cudaStream_t s2 = nullptr, s3 = nullptr;
    cudaEvent_t *ev_pre = nullptr, *ev_q = nullptr, *ev_g = nullptr, *ev_se = nullptr;
    CQ_TRY(cached_stream("wf.s2", 1, &s2));
    CQ_TRY(cached_stream("wf.s3", 2, &s3));
    CQ_TRY(cached_events("wf.pre", (size_t)nsub, &ev_pre));
    CQ_TRY(cached_events("wf.q", (size_t)nsub, &ev_q));
    CQ_TRY(cached_events("wf.g", (size_t)nw, &ev_g));
    CQ_TRY(cached_events("wf.se", 2, &ev_se));
    cudaEvent_t ev_start = ev_se[0], ev_end = ev_se[1];
    // CQRRPT_WF_TRACE=1: print when each Q block is formed and downloaded
    static const bool trace = std::getenv("CQRRPT_WF_TRACE") != nullptr;
    std::vector<cudaEvent_t> tq, td;
    cudaEvent_t t0 = nullptr;
    auto tev = [&](std::vector<cudaEvent_t> &v, cudaStream_t on) -> int {
        cudaEvent_t e;
        CQ_CUDA(cudaEventCreate(&e), "trace event");
        CQ_CUDA(cudaEventRecord(e, on), "trace record");
        v.push_back(e);
        return 0;
    };
    if (trace) {
        CQ_CUDA(cudaEventCreate(&t0), "trace event");
        CQ_CUDA(cudaEventRecord(t0, st), "trace record");
    }
    // st is idle here (stage 1 synchronised), so the pageable upload is cheap
    CQ_CUDA(cudaMemcpyAsync(tiles, tiles_h.data(), sizeof(int2) * tiles_h.size(), cudaMemcpyHostToDevice, st),
            "wavefront tiles h2d");
    CQ_CUDA(cudaMemsetAsync(fail, 0, sizeof(int64_t), st), "wavefront fail flag");
    CQ_CUDA(cudaEventRecord(ev_start, st), "wavefront start");
    CQ_CUDA(cudaStreamWaitEvent(s2, ev_start, 0), "wavefront start wait");
    CQ_CUDA(cudaStreamWaitEvent(s3, ev_start, 0), "wavefront start wait");
    // precondition M_pre = M[:, J[:k0]] A_sk^{-1} on st, an event per 64 columns
    CQ_TRY(trsm_right(m, k0, A, lda, jd, rsk, ldk, mpre, ldp, st, nullptr, true, ev_pre));
    clk.mark(PH_PRE);
    if (inplace) CQ_CUDA(cudaStreamWaitEvent(s2, ev_pre[(size_t)(nsub - 1)], 0), "wavefront wait precondition");
    for (int64_t b = 0; b < nw; ++b) {  // Gram columns, as soon as M_pre's columns exist
        const int64_t w1 = std::min(k0, (b + 1) * WB);
        CQ_CUDA(cudaStreamWaitEvent(s3, ev_pre[(size_t)((w1 - 1) / NB)], 0), "wavefront wait block");
        CQ_TRY(gram_cols(m, k0, w1, tiles + toff[(size_t)b], toff[(size_t)b + 1] - toff[(size_t)b], mpre, ldp, gmat,
                         k0, part, s3));
        CQ_CUDA(cudaEventRecord(ev_g[(size_t)b], s3), "wavefront gram event");
    }
    for (int64_t b = 0; b < nw; ++b) {
        const int64_t w0 = b * WB, w1 = std::min(k0, w0 + WB);
        CQ_CUDA(cudaStreamWaitEvent(s2, ev_g[(size_t)b], 0), "wavefront wait gram");
        for (int64_t c0 = w0; c0 < w1; c0 += NB) {
            const int64_t c1 = std::min(w1, c0 + NB), sb = c0 / NB;
            CQ_TRY(potrf_cols(k0, gmat, k0, c0, c1, fail, s2));
            CQ_TRY(trtri_diag_blocks(c1 - c0, gmat + c0 * k0 + c0, k0, dinv + sb * NB * NB, s2));
            CQ_TRY(trsm_block(m, k0, c0, mpre, ldp, nullptr, gmat, k0, dinv + sb * NB * NB, qws, ldq, s2));
            if (trace) CQ_TRY(tev(tq, s2));
            if (!sink) continue;
            CQ_CUDA(cudaEventRecord(ev_q[(size_t)sb], s2), "wavefront q event");
            CQ_CUDA(cudaStreamWaitEvent(sink->copy, ev_q[(size_t)sb], 0), "wavefront sink wait");
            CQ_CUDA(cudaMemcpy2DAsync(sink->host + c0 * sink->ldh, sizeof(double) * sink->ldh, qws + c0 * ldq,
                                      sizeof(double) * ldq, sizeof(double) * m, c1 - c0, cudaMemcpyDeviceToHost,
                                      sink->copy),
                    "wavefront q d2h");
            if (trace) CQ_TRY(tev(td, sink->copy));
        }
    }
    CQ_CUDA(cudaEventRecord(ev_end, s2), "wavefront end");
    CQ_CUDA(cudaStreamWaitEvent(st, ev_end, 0), "wavefront join");
    CQ_TRY(zero_strict_lower(k0, gmat, k0, st));
    CQ_CUDA(cudaMemcpyAsync(fi, fail, sizeof(int64_t), cudaMemcpyDeviceToHost, st), "wavefront fail d2h");
    CQ_CUDA(cudaStreamSynchronize(st), "wavefront sync");
    if (trace) {
        if (sink) CQ_CUDA(cudaStreamSynchronize(sink->copy), "trace sync");
        for (size_t i = 0; i < tq.size(); ++i) {
            float a = 0.f, b = 0.f;
            cudaEventElapsedTime(&a, t0, tq[i]);
            if (i < td.size()) cudaEventElapsedTime(&b, t0, td[i]);
            std::fprintf(stderr, "wavefront block %zu: Q formed %.3f ms, downloaded %.3f ms\n", i, a, b);
            cudaEventDestroy(tq[i]);
            if (i < td.size()) cudaEventDestroy(td[i]);
        }
        cudaEventDestroy(t0);
    }
    *done = true;
    return 0;
}

// ---- rank_stage2's attempt loop (cqrrpt.cc:160-193) -------------------------
// M_pre = B[:, cols[:k0]] A_sk^{-1} (gather fused into the TRSM), G = M_pre^T
// M_pre (allreduced across ranks), upper Cholesky of G in place. fi: 0 or the
// 1-based first failing minor.
int precondition_factor(int64_t m, int64_t k0, const double *B, int64_t ldb, const int64_t *cols, const double *a_sk,
                        int64_t ldas, double *mpre, int64_t ldp, double *g, int64_t ldg, int64_t *fi,
                        cqrrpt_gpu_ctx *ctx, PhaseClock *clk, Workspace &ws, cudaStream_t st) {
    CQ_TRY(trsm_right(m, k0, B, ldb, cols, a_sk, ldas, mpre, ldp, st));
    if (clk) clk->mark(PH_PRE);
    CQ_TRY(gram(m, k0, mpre, ldp, g, ldg, ws, st));
    if (clk) clk->mark(PH_CHOL);
    if (ctx) CQ_TRY(do_allreduce(ctx, g, (size_t)(k0 * ldg), st));
    if (clk) clk->mark(PH_COMM);
    return potrf(k0, g, ldg, fi, ws, st);
}

// A failure at minor fi shrinks k0 to fi - 1. The retry on the leading fi-1
// columns recomputes bitwise the same M_pre columns, Gram block (the Gram has
// the leading-block property) and factor (cqrrpt.cc:162-164), so it always
// succeeds: one retry, k0_final = fi - 1 (0 means rank 0, cqrrpt.cc:178-182).
void shrink_after_failure(int64_t k0, int64_t fi, int64_t *k0f, int *retries) {
    *k0f = k0;
    *retries = 0;
    if (fi > 0) {
        *retries = 1;
        *k0f = fi - 1;
    }
}

// ---- rank_stage2's selection (cqrrpt.cc:195-207) ----------------------------
// On the Cholesky factor R_pre (leading k0f x k0f block of rfull, ld ldf):
// the largest leading block whose NestedCondEstimator value is <=
// sqrt(eps_tol/u). Fast accept (exact): if every probe of the
// all-pass search path has tau >= 1 at its first power iterate (so the
// reference's identity_deviation is +inf and it falls back to krylov_bounds)
// and ||R||_F ||R^-1||_F (1+1e-5) <= threshold bounds every krylov estimate,
// every probe passes and k = k0f; otherwise the reference's binary search
// runs on the device. rinv (k0f x k0f) = R_pre^{-1} stays valid in ws.
struct Stage2Out {
    int64_t k = 0;
    double cond = NAN;   // est.at(k) when the search ran, NaN on the fast path
    int exact = 0;       // 1 if the binary search ran
    double bound = 0.0;  // ||R||_F ||R^-1||_F
};

static void all_pass_probes(int64_t k0f, std::vector<int64_t> &ells) {
    ells.clear();
    for (int64_t lo = 0, hi = k0f; lo < hi;) {  // cqrrpt.cc:197-204 when every probe passes
        const int64_t mid = lo + (hi - lo + 1) / 2;
        ells.push_back(mid);
        lo = mid;
    }
}

static int nested_method(int method) {
    // identity_deviation with the nested krylov fallback (cqrrpt.cc:57-58)
    return (method == CQRRPT_COND_IDENTITY_DEVIATION) ? CQRRPT_COND_NESTED_IDENTITY_DEVIATION : method;
}

int stage2_select(int64_t k0f, const double *rfull, int64_t ldf, double eps_tol, int method, bool force_exact,
                  Workspace &ws, cudaStream_t s, Stage2Out *out, double **rinv_out) {
    const double threshold = std::sqrt(eps_tol / kUnitRoundoff);
    double *rinv = ws.get<double>("drv.rinv", (size_t)(k0f * k0f));
    if (!rinv) return fail_nomem("rinv");
    *rinv_out = rinv;
    CQ_TRY(trtri_upper(k0f, rfull, ldf, rinv, k0f, ws, s));  // leading blocks of R^-1 = leading inverses
    bool exact = force_exact;
    out->k = k0f;
    if (!exact) {
        std::vector<int64_t> ells;
        all_pass_probes(k0f, ells);
        if (method == CQRRPT_COND_IDENTITY_DEVIATION) {
            // power_iterate keeps est = max(est, ...) (linalg.cc:455): tau >= 1
            // at the first iterate means +inf whatever the later iterates
            std::vector<double> first(ells.size());
            CQ_TRY(identity_deviation_first(rfull, ldf, ells.data(), (int)ells.size(), first.data(), ws, s));
            for (double v : first)
                if (!(v * (1.0 + 1e-6) >= 1.0)) exact = true;
        }
        double fr = 0.0, fi = 0.0;
        CQ_TRY(frob_norm_upper(k0f, rfull, ldf, &fr, ws, s));
        CQ_TRY(frob_norm_upper(k0f, rinv, k0f, &fi, ws, s));
        out->bound = fr * fi;  // >= cond_2(R_ell) for every leading block
        if (!(out->bound * (1.0 + 1e-5) <= threshold)) exact = true;
    }
    out->exact = exact ? 1 : 0;
    if (!exact) return 0;
    // NestedCondEstimator (cqrrpt.cc:47-71): memoised raw estimates, running max
    std::map<int64_t, double> raw;
    auto at = [&](int64_t ell, double *v) -> int {
        if (ell <= 0) {
            *v = 1.0;
            return 0;
        }
        if (!raw.count(ell)) {
            double e = 1.0;
            CQ_TRY(cond_estimate(ell, rfull, ldf, rinv, k0f, nested_method(method), &e, ws, s));
            raw[ell] = e;
        }
        double e = 1.0;
        for (auto &kv : raw)
            if (kv.first <= ell) e = std::max(e, kv.second);
        *v = e;
        return 0;
    };
    // The search's all-pass prefix in one batched launch (the estimates do
    // not depend on the batch): probes are memoised up to and including the
    // first one whose running max fails -- exactly the probes the reference
    // evaluates before its search turns; the rest of the search continues
    // probe by probe.
    {
        std::vector<int64_t> ells;
        all_pass_probes(k0f, ells);
        if (ells.size() > 1) {
            std::vector<double> est(ells.size(), 1.0);
            CQ_TRY(cond_estimate_batch((int)ells.size(), ells.data(), rfull, ldf, rinv, k0f, nested_method(method),
                                       est.data(), ws, s));
            double run = 1.0;
            for (size_t q = 0; q < ells.size(); ++q) {
                raw[ells[q]] = est[q];
                run = std::max(run, est[q]);
                if (!(run <= threshold)) break;
            }
        }
    }
    int64_t lo = 0, hi = k0f;  // binary search (cqrrpt.cc:197-207)
    while (lo < hi) {
        const int64_t mid = lo + (hi - lo + 1) / 2;
        double e = 0.0;
        CQ_TRY(at(mid, &e));
        if (e <= threshold) lo = mid;
        else hi = mid - 1;
    }
    out->k = lo;
    double c = 1.0;
    if (lo > 0) CQ_TRY(at(lo, &c));
    out->cond = c;
    return 0;
}

// est.at(k0f) after an all-pass search: the running max of the probes' raw
// nested estimates (what the reference reports as cond_m_pre on that path)
int probe_cond(int64_t k0f, const double *rfull, int64_t ldf, const double *rinv, int method, Workspace &ws,
               cudaStream_t s, double *cond) {
    std::vector<int64_t> ells;
    all_pass_probes(k0f, ells);
    std::vector<double> est(ells.size(), 1.0);
    CQ_TRY(cond_estimate_batch((int)ells.size(), ells.data(), rfull, ldf, rinv, k0f, nested_method(method), est.data(),
                               ws, s));
    double c = 1.0;
    for (double e : est) c = std::max(c, e);
    *cond = (k0f > 0) ? c : 1.0;
    return 0;
}

// The driver; `qsink` (optional) downloads Q block by block during the final TRSM.
constexpr int kInputChunks = 4;  // H2D row chunks of the host-buffer entry point

int dgeqpt_impl(int64_t m, int64_t n, double *A, int64_t lda, double d_factor, int64_t nnz, uint64_t seed,
                double eps_tol, double *R, int64_t ldr, int64_t *J, int64_t *k_out, int64_t *k0_out,
                cqrrpt_gpu_ctx *ctx, const BlockSink *qsink, const InputChunks *ichunks = nullptr) {
    cqrrpt_gpu_ctx local;
    if (!ctx) {
        cqrrpt_gpu_ctx_init(&local);
        ctx = &local;
    }
    // ---- argument checks (check_config cqrrpt.cc:38-42 first, as the reference does)
    if (!(d_factor >= 1.0)) return set_error("d_factor must be >= 1"), -5;
    if (!(eps_tol > kUnitRoundoff)) return set_error("eps_tol must exceed the unit roundoff"), -8;
    if (m < 0) return set_error("m < 0"), -1;
    if (n < 0) return set_error("n < 0"), -2;
    if (!k_out) return -12;
    if (!k0_out) return -13;
    *k_out = 0;
    *k0_out = 0;
    if (n == 0) return 0;  // cqrrpt.cc:319-324
    const bool multi = ctx->nranks > 1;
    if (!multi && m < 1) return set_error("sample_sketch: need m >= 1"), -1;  // sketch.cc:54
    if (m > 0 && !A) return -3;
    if (m > 0 && lda < m) return set_error("lda < m"), -4;
    const int64_t d = ctx->sketch_rows > 0 ? ctx->sketch_rows : cqrrpt_gpu_sketch_rows(d_factor, n);
    if (ctx->sketch_family != CQRRPT_SKETCH_SASO && ctx->sketch_family != CQRRPT_SKETCH_GAUSSIAN &&
        ctx->sketch_family != CQRRPT_SKETCH_SRFT)
        return set_error("unknown sketch family"), -14;  // the reference throws std::logic_error
    const bool gaussian = ctx->sketch_family == CQRRPT_SKETCH_GAUSSIAN;
    const bool srft = ctx->sketch_family == CQRRPT_SKETCH_SRFT;
    const bool saso = !gaussian && !srft;
    if (saso && (nnz < 1 || nnz > d)) return set_error("SASO needs 1 <= nnz <= d"), -6;  // sketch.cc:74-75
    if (srft && d > m) return set_error("sample_sketch: SRFT needs d <= m"), -6;         // sketch.cc:101
    if (srft && multi) return set_error("the SRFT family needs the whole matrix on one rank"), -14;
    if (!R) return -9;
    if (ldr < n) return set_error("ldr < n"), -10;
    if (!J) return -11;

    cudaStream_t st = (cudaStream_t)ctx->stream;
    Workspace &ws = workspace();
    const bool host_out = (ctx->flags & CQRRPT_GPU_OUTPUTS_ON_HOST) != 0;
    PhaseClock clk;
    clk.start((ctx->flags & CQRRPT_GPU_TIMINGS) != 0, st);
    ctx->d = d;
    ctx->retries = 0;
    ctx->stage2_exact = 0;
    ctx->cond_m_pre = NAN;
    ctx->cond_upper_bound = 0.0;
    ctx->truncation_ratio = 0.0;

    // ---- sketch ------------------------------------------------------------
    double *msk = ws.get<double>("drv.msk", (size_t)(d * n));
    if (!msk) return fail_nomem("sketch");
    if (ichunks && !saso)  // A still arriving: only the exact SASO sketch follows the chunks
        for (int c = 0; c < ichunks->count; ++c) CQ_CUDA(cudaStreamWaitEvent(st, ichunks->ev[c], 0), "wait input");
    if (gaussian)
        CQ_TRY(gaussian_sketch(m, n, A, lda, d, seed, ctx->global_row_offset, msk, d, ws, st));
    else if (srft)
        CQ_TRY(srft_sketch(m, n, A, lda, d, seed, msk, d, ws, st));
    else
        CQ_TRY(saso_sketch(m, n, A, lda, d, nnz, seed, ctx->global_row_offset, msk, d, ws, st,
                           (ctx->flags & CQRRPT_GPU_FAST_SKETCH) != 0, ichunks));
    clk.mark(PH_SKETCH);
    CQ_TRY(do_allreduce(ctx, msk, (size_t)(d * n), st));
    clk.mark(PH_COMM);

    // ---- QRCP of the sketch -------------------------------------------------
    const int64_t ldk = n;  // R_sk buffer: n x n
    double *rsk = ws.get<double>("drv.rsk", (size_t)(n * n));
    int64_t *jd = ws.get<int64_t>("drv.j", (size_t)n);
    if (!rsk || !jd) return fail_nomem("rsk");
    int64_t k_sk = 0;
    CQ_TRY(qrcp(d, n, msk, d, -1.0, rsk, ldk, jd, &k_sk, ws, st));
    ctx->k_sk = k_sk;
    clk.mark(PH_QRCP);

    // ---- stage 1 ------------------------------------------------------------
    int64_t k0 = k_sk;
    if (!(ctx->flags & CQRRPT_GPU_NO_STAGE1)) CQ_TRY(rank_stage1(k_sk, n, rsk, ldk, &k0, ws, st));
    *k0_out = k0;
    clk.mark(PH_RANK);
    auto emit_pivots = [&]() -> int {
        if (host_out) {
            CQ_CUDA(cudaMemcpyAsync(J, jd, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, st), "J d2h");
        } else {
            CQ_CUDA(cudaMemcpyAsync(J, jd, sizeof(int64_t) * n, cudaMemcpyDeviceToDevice, st), "J d2d");
        }
        CQ_CUDA(cudaStreamSynchronize(st), "final sync");
        return 0;
    };
    auto finish_diag = [&](int64_t k) {
        // sketch_flops (sketch.cc:211-224): SASO 2 nnz m n, Gaussian 2 d m n,
        // SRFT n (m + P log2 P + d)
        double csk = 2.0 * (double)(gaussian ? d : nnz) * (double)m * (double)n;
        if (srft) {
            double P = 1.0;
            while (P < (double)m) P *= 2.0;
            csk = (double)n * ((double)m + P * std::log2(P) + (double)d);
        }
        ctx->flop_estimate = cqrrpt_gpu_flop_model(m, n, k, d, csk);
        if (k == 0) ctx->cond_m_pre = 1.0;  // CqrrptDiagnostics default (cqrrpt.hh:118) on rank-0 outputs
        clk.finish(ctx->timings_ms);
    };
    if (k0 == 0) {  // cqrrpt.cc:257-260
        CQ_TRY(emit_pivots());
        finish_diag(0);
        return 0;
    }

    // ---- precondition: M_pre = M[:, J[:k0]] * A_sk^{-1} ----------------------
    const int64_t ldp = std::max<int64_t>(m, 1);
    double *mpre = ws.get<double>("drv.mpre", (size_t)(ldp * k0));
    if (!mpre) return fail_nomem("M_pre workspace");
    double *gmat = ws.get<double>("drv.gram", (size_t)(k0 * k0));
    if (!gmat) return fail_nomem("gram");
    int64_t fi = 0;
    bool wave = false;  // Q already computed (k = k0) and downloaded by the wavefront
    // The wavefront pays off when Q leaves over PCIe (host entry point). On the
    // device entry point it was measured slower (C2 25.0 -> 29.8 ms: Q's
    // blocks must wait for the whole precondition, which the Gram columns
    // then starve), so it is used there only on request (CQRRPT_GPU_WAVEFRONT).
    const bool want_wave = qsink ? !(ctx->flags & CQRRPT_GPU_NO_WAVEFRONT) : (ctx->flags & CQRRPT_GPU_WAVEFRONT) != 0;
    if (!multi && want_wave && m >= 1)
        CQ_TRY(wavefront_q(m, k0, A, lda, jd, rsk, ldk, mpre, ldp, gmat, qsink, &fi, &wave, clk, ws, st));
    if (wave) {
        clk.mark(PH_CHOL);
    } else {
        CQ_TRY(precondition_factor(m, k0, A, lda, jd, rsk, ldk, mpre, ldp, gmat, k0, &fi, ctx, &clk, ws, st));
    }
    int64_t k0f = k0;
    int retries = 0;
    shrink_after_failure(k0, fi, &k0f, &retries);
    ctx->retries = retries;
    if (fi > 0) {
        if (k0f <= 0) {
            ctx->k0_final = 0;
            CQ_TRY(emit_pivots());
            finish_diag(0);
            return 0;
        }
    }
    ctx->k0_final = k0f;
    const double *rfull = gmat;  // upper triangle, ld k0
    clk.mark(PH_CHOL);

    // Device entry point: the final solve Q = M_pre R_pre^{-1} is speculated
    // on k = k0_final and runs on a side stream while stage 2 (R^{-1}, the
    // condition bounds, their host round trips) decides k on st; it is redone
    // for k columns in the rare case stage 2 truncates (A[:, k:k0] then holds
    // speculative columns). The side stream touches only M_pre, R_pre, A and
    // the TRSM's own block inverses, none of which stage 2 writes.
    const bool spec_q = !wave && !qsink && !(ctx->flags & CQRRPT_GPU_NO_WAVEFRONT);
    cudaStream_t sq = nullptr, shi = nullptr;
    cudaEvent_t *ev_side = nullptr;
    if (spec_q) {
        CQ_TRY(cached_stream("drv.sq", 0, &sq));
        CQ_TRY(cached_stream("drv.shi", 1, &shi));
        CQ_TRY(cached_events("drv.side", 3, &ev_side));
    }
    cudaEvent_t ev_sq0 = spec_q ? ev_side[0] : nullptr, ev_sq1 = spec_q ? ev_side[1] : nullptr,
                ev_hi = spec_q ? ev_side[2] : nullptr;
    // On an error return after the fork, wait for the side streams before
    // handing control back: the speculative solve writes into A.
    struct SideJoin {
        cudaEvent_t sq_done = nullptr, hi_done = nullptr;
        cudaStream_t shi = nullptr;
        bool armed = false;
        ~SideJoin() {
            if (!armed) return;
            if (shi && hi_done && cudaEventRecord(hi_done, shi) == cudaSuccess) cudaEventSynchronize(hi_done);
            if (sq_done) cudaEventSynchronize(sq_done);
            cudaGetLastError();
        }
    } side_join;
    if (spec_q) {
        CQ_CUDA(cudaEventRecord(ev_sq0, st), "final solve fork");
        CQ_CUDA(cudaStreamWaitEvent(sq, ev_sq0, 0), "final solve fork wait");
        side_join.armed = true;
        side_join.shi = shi;
        side_join.hi_done = ev_hi;
        CQ_TRY(trsm_right(m, k0f, mpre, ldp, nullptr, rfull, k0, A, lda, sq, nullptr, /*check_diag=*/false));
        CQ_CUDA(cudaEventRecord(ev_sq1, sq), "final solve join");
        side_join.sq_done = ev_sq1;
    }
    auto join_spec = [&]() -> int {
        if (spec_q) CQ_CUDA(cudaStreamWaitEvent(st, ev_sq1, 0), "final solve join wait");
        side_join.armed = false;  // st now orders everything after the side streams
        return 0;
    };

    // ---- stage 2: largest leading block with cond <= sqrt(eps_tol/u) -------
    // with the speculative final solve in flight, stage 2 runs on a
    // high-priority stream so its small kernels are not queued behind the
    // solve's CTAs
    cudaStream_t s2st = st;
    if (spec_q) {
        CQ_CUDA(cudaStreamWaitEvent(shi, ev_sq0, 0), "stage-2 fork");
        s2st = shi;
    }
    Stage2Out s2o;
    double *rinv = nullptr;
    CQ_TRY(stage2_select(k0f, rfull, k0, eps_tol, ctx->cond_method, (ctx->flags & CQRRPT_GPU_EXACT_STAGE2) != 0, ws,
                         s2st, &s2o, &rinv));
    const int64_t k = s2o.k;
    ctx->cond_upper_bound = s2o.bound;
    ctx->stage2_exact = s2o.exact;
    ctx->cond_m_pre = s2o.cond;  // NaN on the fast-accept path until the diagnostics below
    if (spec_q) {
        CQ_CUDA(cudaEventRecord(ev_hi, shi), "stage-2 join");
        CQ_CUDA(cudaStreamWaitEvent(st, ev_hi, 0), "stage-2 join wait");
        side_join.shi = nullptr;  // joined
    }
    clk.mark(PH_RANK);
    *k_out = k;
    if (k == 0) {
        CQ_TRY(join_spec());
        CQ_TRY(emit_pivots());
        finish_diag(0);
        return 0;
    }

    // ---- Q = M_pre[:, :k] R_pre^{-1}, in place into A[:, :k] ----------------
    CQ_TRY(join_spec());
    if (!(wave && fi == 0 && k == k0) && !(spec_q && k == k0f))
        CQ_TRY(trsm_right(m, k, mpre, ldp, nullptr, rfull, k0, A, lda, st, qsink, /*check_diag=*/false));
    clk.mark(PH_CHOL);

    // ---- R = R_pre R_sk[:k, :] (upper-trapezoidal) --------------------------
    if (host_out) {
        double *rk = ws.get<double>("drv.rout", (size_t)(k * n));
        if (!rk) return fail_nomem("rout");
        CQ_TRY(gemm_fill(false, k, n, k, 1.0, rfull, k0, rsk, ldk, 0.0, rk, k, ws, st));
        clk.mark(PH_UNDO);
        CQ_CUDA(cudaMemcpy2DAsync(R, sizeof(double) * ldr, rk, sizeof(double) * k, sizeof(double) * k, n,
                                  cudaMemcpyDeviceToHost, st),
                "R d2h");
    } else {
        CQ_TRY(gemm_fill(false, k, n, k, 1.0, rfull, k0, rsk, ldk, 0.0, R, ldr, ws, st));
        clk.mark(PH_UNDO);
    }
    CQ_TRY(emit_pivots());

    // ---- diagnostics (outside the profiled phases, cqrrpt.cc:298-303) -------
    finish_diag(k);
    if (ctx->flags & CQRRPT_GPU_DIAGNOSTICS) {
        // cond_m_pre (cqrrpt.cc:205,298): on the fast-accept path every probe
        // of the binary search passed, so est.at(k) is the running max of the
        // probes' nested estimates -- evaluated here, outside the timed phases
        if (!s2o.exact) CQ_TRY(probe_cond(k0f, rfull, k0, rinv, ctx->cond_method, ws, st, &ctx->cond_m_pre));
        std::vector<double> hr((size_t)(n * n));
        CQ_CUDA(cudaMemcpyAsync(hr.data(), rsk, sizeof(double) * n * n, cudaMemcpyDeviceToHost, st), "rsk d2h");
        CQ_CUDA(cudaStreamSynchronize(st), "diag sync");
        double ck = 0.0;
        for (int64_t j = k; j < n; ++j)
            for (int64_t i = k; i < k_sk; ++i) ck += hr[j * n + i] * hr[j * n + i];
        double rn = 0.0;
        CQ_TRY(spectral_norm_estimate(k_sk, n, rsk, ldk, &rn, ws, st));
        ctx->truncation_ratio = (rn > 0.0) ? std::sqrt(ck) / rn : 0.0;
    }
    return 0;
}
}  // namespace

extern "C" {

int cqrrpt_gpu_dgeqpt(int64_t m, int64_t n, double *A, int64_t lda, double d_factor, int64_t nnz, uint64_t seed,
                      double eps_tol, double *R, int64_t ldr, int64_t *J, int64_t *k_out, int64_t *k0_out,
                      cqrrpt_gpu_ctx *ctx) {
    return dgeqpt_impl(m, n, A, lda, d_factor, nnz, seed, eps_tol, R, ldr, J, k_out, k0_out, ctx, nullptr);
}

int cqrrpt_gpu_dgeqpt_host(int64_t m, int64_t n, const double *A_host, int64_t lda, double d_factor, int64_t nnz,
                           uint64_t seed, double eps_tol, double *Q_host, int64_t ldq, double *R_host, int64_t ldr,
                           int64_t *J_host, int64_t *k_out, int64_t *k0_out, cqrrpt_gpu_ctx *ctx) {
    cqrrpt_gpu_ctx local;
    if (!ctx) {
        cqrrpt_gpu_ctx_init(&local);
        ctx = &local;
    }
    if (m < 0) return -1;
    if (n < 0) return -2;
    if (m > 0 && n > 0 && !A_host) return -3;
    if (m > 0 && lda < m) return -4;
    if (m > 0 && n > 0 && (!Q_host || ldq < m)) return -10;
    cudaStream_t st = (cudaStream_t)ctx->stream;
    Workspace &ws = workspace();
    double *dA = (m > 0 && n > 0) ? ws.get<double>("host.a", (size_t)(m * n)) : nullptr;
    if (m > 0 && n > 0 && !dA) return fail_nomem("device copy of A");
    cudaStream_t copy = nullptr;
    CQ_TRY(cached_stream("host.copy", 0, &copy));
    // H2D of A in row chunks on the copy stream; the exact sketch consumes
    // each chunk as it lands (its FMA chains run in row order), so only the
    // last chunk's share of the sketch remains after the transfer
    cudaEvent_t *in_ev = nullptr;
    CQ_TRY(cached_events("host.in", kInputChunks, &in_ev));
    int64_t row_end[kInputChunks];
    int nch = 0;
    if (dA) {
        const int64_t tiles = (m + 255) / 256;
        nch = (int)std::max<int64_t>(1, std::min<int64_t>(kInputChunks, tiles / 64));
        CQ_CUDA(cudaEventRecord(in_ev[0], st), "input order");  // A's buffer is free once st reaches here
        CQ_CUDA(cudaStreamWaitEvent(copy, in_ev[0], 0), "input order wait");
        int64_t r0 = 0;
        for (int c = 0; c < nch; ++c) {
            const int64_t r1 = (c + 1 == nch) ? m : ((tiles * (c + 1) / nch) * 256);
            CQ_CUDA(cudaMemcpy2DAsync(dA + r0, sizeof(double) * m, A_host + r0, sizeof(double) * lda,
                                      sizeof(double) * (r1 - r0), n, cudaMemcpyHostToDevice, copy),
                    "A h2d");
            CQ_CUDA(cudaEventRecord(in_ev[c], copy), "input chunk event");
            row_end[c] = r1;
            r0 = r1;
        }
    }
    const InputChunks chunks{nch, in_ev, row_end};
    BlockSink sink{copy, Q_host, ldq};
    const int32_t flags = ctx->flags;
    ctx->flags |= CQRRPT_GPU_OUTPUTS_ON_HOST;
    const int rc = dgeqpt_impl(m, n, dA, std::max<int64_t>(m, 1), d_factor, nnz, seed, eps_tol, R_host, ldr, J_host,
                               k_out, k0_out, ctx, dA ? &sink : nullptr, dA ? &chunks : nullptr);
    if (dA) CQ_CUDA(cudaStreamWaitEvent(st, in_ev[nch - 1], 0), "input join");  // early returns
    ctx->flags = flags;
    CQ_CUDA(cudaStreamSynchronize(copy), "Q d2h");
    return rc;
}

// ---------------------------------------------------------------------------
// phase-level entry points
// ---------------------------------------------------------------------------
int cqrrpt_gpu_saso_plan(int64_t d, int64_t c0, int64_t count, int64_t nnz, uint64_t seed, uint32_t *plan,
                         void *stream) {
    if (d < 1) return -1;
    if (count < 0) return -3;
    if (nnz < 1 || nnz > d) return -4;
    return saso_plan(d, c0, count, nnz, seed, plan, (cudaStream_t)stream);
}

int cqrrpt_gpu_saso_sketch(int64_t m, int64_t n, const double *A, int64_t lda, int64_t d, int64_t nnz, uint64_t seed,
                           int64_t c0, double *Msk, int64_t ldm, void *stream) {
    if (m < 0) return -1;
    if (n < 0) return -2;
    if (m > 0 && lda < m) return -4;
    if (d < 1) return -5;
    if (nnz < 1 || nnz > d) return -6;
    if (ldm < d) return -10;
    return saso_sketch(m, n, A, lda, d, nnz, seed, c0, Msk, ldm, workspace(), (cudaStream_t)stream);
}

int cqrrpt_gpu_gaussian_sketch(int64_t m, int64_t n, const double *A, int64_t lda, int64_t d, uint64_t seed,
                               int64_t c0, double *Msk, int64_t ldm, void *stream) {
    if (m < 0) return -1;
    if (n < 0) return -2;
    if (m > 0 && lda < m) return -4;
    if (d < 1) return -5;
    if (ldm < d) return -9;
    return gaussian_sketch(m, n, A, lda, d, seed, c0, Msk, ldm, workspace(), (cudaStream_t)stream);
}

int cqrrpt_gpu_srft_sketch(int64_t m, int64_t n, const double *A, int64_t lda, int64_t d, uint64_t seed,
                           double *Msk, int64_t ldm, void *stream) {
    if (m < 1) return -1;
    if (n < 0) return -2;
    if (lda < m) return -4;
    if (d < 1 || d > m) return -5;  // sample_sketch: SRFT needs d <= m (sketch.cc:101)
    if (ldm < d) return -8;
    return srft_sketch(m, n, A, lda, d, seed, Msk, ldm, workspace(), (cudaStream_t)stream);
}

int cqrrpt_gpu_saso_sketch_ex(int64_t m, int64_t n, const double *A, int64_t lda, int64_t d, int64_t nnz,
                              uint64_t seed, int64_t c0, double *Msk, int64_t ldm, uint32_t flags, void *stream) {
    if (m < 0) return -1;
    if (n < 0) return -2;
    if (m > 0 && lda < m) return -4;
    if (d < 1) return -5;
    if (nnz < 1 || nnz > d) return -6;
    if (ldm < d) return -10;
    return saso_sketch(m, n, A, lda, d, nnz, seed, c0, Msk, ldm, workspace(), (cudaStream_t)stream,
                       (flags & CQRRPT_GPU_FAST_SKETCH) != 0);
}

int cqrrpt_gpu_qrcp(int64_t d, int64_t n, double *Msk, int64_t ldm, double rank_tol, double *Rsk, int64_t ldr,
                    int64_t *J, int64_t *k_sk, void *stream) {
    if (d < 1) return set_error("qrcp_maxnorm: need at least one row"), -1;  // qrcp.cc:37
    if (n < 0) return -2;
    if (ldm < d) return -4;
    if (ldr < n) return -7;
    *k_sk = 0;
    if (n == 0) return 0;
    return qrcp(d, n, Msk, ldm, rank_tol, Rsk, ldr, J, k_sk, workspace(), (cudaStream_t)stream);
}

int cqrrpt_gpu_rank_stage1(int64_t k, int64_t n, const double *R, int64_t ldr, int64_t *k0, void *stream) {
    if (k < 0 || n < 0) return -1;
    return rank_stage1(k, n, R, ldr, k0, workspace(), (cudaStream_t)stream);
}

int cqrrpt_gpu_rank_stage2(int64_t m, int64_t k0, const double *M_k0, int64_t ldm, const double *A_sk, int64_t ldas,
                           double eps_tol, int32_t cond_method, int32_t flags, double *M_pre, int64_t ldp, double *R_pre,
                           int64_t ldr, int64_t *rank, int64_t *k0_final, int32_t *retries, double *cond_at_rank,
                           void *stream) {
    if (m < 0) return -1;
    if (k0 < 1) return set_error("rank_stage2: requires k0 >= 1"), -2;  // cqrrpt.cc:153
    if (!M_k0 && m > 0) return -3;
    if (m > 0 && ldm < m) return -4;
    if (!A_sk) return -5;
    if (ldas < k0) return -6;
    if (!(eps_tol > kUnitRoundoff)) return -7;
    if (cond_method < 0 || cond_method > 3) return -8;
    if (!M_pre && m > 0) return -10;
    if (m > 0 && ldp < m) return -11;
    if (!R_pre) return -12;
    if (ldr < k0) return -13;
    if (!rank || !k0_final || !retries || !cond_at_rank) return -14;
    cudaStream_t st = (cudaStream_t)stream;
    Workspace &ws = workspace();
    int64_t fi = 0;
    CQ_TRY(precondition_factor(m, k0, M_k0, ldm, nullptr, A_sk, ldas, M_pre, std::max<int64_t>(ldp, 1), R_pre, ldr, &fi,
                               nullptr, nullptr, ws, st));
    int64_t k0f = k0;
    int rt = 0;
    shrink_after_failure(k0, fi, &k0f, &rt);
    *retries = rt;
    *k0_final = k0f;
    *rank = 0;
    *cond_at_rank = 1.0;
    if (k0f <= 0) {
        *k0_final = 0;
        return 0;
    }
    Stage2Out s2o;
    double *rinv = nullptr;
    CQ_TRY(stage2_select(k0f, R_pre, ldr, eps_tol, cond_method, (flags & CQRRPT_GPU_EXACT_STAGE2) != 0, ws, st, &s2o,
                         &rinv));
    *rank = s2o.k;
    if (s2o.k > 0) {
        if (s2o.exact) *cond_at_rank = s2o.cond;
        else CQ_TRY(probe_cond(k0f, R_pre, ldr, rinv, cond_method, ws, st, cond_at_rank));
    }
    CQ_CUDA(cudaStreamSynchronize(st), "rank_stage2 sync");
    return 0;
}

int cqrrpt_gpu_trsm_engine(int64_t m, int64_t k) { return trsm_use_ozaki(m, k) ? 1 : 0; }

int cqrrpt_gpu_trsm_right(int64_t m, int64_t k, const double *B, int64_t ldb, const int64_t *cols, const double *U,
                          int64_t ldu, double *X, int64_t ldx, void *stream) {
    if (m < 0) return -1;
    if (k < 0) return -2;
    if (ldu < k) return -7;
    if (ldx < m) return -9;
    return trsm_right(m, k, B, ldb, cols, U, ldu, X, ldx, (cudaStream_t)stream);
}

int cqrrpt_gpu_gram(int64_t m, int64_t k, const double *X, int64_t ldx, double *G, int64_t ldg, void *stream) {
    if (m < 0 || k < 0) return -1;
    if (ldg < k) return -6;
    return gram(m, k, X, ldx, G, ldg, workspace(), (cudaStream_t)stream);
}

int cqrrpt_gpu_potrf(int64_t n, double *G, int64_t ldg, int64_t *failure_index, void *stream) {
    if (n < 0) return -1;
    if (ldg < n) return -3;
    return potrf(n, G, ldg, failure_index, workspace(), (cudaStream_t)stream);
}

int cqrrpt_gpu_cond_estimate(int64_t ell, const double *R, int64_t ldr, int32_t method, double *value, void *stream) {
    if (ell < 0) return -1;
    if (method < 0 || method > 3) return -4;
    cudaStream_t st = (cudaStream_t)stream;
    Workspace &ws = workspace();
    double *rinv = nullptr;
    if (method != CQRRPT_COND_DIAG_RATIO && ell > 0) {
        rinv = ws.get<double>("ce.rinv", (size_t)(ell * ell));
        if (!rinv) return fail_nomem("cond rinv");
        // zero diagonal: inverse_norm_estimate returns +inf (linalg.cc:489-490);
        // the kernel handles that case without reading rinv
        CQ_TRY(trtri_upper(ell, R, ldr, rinv, ell, ws, st));
    }
    return cond_estimate(ell, R, ldr, rinv, ell, method, value, ws, st);
}

// ---- CholeskyQR / CholeskyQR2 (cqrrpt.cc:75-90) ------------------------------
namespace {
// one pass in place: G = A^T A (into r), r = chol(G), A <- A r^{-1}
int cholqr_pass(int64_t m, int64_t n, double *A, int64_t lda, double *r, int64_t ldr, int64_t *failure_index,
                Workspace &ws, cudaStream_t st) {
    CQ_TRY(gram(m, n, A, lda, r, ldr, ws, st));
    CQ_TRY(potrf(n, r, ldr, failure_index, ws, st));
    if (*failure_index > 0) return 0;
    // in place (block jb reads B[:, jb] first); r is potrf's factor: no zero diagonal
    return trsm_right(m, n, A, lda, nullptr, r, ldr, A, lda, st, nullptr, /*check_diag=*/false);
}
}  // namespace

int cqrrpt_gpu_cholesky_qr(int64_t m, int64_t n, double *A, int64_t lda, double *R, int64_t ldr, int32_t twice,
                           int64_t *failure_index, void *stream) {
    if (m < 0) return -1;
    if (n < 0 || m < n) return -2;  // cholesky_qr: requires rows >= cols (cqrrpt.cc:76-77)
    if (n > 0 && lda < m) return -4;
    if (n > 0 && ldr < n) return -6;
    if (!failure_index) return -8;
    *failure_index = 0;
    if (n == 0) return 0;
    cudaStream_t st = (cudaStream_t)stream;
    Workspace &ws = workspace();
    if (!twice) return cholqr_pass(m, n, A, lda, R, ldr, failure_index, ws, st);
    double *r1 = ws.get<double>("cholqr2.r1", (size_t)(n * n));
    double *r2 = ws.get<double>("cholqr2.r2", (size_t)(n * n));
    if (!r1 || !r2) return fail_nomem("cholesky_qr2");
    CQ_TRY(cholqr_pass(m, n, A, lda, r1, n, failure_index, ws, st));
    if (*failure_index > 0) return 0;
    CQ_TRY(cholqr_pass(m, n, A, lda, r2, n, failure_index, ws, st));
    if (*failure_index > 0) return 0;
    return gemm_fill(false, n, n, n, 1.0, r2, n, r1, n, 0.0, R, ldr, ws, st);  // R = R2 R1 (cqrrpt.cc:88)
}

int cqrrpt_gpu_trtri_upper(int64_t k, const double *R, int64_t ldr, double *X, int64_t ldx, void *stream) {
    if (k < 0) return -1;
    if (k > 0 && (ldr < k || ldx < k)) return -3;
    return trtri_upper(k, R, ldr, X, ldx, workspace(), (cudaStream_t)stream);
}

int cqrrpt_gpu_trmm_upper(int64_t k, int64_t n, const double *A, int64_t lda, const double *B, int64_t ldb, double *C,
                          int64_t ldc, void *stream) {
    if (k < 0 || n < 0) return -1;
    return gemm_fill(false, k, n, k, 1.0, A, lda, B, ldb, 0.0, C, ldc, workspace(), (cudaStream_t)stream);
}

// ---- device validator ------------------------------------------------------
namespace {
__global__ void sub_identity_kernel(int64_t k, double *a, int64_t lda) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < k) a[i * lda + i] -= 1.0;
}
__global__ void colsq_kernel(int64_t m, int64_t n, const double *a, int64_t lda, const int64_t *cols,
                             const double *b, int64_t ldb, double *colsq) {
    __shared__ double sc[32];
    int64_t j = blockIdx.x;
    const double *aj = a + (cols ? cols[j] : j) * lda;
    double s = 0.0;
    for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
        double v = aj[i] - (b ? b[j * ldb + i] : 0.0);
        s = fma(v, v, s);
    }
    s = block_sum(s, sc);
    if (threadIdx.x == 0) colsq[j] = s;
}
__global__ void sum1_kernel(int64_t n, const double *v, double *out) {
    __shared__ double sc[32];
    double s = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += v[i];
    s = block_sum(s, sc);
    if (threadIdx.x == 0) out[0] = s;
}
int frob_cols(int64_t m, int64_t n, const double *a, int64_t lda, const int64_t *cols, const double *b, int64_t ldb,
              double *out, Workspace &ws, cudaStream_t st) {
    double *cs = ws.get<double>("val.cs", (size_t)std::max<int64_t>(n, 1));
    double *tot = ws.get<double>("val.tot", 1);
    if (n <= 0) {
        *out = 0.0;
        return 0;
    }
    colsq_kernel<<<(unsigned)n, 256, 0, st>>>(m, n, a, lda, cols, b, ldb, cs);
    note_launch();
    sum1_kernel<<<1, 1024, 0, st>>>(n, cs, tot);
    note_launch();
    CQ_TRY(check_launch("frob_cols"));
    double h = 0.0;
    CQ_CUDA(cudaMemcpyAsync(&h, tot, sizeof(double), cudaMemcpyDeviceToHost, st), "frob d2h");
    CQ_CUDA(cudaStreamSynchronize(st), "frob sync");
    *out = std::sqrt(h);
    return 0;
}
}  // namespace

int cqrrpt_gpu_validate(int64_t m, int64_t n, int64_t k, const double *A, int64_t lda, const double *Q, int64_t ldq,
                        const double *R, int64_t ldr, const int64_t *J, double *orth_fro, double *orth_2, double *recon,
                        void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    Workspace &ws = workspace();
    *orth_fro = 0.0;
    *orth_2 = 0.0;
    if (k > 0) {
        double *qtq = ws.get<double>("val.qtq", (size_t)(k * k));
        CQ_TRY(gram(m, k, Q, ldq, qtq, k, ws, st));
        sub_identity_kernel<<<(unsigned)((k + 255) / 256), 256, 0, st>>>(k, qtq, k);
        note_launch();
        CQ_TRY(frob_cols(k, k, qtq, k, nullptr, nullptr, 0, orth_fro, ws, st));
        CQ_TRY(spectral_norm_estimate(k, k, qtq, k, orth_2, ws, st));
    }
    double an = 0.0, dn = 0.0;
    CQ_TRY(frob_cols(m, n, A, lda, nullptr, nullptr, 0, &an, ws, st));
    double *qr = ws.get<double>("val.qr", (size_t)(std::max<int64_t>(m, 1) * n));
    if (!qr) return fail_nomem("validate QR");
    if (k > 0) CQ_TRY(gemm(false, m, n, k, 1.0, Q, ldq, R, ldr, 0.0, qr, std::max<int64_t>(m, 1), st));
    else CQ_CUDA(cudaMemsetAsync(qr, 0, sizeof(double) * std::max<int64_t>(m, 1) * n, st), "memset qr");
    CQ_TRY(frob_cols(m, n, A, lda, J, qr, std::max<int64_t>(m, 1), &dn, ws, st));
    *recon = (an > 0.0) ? dn / an : (dn > 0.0 ? INFINITY : 0.0);  // qrcp.cc:182
    return 0;
}

// ---- NCCL --------------------------------------------------------------------
int cqrrpt_gpu_comm_unique_id(unsigned char id[128]) {
    NcclApi &api = nccl();
    if (!api.get_id) return set_error("libnccl.so.2 not found"), CQRRPT_GPU_ERR_NCCL;
    int rc = api.get_id(id);
    if (rc) return set_error("ncclGetUniqueId failed"), CQRRPT_GPU_ERR_NCCL;
    return 0;
}

int cqrrpt_gpu_comm_init(int32_t nranks, int32_t rank, const unsigned char id[128], cqrrpt_gpu_comm **comm) {
    NcclApi &api = nccl();
    if (!api.init_rank) return set_error("libnccl.so.2 not found"), CQRRPT_GPU_ERR_NCCL;
    NcclId uid;
    std::memcpy(uid.internal, id, 128);
    cqrrpt_gpu_comm *c = new cqrrpt_gpu_comm();
    int rc = api.init_rank(&c->comm, nranks, uid, rank);
    if (rc) {
        delete c;
        set_error(std::string("ncclCommInitRank: ") + (api.errstr ? api.errstr(rc) : "error"));
        return CQRRPT_GPU_ERR_NCCL;
    }
    c->nranks = nranks;
    c->rank = rank;
    *comm = c;
    return 0;
}

int cqrrpt_gpu_comm_allreduce(cqrrpt_gpu_comm *comm, double *buf, size_t count, void *stream) {
    NcclApi &api = nccl();
    if (!comm || !api.allreduce) return set_error("no NCCL communicator"), CQRRPT_GPU_ERR_NCCL;
    int rc = api.allreduce(buf, buf, count, /*ncclDouble*/ 8, /*ncclSum*/ 0, comm->comm, (cudaStream_t)stream);
    if (rc) {
        set_error(std::string("ncclAllReduce: ") + (api.errstr ? api.errstr(rc) : "error"));
        return CQRRPT_GPU_ERR_NCCL;
    }
    return 0;
}

void cqrrpt_gpu_comm_destroy(cqrrpt_gpu_comm *comm) {
    if (!comm) return;
    NcclApi &api = nccl();
    if (api.destroy && comm->comm) api.destroy(comm->comm);
    delete comm;
}

void cqrrpt_gpu_release_workspace(void) { release_workspace(); }

// ---- helpers for caller-supplied collectives -------------------------------
namespace {
__global__ void add_kernel(double *y, const double *x, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        y[i] += x[i];
}
}  // namespace

int cqrrpt_gpu_add(double *y, const double *x, size_t n, void *stream) {
    if (n == 0) return 0;
    add_kernel<<<(unsigned)std::min<size_t>((n + 255) / 256, 4096), 256, 0, (cudaStream_t)stream>>>(y, x, n);
    note_launch();
    return check_launch("add_kernel");
}

int cqrrpt_gpu_copy(void *dst, const void *src, size_t bytes, void *stream) {
    CQ_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, (cudaStream_t)stream), "copy");
    CQ_CUDA(cudaStreamSynchronize((cudaStream_t)stream), "copy sync");
    return 0;
}

int cqrrpt_gpu_stream_sync(void *stream) {
    CQ_CUDA(cudaStreamSynchronize((cudaStream_t)stream), "stream sync");
    return 0;
}

}  // extern "C"

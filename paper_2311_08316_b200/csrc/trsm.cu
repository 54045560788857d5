// K5a / K8: fused pivoted-gather + right triangular solve on FP64 tensor cores.
//
//   X (m x k) = B[:, cols] * U^{-1},   U upper-triangular k x k
//
// Reference: trsm_right (linalg.cc:244-277) applied to M.select_columns(J[:k0])
// (dense_matrix.hh:70-80, cqrrpt.cc:262,165) and to M_pre (cqrrpt.cc:280).
//
// Left-looking blocked algorithm, one launch per 64-wide column block jb:
//   X[:, jb] = (B[:, cols(jb)] - X[:, <jb] U[<jb, jb]) U[jb, jb]^{-1}
// A CTA owns a 64 x 64 tile (4 warps, 32 x 32 DMMA accumulators each). The
// accumulator is initialised with the gathered source columns (their loads
// overlap the main loop) and accumulates B - X U over K = 64*jb with
// mma.sync.m8n8k4.f64 (DMMA.8x8x4), K streaming in 16-deep chunks through a
// 3-stage cp.async pipeline of XOR-swizzled (conflict-free, unpadded) tiles.
// The epilogue multiplies by the inverse of the 64 x 64 diagonal block
// (all block inverses are formed once per solve, trtri.cu), so the whole
// solve runs on the tensor cores; the reference substitutes element by
// element (linalg.cc:262-274). The blocks of a well-conditioned
// preconditioner are well conditioned; the parity tests bound the difference.
// Algorithmic flops: m*k^2 (the reference's count, flop_model term).
#include <vector>

#include "common.cuh"
#include "internal.hh"

namespace cqg {

constexpr int kBM = 64;    // rows per CTA
constexpr int kNB = 64;    // column block
constexpr int kBK = 16;    // K chunk
constexpr int kStages = 3;
constexpr int kThreads = 128;
constexpr int kLdT = kNB + 2;  // 66: conflict-free double2 row access

constexpr size_t kPipeBytes = sizeof(double) * kStages * (kBM + kNB) * kBK;
constexpr size_t kEpiBytes = sizeof(double) * (kBM * kLdT + kNB * kLdT);
constexpr size_t kTrsmSmem = kPipeBytes > kEpiBytes ? kPipeBytes : kEpiBytes;

CQ_DEVI int sw_km(int k, int m) { return k * kBM + (m ^ ((k & 1) << 3)); }   // A tile [k][m]
CQ_DEVI int sw_rk(int r, int k) { return r * kBK + (k ^ ((r & 3) << 2)); }  // B tile [n][k]

__global__ void __launch_bounds__(kThreads, 3)
    trsm_block_kernel(int64_t m, int64_t k, int64_t c0, const double *__restrict__ b, int64_t ldb,
                      const int64_t *__restrict__ cols, const double *__restrict__ u, int64_t ldu,
                      const double *__restrict__ dinv_blk, double *__restrict__ x, int64_t ldx) {
    extern __shared__ __align__(16) double sm[];
    double *As = sm;                        // [stages][16][64] swizzled
    double *Bs = sm + kStages * kBK * kBM;  // [stages][64][16] swizzled
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int wm = warp & 1, wn = warp >> 1;
    const int64_t row0 = (int64_t)blockIdx.x * kBM;
    const int nbw = (int)cmin<int64_t>(kNB, k - c0);

    // accumulator <- gathered right-hand side B[:, cols(c0 + c)]
    double acc[4][4][2];
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
            const int c = wn * 32 + ni * 8 + 2 * t + v;
            const double *bc = (c < nbw) ? b + (cols ? __ldg(cols + c0 + c) : (c0 + c)) * ldb : nullptr;
#pragma unroll
            for (int mi = 0; mi < 4; ++mi) {
                const int64_t row = row0 + wm * 32 + mi * 8 + g;
                acc[mi][ni][v] = (bc && row < m) ? __ldg(bc + row) : 0.0;
            }
        }

    // Programmatic dependent launch: the next block's grid may start as soon
    // as every CTA of this one has started; its CTAs gather their source
    // columns (independent of earlier blocks) and then wait for this grid's
    // completion before reading X[:, <c0]. No-ops without the launch attribute.
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int nchunks = (int)(c0 / kBK);  // c0 is a multiple of 64
    // 16-byte copies of element pairs when X and U are 16-byte aligned with
    // even leading dimensions (the swizzles keep pairs adjacent)
    const bool vec16 = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(u)) & 15) == 0 &&
                       ((ldx | ldu) & 1) == 0;
    auto load_chunk = [&](int kc, int stage) {
        const int64_t kb = (int64_t)kc * kBK;
        double *as = As + stage * kBK * kBM;
        double *bs = Bs + stage * kNB * kBK;
        if (vec16) {
#pragma unroll
            for (int it = 0; it < (kBK * kBM) / 2 / kThreads; ++it) {  // A: X[row0 + mm .. +1][kb + kk]
                const int q = it * kThreads + tid;
                const int kk = q / (kBM / 2), mm = (q % (kBM / 2)) * 2;
                const int64_t row = row0 + mm;
                cp_async16_zfill(as + sw_km(kk, mm), x + (kb + kk) * ldx + (row < m ? row : 0),
                                 row < m ? (row + 1 < m ? 16 : 8) : 0);
            }
#pragma unroll
            for (int it = 0; it < (kBK * kNB) / 2 / kThreads; ++it) {  // B: U[kb + kk .. +1][c0 + nn]
                const int q = it * kThreads + tid;
                const int nn = q / (kBK / 2), kk = (q % (kBK / 2)) * 2;
                const bool ok = nn < nbw;
                cp_async16_zfill(bs + sw_rk(nn, kk), u + (c0 + (ok ? nn : 0)) * ldu + kb + kk, ok ? 16 : 0);
            }
            return;
        }
#pragma unroll
        for (int it = 0; it < (kBK * kBM) / kThreads; ++it) {  // A: X[row0 + mm][kb + kk]
            int q = it * kThreads + tid;
            int kk = q / kBM, mm = q % kBM;
            int64_t row = row0 + mm;
            cp_async8_zfill(as + sw_km(kk, mm), x + (kb + kk) * ldx + (row < m ? row : 0), row < m ? 8 : 0);
        }
#pragma unroll
        for (int it = 0; it < (kBK * kNB) / kThreads; ++it) {  // B: U[kb + kk][c0 + nn]
            int q = it * kThreads + tid;
            int nn = q / kBK, kk = q % kBK;
            bool ok = nn < nbw;
            cp_async8_zfill(bs + sw_rk(nn, kk), u + (c0 + (ok ? nn : 0)) * ldu + kb + kk, ok ? 8 : 0);
        }
    };

    if (nchunks > 0) {
#pragma unroll
        for (int s = 0; s < kStages - 1; ++s) {
            if (s < nchunks) load_chunk(s, s);
            cp_async_commit();
        }
        for (int kc = 0; kc < nchunks; ++kc) {
            cp_async_wait<kStages - 2>();
            __syncthreads();
            {
                int nk = kc + kStages - 1;
                if (nk < nchunks) load_chunk(nk, nk % kStages);
                cp_async_commit();
            }
            const double *as = As + (kc % kStages) * kBK * kBM;
            const double *bs = Bs + (kc % kStages) * kNB * kBK;
            const int mb = wm * 32 + g, nb = wn * 32 + g;
#pragma unroll
            for (int kk = 0; kk < kBK; kk += 4) {
                double af[4], bf[4];
#pragma unroll
                for (int mi = 0; mi < 4; ++mi) af[mi] = -as[sw_km(kk + t, mb + 8 * mi)];  // B - X U
#pragma unroll
                for (int ni = 0; ni < 4; ++ni) bf[ni] = bs[sw_rk(nb + 8 * ni, kk + t)];
#pragma unroll
                for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                    for (int ni = 0; ni < 4; ++ni) dmma884(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
            }
        }
        cp_async_wait<0>();
    }
    __syncthreads();  // pipeline buffers are reused by the epilogue

    // ---- epilogue: X_jb = T U_jb^{-1} on the tensor cores ----------------
    // T = B[:, cols] - X[:, <jb] U[<jb, jb] (the accumulators); U_jb^{-1} is
    // the precomputed inverse of the 64 x 64 diagonal block (dinv_blk).
    double *Ts = sm;               // [64 r][66]: T
    double *Ds = sm + kBM * kLdT;  // [64 c][66]: Ds[c][s] = U_jb^{-1}(s, c)
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) {
            int r = wm * 32 + mi * 8 + g, c = wn * 32 + ni * 8 + 2 * t;
            *reinterpret_cast<double2 *>(Ts + r * kLdT + c) = make_double2(acc[mi][ni][0], acc[mi][ni][1]);
        }
    for (int q = tid; q < kNB * kNB; q += kThreads) {
        const int cc = q / kNB, ss = q % kNB;  // coalesced over ss (a column of the inverse)
        Ds[cc * kLdT + ss] = __ldg(dinv_blk + q);
    }
    __syncthreads();
    // U_jb^{-1} is upper triangular: the 8-column block nb only takes the
    // k-steps kk <= 8 nb + 4 (2 nb + 2 of 16). Warp w computes the column
    // blocks w and 7 - w for all 64 rows, so every warp issues 144 DMMAs
    // instead of 256 (the all-zero k-steps are skipped, balanced).
    const int nbA = warp, nbB = 7 - warp;
    double ep[8][2][2];
#pragma unroll
    for (int mi = 0; mi < 8; ++mi)
#pragma unroll
        for (int b2 = 0; b2 < 2; ++b2) ep[mi][b2][0] = ep[mi][b2][1] = 0.0;
#pragma unroll
    for (int kk = 0; kk < kNB; kk += 4) {
        if (kk > 8 * nbB + 4) break;  // nbB >= 4 > nbA: the longer of the two (warp-uniform)
        double af[8];
#pragma unroll
        for (int mi = 0; mi < 8; ++mi) af[mi] = Ts[(mi * 8 + g) * kLdT + kk + t];
        const double bfB = Ds[(nbB * 8 + g) * kLdT + kk + t];
#pragma unroll
        for (int mi = 0; mi < 8; ++mi) dmma884(ep[mi][1][0], ep[mi][1][1], af[mi], bfB);
        if (kk <= 8 * nbA + 4) {
            const double bfA = Ds[(nbA * 8 + g) * kLdT + kk + t];
#pragma unroll
            for (int mi = 0; mi < 8; ++mi) dmma884(ep[mi][0][0], ep[mi][0][1], af[mi], bfA);
        }
    }
    __syncthreads();  // Ts is reused for the output staging
    double *Os = sm;  // [64 c][65 r]
#pragma unroll
    for (int mi = 0; mi < 8; ++mi)
#pragma unroll
        for (int b2 = 0; b2 < 2; ++b2)
#pragma unroll
            for (int v = 0; v < 2; ++v) {
                const int r = mi * 8 + g, c = (b2 ? nbB : nbA) * 8 + 2 * t + v;
                Os[c * (kBM + 1) + r] = ep[mi][b2][v];
            }
    __syncthreads();
    for (int q = tid; q < kNB * kBM; q += kThreads) {  // coalesced column writes
        const int c = q / kBM, r = q % kBM;
        const int64_t row = row0 + r;
        if (c < nbw && row < m) x[(c0 + c) * ldx + row] = Os[c * (kBM + 1) + r];
    }
}

__global__ void diag_zero_check_kernel(int64_t k, const double *__restrict__ u, int64_t ldu, int *__restrict__ flag) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < k && u[i * ldu + i] == 0.0) atomicExch(flag, 1);
}

int trsm_block(int64_t m, int64_t k, int64_t c0, const double *b, int64_t ldb, const int64_t *cols, const double *u,
               int64_t ldu, const double *dinv_blk, double *x, int64_t ldx, cudaStream_t st, bool pdl) {
    if (m <= 0 || c0 >= k) return 0;
    static thread_local int attr_dev = -1;
    if (attr_dev != current_device()) {
        CQ_CUDA(cudaFuncSetAttribute(trsm_block_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTrsmSmem),
                "trsm smem attr");
        attr_dev = current_device();
    }
    // pdl: programmatic dependent launch after a trsm_block of the same solve
    // (the gather of this block's source columns overlaps its tail)
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.gridDim = dim3((unsigned)((m + kBM - 1) / kBM));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = kTrsmSmem;
    cfg.stream = st;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    CQ_CUDA(cudaLaunchKernelEx(&cfg, trsm_block_kernel, m, k, c0, b, ldb, cols, u, ldu, dinv_blk, x, ldx),
            "trsm block launch");
    note_launch();
    return check_launch("trsm_block_kernel");
}

int trsm_right(int64_t m, int64_t k, const double *b, int64_t ldb, const int64_t *cols, const double *u,
               int64_t ldu, double *x, int64_t ldx, cudaStream_t st, const BlockSink *sink, bool check_diag,
               const cudaEvent_t *block_ev) {
    if (m <= 0 || k <= 0) return 0;
    if (check_diag) {
        // zero diagonal -> the reference throws std::domain_error (linalg.cc:250-252)
        int *flag = workspace().get<int>("trsm.flag", 1);
        CQ_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), st), "memset flag");
        diag_zero_check_kernel<<<(unsigned)((k + 255) / 256), 256, 0, st>>>(k, u, ldu, flag);
        note_launch();
        int hflag = 0;
        CQ_CUDA(cudaMemcpyAsync(&hflag, flag, sizeof(int), cudaMemcpyDeviceToHost, st), "flag d2h");
        CQ_CUDA(cudaStreamSynchronize(st), "trsm sync");
        if (hflag) {
            set_error("trsm_right: singular preconditioner (zero diagonal)");
            return CQRRPT_GPU_ERR_SINGULAR;
        }
    }
    CQ_CUDA(cudaFuncSetAttribute(trsm_block_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTrsmSmem),
            "trsm smem attr");
    const int64_t nblk = (k + kNB - 1) / kNB;
    double *dinv = workspace().get<double>("trsm.dinv", (size_t)(nblk * kNB * kNB));
    if (!dinv) return fail_nomem("trsm diagonal-block inverses");
    CQ_TRY(trtri_diag_blocks(k, u, ldu, dinv, st));
    // the INT8 engine stages right-hand-side columns with 16-byte bulk copies
    // and tensor-map boxes, whose row bound is applied at 16-byte granularity
    // (measured: an odd m lets the store write row m): even m, even leading
    // dimensions, 16-byte aligned bases
    const bool aligned = ((reinterpret_cast<uintptr_t>(b) | reinterpret_cast<uintptr_t>(x)) & 15) == 0 &&
                         ((ldb | ldx | m) & 1) == 0;
    if (aligned && trsm_use_ozaki(m, k))
        return trsm_right_oz(m, k, b, ldb, cols, u, ldu, x, ldx, st, sink, dinv, block_ev);
    const unsigned grid = (unsigned)((m + kBM - 1) / kBM);
    cudaEvent_t *evs = nullptr;  // one per block, reused across calls (per device)
    if (sink) CQ_TRY(cached_events("trsm.sink", (size_t)((k + kNB - 1) / kNB), &evs));
    for (int64_t c0 = 0; c0 < k; c0 += kNB) {
        {
            cudaLaunchConfig_t cfg = {};
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.gridDim = dim3(grid);
            cfg.blockDim = dim3(kThreads);
            cfg.dynamicSmemBytes = kTrsmSmem;
            cfg.stream = st;
            cfg.attrs = at;
            cfg.numAttrs = c0 > 0 ? 1 : 0;  // the first block follows trtri_diag normally
            CQ_CUDA(cudaLaunchKernelEx(&cfg, trsm_block_kernel, m, k, c0, b, ldb, cols, u, ldu,
                                       (const double *)(dinv + (c0 / kNB) * kNB * kNB), x, ldx),
                    "trsm launch");
        }
        note_launch();
        if (block_ev) CQ_CUDA(cudaEventRecord(block_ev[c0 / kNB], st), "trsm block event");
        if (sink) {  // block c0 is final: download it while the next blocks run
            const size_t e = (size_t)(c0 / kNB);
            CQ_CUDA(cudaEventRecord(evs[e], st), "trsm sink record");
            CQ_CUDA(cudaStreamWaitEvent(sink->copy, evs[e], 0), "trsm sink wait");
            const int64_t nb = std::min<int64_t>(kNB, k - c0);
            CQ_CUDA(cudaMemcpy2DAsync(sink->host + c0 * sink->ldh, sizeof(double) * sink->ldh, x + c0 * ldx,
                                      sizeof(double) * ldx, sizeof(double) * m, nb, cudaMemcpyDeviceToHost,
                                      sink->copy),
                    "trsm sink copy");
        }
    }
    return check_launch("trsm_block_kernel");
}

}  // namespace cqg

// K5b: Gram (SYRK) and a general FP64 DMMA GEMM.
//
// gram: G = X^T X (reference gram, linalg.cc:298-307): upper-triangle 64x64
// tiles, split-K over the m rows into fixed slices; each (tile, slice) CTA
// writes a partial, a second kernel sums the slices in fixed order and
// mirrors the upper triangle, so G is deterministic and bitwise symmetric
// (the property test_linalg.cc:179-189 pins). Because every entry's
// arithmetic depends only on its own two columns and the slice partition of
// m, the leading j x j block of G equals gram(X[:, :j]) bitwise — which is
// what makes the reference's Cholesky-failure retry free (cqrrpt.cc:162-164).
//
// gemm: C = alpha op(A) B + beta C with op(A) in {A, A^T}, used by the
// blocked Cholesky trailing update, the R = R_pre R_sk product and the
// device validator.
//
// Both: 128 threads, 64 x 64 CTA tile (2 x 2 warps of 32 x 32 = 16 DMMA
// accumulators each), K chunks of 32 through a 3-stage cp.async pipeline,
// operand tiles padded so every m8n8k4 fragment load is conflict-free.
#include "common.cuh"
#include "internal.hh"

namespace cqg {

constexpr int kGT = 64;        // tile
constexpr int kGBK = 32;       // K chunk
constexpr int kGStages = 3;
constexpr int kGThreads = 128;
constexpr int kLdK = kGBK + 4;   // [mn][k] layout, 36 = 4 mod 16
constexpr int kLdM = kGT + 8;    // [k][mn] layout, 72 = 8 mod 16
constexpr size_t kGemmSmem = sizeof(double) * kGStages * (kGBK * kLdM + kGT * kLdK);  // covers both A layouts
constexpr size_t kSyrkSmem = sizeof(double) * kGStages * 2 * kGT * kLdK;

// ---------------------------------------------------------------------------
// loaders (8-byte cp.async, zero fill outside the matrix)
// ---------------------------------------------------------------------------
// tile[mn][k] <- src[(c0+mn)*ld + k0 + k]   (column mn contiguous along k)
CQ_DEVI void load_mn_k(double *tile, const double *src, int64_t ld, int64_t c0, int64_t ncols, int64_t k0,
                       int64_t kmax, int tid) {
#pragma unroll
    for (int it = 0; it < (kGT * kGBK) / kGThreads; ++it) {
        int q = it * kGThreads + tid;
        int mn = q / kGBK, kk = q % kGBK;
        bool ok = (c0 + mn < ncols) && (k0 + kk < kmax);
        const double *p = src + (ok ? (c0 + mn) * ld + k0 + kk : 0);
        cp_async8_zfill(tile + mn * kLdK + kk, p, ok ? 8 : 0);
    }
}
// tile[k][mn] <- src[(k0+k)*ld + r0 + mn]   (column k contiguous along mn)
CQ_DEVI void load_k_mn(double *tile, const double *src, int64_t ld, int64_t r0, int64_t nrows, int64_t k0,
                       int64_t kmax, int tid) {
#pragma unroll
    for (int it = 0; it < (kGT * kGBK) / kGThreads; ++it) {
        int q = it * kGThreads + tid;
        int kk = q / kGT, mn = q % kGT;
        bool ok = (r0 + mn < nrows) && (k0 + kk < kmax);
        const double *p = src + (ok ? (k0 + kk) * ld + r0 + mn : 0);
        cp_async8_zfill(tile + kk * kLdM + mn, p, ok ? 8 : 0);
    }
}

// 32x32 warp tile on a 4-deep k step. a_at(mi) / b_at(ni) give the fragment.
#define DMMA_WARP_STEP(acc, A_EXPR, B_EXPR)                                         \
    {                                                                               \
        double af[4], bf[4];                                                        \
        _Pragma("unroll") for (int mi = 0; mi < 4; ++mi) af[mi] = (A_EXPR);         \
        _Pragma("unroll") for (int ni = 0; ni < 4; ++ni) bf[ni] = (B_EXPR);         \
        _Pragma("unroll") for (int mi = 0; mi < 4; ++mi)                            \
            _Pragma("unroll") for (int ni = 0; ni < 4; ++ni)                        \
                dmma884(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);            \
    }

// ---------------------------------------------------------------------------
// SYRK partials: tile list (ti, tj) with ti <= tj, split-K slices.
// part[(slice * ntiles + tile) * 64*64 + c*64 + r] (col-major 64 x 64)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kGThreads, 2)
    syrk_partial_kernel(int64_t m, int64_t k, const double *__restrict__ x, int64_t ldx, int64_t rows_per_slice,
                        const int2 *__restrict__ tiles, int64_t ntiles, double *__restrict__ part) {
    extern __shared__ __align__(16) double sm[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int wm = warp >> 1, wn = warp & 1;
    const int64_t tile = blockIdx.x, slice = blockIdx.y;
    const int2 tt = tiles[tile];
    const int64_t ci = (int64_t)tt.x * kGT, cj = (int64_t)tt.y * kGT;
    const int64_t kbeg = slice * rows_per_slice;
    const int64_t kend = cmin<int64_t>(kbeg + rows_per_slice, m);
    const int nchunks = (int)((kend - kbeg + kGBK - 1) / kGBK);

    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    auto As = [&](int s) { return sm + s * 2 * kGT * kLdK; };
    auto Bs = [&](int s) { return sm + s * 2 * kGT * kLdK + kGT * kLdK; };
    auto load = [&](int kc, int s) {
        int64_t k0 = kbeg + (int64_t)kc * kGBK;
        load_mn_k(As(s), x, ldx, ci, k, k0, kend, tid);
        load_mn_k(Bs(s), x, ldx, cj, k, k0, kend, tid);
    };
#pragma unroll
    for (int s = 0; s < kGStages - 1; ++s) {
        if (s < nchunks) load(s, s);
        cp_async_commit();
    }
    for (int kc = 0; kc < nchunks; ++kc) {
        cp_async_wait<kGStages - 2>();
        __syncthreads();
        {
            int nk = kc + kGStages - 1;
            if (nk < nchunks) load(nk, nk % kGStages);
            cp_async_commit();
        }
        const double *as = As(kc % kGStages) + (wm * 32 + g) * kLdK + t;
        const double *bs = Bs(kc % kGStages) + (wn * 32 + g) * kLdK + t;
#pragma unroll
        for (int kk = 0; kk < kGBK; kk += 4)
            DMMA_WARP_STEP(acc, as[mi * 8 * kLdK + kk], bs[ni * 8 * kLdK + kk]);
    }
    cp_async_wait<0>();
    double *out = part + (slice * ntiles + tile) * (int64_t)(kGT * kGT);
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) {
            int r = wm * 32 + mi * 8 + g, c = wn * 32 + ni * 8 + 2 * t;
            out[c * kGT + r] = acc[mi][ni][0];
            out[(c + 1) * kGT + r] = acc[mi][ni][1];
        }
}

// G[i][j] = sum_s part[s][tile(i,j)] for i <= j (upper), mirrored below.
__global__ void syrk_reduce_kernel(int64_t k, int64_t nslices, const int2 *__restrict__ tiles, int64_t ntiles,
                                   const double *__restrict__ part, double *__restrict__ gmat, int64_t ldg) {
    const int64_t tile = blockIdx.x;
    const int2 tt = tiles[tile];
    for (int q = threadIdx.x; q < kGT * kGT; q += blockDim.x) {
        int c = q / kGT, r = q % kGT;
        int64_t i = (int64_t)tt.x * kGT + r, j = (int64_t)tt.y * kGT + c;
        if (i >= k || j >= k || i > j) continue;
        double s = 0.0;
        for (int64_t sl = 0; sl < nslices; ++sl) s += part[(sl * ntiles + tile) * (int64_t)(kGT * kGT) + q];
        gmat[j * ldg + i] = s;
        gmat[i * ldg + j] = s;
    }
}

int gram(int64_t m, int64_t k, const double *x, int64_t ldx, double *gmat, int64_t ldg, Workspace &ws,
         cudaStream_t st) {
    if (k <= 0) return 0;
    const int64_t nt = (k + kGT - 1) / kGT;
    const int64_t ntiles = nt * (nt + 1) / 2;
    int2 *tiles = ws.get<int2>("gram.tiles", ntiles);
    std::vector<int2> h((size_t)ntiles);
    {
        size_t q = 0;
        for (int64_t j = 0; j < nt; ++j)
            for (int64_t i = 0; i <= j; ++i) h[q++] = make_int2((int)i, (int)j);
    }
    // slices: fill >= 2 waves of 2 CTAs/SM, slices at least 256 rows
    const int sms = num_sms();
    int64_t want = std::max<int64_t>(1, (4 * (int64_t)sms + ntiles - 1) / ntiles);
    int64_t max_slices = std::max<int64_t>(1, m / 256);
    int64_t nslices = std::min(want, max_slices);
    int64_t rps = ((m + nslices - 1) / nslices + kGBK - 1) / kGBK * kGBK;
    nslices = std::max<int64_t>(1, (m + rps - 1) / rps);
    double *part = ws.get<double>("gram.part", (size_t)(nslices * ntiles * kGT * kGT));
    if (!tiles || !part) return fail_nomem("gram workspace");
    CQ_CUDA(cudaMemcpyAsync(tiles, h.data(), sizeof(int2) * ntiles, cudaMemcpyHostToDevice, st), "tiles h2d");
    CQ_CUDA(cudaFuncSetAttribute(syrk_partial_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSyrkSmem),
            "syrk smem attr");
    if (m > 0) {
        syrk_partial_kernel<<<dim3((unsigned)ntiles, (unsigned)nslices), kGThreads, kSyrkSmem, st>>>(
            m, k, x, ldx, rps, tiles, ntiles, part);
        note_launch();
    } else {
        CQ_CUDA(cudaMemsetAsync(part, 0, sizeof(double) * ntiles * kGT * kGT, st), "memset part");
        nslices = 1;
    }
    syrk_reduce_kernel<<<(unsigned)ntiles, 256, 0, st>>>(k, nslices, tiles, ntiles, part, gmat, ldg);
    note_launch();
    // the host vector must outlive the async copy
    CQ_CUDA(cudaStreamSynchronize(st), "gram sync");
    return check_launch("syrk kernels");
}

// ---------------------------------------------------------------------------
// general GEMM: C (M x N) = alpha op(A) B + beta C. UPPER_ONLY skips tiles
// strictly below the diagonal (ti > tj) and entries i > j inside diagonal tiles.
// ---------------------------------------------------------------------------
template <bool TRANS_A, bool UPPER_ONLY>
__global__ void __launch_bounds__(kGThreads, 2)
    gemm_kernel(int64_t M, int64_t N, int64_t K, double alpha, const double *__restrict__ a, int64_t lda,
                const double *__restrict__ b, int64_t ldb, double beta, double *__restrict__ c, int64_t ldc,
                const int64_t *__restrict__ skip_flag) {
    if (skip_flag && *skip_flag) return;
    const int64_t ti = blockIdx.x, tj = blockIdx.y;
    if (UPPER_ONLY && ti > tj) return;
    extern __shared__ __align__(16) double sm[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int wm = warp >> 1, wn = warp & 1;
    const int64_t r0 = ti * kGT, c0 = tj * kGT;
    constexpr int aStride = TRANS_A ? kGT * kLdK : kGBK * kLdM;
    auto As = [&](int s) { return sm + s * (aStride + kGT * kLdK); };
    auto Bs = [&](int s) { return sm + s * (aStride + kGT * kLdK) + aStride; };
    const int nchunks = (int)((K + kGBK - 1) / kGBK);

    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    auto load = [&](int kc, int s) {
        int64_t k0 = (int64_t)kc * kGBK;
        if (TRANS_A) load_mn_k(As(s), a, lda, r0, M, k0, K, tid);   // A is K x M
        else load_k_mn(As(s), a, lda, r0, M, k0, K, tid);           // A is M x K
        load_mn_k(Bs(s), b, ldb, c0, N, k0, K, tid);
    };
#pragma unroll
    for (int s = 0; s < kGStages - 1; ++s) {
        if (s < nchunks) load(s, s);
        cp_async_commit();
    }
    for (int kc = 0; kc < nchunks; ++kc) {
        cp_async_wait<kGStages - 2>();
        __syncthreads();
        {
            int nk = kc + kGStages - 1;
            if (nk < nchunks) load(nk, nk % kGStages);
            cp_async_commit();
        }
        const double *bs = Bs(kc % kGStages) + (wn * 32 + g) * kLdK + t;
        if (TRANS_A) {
            const double *as = As(kc % kGStages) + (wm * 32 + g) * kLdK + t;
#pragma unroll
            for (int kk = 0; kk < kGBK; kk += 4)
                DMMA_WARP_STEP(acc, as[mi * 8 * kLdK + kk], bs[ni * 8 * kLdK + kk]);
        } else {
            const double *as = As(kc % kGStages) + t * kLdM + wm * 32 + g;
#pragma unroll
            for (int kk = 0; kk < kGBK; kk += 4)
                DMMA_WARP_STEP(acc, as[kk * kLdM + mi * 8], bs[ni * 8 * kLdK + kk]);
        }
    }
    cp_async_wait<0>();
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni)
#pragma unroll
            for (int v = 0; v < 2; ++v) {
                int64_t i = r0 + wm * 32 + mi * 8 + g, j = c0 + wn * 32 + ni * 8 + 2 * t + v;
                if (i < M && j < N && (!UPPER_ONLY || i <= j)) {
                    double val = alpha * acc[mi][ni][v];
                    if (beta != 0.0) val = fma(beta, c[j * ldc + i], val);
                    c[j * ldc + i] = val;
                }
            }
}

template <bool TA, bool UP>
static int launch_gemm(int64_t M, int64_t N, int64_t K, double alpha, const double *a, int64_t lda,
                       const double *b, int64_t ldb, double beta, double *c, int64_t ldc, const int64_t *skip,
                       cudaStream_t st) {
    auto kern = gemm_kernel<TA, UP>;
    CQ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGemmSmem), "gemm attr");
    dim3 grid((unsigned)((M + kGT - 1) / kGT), (unsigned)((N + kGT - 1) / kGT));
    kern<<<grid, kGThreads, kGemmSmem, st>>>(M, N, K, alpha, a, lda, b, ldb, beta, c, ldc, skip);
    note_launch();
    return check_launch("gemm_kernel");
}

int gemm(bool trans_a, int64_t M, int64_t N, int64_t K, double alpha, const double *a, int64_t lda,
         const double *b, int64_t ldb, double beta, double *c, int64_t ldc, cudaStream_t st) {
    if (M <= 0 || N <= 0) return 0;
    return trans_a ? launch_gemm<true, false>(M, N, K, alpha, a, lda, b, ldb, beta, c, ldc, nullptr, st)
                   : launch_gemm<false, false>(M, N, K, alpha, a, lda, b, ldb, beta, c, ldc, nullptr, st);
}

// upper-triangle-only C -= A^T B (Cholesky trailing update), skipped when
// *skip_flag != 0 (a failure was already found)
int gemm_tn_upper(int64_t N, int64_t K, double alpha, const double *a, int64_t lda, const double *b, int64_t ldb,
                  double beta, double *c, int64_t ldc, const int64_t *skip_flag, cudaStream_t st) {
    if (N <= 0) return 0;
    return launch_gemm<true, true>(N, N, K, alpha, a, lda, b, ldb, beta, c, ldc, skip_flag, st);
}

}  // namespace cqg

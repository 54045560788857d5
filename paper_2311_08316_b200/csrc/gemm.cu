// FP64 DMMA GEMM engine shared by the contraction passes.
//
//   C_out = alpha * op(A) * B + beta * C_in        op(A) in {A, A^T}
//
// Used by: the recursive TRSM updates (K5a/K8, trsm.cu), the Gram SYRK (K5b,
// split-K partials), the blocked Cholesky trailing update (K6), the
// R = R_pre R_sk product (K9) and the device validator.
//
// sm_100a has no FP64 tcgen05 kind, so the MMA is warp-level
// mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4). CTA = 4 warps, tile 64x128 or
// 128x64, every warp owns a 32x64 accumulator block (32 DMMAs per 4-deep k
// step against 12 fragment loads). K streams in 16-deep chunks through a
// 3-stage cp.async pipeline; the shared tiles are unpadded and XOR-swizzled
// so all fragment loads and async fills are bank-conflict free, which keeps a
// stage at 24 KB and allows 3 CTAs (12 warps) per SM.
#include <cstdlib>
#include <string>

#include "common.cuh"
#include "gemm.cuh"
#include "internal.hh"

namespace cqg {

constexpr int kBK = 16;
constexpr int kStages = 3;
constexpr int kThreads = 128;

// swizzled offsets (doubles) inside a stage tile
// [k][m] layout (A, not transposed): BM doubles per k row
template <int BM>
CQ_DEVI int sw_km(int k, int m) {
    return k * BM + (m ^ ((k & 1) << 3));
}
// [r][k] layout (B, and A transposed): 16 doubles per row
CQ_DEVI int sw_rk(int r, int k) { return r * kBK + (k ^ ((r & 3) << 2)); }

template <int BM, int BN, bool TA, bool BATCH>
__global__ void __launch_bounds__(kThreads, 3) dgemm_kernel(GemmArgs P) {
    constexpr int WM = BM / 32;  // warps along M
    static_assert(WM * (BN / 64) == 4, "4 warps of 32x64");
    extern __shared__ __align__(16) double sm[];
    if (P.skip_flag && *P.skip_flag) return;
    int64_t tm, tn;
    if (P.tiles) {
        const int2 tt = P.tiles[blockIdx.x];
        tm = tt.x;
        tn = tt.y;
    } else {
        tm = blockIdx.x;
        tn = blockIdx.y;
    }
    const int64_t r0 = tm * BM, c0 = P.tile_n64 ? tn * 64 : tn * BN;
    if (P.upper_only && r0 > c0 + BN - 1) return;
    const int64_t z = blockIdx.z;
    // BATCH: grid.z indexes independent problems (element offsets below);
    // otherwise it is the split-K slice
    const int64_t za = BATCH ? z * P.bs_a : 0, zb = BATCH ? z * P.bs_b : 0;
    const int64_t kbeg = BATCH ? 0 : z * P.k_per_split;
    const int64_t kend = BATCH ? P.K : cmin<int64_t>(kbeg + P.k_per_split, P.K);
    const int nchunks = (int)((kend - kbeg + kBK - 1) / kBK);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int wm = warp % WM, wn = warp / WM;
    double *const As0 = sm;
    double *const Bs0 = sm + kStages * BM * kBK;

    double acc[4][8][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    auto load = [&](int kc, int s) {
        const int64_t k0 = kbeg + (int64_t)kc * kBK;
        double *as = As0 + s * BM * kBK;
        double *bs = Bs0 + s * BN * kBK;
        if (P.vec16) {  // element pairs (16-byte copies; the swizzles keep pairs adjacent)
            if (!TA) {  // A tile [k][m]: pairs along m
#pragma unroll
                for (int it = 0; it < BM * kBK / 2 / kThreads; ++it) {
                    const int q = it * kThreads + tid;
                    const int kk = q / (BM / 2), mm = (q % (BM / 2)) * 2;
                    const bool ok = (r0 + mm < P.M) && (k0 + kk < kend);
                    const double *src = P.A + za + (ok ? (k0 + kk) * P.lda + r0 + mm : 0);
                    cp_async16_zfill(as + sw_km<BM>(kk, mm), src, ok ? (r0 + mm + 1 < P.M ? 16 : 8) : 0);
                }
            } else {  // A^T tile [m][k]: pairs along k
#pragma unroll
                for (int it = 0; it < BM * kBK / 2 / kThreads; ++it) {
                    const int q = it * kThreads + tid;
                    const int mm = q / (kBK / 2), kk = (q % (kBK / 2)) * 2;
                    const bool ok = (r0 + mm < P.M) && (k0 + kk < kend);
                    const double *src = P.A + za + (ok ? (r0 + mm) * P.lda + k0 + kk : 0);
                    cp_async16_zfill(as + sw_rk(mm, kk), src, ok ? (k0 + kk + 1 < kend ? 16 : 8) : 0);
                }
            }
#pragma unroll
            for (int it = 0; it < BN * kBK / 2 / kThreads; ++it) {  // B tile [n][k]: pairs along k
                const int q = it * kThreads + tid;
                const int nn = q / (kBK / 2), kk = (q % (kBK / 2)) * 2;
                const bool ok = (c0 + nn < P.N) && (k0 + kk < kend);
                const double *src = P.B + zb + (ok ? (c0 + nn) * P.ldb + k0 + kk : 0);
                cp_async16_zfill(bs + sw_rk(nn, kk), src, ok ? (k0 + kk + 1 < kend ? 16 : 8) : 0);
            }
            return;
        }
        if (!TA) {  // A: M x K col-major, tile [k][m]
#pragma unroll
            for (int it = 0; it < BM * kBK / kThreads; ++it) {
                int q = it * kThreads + tid;
                int kk = q / BM, mm = q % BM;
                bool ok = (r0 + mm < P.M) && (k0 + kk < kend);
                const double *src = P.A + za + (ok ? (k0 + kk) * P.lda + r0 + mm : 0);
                cp_async8_zfill(as + sw_km<BM>(kk, mm), src, ok ? 8 : 0);
            }
        } else {  // A: K x M col-major (op = A^T), tile [m][k]
#pragma unroll
            for (int it = 0; it < BM * kBK / kThreads; ++it) {
                int q = it * kThreads + tid;
                int mm = q / kBK, kk = q % kBK;
                bool ok = (r0 + mm < P.M) && (k0 + kk < kend);
                const double *src = P.A + za + (ok ? (r0 + mm) * P.lda + k0 + kk : 0);
                cp_async8_zfill(as + sw_rk(mm, kk), src, ok ? 8 : 0);
            }
        }
#pragma unroll
        for (int it = 0; it < BN * kBK / kThreads; ++it) {  // B: K x N col-major, tile [n][k]
            int q = it * kThreads + tid;
            int nn = q / kBK, kk = q % kBK;
            bool ok = (c0 + nn < P.N) && (k0 + kk < kend);
            const double *src = P.B + zb + (ok ? (c0 + nn) * P.ldb + k0 + kk : 0);
            cp_async8_zfill(bs + sw_rk(nn, kk), src, ok ? 8 : 0);
        }
    };

#pragma unroll
    for (int s = 0; s < kStages - 1; ++s) {
        if (s < nchunks) load(s, s);
        cp_async_commit();
    }
    for (int kc = 0; kc < nchunks; ++kc) {
        cp_async_wait<kStages - 2>();
        __syncthreads();
        {
            int nk = kc + kStages - 1;
            if (nk < nchunks) load(nk, nk % kStages);
            cp_async_commit();
        }
        const double *as = As0 + (kc % kStages) * BM * kBK;
        const double *bs = Bs0 + (kc % kStages) * BN * kBK;
        const int mb = wm * 32 + g, nb = wn * 64 + g;
#pragma unroll
        for (int kk = 0; kk < kBK; kk += 4) {
            double af[4], bf[8];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
                af[mi] = TA ? as[sw_rk(mb + 8 * mi, kk + t)] : as[sw_km<BM>(kk + t, mb + 8 * mi)];
#pragma unroll
            for (int ni = 0; ni < 8; ++ni) bf[ni] = bs[sw_rk(nb + 8 * ni, kk + t)];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                for (int ni = 0; ni < 8; ++ni) dmma884(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
        }
    }
    cp_async_wait<0>();

    // ---- epilogue ------------------------------------------------------------
    if (P.part) {  // split-K partial tile, column-major BM x BN
        const int64_t tix = P.tiles ? (int64_t)blockIdx.x : (int64_t)blockIdx.y * gridDim.x + blockIdx.x;
        double *out = P.part + ((int64_t)z * P.ntiles_part + tix) * (int64_t)(BM * BN);
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
            for (int ni = 0; ni < 8; ++ni)
#pragma unroll
                for (int v = 0; v < 2; ++v) {
                    int r = wm * 32 + mi * 8 + g, c = wn * 64 + ni * 8 + 2 * t + v;
                    out[c * BM + r] = acc[mi][ni][v];
                }
        return;
    }
#pragma unroll
    for (int ni = 0; ni < 8; ++ni)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
            const int64_t j = c0 + wn * 64 + ni * 8 + 2 * t + v;
            if (j >= P.N) continue;
            const double *cin = nullptr;
            if (P.beta != 0.0) cin = P.Cin + (BATCH ? z * P.bs_cin : 0) + (P.cin_cols ? P.cin_cols[j] : j) * P.ldcin;
            double *cout = P.Cout + (BATCH ? z * P.bs_c : 0) + j * P.ldc;
#pragma unroll
            for (int mi = 0; mi < 4; ++mi) {
                const int64_t i = r0 + wm * 32 + mi * 8 + g;
                if (i < P.M && (!P.upper_only || i <= j)) {
                    double val = P.alpha * acc[mi][ni][v];
                    if (cin) val = fma(P.beta, cin[i], val);
                    cout[i] = val;
                }
            }
        }
}

template <int BM, int BN>
size_t gemm_smem() {
    return sizeof(double) * kStages * (BM + BN) * kBK;
}

template <int BM, int BN, bool TA, bool BATCH>
static int launch(const GemmArgs &P, dim3 grid, cudaStream_t st) {
    auto kern = dgemm_kernel<BM, BN, TA, BATCH>;
    const size_t smem = gemm_smem<BM, BN>();
    static thread_local int configured[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && !configured[dev]) {
        CQ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "gemm attr");
        configured[dev] = 1;
    }
    kern<<<grid, kThreads, smem, st>>>(P);
    note_launch();
    return check_launch("dgemm_kernel");
}

template <int BM, int BN>
static int launch_shape(bool trans_a, bool batch, const GemmArgs &P, dim3 grid, cudaStream_t st) {
    if (batch) return trans_a ? launch<BM, BN, true, true>(P, grid, st) : launch<BM, BN, false, true>(P, grid, st);
    return trans_a ? launch<BM, BN, true, false>(P, grid, st) : launch<BM, BN, false, false>(P, grid, st);
}

// Tile shape: 128x64 for tall-skinny outputs (N <= 64), 64x128 otherwise.
int gemm_ex(bool trans_a, GemmArgs P, int64_t splits, cudaStream_t st) {
    if (P.M <= 0 || P.N <= 0) return 0;
    if (splits < 1) splits = 1;
    if (P.batch > 1) {
        if (P.part) return fail_internal("gemm_ex: batched split-K is not supported");
        splits = P.batch;  // grid.z = problems
    } else if (P.k_per_split <= 0) {
        P.k_per_split = (P.K + splits - 1) / splits;
    }
    const bool tall = P.N <= 64;
    const int BM = tall ? 128 : 64, BN = tall ? 64 : 128;
    {  // 16-byte staging: 16-byte aligned operands, even strides and split starts
        auto al = [](const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
        P.vec16 = al(P.A) && al(P.B) && P.lda % 2 == 0 && P.ldb % 2 == 0 &&
                  (P.batch <= 1 || (P.bs_a % 2 == 0 && P.bs_b % 2 == 0)) && (splits <= 1 || P.k_per_split % 2 == 0);
    }
    dim3 grid;
    if (P.tiles) grid = dim3((unsigned)P.ntiles_part, 1, (unsigned)splits);
    else grid = dim3((unsigned)((P.M + BM - 1) / BM), (unsigned)((P.N + BN - 1) / BN), (unsigned)splits);
    const bool batch = P.batch > 1;
    if (tall) return launch_shape<128, 64>(trans_a, batch, P, grid, st);
    return launch_shape<64, 128>(trans_a, batch, P, grid, st);
}

// Split-K reduction: C = alpha * sum_s part[s] (+ beta C), slices in order.
template <int BM, int BN>
__global__ void __launch_bounds__(256) splitk_reduce_kernel(int64_t M, int64_t N, int64_t ntm, int64_t ntiles,
                                                            int64_t splits, const double *__restrict__ part,
                                                            double alpha, double beta, double *__restrict__ c,
                                                            int64_t ldc) {
    const int64_t tix = blockIdx.x;
    const int64_t tm = tix % ntm, tn = tix / ntm;
    for (int e = threadIdx.x; e < BM * BN; e += blockDim.x) {
        const int r = e % BM, cc = e / BM;
        const int64_t i = tm * BM + r, j = tn * BN + cc;
        if (i >= M || j >= N) continue;
        double s = 0.0;
        for (int64_t k = 0; k < splits; ++k) s += part[(k * ntiles + tix) * (int64_t)(BM * BN) + e];
        double v = alpha * s;
        if (beta != 0.0) v = fma(beta, c[j * ldc + i], v);
        c[j * ldc + i] = v;
    }
}

int gemm_splitk(bool trans_a, int64_t M, int64_t N, int64_t K, double alpha, const double *a, int64_t lda,
                const double *b, int64_t ldb, double beta, double *c, int64_t ldc, int64_t splits, Workspace &ws,
                cudaStream_t st) {
    if (M <= 0 || N <= 0) return 0;
    const bool tall = N <= 64;  // gemm_ex's tile choice
    const int BM = tall ? 128 : 64, BN = tall ? 64 : 128;
    const int64_t ntm = (M + BM - 1) / BM, ntn = (N + BN - 1) / BN, ntiles = ntm * ntn;
    splits = std::max<int64_t>(1, std::min<int64_t>(splits, (K + kBK - 1) / kBK));
    const int64_t kps = ((K + splits - 1) / splits + kBK - 1) / kBK * kBK;
    splits = (K + kps - 1) / kps;
    double *part = ws.get<double>("gemm.splitk", (size_t)(splits * ntiles * BM * BN));
    if (!part) return fail_nomem("gemm split-K partials");
    GemmArgs P{};
    P.M = M;
    P.N = N;
    P.K = K;
    P.A = a;
    P.lda = lda;
    P.B = b;
    P.ldb = ldb;
    P.Cin = c;
    P.ldcin = ldc;
    P.Cout = c;
    P.ldc = ldc;
    P.alpha = 1.0;
    P.beta = 0.0;
    P.k_per_split = kps;
    P.part = part;
    P.ntiles_part = ntiles;
    CQ_TRY(gemm_ex(trans_a, P, splits, st));
    if (tall)
        splitk_reduce_kernel<128, 64><<<(unsigned)ntiles, 256, 0, st>>>(M, N, ntm, ntiles, splits, part, alpha, beta,
                                                                        c, ldc);
    else
        splitk_reduce_kernel<64, 128><<<(unsigned)ntiles, 256, 0, st>>>(M, N, ntm, ntiles, splits, part, alpha, beta,
                                                                        c, ldc);
    note_launch();
    return check_launch("splitk_reduce_kernel");
}

int gemm(bool trans_a, int64_t M, int64_t N, int64_t K, double alpha, const double *a, int64_t lda,
         const double *b, int64_t ldb, double beta, double *c, int64_t ldc, cudaStream_t st) {
    GemmArgs P{};
    P.M = M;
    P.N = N;
    P.K = K;
    P.A = a;
    P.lda = lda;
    P.B = b;
    P.ldb = ldb;
    P.Cin = c;
    P.ldcin = ldc;
    P.Cout = c;
    P.ldc = ldc;
    P.alpha = alpha;
    P.beta = beta;
    return gemm_ex(trans_a, P, 1, st);
}

// Plain GEMM when its tiles fill the GPU, else split-K (fixed-order reduce)
// to about three CTAs per SM, K slices of >= 128.
int gemm_fill(bool trans_a, int64_t M, int64_t N, int64_t K, double alpha, const double *a, int64_t lda,
              const double *b, int64_t ldb, double beta, double *c, int64_t ldc, Workspace &ws, cudaStream_t st) {
    if (M <= 0 || N <= 0) return 0;
    const bool tall = N <= 64;
    const int BM = tall ? 128 : 64, BN = tall ? 64 : 128;
    const int64_t tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
    const int64_t sms = num_sms();
    const int64_t splits = std::min<int64_t>({(3 * sms + tiles - 1) / tiles, K / 128, 16});
    if (tiles >= sms || splits < 2) return gemm(trans_a, M, N, K, alpha, a, lda, b, ldb, beta, c, ldc, st);
    return gemm_splitk(trans_a, M, N, K, alpha, a, lda, b, ldb, beta, c, ldc, splits, ws, st);
}

int gemm_tn_upper(int64_t N, int64_t K, double alpha, const double *a, int64_t lda, const double *b, int64_t ldb,
                  double beta, double *c, int64_t ldc, const int64_t *skip_flag, cudaStream_t st) {
    GemmArgs P{};
    P.M = N;
    P.N = N;
    P.K = K;
    P.A = a;
    P.lda = lda;
    P.B = b;
    P.ldb = ldb;
    P.Cin = c;
    P.ldcin = ldc;
    P.Cout = c;
    P.ldc = ldc;
    P.alpha = alpha;
    P.beta = beta;
    P.upper_only = 1;
    P.skip_flag = skip_flag;
    return gemm_ex(true, P, 1, st);
}

// ---------------------------------------------------------------------------
// Gram: G = X^T X (reference gram, linalg.cc:298-307). 64x128 tiles covering
// the upper triangle, split-K over m into fixed slices, then a fixed-order
// slice sum that mirrors the upper triangle -> deterministic and bitwise
// symmetric (test_linalg.cc:179-189). Every entry depends only on its two
// columns and the (k0-independent) slice partition of m, so the leading j x j
// block of G equals gram(X[:, :j]) bitwise — the reference's Cholesky-retry
// property (cqrrpt.cc:162-164) holds without recomputation.
// ---------------------------------------------------------------------------
// Fixed-order sum of the split-K slices (slice 0 first, as before), one CTA per
// (tile, 16-column strip): the slice loads are issued four at a time, and both
// triangles are written coalesced through a shared 64 x 16 block.
constexpr int kRedSW = 16;
__global__ void __launch_bounds__(256) gram_reduce_kernel(int64_t k, int64_t nslices, const int2 *__restrict__ tiles,
                                                          int64_t ntiles, const double *__restrict__ part,
                                                          double *__restrict__ gmat, int64_t ldg) {
    constexpr int BM = 64, BN = 128;
    __shared__ double sblk[kRedSW][BM + 1];
    const int64_t tile = blockIdx.x;
    const int2 tt = tiles[tile];
    const int64_t i0 = (int64_t)tt.x * BM, j0 = (int64_t)tt.y * 64 + (int64_t)blockIdx.y * kRedSW;
    if (i0 >= k || j0 >= k || i0 > j0 + kRedSW - 1) return;  // strip entirely outside the upper triangle
    const int64_t sstride = ntiles * (int64_t)(BM * BN);
    for (int q = threadIdx.x; q < BM * kRedSW; q += blockDim.x) {
        const int c = q / BM, r = q % BM;  // part element (r, c) of the tile at c * BM + r
        const double *pp = part + tile * (int64_t)(BM * BN) + (int64_t)(blockIdx.y * kRedSW + c) * BM + r;
        double sum = 0.0;
        int64_t sl = 0;
        for (; sl + 4 <= nslices; sl += 4) {
            const double a0 = pp[sl * sstride], a1 = pp[(sl + 1) * sstride], a2 = pp[(sl + 2) * sstride],
                         a3 = pp[(sl + 3) * sstride];
            sum += a0;
            sum += a1;
            sum += a2;
            sum += a3;
        }
        for (; sl < nslices; ++sl) sum += pp[sl * sstride];
        sblk[c][r] = sum;
    }
    __syncthreads();
    for (int q = threadIdx.x; q < BM * kRedSW; q += blockDim.x) {  // upper: column j, rows i0.. (coalesced)
        const int c = q / BM, r = q % BM;
        const int64_t i = i0 + r, j = j0 + c;
        if (i < k && j < k && i <= j) gmat[j * ldg + i] = sblk[c][r];
    }
    for (int q = threadIdx.x; q < BM * kRedSW; q += blockDim.x) {  // mirror: column i, rows j0..j0+15
        const int r = q / kRedSW, c = q % kRedSW;
        const int64_t i = i0 + r, j = j0 + c;
        if (i < k && j < k && i < j) gmat[i * ldg + j] = sblk[c][r];
    }
}

// Split-K slices over m (>= 512 rows each) of gram(m, k): every CTA does the
// same work, so the time is waves(ns) * m / ns with waves = ceil(ntiles*ns /
// resident slots); pick the fewest slices within 2% of the best (no ragged
// last wave). Depends on (m, k) only, so a column block (gram_cols) uses the
// same slices as the full Gram and reproduces its entries bitwise.
// min_slices > 0 (the wavefront's Gram columns, gram_cols): that many slices
// (at most m / 512), so the first column blocks, which have only a few tiles,
// still fill the GPU.
static int gram_slices(int64_t m, int64_t k, int64_t *rps_out, int64_t *nslices_out, int64_t min_slices = 0) {
    constexpr int BM = 64, BN = 128;
    const int64_t tm = (k + BM - 1) / BM;
    int64_t ntiles = 0;
    for (int64_t i = 0; i < tm; ++i) ntiles += (k - i * BM + BN - 1) / BN;
    const int sms = num_sms();
    int per_sm = 0;
    CQ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dgemm_kernel<64, 128, true, false>, kThreads,
                                                          gemm_smem<64, 128>()),
            "gram occupancy");
    const int64_t slots = (int64_t)std::max(1, per_sm) * sms;
    const int64_t max_slices = std::max<int64_t>(1, std::min<int64_t>(64, m / 512));
    int64_t nslices = 1;
    {
        double best = 1e300;
        for (int64_t ns = 1; ns <= max_slices; ++ns) {
            const double cost = (double)((ntiles * ns + slots - 1) / slots) / (double)ns;
            if (cost < best * 0.98) {
                best = cost;
                nslices = ns;
            }
        }
    }
    if (min_slices > 0) nslices = std::max<int64_t>(1, std::min<int64_t>(min_slices, m / 512));
    const int64_t rps = ((m + nslices - 1) / nslices + kBK - 1) / kBK * kBK;
    *rps_out = rps;
    *nslices_out = std::max<int64_t>(1, (m + rps - 1) / rps);
    return 0;
}

// Engine choice (CQRRPT_GPU_GRAM=dmma|ozaki overrides): the INT8 emulation
// when cuBLASLt is loadable and the product is large enough to amortise its
// residue passes, else the DMMA SYRK below.
int gram(int64_t m, int64_t k, const double *x, int64_t ldx, double *gmat, int64_t ldg, Workspace &ws,
         cudaStream_t st) {
    const char *env = getenv("CQRRPT_GPU_GRAM");
    const bool force_dmma = env && std::string(env) == "dmma";
    const bool force_oz = env && std::string(env) == "ozaki";
    // at narrow k the int8 GEMMs (one 256 x 256 IMMA tile per modulus and
    // column block) cannot fill the GPU: C5-256's Gram is faster on DMMA (26.8
    // vs 33.2 ms for Gram + potrf + Q), C5-512's on INT8 (75.1 vs 81.3 ms)
    const bool big = (k >= 1024 && m >= 65536) || (k >= 512 && m >= 1048576);
    const bool oz = !force_dmma && (force_oz || big) && gram_ozaki_available();
    if (oz) return gram_ozaki(m, k, x, ldx, gmat, ldg, ws, st);
    return gram_dmma(m, k, x, ldx, gmat, ldg, ws, st);
}

int gram_dmma(int64_t m, int64_t k, const double *x, int64_t ldx, double *gmat, int64_t ldg, Workspace &ws,
              cudaStream_t st) {
    if (k <= 0) return 0;
    constexpr int BM = 64, BN = 128;
    const int64_t tm = (k + BM - 1) / BM;
    // Row tile i (64 rows) takes 128-wide column tiles starting at its own
    // diagonal (columns 64i, 64i+128, ...; tile.y in units of 64 columns):
    // only the lower half of each row's first 64 x 64 block lies below the
    // diagonal (~6% of the work instead of ~12% with a fixed 128-column grid).
    // An entry's DMMA summation order does not depend on its tile, so G is
    // bitwise the same.
    static thread_local std::vector<int2> h;  // outlives the async upload below
    h.clear();
    for (int64_t i = 0; i < tm; ++i)
        for (int64_t c0 = i * BM; c0 < k; c0 += BN) h.push_back(make_int2((int)i, (int)(c0 / 64)));
    const int64_t ntiles = (int64_t)h.size();
    int64_t rps = 0, nslices = 0;
    CQ_TRY(gram_slices(m, k, &rps, &nslices));
    int2 *tiles = ws.get<int2>("gram.tiles", (size_t)ntiles);
    double *part = ws.get<double>("gram.part", (size_t)(nslices * ntiles * BM * BN));
    if (!tiles || !part) return fail_nomem("gram workspace");
    CQ_CUDA(cudaMemcpyAsync(tiles, h.data(), sizeof(int2) * ntiles, cudaMemcpyHostToDevice, st), "tiles h2d");
    if (m > 0) {
        GemmArgs P{};
        P.M = k;
        P.N = k;
        P.K = m;
        P.A = x;
        P.lda = ldx;
        P.B = x;
        P.ldb = ldx;
        P.alpha = 1.0;
        P.k_per_split = rps;
        P.part = part;
        P.ntiles_part = ntiles;
        P.tiles = tiles;
        P.tile_n64 = 1;
        // 16-byte staging (as gemm_ex): aligned X, even ld and slice starts
        P.vec16 = (reinterpret_cast<uintptr_t>(x) & 15) == 0 && ldx % 2 == 0 && rps % 2 == 0;
        GemmArgs *pp = &P;
        dim3 grid((unsigned)ntiles, 1, (unsigned)nslices);
        CQ_TRY((launch<64, 128, true, false>(*pp, grid, st)));
    } else {
        CQ_CUDA(cudaMemsetAsync(part, 0, sizeof(double) * ntiles * BM * BN, st), "memset part");
        nslices = 1;
    }
    gram_reduce_kernel<<<dim3((unsigned)ntiles, (unsigned)(BN / kRedSW)), 256, 0, st>>>(k, nslices, tiles, ntiles,
                                                                                       part, gmat, ldg);
    note_launch();
    return check_launch("gram_reduce_kernel");
}

// Tiles of column block [c0, c1): row tiles 0 .. (c1-1)/64, 128-wide column
// tiles from c0 (an entry's DMMA order does not depend on its tile). The m
// slices are num_sms() of them (gram_slices), whatever the block, so all
// blocks of one factorization agree with each other (not with gram()'s
// fewer slices: a different fixed summation order).
void gram_col_tiles(int64_t c0, int64_t c1, std::vector<int2> &tiles) {
    for (int64_t i = 0; i * 64 < c1; ++i)
        for (int64_t j = c0; j < c1; j += 128) tiles.push_back(make_int2((int)i, (int)(j / 64)));
}

size_t gram_col_part_size(int64_t m, int64_t k, int64_t ntiles) {
    int64_t rps = 0, nslices = 0;
    if (gram_slices(m, k, &rps, &nslices, num_sms())) return 0;
    return (size_t)(nslices * ntiles * 64 * 128);
}

int gram_cols(int64_t m, int64_t k, int64_t c1, const int2 *tiles, int64_t ntiles, const double *x, int64_t ldx,
              double *gmat, int64_t ldg, double *part, cudaStream_t st) {
    if (ntiles <= 0 || m <= 0) return 0;
    int64_t rps = 0, nslices = 0;
    CQ_TRY(gram_slices(m, k, &rps, &nslices, num_sms()));
    GemmArgs P{};
    P.M = c1;
    P.N = c1;
    P.K = m;
    P.A = x;
    P.lda = ldx;
    P.B = x;
    P.ldb = ldx;
    P.alpha = 1.0;
    P.k_per_split = rps;
    P.part = part;
    P.ntiles_part = ntiles;
    P.tiles = tiles;
    P.tile_n64 = 1;
    P.vec16 = (reinterpret_cast<uintptr_t>(x) & 15) == 0 && ldx % 2 == 0 && rps % 2 == 0;
    CQ_TRY((launch<64, 128, true, false>(P, dim3((unsigned)ntiles, 1, (unsigned)nslices), st)));
    gram_reduce_kernel<<<dim3((unsigned)ntiles, (unsigned)(128 / kRedSW)), 256, 0, st>>>(c1, nslices, tiles, ntiles,
                                                                                       part, gmat, ldg);
    note_launch();
    return check_launch("gram_reduce_kernel");
}

}  // namespace cqg

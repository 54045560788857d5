// K5a / K8: fused pivoted-gather + right triangular solve on FP64 tensor cores.
//
//   X (m x k) = B[:, cols] * U^{-1},   U upper-triangular k x k
//
// Reference: trsm_right (linalg.cc:244-277) applied to M.select_columns(J[:k0])
// (dense_matrix.hh:70-80, cqrrpt.cc:262,165) and to M_pre (cqrrpt.cc:280).
//
// Left-looking blocked algorithm, one launch per 64-wide column block jb:
//   X[:, jb] = (B[:, cols(jb)] - X[:, <jb] * U[<jb, jb]) * U[jb, jb]^{-1}
// The update is a DMMA GEMM (mma.sync.m8n8k4.f64 -> DMMA.8x8x4): a CTA owns a
// 128 x 64 tile (4 warps x 32 rows x 64 cols, 32 DMMA accumulators / warp),
// K streams through a 3-stage cp.async pipeline in 16-deep chunks. The
// epilogue stages the accumulator in shared memory, gathers the pivoted
// source columns (coalesced: thread = row), and solves the 64 x 64 diagonal
// block by row substitution in registers with the reference's per-element
// order (subtract U(s,c) x_s for s ascending, then multiply by 1/U(c,c)).
// Algorithmic flops: m*k^2 (the reference's count, flop_model term).
#include "common.cuh"
#include "internal.hh"

namespace cqg {

constexpr int kTBM = 128;  // rows per CTA
constexpr int kTNB = 64;   // column block
constexpr int kTBK = 16;   // K chunk
constexpr int kTStages = 3;
constexpr int kTThreads = 128;
constexpr int kLdA = kTBM + 8;  // 136 = 8 mod 16 -> conflict-free A fragments
constexpr int kLdB = kTBK + 4;  // 20  = 4 mod 16 -> conflict-free B fragments
constexpr int kLdT = kTNB + 1;

constexpr size_t kPipeBytes = sizeof(double) * kTStages * (kTBK * kLdA + kTNB * kLdB);
constexpr size_t kEpiBytes = sizeof(double) * (kTBM * kLdT + kTNB * kTNB + kTNB);
constexpr size_t kTrsmSmem = (kPipeBytes > kEpiBytes) ? kPipeBytes : kEpiBytes;

__global__ void __launch_bounds__(kTThreads, 2)
    trsm_block_kernel(int64_t m, int64_t k, int64_t c0, const double *__restrict__ b, int64_t ldb,
                      const int64_t *__restrict__ cols, const double *__restrict__ u, int64_t ldu,
                      double *__restrict__ x, int64_t ldx) {
    extern __shared__ __align__(16) double sm[];
    double *As = sm;                                 // [stages][16][136]
    double *Bs = sm + kTStages * kTBK * kLdA;        // [stages][64][20]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int64_t row0 = (int64_t)blockIdx.x * kTBM;
    const int nbw = (int)cmin<int64_t>(kTNB, k - c0);

    double acc[4][8][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    const int nchunks = (int)(c0 / kTBK);  // c0 is a multiple of 64
    auto load_chunk = [&](int kc, int stage) {
        const int64_t kb = (int64_t)kc * kTBK;
        double *as = As + stage * kTBK * kLdA;
        double *bs = Bs + stage * kTNB * kLdB;
        // A: X[row0 + mm][kb + kk], 16 x 128, lanes along mm
#pragma unroll
        for (int it = 0; it < (kTBK * kTBM) / kTThreads; ++it) {
            int q = it * kTThreads + tid;
            int kk = q / kTBM, mm = q % kTBM;
            int64_t row = row0 + mm;
            const double *src = x + (kb + kk) * ldx + (row < m ? row : 0);
            cp_async8_zfill(as + kk * kLdA + mm, src, row < m ? 8 : 0);
        }
        // B: U[kb + kk][c0 + nn], 16 x 64, lanes along kk
#pragma unroll
        for (int it = 0; it < (kTBK * kTNB) / kTThreads; ++it) {
            int q = it * kTThreads + tid;
            int nn = q / kTBK, kk = q % kTBK;
            bool ok = nn < nbw;
            const double *src = u + (c0 + (ok ? nn : 0)) * ldu + kb + kk;
            cp_async8_zfill(bs + nn * kLdB + kk, src, ok ? 8 : 0);
        }
    };

    if (nchunks > 0) {
#pragma unroll
        for (int s = 0; s < kTStages - 1; ++s) {
            if (s < nchunks) load_chunk(s, s);
            cp_async_commit();
        }
        for (int kc = 0; kc < nchunks; ++kc) {
            cp_async_wait<kTStages - 2>();
            __syncthreads();
            {
                int nk = kc + kTStages - 1;
                if (nk < nchunks) load_chunk(nk, nk % kTStages);
                cp_async_commit();
            }
            const double *as = As + (kc % kTStages) * kTBK * kLdA + warp * 32 + g;
            const double *bs = Bs + (kc % kTStages) * kTNB * kLdB + g * kLdB + t;
#pragma unroll
            for (int kk = 0; kk < kTBK; kk += 4) {
                double af[4], bf[8];
#pragma unroll
                for (int mi = 0; mi < 4; ++mi) af[mi] = as[(kk + t) * kLdA + mi * 8];
#pragma unroll
                for (int ni = 0; ni < 8; ++ni) bf[ni] = bs[ni * 8 * kLdB + kk];
#pragma unroll
                for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                    for (int ni = 0; ni < 8; ++ni) dmma884(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
            }
        }
        cp_async_wait<0>();
    }
    __syncthreads();  // pipeline buffers are reused by the epilogue

    // ---- epilogue -------------------------------------------------------
    double *Ts = sm;                       // [128][65]
    double *Uj = sm + kTBM * kLdT;         // [64 cols][64 rows] col-major
    double *inv = Uj + kTNB * kTNB;        // [64]
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 8; ++ni) {
            int r = warp * 32 + mi * 8 + g, c = ni * 8 + 2 * t;
            Ts[r * kLdT + c] = acc[mi][ni][0];
            Ts[r * kLdT + c + 1] = acc[mi][ni][1];
        }
    for (int q = tid; q < kTNB * kTNB; q += kTThreads) {
        int cc = q / kTNB, ss = q % kTNB;  // Uj[cc][ss] = U[c0+ss][c0+cc]
        double v;
        if (cc < nbw) v = (ss <= cc) ? u[(c0 + cc) * ldu + c0 + ss] : 0.0;
        else v = (ss == cc) ? 1.0 : 0.0;
        Uj[cc * kTNB + ss] = v;
    }
    __syncthreads();
    if (tid < kTNB) inv[tid] = 1.0 / Uj[tid * kTNB + tid];  // linalg.cc:272
    __syncthreads();

    const int64_t row = row0 + tid;
    if (row < m) {
        double tv[kTNB];
#pragma unroll
        for (int c = 0; c < kTNB; ++c) {
            double bv = 0.0;
            if (c < nbw) {
                int64_t col = cols ? cols[c0 + c] : (c0 + c);
                bv = b[col * ldb + row];
            }
            tv[c] = bv - Ts[tid * kLdT + c];
        }
#pragma unroll
        for (int s = 0; s < kTNB; ++s) {
            const double xs = tv[s] * inv[s];
            tv[s] = xs;
#pragma unroll
            for (int c = s + 1; c < kTNB; ++c) tv[c] = fma(-Uj[c * kTNB + s], xs, tv[c]);
        }
#pragma unroll
        for (int c = 0; c < kTNB; ++c)
            if (c < nbw) x[(c0 + c) * ldx + row] = tv[c];
    }
}

__global__ void diag_zero_check_kernel(int64_t k, const double *__restrict__ u, int64_t ldu, int *__restrict__ flag) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < k && u[i * ldu + i] == 0.0) atomicExch(flag, 1);
}

int trsm_right(int64_t m, int64_t k, const double *b, int64_t ldb, const int64_t *cols, const double *u,
               int64_t ldu, double *x, int64_t ldx, cudaStream_t st) {
    if (m <= 0 || k <= 0) return 0;
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
    static bool attr = false;
    if (!attr) {
        CQ_CUDA(cudaFuncSetAttribute(trsm_block_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTrsmSmem),
                "trsm smem attr");
        attr = true;
    }
    const unsigned grid = (unsigned)((m + kTBM - 1) / kTBM);
    for (int64_t c0 = 0; c0 < k; c0 += kTNB) {
        trsm_block_kernel<<<grid, kTThreads, kTrsmSmem, st>>>(m, k, c0, b, ldb, cols, u, ldu, x, ldx);
        note_launch();
    }
    return check_launch("trsm_block_kernel");
}

}  // namespace cqg

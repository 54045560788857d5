// K6: blocked upper Cholesky G = R^T R with the reference's failure index.
//
// Reference: cholesky (linalg.cc:223-242): column j fails when
// d = g(j,j) - sum_t r(t,j)^2 is <= 0 or non-finite; the 1-based index j+1 is
// reported and the leading j x j factor is valid. Right-looking blocked
// variant with 64-wide panels: diagonal block factor (1 CTA, shared memory),
// panel solve R_jj^{-T} G[jb, >jb] (thread per column), DMMA trailing update
// of the upper triangle. After a failure, later launches see the device flag
// and exit, so the leading block is exactly what was computed before it.
#include "common.cuh"
#include "internal.hh"

namespace cqg {

int gemm_tn_upper(int64_t N, int64_t K, double alpha, const double *a, int64_t lda, const double *b, int64_t ldb,
                  double beta, double *c, int64_t ldc, const int64_t *skip_flag, cudaStream_t st);

constexpr int kPB = 64;

// Diagonal block: 4 threads per column (thread (c, q) keeps rows i = 4s + q of
// column c in registers, static indices only), so a step is 16 predicated
// FMAs per thread across 8 warps. Two barriers per step (rrow is double
// buffered).
constexpr int kPQ = 4;               // threads per column
constexpr int kPS = kPB / kPQ;       // rows per thread
constexpr int kDiagThreads = kPB * kPQ;

__global__ void __launch_bounds__(kDiagThreads) potrf_diag_kernel(int64_t n, double *__restrict__ g, int64_t ldg,
                                                                  int64_t j0, int64_t *__restrict__ fail) {
    if (*fail) return;
    __shared__ double rmat[kPB][kPB + 1];  // R block, [col][row]
    __shared__ double rrow[2][kPB];
    __shared__ double s_rjj;
    __shared__ int s_fail;
    const int nb = (int)cmin<int64_t>(kPB, n - j0);
    const int c = threadIdx.x >> 2, q = threadIdx.x & 3;
    double a[kPS];
    const double *col = g + (j0 + c) * ldg + j0;
#pragma unroll
    for (int s = 0; s < kPS; ++s) {
        const int i = kPQ * s + q;
        a[s] = (c < nb && i <= c) ? col[i] : 0.0;
    }
    if (threadIdx.x == 0) s_fail = 0;
    __syncthreads();
    int base = 0;  // a[s] holds row 4 * (base + s) + q: the window slides so row j is in a[0]
    for (int j = 0; j < nb; ++j) {
        if ((j >> 2) != base) {
#pragma unroll
            for (int s = 0; s + 1 < kPS; ++s) a[s] = a[s + 1];
            a[kPS - 1] = 0.0;
            ++base;
        }
        const bool holder = (q == (j & 3));  // this thread holds row j of its column
        const double ajc = a[0];             // (holder) g(j,c) - sum_{t<j} r(t,j) r(t,c)
        if (holder && c == j) {
            if (ajc <= 0.0 || !isfinite(ajc)) s_fail = j + 1;
            else s_rjj = sqrt(ajc);
        }
        __syncthreads();
        if (s_fail) break;
        double *rr = rrow[j & 1];
        if (holder) {
            // division, not a reciprocal product: on exactly singular Grams the
            // sign of the last Schur complement (the failure index) follows it
            const double rjc = c > j ? ajc / s_rjj : (c == j ? s_rjj : 0.0);
            rr[c] = rjc;
            rmat[c][j] = rjc;
        }
        __syncthreads();
        if (c > j) {
            const double rjc = rr[c];
#pragma unroll
            for (int s = 0; s < kPS; ++s) {
                const int i = kPQ * (base + s) + q;
                if (i > j && i <= c && i < kPB) a[s] = fma(-rr[i], rjc, a[s]);
            }
        }
    }
    const int f = s_fail;
    const int ncols = f ? f - 1 : nb;
    for (int e = threadIdx.x; e < kPB * kPB; e += blockDim.x) {
        int cc = e / kPB, r = e % kPB;
        if (cc < ncols && r <= cc) g[(j0 + cc) * ldg + j0 + r] = rmat[cc][r];
    }
    if (threadIdx.x == 0 && f) *fail = j0 + f;  // 1-based global index
}

// Panel: X = R_jj^{-T} G[j0:j0+nb, cols] for the columns right of the block.
// One warp per column: lane l owns rows l and l+32; at step t the solved x_t
// is broadcast by shuffle and every lane updates its rows below t.
constexpr int kPanelWarps = 8;

__global__ void __launch_bounds__(kPanelWarps * 32) potrf_panel_kernel(int64_t n, double *__restrict__ g,
                                                                      int64_t ldg, int64_t j0,
                                                                      const int64_t *__restrict__ fail) {
    if (*fail) return;
    __shared__ double r[kPB][kPB + 1];  // r[col][row] of R_jj
    const int nb = (int)cmin<int64_t>(kPB, n - j0);
    for (int e = threadIdx.x; e < kPB * kPB; e += blockDim.x) {
        int cc = e / kPB, rr = e % kPB;
        r[cc][rr] = (cc < nb && rr <= cc) ? g[(j0 + cc) * ldg + j0 + rr] : 0.0;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t col = j0 + nb + (int64_t)blockIdx.x * kPanelWarps + w;
    if (col >= n) return;
    double *gc = g + col * ldg + j0;
    const int l0 = lane, l1 = lane + 32;
    double x0 = l0 < nb ? gc[l0] : 0.0, x1 = l1 < nb ? gc[l1] : 0.0;
    for (int t = 0; t < nb; ++t) {
        const double cur = __shfl_sync(0xffffffffu, t < 32 ? x0 : x1, t & 31);
        const double xt = cur / r[t][t];
        if (lane == (t & 31)) {
            if (t < 32) x0 = xt;
            else x1 = xt;
        }
        if (l0 > t && l0 < nb) x0 = fma(-r[l0][t], xt, x0);
        if (l1 > t && l1 < nb) x1 = fma(-r[l1][t], xt, x1);
    }
    if (l0 < nb) gc[l0] = x0;
    if (l1 < nb) gc[l1] = x1;
}

__global__ void zero_strict_lower_kernel(int64_t n, double *__restrict__ a, int64_t lda) {
    int64_t j = blockIdx.x;
    for (int64_t i = j + 1 + threadIdx.x; i < n; i += blockDim.x) a[j * lda + i] = 0.0;
}

int zero_strict_lower(int64_t n, double *a, int64_t lda, cudaStream_t st) {
    if (n <= 1) return 0;
    zero_strict_lower_kernel<<<(unsigned)n, 128, 0, st>>>(n, a, lda);
    note_launch();
    return check_launch("zero_strict_lower");
}

int potrf(int64_t n, double *g, int64_t ldg, int64_t *failure_index, Workspace &ws, cudaStream_t st) {
    *failure_index = 0;
    if (n <= 0) return 0;
    int64_t *fail = ws.get<int64_t>("potrf.fail", 1);
    if (!fail) return fail_nomem("potrf workspace");
    CQ_CUDA(cudaMemsetAsync(fail, 0, sizeof(int64_t), st), "memset fail");
    for (int64_t j0 = 0; j0 < n; j0 += kPB) {
        const int64_t nb = std::min<int64_t>(kPB, n - j0);
        potrf_diag_kernel<<<1, kDiagThreads, 0, st>>>(n, g, ldg, j0, fail);
        note_launch();
        const int64_t rest = n - j0 - nb;
        if (rest > 0) {
            potrf_panel_kernel<<<(unsigned)((rest + kPanelWarps - 1) / kPanelWarps), kPanelWarps * 32, 0, st>>>(
                n, g, ldg, j0, fail);
            note_launch();
            // G[t0:, t0:] -= P^T P, P = R[j0:j0+nb, t0:]
            const int64_t t0 = j0 + nb;
            CQ_TRY(gemm_tn_upper(rest, nb, -1.0, g + t0 * ldg + j0, ldg, g + t0 * ldg + j0, ldg, 1.0,
                                 g + t0 * ldg + t0, ldg, fail, st));
        }
    }
    CQ_TRY(check_launch("potrf kernels"));
    CQ_CUDA(cudaMemcpyAsync(failure_index, fail, sizeof(int64_t), cudaMemcpyDeviceToHost, st), "fail d2h");
    CQ_CUDA(cudaStreamSynchronize(st), "potrf sync");
    return zero_strict_lower(n, g, ldg, st);
}

}  // namespace cqg

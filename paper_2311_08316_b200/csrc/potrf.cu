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

__global__ void __launch_bounds__(256) potrf_diag_kernel(int64_t n, double *__restrict__ g, int64_t ldg, int64_t j0,
                                                         int64_t *__restrict__ fail) {
    if (*fail) return;
    __shared__ double a[kPB][kPB + 1];  // a[col][row]
    __shared__ int s_fail;
    const int nb = (int)cmin<int64_t>(kPB, n - j0);
    for (int q = threadIdx.x; q < kPB * kPB; q += blockDim.x) {
        int c = q / kPB, r = q % kPB;
        a[c][r] = (c < nb && r < nb && r <= c) ? g[(j0 + c) * ldg + j0 + r] : 0.0;
    }
    if (threadIdx.x == 0) s_fail = 0;
    __syncthreads();
    for (int j = 0; j < nb; ++j) {
        // a[j][j] now holds g(j,j) - sum_{t<j} r(t,j)^2
        if (threadIdx.x == 0) {
            double d = a[j][j];
            if (d <= 0.0 || !isfinite(d)) {
                s_fail = j + 1;
            } else {
                a[j][j] = sqrt(d);
            }
        }
        __syncthreads();
        if (s_fail) break;
        const double rjj = a[j][j];
        // row j of R: r(j,c) = a(j,c) / r(j,j) for c > j
        for (int c = j + 1 + threadIdx.x; c < nb; c += blockDim.x) a[c][j] = a[c][j] / rjj;
        __syncthreads();
        // trailing: a(i,c) -= r(j,i) r(j,c) for j < i <= c
        for (int q = threadIdx.x; q < kPB * kPB; q += blockDim.x) {
            int c = q / kPB, i = q % kPB;
            if (c > j && c < nb && i > j && i <= c) a[c][i] = fma(-a[i][j], a[c][j], a[c][i]);
        }
        __syncthreads();
    }
    const int f = s_fail;
    // write back the factored part (all columns before the failure)
    const int ncols = f ? f - 1 : nb;
    for (int q = threadIdx.x; q < kPB * kPB; q += blockDim.x) {
        int c = q / kPB, r = q % kPB;
        if (c < ncols && r <= c) g[(j0 + c) * ldg + j0 + r] = a[c][r];
    }
    if (threadIdx.x == 0 && f) *fail = j0 + f;  // 1-based global index
}

// panel: for each column c >= j0+nb: x = R_jj^{-T} g[j0:j0+nb, c] (forward substitution)
__global__ void __launch_bounds__(128) potrf_panel_kernel(int64_t n, double *__restrict__ g, int64_t ldg, int64_t j0,
                                                          const int64_t *__restrict__ fail) {
    if (*fail) return;
    __shared__ double r[kPB][kPB + 1];  // r[col][row]
    const int nb = (int)cmin<int64_t>(kPB, n - j0);
    for (int q = threadIdx.x; q < kPB * kPB; q += blockDim.x) {
        int c = q / kPB, rr = q % kPB;
        r[c][rr] = (c < nb && rr <= c) ? g[(j0 + c) * ldg + j0 + rr] : (c == rr ? 1.0 : 0.0);
    }
    __syncthreads();
    const int64_t col = j0 + nb + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (col >= n) return;
    double *gc = g + col * ldg + j0;
    double x[kPB];
#pragma unroll
    for (int i = 0; i < kPB; ++i) x[i] = (i < nb) ? gc[i] : 0.0;
#pragma unroll
    for (int i = 0; i < kPB; ++i) {
        double s = x[i];
#pragma unroll
        for (int t = 0; t < i; ++t) s = fma(-r[i][t], x[t], s);
        x[i] = s / r[i][i];
    }
#pragma unroll
    for (int i = 0; i < kPB; ++i)
        if (i < nb) gc[i] = x[i];
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
    CQ_CUDA(cudaMemsetAsync(fail, 0, sizeof(int64_t), st), "memset fail");
    for (int64_t j0 = 0; j0 < n; j0 += kPB) {
        const int64_t nb = std::min<int64_t>(kPB, n - j0);
        potrf_diag_kernel<<<1, 256, 0, st>>>(n, g, ldg, j0, fail);
        note_launch();
        const int64_t rest = n - j0 - nb;
        if (rest > 0) {
            potrf_panel_kernel<<<(unsigned)((rest + 127) / 128), 128, 0, st>>>(n, g, ldg, j0, fail);
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

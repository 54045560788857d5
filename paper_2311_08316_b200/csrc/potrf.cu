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
#include "gemm.cuh"
#include "internal.hh"

namespace cqg {

int gemm_tn_upper(int64_t N, int64_t K, double alpha, const double *a, int64_t lda, const double *b, int64_t ldb,
                  double beta, double *c, int64_t ldc, const int64_t *skip_flag, cudaStream_t st);

constexpr int kPB = 64;

// Diagonal block, unblocked right-looking, 64 threads (thread = column): the
// column lives in registers, shifted up one row per step so the active row
// is always a[0]; R(j, :) is exchanged through shared memory with one CTA
// barrier per side. Every entry receives the right-looking FMAs in column
// order (as the earlier one-warp 32 x 32 sub-block scheme did: R11, R12,
// A22 -= R12^T R12, R22), with the reference's failure rule; the critical
// path per column is one sqrt, one division and one FMA (C2's 1024 x 1024
// factor: 1.32 -> 1.13 ms with this kernel).
__global__ void __launch_bounds__(kPB) potrf_diag64_kernel(int64_t n, double *__restrict__ g, int64_t ldg,
                                                          int64_t j0, int64_t *__restrict__ fail) {
    if (*fail) return;
    __shared__ double blk[kPB][kPB + 1];  // [col][row]: the factor, written row by row
    __shared__ double srow[2 * kPB];      // R(j, :) of the current step (+ zero pad)
    __shared__ double sd;
    const int nb = (int)cmin<int64_t>(kPB, n - j0);
    const int c = threadIdx.x;
    double a[kPB];
#pragma unroll
    for (int t = 0; t < kPB; ++t)  // column c, rows 0..63 (identity padded past nb)
        a[t] = (c < nb && t <= c) ? g[(j0 + c) * ldg + j0 + t] : (c == t ? 1.0 : 0.0);
    srow[kPB + c] = 0.0;
    int f = 0;
#pragma unroll 1
    for (int j = 0; j < kPB; ++j) {
        if (c == j) sd = a[0];  // g(j,j) - sum_{t<j} r(t,j)^2
        __syncthreads();
        const double d = sd;
        if (d <= 0.0 || !isfinite(d)) {  // CTA-uniform
            f = j + 1;
            break;
        }
        const double rjj = sqrt(d);
        const double q = a[0] / rjj;
        const double rjc = c == j ? rjj : q;
        blk[c][j] = rjc;
        srow[c] = rjc;
        __syncthreads();
#pragma unroll
        for (int t = 1; t < kPB; ++t) a[t] = fma(-srow[j + t], rjc, a[t]);  // row j + t (pad: zero)
#pragma unroll
        for (int t = 0; t + 1 < kPB; ++t) a[t] = a[t + 1];
    }
    __syncthreads();
    const int ncols = f ? f - 1 : nb;
    for (int q = c; q < kPB * kPB; q += kPB) {  // factored columns, rows <= col
        const int cc = q / kPB, r = q % kPB;
        if (cc < ncols && r <= cc) g[(j0 + cc) * ldg + j0 + r] = blk[cc][r];
    }
    if (c == 0 && f) *fail = j0 + f;  // 1-based global index
}

// Panel: X = R_jj^{-T} G[j0:j0+nb, cols] for the columns right of the block.
// One warp per column: lane l owns rows l and l+32; at step t the solved x_t
// is broadcast by shuffle and every lane updates its rows below t.
constexpr int kPanelWarps = 8;

__global__ void __launch_bounds__(kPanelWarps * 32) potrf_panel_kernel(int64_t n, double *__restrict__ g,
                                                                      int64_t ldg, int64_t j0, int64_t c_begin,
                                                                      int64_t c_end,
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
    const int64_t col = c_begin + (int64_t)blockIdx.x * kPanelWarps + w;
    if (col >= c_end) return;
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

// One-block lookahead on two streams. Step jb: diag(jb), panel(jb) and C1(jb)
// = the update of row block jb+1 (G[t0:t1, t0:] -= P[:, :nb1]^T P) run on the
// aux stream; C2(jb) = the rest of the trailing update (rows >= t1) runs on
// the caller's stream, so diag(jb+1) and panel(jb+1) overlap it. C1(jb+1)
// waits for C2(jb) (both touch row block jb+2). Every entry still receives
// its updates in block order, so the factor is unchanged.
int potrf(int64_t n, double *g, int64_t ldg, int64_t *failure_index, Workspace &ws, cudaStream_t st) {
    *failure_index = 0;
    if (n <= 0) return 0;
    int64_t *fail = ws.get<int64_t>("potrf.fail", 1);
    if (!fail) return fail_nomem("potrf workspace");
    cudaStream_t aux = nullptr;
    cudaEvent_t *pev = nullptr;
    CQ_TRY(cached_stream("potrf.aux", 0, &aux));
    CQ_TRY(cached_events("potrf.ev", 3, &pev));
    cudaEvent_t ev_in = pev[0], ev_c1 = pev[1], ev_c2 = pev[2];
    CQ_CUDA(cudaMemsetAsync(fail, 0, sizeof(int64_t), st), "memset fail");
    CQ_CUDA(cudaEventRecord(ev_in, st), "potrf record");
    CQ_CUDA(cudaStreamWaitEvent(aux, ev_in, 0), "potrf wait");
    for (int64_t j0 = 0; j0 < n; j0 += kPB) {
        const int64_t nb = std::min<int64_t>(kPB, n - j0);
        potrf_diag64_kernel<<<1, kPB, 0, aux>>>(n, g, ldg, j0, fail);
        note_launch();
        const int64_t rest = n - j0 - nb;
        if (rest <= 0) break;
        potrf_panel_kernel<<<(unsigned)((rest + kPanelWarps - 1) / kPanelWarps), kPanelWarps * 32, 0, aux>>>(
            n, g, ldg, j0, j0 + nb, n, fail);
        note_launch();
        const int64_t t0 = j0 + nb, nb1 = std::min<int64_t>(kPB, rest), t1 = t0 + nb1;
        if (j0 > 0) CQ_CUDA(cudaStreamWaitEvent(aux, ev_c2, 0), "potrf wait c2");  // C2(jb-1) -> row block jb+1
        {  // C1: G[t0:t1, t0:n] -= P[:, 0:nb1]^T P, P = R[j0:j0+nb, t0:n]
            GemmArgs P{};
            P.M = nb1;
            P.N = rest;
            P.K = nb;
            P.A = g + t0 * ldg + j0;
            P.lda = ldg;
            P.B = g + t0 * ldg + j0;
            P.ldb = ldg;
            P.Cin = g + t0 * ldg + t0;
            P.ldcin = ldg;
            P.Cout = g + t0 * ldg + t0;
            P.ldc = ldg;
            P.alpha = -1.0;
            P.beta = 1.0;
            P.skip_flag = fail;
            CQ_TRY(gemm_ex(true, P, 1, aux));
        }
        CQ_CUDA(cudaEventRecord(ev_c1, aux), "potrf record c1");
        if (rest > nb1) {  // C2: G[t1:, t1:] -= P[:, nb1:]^T P[:, nb1:] (upper)
            CQ_CUDA(cudaStreamWaitEvent(st, ev_c1, 0), "potrf wait c1");  // panel(jb) done
            CQ_TRY(gemm_tn_upper(rest - nb1, nb, -1.0, g + t1 * ldg + j0, ldg, g + t1 * ldg + j0, ldg, 1.0,
                                 g + t1 * ldg + t1, ldg, fail, st));
            CQ_CUDA(cudaEventRecord(ev_c2, st), "potrf record c2");
        }
    }
    CQ_CUDA(cudaEventRecord(ev_c1, aux), "potrf record end");
    CQ_CUDA(cudaStreamWaitEvent(st, ev_c1, 0), "potrf join");
    CQ_TRY(check_launch("potrf kernels"));
    CQ_CUDA(cudaMemcpyAsync(failure_index, fail, sizeof(int64_t), cudaMemcpyDeviceToHost, st), "fail d2h");
    CQ_CUDA(cudaStreamSynchronize(st), "potrf sync");
    return zero_strict_lower(n, g, ldg, st);
}

int potrf_cols(int64_t n, double *g, int64_t ldg, int64_t c0, int64_t c1, int64_t *fail, cudaStream_t st) {
    if (c1 <= c0) return 0;
    const int64_t w = c1 - c0;
    for (int64_t j0 = 0; j0 < c0; j0 += kPB) {
        // panel(j): R[j, c0:c1] = R_jj^{-T} G[j, c0:c1]
        potrf_panel_kernel<<<(unsigned)((w + kPanelWarps - 1) / kPanelWarps), kPanelWarps * 32, 0, st>>>(
            n, g, ldg, j0, c0, c1, fail);
        note_launch();
        // update(j): G[t0:c1, c0:c1] -= R[j, t0:c1]^T R[j, c0:c1] (potrf's C1/C2 entries of these columns)
        const int64_t t0 = j0 + kPB;
        GemmArgs P{};
        P.M = c1 - t0;
        P.N = w;
        P.K = kPB;
        P.A = g + t0 * ldg + j0;
        P.lda = ldg;
        P.B = g + c0 * ldg + j0;
        P.ldb = ldg;
        P.Cin = g + c0 * ldg + t0;
        P.ldcin = ldg;
        P.Cout = g + c0 * ldg + t0;
        P.ldc = ldg;
        P.alpha = -1.0;
        P.beta = 1.0;
        P.skip_flag = fail;
        CQ_TRY(gemm_ex(true, P, 1, st));
    }
    potrf_diag64_kernel<<<1, kPB, 0, st>>>(n, g, ldg, c0, fail);
    note_launch();
    return check_launch("potrf_cols");
}

}  // namespace cqg

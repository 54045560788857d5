// X = R^{-1} for an upper-triangular k x k R, in log depth.
//
// Used by stage 2 (rank_stage2, cqrrpt.cc:160-207): the condition estimators
// apply R_ell^{-1} to vectors, and the fast accept needs ||R^{-1}||_F. The
// reference solves with R on every power iteration; here the inverse is formed
// once and every leading block's inverse is its leading block.
//
// Recursive blocking: the 64 x 64 diagonal blocks are inverted in one launch
// (one CTA each, thread per column, back substitution in shared memory), then
// for s = 64, 128, ...: every pair of neighbouring s-blocks [A B; 0 C] gets its
// off-diagonal block -A^{-1} B C^{-1} from two batched DMMA GEMMs. log2(k/64)
// levels, two launches each (plus one for a ragged last pair).
#include "common.cuh"
#include "gemm.cuh"
#include "internal.hh"

namespace cqg {

constexpr int kTB = 64;

// compact = true: block b's inverse goes to x + b*64*64 (column-major, ld 64)
__global__ void __launch_bounds__(kTB) trtri_diag_kernel(int64_t k, const double *__restrict__ r, int64_t ldr,
                                                         double *__restrict__ x, int64_t ldx, bool compact) {
    // rs[col][row]: R_bb in the upper triangle (row <= col); y(i, c) of X_bb
    // (i <= c) lives in the unused strictly-lower slot rs[i][c + 1].
    __shared__ double rs[kTB][kTB + 1];
    __shared__ double inv[kTB];
    const int64_t o = (int64_t)blockIdx.x * kTB;
    const int s = (int)cmin<int64_t>(kTB, k - o);
    for (int e = threadIdx.x; e < kTB * kTB; e += blockDim.x) {
        int c = e / kTB, i = e % kTB;
        rs[c][i] = (c < s && i <= c) ? r[(o + c) * ldr + o + i] : 0.0;
    }
    __syncthreads();
    if (threadIdx.x < s) inv[threadIdx.x] = 1.0 / rs[threadIdx.x][threadIdx.x];
    __syncthreads();
    const int c = threadIdx.x;
    if (c < s) {  // column c: R y = e_c by back substitution
        rs[c][c + 1] = inv[c];
        for (int i = c - 1; i >= 0; --i) {  // four partial sums: no dependent chain of length c
            double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
            int t = i + 1;
            for (; t + 3 <= c; t += 4) {
                a0 = fma(rs[t][i], rs[t][c + 1], a0);
                a1 = fma(rs[t + 1][i], rs[t + 1][c + 1], a1);
                a2 = fma(rs[t + 2][i], rs[t + 2][c + 1], a2);
                a3 = fma(rs[t + 3][i], rs[t + 3][c + 1], a3);
            }
            for (; t <= c; ++t) a0 = fma(rs[t][i], rs[t][c + 1], a0);
            rs[i][c + 1] = -((a0 + a1) + (a2 + a3)) * inv[i];
        }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < kTB * kTB; e += blockDim.x) {
        int cc = e / kTB, i = e % kTB;
        if (compact) x[o * kTB + cc * kTB + i] = (cc < s && i <= cc) ? rs[i][cc + 1] : (cc == i ? 1.0 : 0.0);
        else if (cc < s && i <= cc) x[(o + cc) * ldx + o + i] = rs[i][cc + 1];
    }
}

int trtri_diag_blocks(int64_t k, const double *r, int64_t ldr, double *dinv, cudaStream_t st) {
    if (k <= 0) return 0;
    trtri_diag_kernel<<<(unsigned)((k + kTB - 1) / kTB), kTB, 0, st>>>(k, r, ldr, dinv, kTB, true);
    note_launch();
    return check_launch("trtri_diag_kernel");
}

// A level's GEMM: batched over the pairs when that fills the GPU, else pair by
// pair with split-K (the top levels have one or two large pairs).
static int level_gemm(const GemmArgs &P, Workspace &ws, cudaStream_t st) {
    const int64_t tiles = ((P.M + 63) / 64) * ((P.N + 127) / 128);
    if (P.batch * tiles >= num_sms() || P.K < 256) return gemm_ex(false, P, 1, st);
    for (int64_t p = 0; p < P.batch; ++p)
        CQ_TRY(gemm_fill(false, P.M, P.N, P.K, P.alpha, P.A + p * P.bs_a, P.lda, P.B + p * P.bs_b, P.ldb, P.beta,
                         P.Cout + p * P.bs_c, P.ldc, ws, st));
    return 0;
}

// One level: pairs p = p0 .. p0+np-1 of s-blocks, C of size cs (cs == s
// except for a ragged last pair). t: s x s scratch per pair.
static int trtri_level(int64_t s, int64_t cs, int64_t p0, int64_t np, const double *r, int64_t ldr, double *x,
                       int64_t ldx, double *t, Workspace &ws, cudaStream_t st) {
    const int64_t o = 2 * s * p0;
    GemmArgs P{};
    // T_p = A_p^{-1} B_p  (s x cs, K = s)
    P.M = s;
    P.N = cs;
    P.K = s;
    P.A = x + o * ldx + o;
    P.lda = ldx;
    P.B = r + (o + s) * ldr + o;
    P.ldb = ldr;
    P.Cin = t;
    P.ldcin = s;
    P.Cout = t;
    P.ldc = s;
    P.alpha = 1.0;
    P.beta = 0.0;
    P.batch = np;
    P.bs_a = 2 * s * (ldx + 1);
    P.bs_b = 2 * s * (ldr + 1);
    P.bs_cin = P.bs_c = s * s;
    CQ_TRY(level_gemm(P, ws, st));
    // X[o:o+s, o+s:o+s+cs] = -T_p C_p^{-1}  (s x cs, K = cs)
    GemmArgs Q{};
    Q.M = s;
    Q.N = cs;
    Q.K = cs;
    Q.A = t;
    Q.lda = s;
    Q.B = x + (o + s) * ldx + o + s;
    Q.ldb = ldx;
    Q.Cout = x + (o + s) * ldx + o;
    Q.Cin = Q.Cout;
    Q.ldcin = ldx;
    Q.ldc = ldx;
    Q.alpha = -1.0;
    Q.beta = 0.0;
    Q.batch = np;
    Q.bs_a = s * s;
    Q.bs_b = 2 * s * (ldx + 1);
    Q.bs_cin = Q.bs_c = 2 * s * (ldx + 1);
    return level_gemm(Q, ws, st);
}

int trtri_upper(int64_t k, const double *r, int64_t ldr, double *x, int64_t ldx, Workspace &ws, cudaStream_t st) {
    if (k <= 0) return 0;
    CQ_CUDA(cudaMemset2DAsync(x, sizeof(double) * ldx, 0, sizeof(double) * k, k, st), "trtri zero");
    const int64_t nblk = (k + kTB - 1) / kTB;
    trtri_diag_kernel<<<(unsigned)nblk, kTB, 0, st>>>(k, r, ldr, x, ldx, false);
    note_launch();
    CQ_TRY(check_launch("trtri_diag_kernel"));
    double *t = nullptr;
    if (k > kTB) {
        t = ws.get<double>("trtri.t", (size_t)k * (size_t)k);  // >= full*s*s + s*cs at every level
        if (!t) return fail_nomem("trtri scratch");
    }
    for (int64_t s = kTB; s < k; s *= 2) {
        const int64_t full = k / (2 * s);  // pairs with a full C block
        if (full > 0) CQ_TRY(trtri_level(s, s, 0, full, r, ldr, x, ldx, t, ws, st));
        const int64_t o = 2 * s * full;
        const int64_t cs = k - o - s;  // ragged last pair
        if (cs > 0) CQ_TRY(trtri_level(s, cs, full, 1, r, ldr, x, ldx, t, ws, st));
    }
    return 0;
}

}  // namespace cqg

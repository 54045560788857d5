// TEST INFRASTRUCTURE ONLY: device restatement of the reference's input
// generators' linear algebra, so the full-size parity tests can rebuild the
// BASELINE inputs bit-for-bit in seconds instead of minutes of serial host
// code. Only tests/ load this library (tests/gen/gen.py); it is never part of
// the product path.
//
// What is restated (same operation order as oracle/cqrrpt_oracle.c, which is
// itself pinned bit-for-bit to the built reference by tests/test_oracle.py):
//   dot            linalg.cc:36-50  (4 accumulators, separately rounded
//                                   products in the 4-lane body, a fused last
//                                   product when one element is left over)
//   make_reflector linalg.cc:110-124
//   apply_reflector linalg.cc:126-136 (contracted axpy)
//   householder_qr / accumulate_q / apply_q_left  linalg.cc:139-197
//   matmul         linalg.cc:52-66  (per column j, t ascending: c = fma(b(t,j), a(:,t), c), b == 0 skipped)
// The Gaussian draws themselves (rng.hh:32-36: log / cos) stay on the host.
// Built with --fmad=false: every fused multiply-add below is an explicit fma().
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

constexpr int kWarps = 8;

// dot(a, b, len) of linalg.cc:36-50 by one warp (all lanes return the value).
// Lane l loads elements 4l..4l+3 of each 128-element chunk; the four
// accumulators then take the chunk's products in index order through
// shuffles (every lane runs the same dependent chain, so no divergence).
__device__ double warp_dot(const double *a, const double *b, int64_t len) {
    const int lane = threadIdx.x & 31;
    const int64_t body = (len / 4) * 4;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    for (int64_t base = 0; base < body; base += 128) {
        const int64_t i = base + 4 * lane;
        double p0 = 0.0, p1 = 0.0, p2 = 0.0, p3 = 0.0;
        if (i < body) {
            p0 = __dmul_rn(a[i], b[i]);
            p1 = __dmul_rn(a[i + 1], b[i + 1]);
            p2 = __dmul_rn(a[i + 2], b[i + 2]);
            p3 = __dmul_rn(a[i + 3], b[i + 3]);
        }
        const int64_t qn = (body - base) / 4 < 32 ? (body - base) / 4 : 32;
        for (int q = 0; q < (int)qn; ++q) {
            s0 = __dadd_rn(s0, __shfl_sync(0xffffffffu, p0, q));
            s1 = __dadd_rn(s1, __shfl_sync(0xffffffffu, p1, q));
            s2 = __dadd_rn(s2, __shfl_sync(0xffffffffu, p2, q));
            s3 = __dadd_rn(s3, __shfl_sync(0xffffffffu, p3, q));
        }
    }
    double s = (body > 0) ? __dadd_rn(__dadd_rn(s0, s1), __dadd_rn(s2, s3)) : 0.0;
    int64_t i = body, rem = len - body;
    if (rem >= 2) {
        s = __dadd_rn(s, __dmul_rn(a[i], b[i]));
        s = __dadd_rn(s, __dmul_rn(a[i + 1], b[i + 1]));
        i += 2;
        rem -= 2;
    }
    if (rem == 1) s = fma(a[i], b[i], s);
    return s;
}

// make_reflector on column j of b (ld), rows `rows`; beta -> betas[j]
__global__ void make_reflector_kernel(double *b, int64_t rows, int64_t ld, int64_t j, double *betas) {
    __shared__ double sh[2];
    double *colj = b + j * ld;
    if (threadIdx.x < 32) {
        const double x0 = colj[j];
        const double tail_sq = warp_dot(colj + j + 1, colj + j + 1, rows - j - 1);
        if (threadIdx.x == 0) {
            const double norm_x = sqrt(fma(x0, x0, tail_sq));
            if (norm_x == 0.0) {
                betas[j] = 0.0;
                sh[0] = 0.0;
            } else {
                const double sign = (x0 >= 0.0) ? 1.0 : -1.0;
                const double alpha = -sign * norm_x;
                sh[0] = __dsub_rn(x0, alpha);  // v0
                sh[1] = alpha;
                betas[j] = __ddiv_rn(__dadd_rn(norm_x, fabs(x0)), norm_x);
            }
        }
    }
    __syncthreads();
    const double v0 = sh[0];
    if (v0 == 0.0) return;
    for (int64_t i = j + 1 + threadIdx.x; i < rows; i += blockDim.x) colj[i] = __ddiv_rn(colj[i], v0);
    __syncthreads();
    if (threadIdx.x == 0) colj[j] = sh[1];
}

// apply_reflector(house col jv, beta = betas[jv]) to target columns [c0, c1),
// rows j..rows-1; one warp per target column
__global__ void apply_reflector_kernel(const double *house, int64_t ldh, int64_t jv, const double *betas, int64_t j,
                                       double *target, int64_t ldt, int64_t c0, int64_t c1, int64_t rows) {
    const double beta = betas[jv];
    if (beta == 0.0) return;
    const int64_t c = c0 + (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
    if (c >= c1) return;
    const int lane = threadIdx.x & 31;
    const double *w = house + jv * ldh;
    double *t = target + c * ldt;
    double tau = t[j];
    tau = __dadd_rn(tau, warp_dot(w + j + 1, t + j + 1, rows - j - 1));
    tau = __dmul_rn(tau, beta);
    __syncwarp();
    if (lane == 0) t[j] = __dsub_rn(t[j], tau);
    for (int64_t i = j + 1 + lane; i < rows; i += 32) t[i] = fma(-tau, w[i], t[i]);
}

// matmul (linalg.cc:52-66): c (m x n, ld m) = a (m x k, lda) b (k x n, ldb)
// Thread = one row i and 8 consecutive columns; t ascending per element.
constexpr int kMmCols = 8;
__global__ void matmul_kernel(int64_t m, int64_t k, int64_t n, const double *a, int64_t lda, const double *b,
                              int64_t ldb, double *c) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t j0 = (int64_t)blockIdx.y * kMmCols;
    double acc[kMmCols];
#pragma unroll
    for (int q = 0; q < kMmCols; ++q) acc[q] = 0.0;
    if (i < m) {
        for (int64_t t = 0; t < k; ++t) {
            const double ait = a[t * lda + i];
#pragma unroll
            for (int q = 0; q < kMmCols; ++q) {
                if (j0 + q < n) {
                    const double btj = b[(j0 + q) * ldb + t];
                    if (btj != 0.0) acc[q] = fma(btj, ait, acc[q]);
                }
            }
        }
#pragma unroll
        for (int q = 0; q < kMmCols; ++q)
            if (j0 + q < n) c[(j0 + q) * m + i] = acc[q];
    }
}

int ok(cudaError_t e) { return e == cudaSuccess ? 0 : (int)e; }

int apply_cols(const double *house, int64_t ldh, int64_t jv, const double *betas, int64_t j, double *target,
               int64_t ldt, int64_t c0, int64_t c1, int64_t rows, cudaStream_t st) {
    if (c1 <= c0) return 0;
    const unsigned grid = (unsigned)((c1 - c0 + kWarps - 1) / kWarps);
    apply_reflector_kernel<<<grid, 32 * kWarps, 0, st>>>(house, ldh, jv, betas, j, target, ldt, c0, c1, rows);
    return ok(cudaGetLastError());
}

}  // namespace

extern "C" {

// householder_qr's reduction (linalg.cc:139-149): b (m x n, ld m) in place,
// betas (device, n)
int gen_householder_reduce(double *b, int64_t m, int64_t n, double *betas, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    for (int64_t j = 0; j < n; ++j) {
        make_reflector_kernel<<<1, 256, 0, st>>>(b, m, m, j, betas);
        if (int e = ok(cudaGetLastError())) return e;
        if (int e = apply_cols(b, m, j, betas, j, b, m, j + 1, n, m, st)) return e;
    }
    return 0;
}

// accumulate_q (linalg.cc:186-197): q (m x k, ld m) = thin Q; q must hold I
int gen_accumulate_q(const double *b, int64_t m, const double *betas, int64_t k, double *q, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    for (int64_t j = k - 1; j >= 0; --j)
        if (int e = apply_cols(b, m, j, betas, j, q, m, j, k, m, st)) return e;
    return 0;
}

// apply_q_left (linalg.cc:151-161): target (m x nt, ld m) = Q target
int gen_apply_q_left(const double *b, int64_t m, int64_t nb, const double *betas, double *target, int64_t nt,
                     void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    for (int64_t j = nb - 1; j >= 0; --j)
        if (int e = apply_cols(b, m, j, betas, j, target, m, 0, nt, m, st)) return e;
    return 0;
}

int gen_matmul(int64_t m, int64_t k, int64_t n, const double *a, int64_t lda, const double *b, int64_t ldb,
               double *c, void *stream) {
    dim3 grid((unsigned)((m + 127) / 128), (unsigned)((n + kMmCols - 1) / kMmCols));
    matmul_kernel<<<grid, 128, 0, (cudaStream_t)stream>>>(m, k, n, a, lda, b, ldb, c);
    return ok(cudaGetLastError());
}

}  // extern "C"

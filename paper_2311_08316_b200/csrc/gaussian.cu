// Gaussian sketch family on device (sketch.cc:62-72 sample, apply = matmul).
//
// S (d x m) has S(i, c) = normal(c*d + i) / sqrt(d) from the stream
// CounterRng(mix_seed(seed, 0x6761757373)), c the GLOBAL row of A, so ranks
// need no communication. S is generated chunk by chunk of A's rows into a
// bounded workspace and multiplied on the FP64 tensor cores by a split-K DMMA
// GEMM whose slices are summed in a fixed order (deterministic). Device
// log/cos are within 1 ulp of the host libm's, so S and the sketch agree with
// the reference's to rounding (J then matches except at near-ties).
#include "common.cuh"
#include "internal.hh"

namespace cqg {

constexpr uint64_t kGaussianSalt = 0x6761757373ULL;  // sketch.cc:18

// S chunk: rows c0 + [0, count) of A -> s (d x count, ld d)
__global__ void gaussian_fill_kernel(int64_t d, int64_t c0, int64_t count, uint64_t stream, double scale,
                                     double *__restrict__ s) {
    const int64_t total = d * count;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = e / d, i = e - c * d;
        s[e] = normal_dev(stream, (uint64_t)((c0 + c) * d + i)) * scale;  // sketch.cc:67-69
    }
}

int gaussian_sketch(int64_t m, int64_t n, const double *a, int64_t lda, int64_t d, uint64_t seed, int64_t c0,
                    double *msk, int64_t ldm, Workspace &ws, cudaStream_t st) {
    if (m <= 0 || n <= 0) {
        for (int64_t j = 0; j < n; ++j)
            CQ_CUDA(cudaMemsetAsync(msk + j * ldm, 0, sizeof(double) * d, st), "gaussian sketch zero");
        return 0;
    }
    const uint64_t stream = mix_seed(seed, kGaussianSalt);
    const double scale = 1.0 / sqrt((double)d);  // sketch.cc:66
    // chunk of A's rows whose S block fits 1 GiB of workspace
    const int64_t mc = std::max<int64_t>(256, std::min<int64_t>(m, ((int64_t)1 << 27) / d));
    double *s = ws.get<double>("gauss.s", (size_t)(d * mc));
    if (!s) return fail_nomem("gaussian sketch operator");
    const int sms = num_sms();
    const int64_t tiles = ((d + 63) / 64) * ((n + 127) / 128);
    const int64_t splits = std::max<int64_t>(1, (3 * (int64_t)sms + tiles - 1) / tiles);
    for (int64_t r0 = 0; r0 < m; r0 += mc) {
        const int64_t cnt = std::min<int64_t>(mc, m - r0);
        const int64_t total = d * cnt;
        const unsigned grid = (unsigned)std::min<int64_t>((total + 255) / 256, (int64_t)sms * 16);
        gaussian_fill_kernel<<<grid, 256, 0, st>>>(d, c0 + r0, cnt, stream, scale, s);
        note_launch();
        CQ_TRY(check_launch("gaussian_fill_kernel"));
        // msk (+)= S_chunk A[r0:r0+cnt, :]
        CQ_TRY(gemm_splitk(false, d, n, cnt, 1.0, s, d, a + r0, lda, r0 == 0 ? 0.0 : 1.0, msk, ldm, splits, ws, st));
    }
    return 0;
}

}  // namespace cqg

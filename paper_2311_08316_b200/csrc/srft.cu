// SRFT sketch family on device (sketch.cc:100-119 sample, 147-166 apply).
//
// out(r, j) = factor * FWHT(signs .* A[:, j] zero-padded to P)[rows[r]],
// P = next_pow2(m), factor = sqrt(P/d) / sqrt(P). The Walsh-Hadamard
// butterflies of one stage are independent, so any schedule that runs the
// stages in the reference's order (half = 1, 2, 4, ...) reproduces its bits:
//   pass 1: stages half < 4096 inside 4096-element blocks in shared memory
//           (the +-1 sign multiply, exact, fused into the load);
//   pass 2: stages half >= 4096 act on the P/4096 elements t, t+4096, ...
//           of each residue t: 8 residues per CTA in shared memory;
//   gather: the d selected coordinates, scaled.
// Sampling: signs in parallel; the selection (a seeded partial Fisher-Yates
// over [0, P)) is sequential by construction -- one thread keeps the first d
// positions in an array and the displaced higher positions in a hash table in
// shared memory. Single rank only (the transform mixes every row).
#include "common.cuh"
#include "internal.hh"

namespace cqg {

constexpr uint64_t kSrftSignSalt = 0x7369676eULL;    // sketch.cc:20
constexpr uint64_t kSrftSelectSalt = 0x73656c65ULL;  // sketch.cc:21
constexpr int kFwBlock = 4096;                       // pass-1 block (32 KB of doubles)
constexpr int kFwThreads = 256;
constexpr int kFwRes = 8;                            // pass-2 residues per CTA

__global__ void srft_signs_kernel(int64_t m, uint64_t stream, double *__restrict__ signs) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        signs[i] = (rng_bits(stream, (uint64_t)i) & 1ULL) ? 1.0 : -1.0;  // sketch.cc:107-108
}

// sketch.cc:110-117: swap(perm[i], perm[i + below(i, P - i)]) for i < d
__global__ void srft_select_kernel(int64_t d, int64_t P, uint64_t stream, int hbits, int64_t *__restrict__ rows) {
    extern __shared__ int32_t ssel[];
    int32_t *low = ssel;               // perm[0 .. d)
    int32_t *hkey = ssel + d;          // hash table for positions >= d: key, value
    int32_t *hval = hkey + (1 << hbits);
    const int hmask = (1 << hbits) - 1;
    for (int64_t i = threadIdx.x; i < d; i += blockDim.x) low[i] = (int32_t)i;
    for (int i = threadIdx.x; i <= hmask; i += blockDim.x) hkey[i] = -1;
    __syncthreads();
    if (threadIdx.x != 0) return;
    auto slot = [&](int32_t key) {
        int h = (int)(((uint32_t)key * 2654435761u) >> (32 - hbits));
        while (hkey[h] != -1 && hkey[h] != key) h = (h + 1) & hmask;
        return h;
    };
    auto get = [&](int64_t pos) -> int32_t {
        if (pos < d) return low[pos];
        const int h = slot((int32_t)pos);
        return hkey[h] == -1 ? (int32_t)pos : hval[h];
    };
    auto set = [&](int64_t pos, int32_t v) {
        if (pos < d) {
            low[pos] = v;
            return;
        }
        const int h = slot((int32_t)pos);
        hkey[h] = (int32_t)pos;
        hval[h] = v;
    };
    for (int64_t i = 0; i < d; ++i) {
        const int64_t j = i + (int64_t)rng_below(stream, (uint64_t)i, (uint64_t)(P - i));
        const int32_t vi = get(i), vj = get(j);
        set(i, vj);
        set(j, vi);
    }
    for (int64_t i = 0; i < d; ++i) rows[i] = low[i];
}

// pass 1: t (P x n, ld P) block b of column j = stages half = 1 .. min(P, 4096)/2
__global__ void __launch_bounds__(kFwThreads) srft_pass1_kernel(int64_t m, int64_t P, const double *__restrict__ a,
                                                                int64_t lda, const double *__restrict__ signs,
                                                                double *__restrict__ t) {
    __shared__ double x[kFwBlock];
    const int64_t j = blockIdx.y;
    const int B = (int)cmin<int64_t>(kFwBlock, P);
    const int64_t base = (int64_t)blockIdx.x * B;
    const double *col = a + j * lda;
    for (int q = threadIdx.x; q < B; q += kFwThreads) {
        const int64_t i = base + q;
        x[q] = (i < m) ? signs[i] * col[i] : 0.0;  // sketch.cc:156-158 (zero padding)
    }
    __syncthreads();
    for (int half = 1; half < B; half <<= 1) {  // fwht, sketch.cc:31-39
        for (int q = threadIdx.x; q < B / 2; q += kFwThreads) {
            const int lo = (q / half) * (2 * half) + (q % half);
            const double u = x[lo], v = x[lo + half];
            x[lo] = u + v;
            x[lo + half] = u - v;
        }
        __syncthreads();
    }
    double *tc = t + j * P + base;
    for (int q = threadIdx.x; q < B; q += kFwThreads) tc[q] = x[q];
}

// pass 2: for residues t0 .. t0+7 of column j, stages half = 4096 .. P/2
__global__ void __launch_bounds__(kFwThreads) srft_pass2_kernel(int64_t P, double *__restrict__ t) {
    extern __shared__ double y[];  // [Ph][kFwRes]
    const int64_t j = blockIdx.y;
    const int64_t t0 = (int64_t)blockIdx.x * kFwRes;
    const int Ph = (int)(P / kFwBlock);
    double *tc = t + j * P;
    for (int q = threadIdx.x; q < Ph * kFwRes; q += kFwThreads) {
        const int k = q / kFwRes, r = q % kFwRes;
        y[q] = tc[(int64_t)k * kFwBlock + t0 + r];
    }
    __syncthreads();
    for (int half = 1; half < Ph; half <<= 1) {  // = global half * 4096, same stage order
        for (int q = threadIdx.x; q < (Ph / 2) * kFwRes; q += kFwThreads) {
            const int p = q / kFwRes, r = q % kFwRes;
            const int lo = (p / half) * (2 * half) + (p % half);
            const double u = y[lo * kFwRes + r], v = y[(lo + half) * kFwRes + r];
            y[lo * kFwRes + r] = u + v;
            y[(lo + half) * kFwRes + r] = u - v;
        }
        __syncthreads();
    }
    for (int q = threadIdx.x; q < Ph * kFwRes; q += kFwThreads) {
        const int k = q / kFwRes, r = q % kFwRes;
        tc[(int64_t)k * kFwBlock + t0 + r] = y[q];
    }
}

__global__ void srft_gather_kernel(int64_t d, int64_t n, int64_t P, const double *__restrict__ t,
                                   const int64_t *__restrict__ rows, double factor, double *__restrict__ out,
                                   int64_t ldo) {
    const int64_t total = d * n;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = e / d, r = e - j * d;
        out[j * ldo + r] = factor * t[j * P + rows[r]];  // sketch.cc:161-162
    }
}

int srft_sketch(int64_t m, int64_t n, const double *a, int64_t lda, int64_t d, uint64_t seed, double *msk,
                int64_t ldm, Workspace &ws, cudaStream_t st) {
    if (d < 1 || m < 1 || d > m) return fail_internal("srft: needs 1 <= d <= m (sketch.cc:101)");
    int64_t P = 1;
    while (P < m) P <<= 1;  // next_pow2 (sketch.cc:23-27)
    if (P > ((int64_t)1 << 30)) return fail_internal("srft: padded length too large");
    if (n == 0) return 0;
    const int64_t Ph = P / kFwBlock;
    if (Ph * kFwRes * (int64_t)sizeof(double) > 200 * 1024) return fail_internal("srft: m too large for pass 2");
    double *signs = ws.get<double>("srft.signs", (size_t)m);
    int64_t *rows = ws.get<int64_t>("srft.rows", (size_t)d);
    double *t = ws.get<double>("srft.t", (size_t)(P * n));
    if (!signs || !rows || !t) return fail_nomem("srft workspace");
    const int sms = num_sms();
    srft_signs_kernel<<<(unsigned)std::min<int64_t>((m + 255) / 256, (int64_t)sms * 8), 256, 0, st>>>(
        m, mix_seed(seed, kSrftSignSalt), signs);
    note_launch();
    int hbits = 4;
    while ((1 << hbits) < 2 * d) ++hbits;
    const size_t sel_smem = sizeof(int32_t) * ((size_t)d + 2 * ((size_t)1 << hbits));
    if (sel_smem > 220 * 1024) return fail_internal("srft: d too large for the selection table");
    CQ_CUDA(cudaFuncSetAttribute(srft_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sel_smem),
            "srft select smem");
    srft_select_kernel<<<1, 256, sel_smem, st>>>(d, P, mix_seed(seed, kSrftSelectSalt), hbits, rows);
    note_launch();
    const int64_t B = std::min<int64_t>(kFwBlock, P);
    srft_pass1_kernel<<<dim3((unsigned)(P / B), (unsigned)n), kFwThreads, 0, st>>>(m, P, a, lda, signs, t);
    note_launch();
    if (P > kFwBlock) {
        const size_t smem2 = sizeof(double) * (size_t)(Ph * kFwRes);
        CQ_CUDA(cudaFuncSetAttribute(srft_pass2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2),
                "srft pass2 smem");
        srft_pass2_kernel<<<dim3((unsigned)(kFwBlock / kFwRes), (unsigned)n), kFwThreads, smem2, st>>>(P, t);
        note_launch();
    }
    const double factor = sqrt((double)P / (double)d) / sqrt((double)P);  // sketch.cc:104,151
    srft_gather_kernel<<<(unsigned)std::min<int64_t>((d * n + 255) / 256, (int64_t)sms * 8), 256, 0, st>>>(
        d, n, P, t, rows, factor, msk, ldm);
    note_launch();
    return check_launch("srft kernels");
}

}  // namespace cqg

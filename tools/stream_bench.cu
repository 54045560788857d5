// Load-side microbenchmark for the sketch's access pattern (no arithmetic):
// a CTA streams a 32-column group of a column-major m x n matrix in 128-row
// tiles through a STAGES-deep cp.async pipeline, as saso_apply_kernel does.
//   mode 0: 8-byte cp.async into [c][33] (the sketch layout)
//   mode 1: 16-byte cp.async (two rows of one column per copy)
//   mode 2: plain streaming LDG.128 of the whole matrix (reference)
// usage: stream_bench m n [splits]
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <stdint.h>

constexpr int TR = 128, LD = 33, THREADS = 512, STAGES = 3;

__device__ __forceinline__ void cpa8(void *s, const void *g, int sz) {
    unsigned sa = (unsigned)__cvta_generic_to_shared(s);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(g), "r"(sz));
}
__device__ __forceinline__ void cpa16(void *s, const void *g, int sz) {
    unsigned sa = (unsigned)__cvta_generic_to_shared(s);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(g), "r"(sz));
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N> __device__ __forceinline__ void waitg() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

template <int MODE>
__global__ void __launch_bounds__(THREADS, 1) tiles(const double *a, int64_t m, int64_t n, int64_t lda,
                                                     int64_t tps, double *sink) {
    extern __shared__ double sm[];
    const int tid = threadIdx.x;
    const int64_t j0 = blockIdx.x * 32;
    const int64_t ntiles = (m + TR - 1) / TR;
    const int64_t t0 = blockIdx.y * tps, t1 = t0 + tps < ntiles ? t0 + tps : ntiles;
    auto issue = [&](int64_t tile, int s) {
        double *dt = sm + s * TR * LD;
        if (MODE == 0) {
            const int cc = tid % TR, jj0 = tid / TR;
            const int64_t row = tile * TR + cc;
            for (int it = 0; it < 8; ++it) {
                const int jj = jj0 + 4 * it;
                const bool ok = row < m && j0 + jj < n;
                cpa8(dt + cc * LD + jj, ok ? a + (j0 + jj) * lda + row : a, ok ? 8 : 0);
            }
        } else {
            const int pr = tid % (TR / 2), jj0 = tid / (TR / 2);  // 64 row pairs x 8 columns per pass
            const int64_t row = tile * TR + 2 * pr;
            for (int it = 0; it < 4; ++it) {
                const int jj = jj0 + 8 * it;
                const bool ok = row + 1 < m && j0 + jj < n;
                cpa16(dt + jj * (TR + 2) + 2 * pr, ok ? a + (j0 + jj) * lda + row : a, ok ? 16 : 0);
            }
        }
    };
    for (int s = 0; s < STAGES - 1; ++s) {
        if (t0 + s < t1) issue(t0 + s, s);
        commit();
    }
    double acc = 0.0;
    for (int64_t t = t0; t < t1; ++t) {
        waitg<STAGES - 2>();
        __syncthreads();
        if (t + STAGES - 1 < t1) issue(t + STAGES - 1, (int)((t + STAGES - 1 - t0) % STAGES));
        commit();
        acc += sm[((t - t0) % STAGES) * TR * LD + tid];
    }
    if (acc == 12345.678) sink[0] = acc;
}

__global__ void stream_ldg(const double2 *a, int64_t n2, double *sink) {
    double s = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2; i += (int64_t)gridDim.x * blockDim.x) {
        double2 v = __ldcs(a + i);
        s += v.x + v.y;
    }
    if (s == 12345.678) sink[0] = s;
}

int main(int argc, char **argv) {
    int64_t m = argc > 1 ? atoll(argv[1]) : 131072, n = argc > 2 ? atoll(argv[2]) : 1024;
    int64_t splits = argc > 3 ? atoll(argv[3]) : 4;
    double *a, *sink;
    cudaMalloc(&a, sizeof(double) * m * n);
    cudaMalloc(&sink, 8);
    cudaMemset(a, 0, sizeof(double) * m * n);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int64_t ntiles = (m + TR - 1) / TR, tps = (ntiles + splits - 1) / splits;
    dim3 grid((unsigned)((n + 31) / 32), (unsigned)splits);
    size_t smem = sizeof(double) * STAGES * TR * LD + 1024;
    cudaFuncSetAttribute(tiles<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(tiles<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const double gb = sizeof(double) * (double)m * n / 1e9;
    for (int mode = 0; mode < 3; ++mode) {
        float best = 1e30f;
        for (int r = 0; r < 4; ++r) {
            cudaEventRecord(e0);
            if (mode == 0) tiles<0><<<grid, THREADS, smem>>>(a, m, n, m, tps, sink);
            else if (mode == 1) tiles<1><<<grid, THREADS, smem>>>(a, m, n, m, tps, sink);
            else stream_ldg<<<sms * 4, 512>>>(reinterpret_cast<const double2 *>(a), m * n / 2, sink);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (r && ms < best) best = ms;
        }
        printf("m=%lld n=%lld splits=%lld ctas=%u mode=%d: %.3f ms  %.0f GB/s  (%s)\n", (long long)m, (long long)n,
               (long long)splits, grid.x * grid.y, mode, best, gb / (best * 1e-3),
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}

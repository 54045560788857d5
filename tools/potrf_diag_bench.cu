// Warm per-launch time of potrf_diag_kernel on one SPD 64 x 64 block, and a
// clock64 breakdown of the warp factorization phases (R11, R12, A22 update, R22).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2311_08316_b200/csrc \
//        tools/potrf_diag_bench.cu -o tools/potrf_diag_bench -Lpaper_2311_08316_b200/_lib -lcqrrpt_gpu
#include "../paper_2311_08316_b200/csrc/potrf.cu"
#include <cstdio>
#include <vector>

using namespace cqg;

__global__ void phases_kernel(const double *g, int64_t ldg, long long *cyc, double *out) {
    __shared__ double blk[kPB][kPB + 1];
    const int c = threadIdx.x;
    for (int q = c; q < kPB * kPB; q += 32) blk[q / kPB][q % kPB] = g[(q / kPB) * ldg + q % kPB];
    __syncwarp();
    double a[kWB];
    long long t0 = clock64();
#pragma unroll
    for (int i = 0; i < kWB; ++i) a[i] = blk[c][i];
    int f = warp_potrf32(a);
    long long t1 = clock64();
#pragma unroll
    for (int i = 0; i < kWB; ++i) blk[c][i] = a[i];
    __syncwarp();
#pragma unroll
    for (int i = 0; i < kWB; ++i) a[i] = blk[kWB + c][i];
#pragma unroll
    for (int t = 0; t < kWB; ++t) {
        a[t] = a[t] / blk[t][t];
#pragma unroll
        for (int i = t + 1; i < kWB; ++i) a[i] = fma(-blk[i][t], a[t], a[i]);
    }
#pragma unroll
    for (int i = 0; i < kWB; ++i) blk[kWB + c][i] = a[i];
    __syncwarp();
    long long t2 = clock64();
#pragma unroll
    for (int i = 0; i < kWB; ++i) a[i] = blk[kWB + c][kWB + i];
#pragma unroll
    for (int k = 0; k < kWB; ++k) {
        const double rkc = blk[kWB + c][k];
#pragma unroll
        for (int i = 0; i < kWB; ++i) a[i] = fma(-blk[kWB + i][k], rkc, a[i]);
    }
    long long t3 = clock64();
    f += warp_potrf32(a);
    long long t4 = clock64();
    double s = f;
#pragma unroll
    for (int i = 0; i < kWB; ++i) s += a[i];
    out[c] = s;
    if (c == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; }
}

int main() {
    const int n = 64;
    std::vector<double> h(n * n);
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) h[j * n + i] = (i == j ? n + 1.0 : 1.0 / (1 + i + j));
    double *g, *g0, *o;
    int64_t *fail;
    long long *cyc, hc[4];
    cudaMalloc(&g, n * n * 8); cudaMalloc(&g0, n * n * 8); cudaMalloc(&o, 256); cudaMalloc(&fail, 8); cudaMalloc(&cyc, 32);
    cudaMemcpy(g0, h.data(), n * n * 8, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
        cudaMemset(fail, 0, 8);
        cudaEventRecord(e0);
        for (int it = 0; it < 100; ++it) {
            cudaMemcpyAsync(g, g0, n * n * 8, cudaMemcpyDeviceToDevice);
            potrf_diag_kernel<<<1, 32>>>(n, g, n, 0, fail);
        }
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        cudaEventRecord(e0);
        for (int it = 0; it < 100; ++it) cudaMemcpyAsync(g, g0, n * n * 8, cudaMemcpyDeviceToDevice);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms0; cudaEventElapsedTime(&ms0, e0, e1);
        phases_kernel<<<1, 32>>>(g0, n, cyc, o);
        cudaMemcpy(hc, cyc, 32, cudaMemcpyDeviceToHost);
        int64_t hf; cudaMemcpy(&hf, fail, 8, cudaMemcpyDeviceToHost);
        if (rep) printf("diag launch %.2f us (copy-only loop %.2f us/iter), fail=%lld; cycles R11 %lld R12 %lld upd %lld R22 %lld\n",
                        ms * 10.0, ms0 * 10.0, (long long)hf, hc[0], hc[1], hc[2], hc[3]);
    }
    return 0;
}

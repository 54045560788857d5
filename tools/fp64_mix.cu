#include <cstdio>
#include <cuda_runtime.h>
// throughput of DADD, DMUL, I2F.F64.S64, and the magic conversion, 8 independent chains per thread
__global__ void kadd(double *out, int iters, double a) {
    double x[8]; for (int j = 0; j < 8; ++j) x[j] = threadIdx.x + j;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = x[j] + a;
    double s = 0; for (int j = 0; j < 8; ++j) s += x[j]; out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void ki2f(double *out, int iters, long long a) {
    long long x[8]; double y[8];
    for (int j = 0; j < 8; ++j) { x[j] = threadIdx.x + j; y[j] = 0; }
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) { y[j] += 0.0 * (double)x[j]; x[j] += a; }
    double s = 0; for (int j = 0; j < 8; ++j) s += y[j]; out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void ki2f_only(double *out, int iters, long long a) {
    long long x[8]; double y[8];
    for (int j = 0; j < 8; ++j) { x[j] = threadIdx.x + j; y[j] = 0; }
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) { y[j] = (double)(x[j] ^ (long long)__double_as_longlong(y[j])); }
    double s = 0; for (int j = 0; j < 8; ++j) s += y[j]; out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <typename K, typename A>
void run(const char *name, K k, A a, int warps_per_sm) {
    double *o; cudaMalloc(&o, 148 * 64 * 1024 * 8);
    int iters = 2048;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int threads = 32 * warps_per_sm;
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        k<<<148, threads>>>(o, iters, a);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double ops = 8.0 * iters * 148.0 * threads;
        if (rep) printf("%s warps/SM=%d: %.1f ops/clk/SM (1.9 GHz)\n", name, warps_per_sm, ops / (ms * 1e-3) / 148 / 1.9e9);
    }
    cudaFree(o);
}
int main() {
    for (int w : {4, 8, 16, 32}) {
        run("DADD", kadd, 0.5, w);
        run("I2F.F64.S64+DFMA", ki2f, 3ll, w);
        run("I2F.F64.S64 chain", ki2f_only, 3ll, w);
    }
}

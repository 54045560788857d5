#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double *out, int iters, double a) {
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
        x0 = fma(x0, a, 1.0); x1 = fma(x1, a, 1.0); x2 = fma(x2, a, 1.0); x3 = fma(x3, a, 1.0);
        x4 = fma(x4, a, 1.0); x5 = fma(x5, a, 1.0); x6 = fma(x6, a, 1.0); x7 = fma(x7, a, 1.0);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void kf(float *out, int iters, float a) {
    float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
        x0 = fmaf(x0, a, 1.f); x1 = fmaf(x1, a, 1.f); x2 = fmaf(x2, a, 1.f); x3 = fmaf(x3, a, 1.f);
        x4 = fmaf(x4, a, 1.f); x5 = fmaf(x5, a, 1.f); x6 = fmaf(x6, a, 1.f); x7 = fmaf(x7, a, 1.f);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
int main() {
    double *o; cudaMalloc(&o, 148 * 8 * 256 * 8);
    int iters = 4096;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        k<<<148 * 8, 256>>>(o, iters, 0.999);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        double fl = 2.0 * 8 * iters * 148.0 * 8 * 256;
        printf("DFMA: %.2f TFLOP/s (%.1f DFMA/clk/SM at 1.9 GHz)\n", fl / ms / 1e9, fl / 2 / (ms * 1e-3) / 148 / 1.9e9);
        cudaEventRecord(a);
        kf<<<148 * 8, 256>>>((float *)o, iters, 0.999f);
        cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("FFMA: %.2f TFLOP/s\n", fl / ms / 1e9);
    }
}

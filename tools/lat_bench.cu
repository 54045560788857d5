// Microbenchmark: dependent-chain latencies of FP64 ops on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double *out, long long *cyc, double a, double b, int n) {
    double s = a, t = b;
    long long c0 = clock64();
    for (int i = 0; i < n; ++i) { s = __dadd_rn(s, t); }
    long long c1 = clock64();
    double f = a;
    for (int i = 0; i < n; ++i) { f = fma(f, b, a); }
    long long c2 = clock64();
    double m = a;
    for (int i = 0; i < n; ++i) { m = __dmul_rn(m, b); }
    long long c3 = clock64();
    __shared__ double sm[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = i * 1e-9;
    __syncthreads();
    double q = 0; int idx = 0;
    long long c4 = clock64();
    for (int i = 0; i < n; ++i) { q = __dadd_rn(q, sm[idx]); idx = (idx + 1) & 1023; }
    long long c5 = clock64();
    out[threadIdx.x] = s + f + m + q;
    if (threadIdx.x == 0) { cyc[0] = c1 - c0; cyc[1] = c2 - c1; cyc[2] = c3 - c2; cyc[3] = c5 - c4; }
}
int main() {
    double *o; long long *c, h[4];
    cudaMalloc(&o, 1024 * 8); cudaMalloc(&c, 32);
    int n = 100000;
    k<<<1, 32>>>(o, c, 1.0, 1.0000001, n);
    cudaDeviceSynchronize();
    k<<<1, 32>>>(o, c, 1.0, 1.0000001, n);
    cudaMemcpy(h, c, 32, cudaMemcpyDeviceToHost);
    printf("DADD chain %.2f cyc, DFMA chain %.2f cyc, DMUL chain %.2f cyc, LDS+DADD chain %.2f cyc per op\n",
           (double)h[0] / n, (double)h[1] / n, (double)h[2] / n, (double)h[3] / n);
    return 0;
}

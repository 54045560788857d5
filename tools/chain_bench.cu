// Ordered FP64 dot-product chains as in the QRCP (lanes 4g+q accumulate
// s_q += a[q+4k]*b[q+4k] for column g): cycles per k-step, by active groups.
#include <cstdio>
#include <cuda_runtime.h>

template <int GROUPS>
__global__ void chain(const double *ga, long long *cyc, double *out, int body) {
    extern __shared__ double sm[];
    double *a = sm;                              // 1312
    auto bcol = [&](int g) { return sm + 1312 + g * 1316; };  // 4 doubles apart mod 16
    for (int i = threadIdx.x; i < 1312; i += blockDim.x) {
        a[i] = ga[i];
        for (int g = 0; g < 8; ++g) bcol(g)[i] = ga[i] * (g + 1);
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, gq = lane >> 2, q = lane & 3;
    double s = 0.0;
    long long c0 = clock64();
    if (threadIdx.x < 32 && gq < GROUPS) {
        const double *cg = bcol(gq);
        int e = q;
        double xa[8], xb[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) { xa[u] = a[e + 4 * u]; xb[u] = cg[e + 4 * u]; }
        for (e += 32; e + 28 < body; e += 32) {
            double na[8], nb[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) { na[u] = a[e + 4 * u]; nb[u] = cg[e + 4 * u]; }
#pragma unroll
            for (int u = 0; u < 8; ++u) s = s + xa[u] * xb[u];
#pragma unroll
            for (int u = 0; u < 8; ++u) { xa[u] = na[u]; xb[u] = nb[u]; }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) s = s + xa[u] * xb[u];
    }
    long long c1 = clock64();
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[0] = c1 - c0;
}

// products pipelined one group ahead of the adds (the DMULs of group k+1 run
// under the DADDs of group k)
template <int GROUPS>
__global__ void chain2(const double *ga, long long *cyc, double *out, int body) {
    extern __shared__ double sm[];
    double *a = sm;
    auto bcol = [&](int g) { return sm + 1312 + g * 1316; };
    for (int i = threadIdx.x; i < 1312; i += blockDim.x) {
        a[i] = ga[i];
        for (int g = 0; g < 8; ++g) bcol(g)[i] = ga[i] * (g + 1);
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, gq = lane >> 2, q = lane & 3;
    double s = 0.0;
    long long c0 = clock64();
    if (threadIdx.x < 32 && gq < GROUPS) {
        const double *cg = bcol(gq);
        const int ng = body - 29 - q >= 0 ? (body - 29 - q) / 32 + 1 : 0;
        double p[8], xa[8], xb[8];
        if (ng > 0) {
#pragma unroll
            for (int u = 0; u < 8; ++u) p[u] = a[q + 4 * u] * cg[q + 4 * u];
            if (ng > 1) {
#pragma unroll
                for (int u = 0; u < 8; ++u) { xa[u] = a[q + 32 + 4 * u]; xb[u] = cg[q + 32 + 4 * u]; }
            }
            for (int k = 0; k < ng; ++k) {
                double na[8], nb[8];
                const int en = q + 32 * (k + 2);
                if (k + 2 < ng) {
#pragma unroll
                    for (int u = 0; u < 8; ++u) { na[u] = a[en + 4 * u]; nb[u] = cg[en + 4 * u]; }
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) s = s + p[u];
#pragma unroll
                for (int u = 0; u < 8; ++u) { p[u] = xa[u] * xb[u]; xa[u] = na[u]; xb[u] = nb[u]; }
            }
        }
        for (int e = q + 32 * ng; e < body; e += 4) s = s + a[e] * cg[e];
    }
    long long c1 = clock64();
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[0] = c1 - c0;
}

// as chain2 but with clamped, unconditional loads (no predication)
template <int GROUPS>
__global__ void chain3(const double *ga, long long *cyc, double *out, int body) {
    extern __shared__ double sm[];
    double *a = sm;
    auto bcol = [&](int g) { return sm + 1312 + g * 1316; };
    for (int i = threadIdx.x; i < 1312; i += blockDim.x) {
        a[i] = ga[i];
        for (int g = 0; g < 8; ++g) bcol(g)[i] = ga[i] * (g + 1);
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, gq = lane >> 2, q = lane & 3;
    double s = 0.0;
    long long c0 = clock64();
    if (threadIdx.x < 32 && gq < GROUPS) {
        const double *cg = bcol(gq);
        const int ng = body - 29 - q >= 0 ? (body - 29 - q) / 32 + 1 : 0;
        if (ng > 0) {
            double p[8], xa[8], xb[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) p[u] = a[q + 4 * u] * cg[q + 4 * u];
            const int e1 = q + 32 * min(1, ng - 1);
#pragma unroll
            for (int u = 0; u < 8; ++u) { xa[u] = a[e1 + 4 * u]; xb[u] = cg[e1 + 4 * u]; }
            for (int k = 0; k < ng; ++k) {
                const int en = q + 32 * min(k + 2, ng - 1);
                double na[8], nb[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) { na[u] = a[en + 4 * u]; nb[u] = cg[en + 4 * u]; }
#pragma unroll
                for (int u = 0; u < 8; ++u) s = s + p[u];
#pragma unroll
                for (int u = 0; u < 8; ++u) { p[u] = xa[u] * xb[u]; xa[u] = na[u]; xb[u] = nb[u]; }
            }
        }
        for (int e = q + 32 * ng; e < body; e += 4) s = s + a[e] * cg[e];
    }
    long long c1 = clock64();
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[0] = c1 - c0;
}

// precomputed products in smem: loads one group ahead, adds only (chain_sum)
__global__ void chain_pre(const double *ga, long long *cyc, double *out, int body) {
    extern __shared__ double sm[];
    for (int i = threadIdx.x; i < 1312; i += blockDim.x) sm[i] = ga[i];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    double s = 0.0;
    long long c0 = clock64();
    if (lane < 4) {
        int e = lane;
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = sm[e + 4 * u];
        for (e += 32; e + 28 < body; e += 32) {
            double nx[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) nx[u] = sm[e + 4 * u];
#pragma unroll
            for (int u = 0; u < 8; ++u) s = s + v[u];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = nx[u];
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) s = s + v[u];
        for (; e < body; e += 4) s = s + sm[e];
    }
    long long c1 = clock64();
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[0] = c1 - c0;
}

// pure dependent DADD chain over values in registers (control)
__global__ void dadd_chain(long long *cyc, double *out, int n) {
    double s = threadIdx.x, t = 1e-9;
    long long c0 = clock64();
#pragma unroll 16
    for (int i = 0; i < n; ++i) s = s + t;
    long long c1 = clock64();
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[0] = c1 - c0;
}

int main() {
    double *a, *o;
    long long *c, h;
    cudaMalloc(&a, 2048 * 8);
    cudaMalloc(&o, 1024 * 8);
    cudaMalloc(&c, 8);
    cudaMemset(a, 0, 2048 * 8);
    const int body = 1280, steps = body / 4;
    const int smem = (1312 + 8 * 1316) * 8;
    cudaFuncSetAttribute(chain<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(chain<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(chain2<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(chain3<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(chain_pre, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int rep = 0; rep < 2; ++rep) {
        chain<1><<<1, 32, smem>>>(a, c, o, body);
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        if (rep) printf("1 group : %.2f cyc/step\n", (double)h / steps);
        chain<8><<<1, 32, smem>>>(a, c, o, body);
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        if (rep) printf("8 groups: %.2f cyc/step\n", (double)h / steps);
        chain<8><<<1, 256, smem>>>(a, c, o, body);
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        if (rep) printf("8 groups, 256-thread CTA: %.2f cyc/step\n", (double)h / steps);
        chain2<8><<<1, 32, smem>>>(a, c, o, body);
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        if (rep) printf("8 groups, products one group ahead: %.2f cyc/step\n", (double)h / steps);
        chain3<8><<<1, 32, smem>>>(a, c, o, body);
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        if (rep) printf("8 groups, products ahead (clamped loads): %.2f cyc/step\n", (double)h / steps);
        chain_pre<<<1, 32, smem>>>(a, c, o, body);
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        if (rep) printf("precomputed products (chain_sum): %.2f cyc/step\n", (double)h / steps);
        dadd_chain<<<1, 32>>>(c, o, 100000);
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        if (rep) printf("register DADD chain: %.2f cyc/add\n", (double)h / 100000);
    }
    return 0;
}

// Microbenchmark: grid-barrier latency of common.cuh's grid_barrier on B200.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2311_08316_b200/csrc/common.cuh"
using namespace cqg;
__device__ __forceinline__ void grid_barrier_spin(unsigned int *bar, unsigned int nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned int *gen = bar + 1;
        unsigned int g = *gen;
        __threadfence();
        unsigned int arrived = atomicAdd(bar, 1u);
        if (arrived == nblocks - 1) { atomicExch(bar, 0u); __threadfence(); atomicAdd(bar + 1, 1u); }
        else { while (*gen == g) {} }
        __threadfence();
    }
    __syncthreads();
}
__global__ void k_sleep(unsigned int *bar, int iters, unsigned long long *t) {
    unsigned long long t0; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int i = 0; i < iters; ++i) grid_barrier(bar, gridDim.x);
    unsigned long long t1; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (blockIdx.x == 0 && threadIdx.x == 0) *t = t1 - t0;
}
__global__ void k_spin(unsigned int *bar, int iters, unsigned long long *t) {
    unsigned long long t0; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int i = 0; i < iters; ++i) grid_barrier_spin(bar, gridDim.x);
    unsigned long long t1; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (blockIdx.x == 0 && threadIdx.x == 0) *t = t1 - t0;
}
int main() {
    unsigned int *bar; unsigned long long *t, ht;
    cudaMalloc(&bar, 16); cudaMalloc(&t, 8);
    int iters = 2000;
    for (int G : {8, 32, 64, 128, 148}) {
        for (int which = 0; which < 2; ++which) {
            cudaMemset(bar, 0, 16);
            void *args[] = {&bar, &iters, &t};
            cudaLaunchCooperativeKernel(which ? (void*)k_spin : (void*)k_sleep, dim3(G), dim3(256), args, 0, 0);
            cudaDeviceSynchronize();
            cudaMemcpy(&ht, t, 8, cudaMemcpyDeviceToHost);
            printf("G=%d %s: %.3f us/barrier\n", G, which ? "spin" : "nanosleep", ht / 1e3 / iters);
        }
    }
    return 0;
}

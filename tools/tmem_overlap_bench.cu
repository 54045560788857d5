// Do tcgen05.ld (TMEM -> registers) and tcgen05.mma.kind::i8 overlap on one SM?
//
// One CTA per SM, all 512 TMEM columns. Warp 1 issues the INT8 update
// kernel's MMA schedule (7 MMAs of N = 128..32, M = 128, 4 K-steps each, SS
// mode, zeroed operands) into TMEM columns [0, 128); warps 2..9 read columns
// [384, 512) with the drain's access pattern (8 x tcgen05.ld.32x32b.x8 per
// warp and "tile", lane quadrant = warp % 4, two warps per quadrant). Modes:
// 1 = MMAs only, 2 = loads only, 3 = both at once (no dependency between
// them). If mode 3 takes max(mode 1, mode 2) they overlap; if it takes the
// sum they do not.
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tmem_overlap_bench tools/tmem_overlap_bench.cu
#include <cstdint>
#include <cstdio>

#include <cuda_runtime.h>

#define DEVI __device__ __forceinline__

DEVI uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
DEVI void mb_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}
DEVI void mb_wait(uint32_t bar, uint32_t parity) {
    uint32_t ok = 0;
    while (!ok)
        asm volatile(
            "{\n.reg .pred p;\n"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            "selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"(bar), "r"(parity)
            : "memory");
}
DEVI void tc_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(bar) : "memory");
}
DEVI uint32_t elect_one() {
    uint32_t pred = 0;
    asm volatile(
        "{\n.reg .b32 rx;\n.reg .pred px;\n"
        "elect.sync rx|px, 0xffffffff;\n"
        "@px mov.s32 %0, 1;\n}\n"
        : "+r"(pred));
    return pred;
}
__host__ __device__ constexpr uint32_t idesc_n(int n) {
    return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
DEVI uint32_t desc_lo(uint32_t addr) { return ((addr >> 4) & 0x3FFFu) | ((128u >> 4) << 16); }
constexpr uint32_t kDescHi = (1024u >> 4) | (1u << 14);

template <uint32_t kIdesc>
DEVI void mma_k128(uint32_t d, uint32_t alo, uint32_t blo, int first) {
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
        const uint32_t acc = (first && ks == 0) ? 0u : 1u;
        asm volatile(
            "{\n.reg .pred q;\n.reg .b64 da, db;\n"
            "setp.ne.b32 q, %3, 0;\n"
            "mov.b64 da, {%1, %4};\nmov.b64 db, {%2, %4};\n"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], da, db, %5, q;\n}\n" ::"r"(d),
            "r"(alo + 16u * ks), "r"(blo + 16u * ks), "r"(acc), "n"(kDescHi), "n"(kIdesc)
            : "memory");
    }
}
// A from TMEM (8 columns per K-step)
template <uint32_t kIdesc>
DEVI void mma_k128_ts(uint32_t d, uint32_t atmem, uint32_t blo, int first) {
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
        const uint32_t acc = (first && ks == 0) ? 0u : 1u;
        asm volatile(
            "{\n.reg .pred q;\n.reg .b64 db;\n"
            "setp.ne.b32 q, %3, 0;\n"
            "mov.b64 db, {%2, %4};\n"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], db, %5, q;\n}\n" ::"r"(d),
            "r"(atmem + 8u * ks), "r"(blo + 16u * ks), "r"(acc), "n"(kDescHi), "n"(kIdesc)
            : "memory");
    }
}
DEVI void tc_cp_128x256b(uint32_t tmem_dst, uint32_t slo) {
    asm volatile(
        "{\n.reg .b64 sd;\n"
        "mov.b64 sd, {%1, %2};\n"
        "tcgen05.cp.cta_group::1.128x256b [%0], sd;\n}\n" ::"r"(tmem_dst),
        "r"(slo), "n"(kDescHi)
        : "memory");
}
DEVI void tmem_ld8(uint32_t taddr, uint32_t (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr)
                 : "memory");
}

constexpr int kThreads = 320;  // warp 0 idle, warp 1 MMA, warps 2..9 loads

__global__ void __launch_bounds__(kThreads, 1) bench_kernel(int mode, int iters, long long *cycles, uint32_t *sink) {
    extern __shared__ __align__(1024) uint8_t smem[];
    // A: 7 slices x 16 KB, B: 8 slices x 2 KB (zeros), barrier, tmem slot
    const uint32_t sA = smem_u32(smem), sB = sA + 7 * 16384;
    const uint32_t bar = sB + 8 * 2048;
    uint32_t *slot = reinterpret_cast<uint32_t *>(smem + 7 * 16384 + 8 * 2048 + 64);
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < (7 * 16384 + 8 * 2048) / 16; i += kThreads)
        reinterpret_cast<uint4 *>(smem)[i] = make_uint4(0x01010101u, 0x01010101u, 0x01010101u, 0x01010101u);
    if (tid == 0) {
        mb_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(slot)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tmem = *slot;
    const long long t0 = clock64();
    if (warp == 1 && (mode & 4)) {  // TS mode: A digits in TMEM columns [0, 224), D in [256, 384)
        if (elect_one()) {
            const uint32_t alo = desc_lo(sA), blo = desc_lo(sB);
            for (int sl = 0; sl < 7; ++sl)
                for (int ks = 0; ks < 4; ++ks)
                    tc_cp_128x256b(tmem + (uint32_t)(sl * 32 + ks * 8), alo + (uint32_t)((sl * 16384 + ks * 256) >> 4));
            for (int it = 0; it < iters; ++it) {
                const uint32_t d0 = tmem + 256u;
                mma_k128_ts<idesc_n(128)>(d0 + 0 * 16, tmem + 0 * 32, blo, 1);
                mma_k128_ts<idesc_n(112)>(d0 + 1 * 16, tmem + 1 * 32, blo, 0);
                mma_k128_ts<idesc_n(96)>(d0 + 2 * 16, tmem + 2 * 32, blo, 0);
                mma_k128_ts<idesc_n(80)>(d0 + 3 * 16, tmem + 3 * 32, blo, 0);
                mma_k128_ts<idesc_n(64)>(d0 + 4 * 16, tmem + 4 * 32, blo, 0);
                mma_k128_ts<idesc_n(48)>(d0 + 5 * 16, tmem + 5 * 32, blo, 0);
                mma_k128_ts<idesc_n(32)>(d0 + 6 * 16, tmem + 6 * 32, blo, 0);
            }
            tc_commit(bar);
        }
        __syncwarp();
        mb_wait(bar, 0);
    }
    if (warp == 1 && (mode & 1)) {
        if (elect_one()) {
            const uint32_t alo = desc_lo(sA), blo = desc_lo(sB);
            constexpr uint32_t sa = 16384 >> 4;
            for (int it = 0; it < iters; ++it) {
                const uint32_t d0 = tmem;  // columns [0, 128)
                mma_k128<idesc_n(128)>(d0 + 0 * 16, alo + 0 * sa, blo, 1);
                mma_k128<idesc_n(112)>(d0 + 1 * 16, alo + 1 * sa, blo, 0);
                mma_k128<idesc_n(96)>(d0 + 2 * 16, alo + 2 * sa, blo, 0);
                mma_k128<idesc_n(80)>(d0 + 3 * 16, alo + 3 * sa, blo, 0);
                mma_k128<idesc_n(64)>(d0 + 4 * 16, alo + 4 * sa, blo, 0);
                mma_k128<idesc_n(48)>(d0 + 5 * 16, alo + 5 * sa, blo, 0);
                mma_k128<idesc_n(32)>(d0 + 6 * 16, alo + 6 * sa, blo, 0);
            }
            tc_commit(bar);
        }
        __syncwarp();
        mb_wait(bar, 0);
    }
    uint32_t acc = 0;
    if (warp >= 2 && (mode & 2)) {
        const int quad = warp & 3, half = ((warp - 2) >> 2) & 1;
        const uint32_t taddr = tmem + 384u + ((uint32_t)(quad * 32) << 16) + (uint32_t)(half * 8);
        for (int it = 0; it < iters; ++it) {
            uint32_t v[8][8];
#pragma unroll
            for (int g = 0; g < 8; ++g) tmem_ld8(taddr + (uint32_t)(g * 16), v[g]);
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
            for (int g = 0; g < 8; ++g)
#pragma unroll
                for (int c = 0; c < 8; ++c) acc ^= v[g][c];
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    const long long t1 = clock64();
    if (tid == 0) cycles[blockIdx.x] = t1 - t0;
    if (acc == 0x12345678u) sink[0] = acc;
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem) : "memory");
    }
}

int main() {
    const int iters = 2000, grid = 148;
    const size_t smem = 7 * 16384 + 8 * 2048 + 256;
    cudaError_t ae = cudaFuncSetAttribute(bench_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (ae != cudaSuccess) printf("attr: %s\n", cudaGetErrorString(ae));
    long long *cyc;
    uint32_t *sink;
    cudaMalloc(&cyc, sizeof(long long) * grid);
    cudaMemset(cyc, 0xff, sizeof(long long) * grid);
    cudaMalloc(&sink, 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    const int modes[] = {1, 2, 3, 4, 6};
    for (int mode : modes) {
        float best = 1e30f;
        for (int rep = 0; rep < 4; ++rep) {
            cudaEventRecord(e0);
            bench_kernel<<<grid, kThreads, smem>>>(mode, iters, cyc, sink);
            cudaEventRecord(e1);
            cudaError_t e = cudaGetLastError();
            if (e == cudaSuccess) e = cudaDeviceSynchronize();
            if (e != cudaSuccess) {
                printf("mode %d: %s\n", mode, cudaGetErrorString(e));
                return 1;
            }
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep && ms < best) best = ms;
        }
        printf("mode %d (%s): %.3f ms for %d tiles = %.0f cycles per tile at %d MHz (28 MMAs x 4 K-steps; 8 warps x 8 "
               "tcgen05.ld.x8 = 64 KB)\n",
               mode, mode == 1 ? "SS MMAs only" : (mode == 2 ? "TMEM loads only" : (mode == 3 ? "SS MMAs + loads" : (mode == 4 ? "TS MMAs only (A in TMEM)" : "TS MMAs + loads"))), best, iters,
               best * 1e-3 * clk_khz * 1e3 / iters, clk_khz / 1000);
    }
    return 0;
}

// Shared device helpers for the sm_100a CQRRPT kernels.
//
// FP64 tensor math: sm_100a has no tcgen05 kind for f64 (the UMMA kinds are
// f16/tf32/f8f6f4/i8/mx*), so the FP64 contractions run on the DMMA pipe via
// warp-level mma.sync.m8n8k4.f64 (SASS: DMMA.8x8x4). Operands are staged in
// shared memory with cp.async and padded leading dimensions chosen so that
// every fragment load is a 2-wavefront (optimal) LDS.64.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#define CQ_DEVI __device__ __forceinline__

namespace cqg {

constexpr double kUnitRoundoff = 1.1102230246251565e-16;  // 2^-53 (cqrrpt.hh:14)

template <class T>
__host__ __device__ __forceinline__ T cmin(T a, T b) {
    return a < b ? a : b;
}
template <class T>
__host__ __device__ __forceinline__ T cmax(T a, T b) {
    return a < b ? b : a;
}

// ---------------------------------------------------------------------------
// DMMA m8n8k4: D(8x8) += A(8x4) * B(4x8).
//   lane = 4*g + t  (g = lane>>2 in 0..7, t = lane&3)
//   a  = A[g][t]        (row-major A fragment)
//   b  = B[t][g]        (column-major B fragment)
//   d0 = D[g][2t], d1 = D[g][2t+1]
// ---------------------------------------------------------------------------
CQ_DEVI void dmma884(double &d0, double &d1, double a, double b) {
    asm volatile(
        "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(d0), "+d"(d1)
        : "d"(a), "d"(b));
}

// ---------------------------------------------------------------------------
// cp.async (LDGSTS) helpers
// ---------------------------------------------------------------------------
CQ_DEVI uint32_t smem_u32(const void *p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

CQ_DEVI void cp_async16(void *smem, const void *gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(smem)), "l"(gmem));
}
// 16-byte copy with zero fill of the bytes past `src_bytes` (0, 8 or 16)
CQ_DEVI void cp_async16_zfill(void *smem, const void *gmem, int src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem),
                 "r"(src_bytes));
}
CQ_DEVI void cp_async8_zfill(void *smem, const void *gmem, int src_bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem),
                 "r"(src_bytes));
}
CQ_DEVI void cp_async4(void *smem, const void *gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(smem)), "l"(gmem));
}
// the same copies addressed by a 32-bit shared-window address
CQ_DEVI void cp_async16_s(uint32_t s, const void *gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
CQ_DEVI void cp_async8_zfill_s(uint32_t s, const void *gmem, int src_bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
CQ_DEVI void cp_async4_s(uint32_t s, const void *gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
}
CQ_DEVI void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
CQ_DEVI void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// L2-coherent loads (bypass the non-coherent L1) for data another CTA of the
// same persistent kernel may have written.
CQ_DEVI double ld_cg(const double *p) { return __ldcg(p); }
CQ_DEVI int32_t ld_cg(const int32_t *p) { return __ldcg(p); }

// ---------------------------------------------------------------------------
// Grid-wide barrier for cooperatively launched (co-resident) kernels.
// Sense-reversing: `bar[0]` counts arrivals, `bar[1]` is the generation.
// ---------------------------------------------------------------------------
CQ_DEVI void grid_barrier(unsigned int *bar, unsigned int nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned int *gen = bar + 1;
        unsigned int g = *gen;
        __threadfence();
        unsigned int arrived = atomicAdd(bar, 1u);
        if (arrived == nblocks - 1) {
            atomicExch(bar, 0u);
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            while (*gen == g) {
                __nanosleep(20);
            }
        }
        __threadfence();
    }
    __syncthreads();
}

// Monotonic-counter barrier: one atomic per CTA, completion = the counter
// reaching `target` (= number of barriers so far x nblocks). The counter is
// zeroed by the host before the launch.
CQ_DEVI void grid_barrier_mono(unsigned long long *counter, unsigned long long target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(counter, 1ULL);
        unsigned long long v;
        do {
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(counter) : "memory");
        } while (v < target);
    }
    __syncthreads();
}

// ---------------------------------------------------------------------------
// Deterministic reductions (fixed shuffle trees)
// ---------------------------------------------------------------------------
CQ_DEVI double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
CQ_DEVI double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Block sum of one double per thread; result valid in every thread.
// `scratch` needs blockDim.x/32 doubles. Deterministic for fixed blockDim.
CQ_DEVI double block_sum(double v, double *scratch) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) scratch[wid] = v;
    __syncthreads();
    double t = (lane < nw) ? scratch[lane] : 0.0;
    t = warp_sum(t);
    return t;
}

// Argmax with the reference's tie rule (qrcp.cc:26-31): larger value wins,
// equal values keep the lower index.
struct ArgMax {
    double v;
    int32_t i;
};
CQ_DEVI ArgMax argmax_combine(ArgMax a, ArgMax b) {
    if (b.v > a.v || (b.v == a.v && b.i < a.i)) return b;
    return a;
}
CQ_DEVI ArgMax warp_argmax(ArgMax a) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        ArgMax b;
        b.v = __shfl_xor_sync(0xffffffffu, a.v, o);
        b.i = __shfl_xor_sync(0xffffffffu, a.i, o);
        a = argmax_combine(a, b);
    }
    return a;
}

// ---------------------------------------------------------------------------
// Counter RNG, bit-identical to the reference (rng.hh:18-53).
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint64_t rng_bits(uint64_t seed, uint64_t counter) {
    uint64_t z = seed + (counter + 1) * 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
CQ_DEVI uint64_t rng_below(uint64_t seed, uint64_t counter, uint64_t bound) {
    return __umul64hi(rng_bits(seed, counter), bound);
}
__host__ __device__ __forceinline__ uint64_t mix_seed(uint64_t seed, uint64_t salt) {
    return rng_bits(seed, 0x5eedULL + salt);
}
// CounterRng::normal (rng.hh:32-36): Box-Muller cosine branch, one value per
// counter; device log/cos are within 1 ulp of the host libm's
CQ_DEVI double normal_dev(uint64_t seed, uint64_t counter) {
    const double u1 = (double)((rng_bits(seed, 2 * counter) >> 11) + 1) * 0x1.0p-53;
    const double u2 = (double)(rng_bits(seed, 2 * counter + 1) >> 11) * 0x1.0p-53;
    return sqrt(-2.0 * log(u1)) * cos(6.283185307179586476925287 * u2);
}

}  // namespace cqg

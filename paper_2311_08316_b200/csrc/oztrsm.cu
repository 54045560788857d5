// K5a / K8, INT8 tensor-core engine: X = B[:, cols] U^{-1} (U upper k x k)
// with the trailing updates on tcgen05 (kind::i8, accumulators in TMEM).
//
// Reference: trsm_right (linalg.cc:244-277) on M.select_columns(J[:k0])
// (dense_matrix.hh:70-80, cqrrpt.cc:262,165) and on M_pre (cqrrpt.cc:280).
// sm_100a has no FP64 tcgen05 kind; the DMMA engine (trsm.cu) runs at ~0.95 of
// the cuBLAS DGEMM rate. This engine moves the GEMM part of the solve to the
// INT8 tensor cores with an exact integer emulation (Ozaki scheme I):
//
// Right-looking blocked solve, 128-column blocks b:
//   X_b = T_b U_bb^{-1}                      DMMA (trsm_block_kernel, 2 x 64)
//   T_>b -= X_b U_b,>b                       INT8 tcgen05 (oz_update_kernel)
// T starts as B[:, cols] (the gather is fused into the first step's reads).
//
// Emulated product of one step: row i of X_b is scaled by 2^(54 - e_i)
// (e_i = exponent of the row's max over the block) and rounded to a 55-bit
// integer, column j of U_b,>b by 2^(54 - f_j); each integer is split into 7
// balanced base-256 digits (int8, most significant first). The products of
// digit slices s, t with s + t = g <= 7 accumulate in int32 (exact: |acc| <=
// 8 pairs * 128 * 2^14 = 2^24) into TMEM group g; the epilogue forms
// sum_g acc_g 2^(-12-8g) in FP64 (smallest group first), scales by
// 2^(e_i + f_j) and subtracts from T in FP64. Dropped pairs (g >= 8) and the
// 54-bit rounding bound the error by ~2^-54 max|X_i,:| max|U_:,j| per term --
// the FP64 GEMM's normwise bound (the parity tests compare with the DMMA
// engine and the oracle).
//
// oz_update_kernel: persistent, one CTA per SM (200 KB shared memory):
//   warp 0   producer: 1-D bulk copies (TMA engine) of the panel's digit
//            slices (128 rows x 128 K x 7 = 112 KB, pre-tiled in the UMMA
//            canonical K-major layout) and a 3-stage ring of N-tiles of U's
//            slices (32 x 128 x 7 = 28 KB);
//   warp 1   TMEM allocator + MMA issuer (one thread): per N tile 34 digit
//            pairs x 4 K-steps of tcgen05.mma M128 N32 K32 into 8 group
//            accumulators, double-buffered (2 x 8 x 32 = 512 TMEM columns);
//   warps 2-5 epilogue: tcgen05.ld of the 8 groups (lane = row), FP64
//            recombination, read-modify-write of T (coalesced column runs).
#include <climits>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "internal.hh"

namespace cqg {
namespace {

constexpr int kW = 128;                    // column block = K of each update
constexpr int kDig = 7;                    // base-256 digits per value
constexpr int kGroups = 8;                 // digit-pair groups g = s + t <= 7
constexpr int kBM = 128;                   // panel rows = MMA M = TMEM lanes
constexpr int kBN = 32;                    // N tile
constexpr int kSliceA = kBM * kW;          // 16384 B per digit slice of a panel
constexpr int kSliceB = kBN * kW;          // 4096 B per digit slice of an N tile
constexpr int kPanelBytes = kDig * kSliceA;  // 114688
constexpr int kTileBBytes = kDig * kSliceB;  // 28672
constexpr int kBStages = 3;
constexpr int kEpiWarps = 8;               // 2 per TMEM lane quadrant, 16 columns each
constexpr int kUpdThreads = 64 + 32 * kEpiWarps;  // producer, MMA, epilogue
constexpr int kTmemCols = 512;             // 2 buffers x 8 groups x 32 columns

constexpr uint32_t kSmemA = 0;
constexpr uint32_t kSmemB = kPanelBytes;
constexpr uint32_t kSmemBar = kSmemB + kBStages * kTileBBytes;  // 200704
constexpr uint32_t kUpdSmem = kSmemBar + 256;

// byte offset of (row r, k kk) in a digit slice laid out as UMMA core matrices
// (8 rows x 16 bytes, K-major, no swizzle): LBO = 128 (next 16 K), SBO = 1024
// (next 8 rows)
__host__ __device__ constexpr uint32_t canon_off(int r, int kk) {
    return (uint32_t)((r >> 3) * 1024 + (kk >> 4) * 128 + (r & 7) * 16 + (kk & 15));
}

// ---------------------------------------------------------------------------
// digit slicing
// ---------------------------------------------------------------------------
CQ_DEVI void digits7(double v, int sh, uint32_t (&w)[kDig], int byte) {
    long long q = __double2ll_rn(ldexp(v, sh));  // |q| <= 2^54
#pragma unroll
    for (int s = kDig - 1; s >= 0; --s) {
        const long long d = ((q + 128) & 255) - 128;  // balanced digit in [-128, 127]
        q = (q - d) >> 8;
        w[s] |= ((uint32_t)(d & 255)) << (8 * byte);
    }
}

// A operand: rows of X_b (m x w, column-major). CTA = one 128-row panel,
// thread = row: exponent of the row max, then 7 digit slices in the canonical
// layout (16-byte stores: 8 consecutive rows write one 128-byte core matrix).
__global__ void __launch_bounds__(kBM) oz_slice_rows_kernel(int64_t m, int w, const double *__restrict__ x,
                                                            int64_t ldx, int8_t *__restrict__ slices,
                                                            double *__restrict__ rscale) {
    const int r = threadIdx.x;
    const int64_t p = blockIdx.x, row = p * kBM + r;
    const bool valid = row < m;
    const double *xr = x + (valid ? row : 0);
    double mx = 0.0;
    bool bad = false;
    if (valid)
        for (int c = 0; c < w; ++c) {
            const double a = fabs(xr[(int64_t)c * ldx]);
            bad |= !(a <= 1.79769313486231570e308);
            mx = fmax(mx, a);
        }
    int e = 0;
    if (mx > 0.0) frexp(mx, &e);  // mx < 2^e
    rscale[row] = bad ? __longlong_as_double(0x7ff8000000000000ll) : ldexp(1.0, e);
    const int sh = 54 - e;
    uint8_t *base = reinterpret_cast<uint8_t *>(slices) + p * (int64_t)kPanelBytes;
#pragma unroll 1
    for (int kc = 0; kc < kW / 16; ++kc) {
        uint32_t wd[4][kDig];
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int s = 0; s < kDig; ++s) wd[q][s] = 0u;
        if (valid && !bad) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const int c = kc * 16 + j;
                const double v = (c < w) ? xr[(int64_t)c * ldx] : 0.0;
                digits7(v, sh, wd[j >> 2], j & 3);
            }
        }
#pragma unroll
        for (int s = 0; s < kDig; ++s)
            *reinterpret_cast<uint4 *>(base + s * kSliceA + canon_off(r, kc * 16)) =
                make_uint4(wd[0][s], wd[1][s], wd[2][s], wd[3][s]);
    }
}

// B operand: columns j of U[b0 : b0 + w, c0 : c0 + N] (column-major U),
// thread = column: exponent of the column max over the block rows, digit
// slices per 32-column N tile in the canonical layout (N = row index there).
__global__ void oz_slice_cols_kernel(int64_t ncols, int w, const double *__restrict__ u, int64_t ldu,
                                     int8_t *__restrict__ slices, double *__restrict__ cscale) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t ntn = (ncols + kBN - 1) / kBN;
    if (j >= ntn * kBN) return;
    const bool valid = j < ncols;
    const double *uc = u + (valid ? j : 0) * ldu;
    double mx = 0.0;
    bool bad = false;
    if (valid)
        for (int t = 0; t < w; ++t) {
            const double a = fabs(uc[t]);
            bad |= !(a <= 1.79769313486231570e308);
            mx = fmax(mx, a);
        }
    int e = 0;
    if (mx > 0.0) frexp(mx, &e);
    cscale[j] = bad ? __longlong_as_double(0x7ff8000000000000ll) : ldexp(1.0, e - 12);  // folds 2^-12 of the groups
    const int sh = 54 - e;
    const int n = (int)(j % kBN);
    uint8_t *base = reinterpret_cast<uint8_t *>(slices) + (j / kBN) * (int64_t)kTileBBytes;
#pragma unroll 1
    for (int kc = 0; kc < kW / 16; ++kc) {
        uint32_t wd[4][kDig];
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int s = 0; s < kDig; ++s) wd[q][s] = 0u;
        if (valid && !bad) {
#pragma unroll
            for (int jj = 0; jj < 16; ++jj) {
                const int t = kc * 16 + jj;
                digits7(t < w ? uc[t] : 0.0, sh, wd[jj >> 2], jj & 3);
            }
        }
#pragma unroll
        for (int s = 0; s < kDig; ++s)
            *reinterpret_cast<uint4 *>(base + s * kSliceB + canon_off(n, kc * 16)) =
                make_uint4(wd[0][s], wd[1][s], wd[2][s], wd[3][s]);
    }
}

// ---------------------------------------------------------------------------
// tcgen05 / mbarrier / bulk-copy primitives
// ---------------------------------------------------------------------------
CQ_DEVI void mb_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}
CQ_DEVI void mb_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
CQ_DEVI void mb_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
// bounded wait: a protocol error traps (the launch fails) instead of hanging
CQ_DEVI void mb_wait(uint32_t bar, uint32_t parity) {
    uint32_t ok = 0;
    for (uint32_t it = 0;; ++it) {
        asm volatile(
            "{\n.reg .pred p;\n"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, 1000000;\n"
            "selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"(bar), "r"(parity)
            : "memory");
        if (ok) return;
        if (it > (1u << 26)) __trap();
    }
}
// whole-warp wait with a warp-uniform exit (keeps the MMA loop's values in
// uniform registers)
CQ_DEVI void mb_wait_warp(uint32_t bar, uint32_t parity) {
    for (uint32_t it = 0;; ++it) {
        uint32_t ok;
        asm volatile(
            "{\n.reg .pred p;\n"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, 1000000;\n"
            "selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"(bar), "r"(parity)
            : "memory");
        if (__all_sync(0xffffffffu, ok)) return;
        if (it > (1u << 26)) __trap();
    }
}
CQ_DEVI void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
CQ_DEVI void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
CQ_DEVI void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
CQ_DEVI void tc_commit(uint32_t bar) {  // by the MMA-issuing thread
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(bar)
                 : "memory");
}
// instruction descriptor: s32 accumulate, s8 x s8, both K-major, N = 32, M = 128
constexpr uint32_t kIdesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kBN >> 3) << 17) |
                            ((uint32_t)(kBM >> 4) << 24);

// Shared-memory matrix descriptor (no swizzle, K-major core matrices): low
// word = start address >> 4 | (LBO = 128) >> 4 << 16, high word = (SBO =
// 1024) >> 4 | version 1 << 14.
CQ_DEVI uint32_t desc_lo(uint32_t addr) { return ((addr >> 4) & 0x3FFFu) | ((128u >> 4) << 16); }
constexpr uint32_t kDescHi = (1024u >> 4) | (1u << 14);

// D[tmem] (+)= A[smem] * B[smem]^T over the 4 K-steps (K = 128) of one digit
// pair, int8 x int8 -> int32, issued by the single elected thread of the MMA
// warp (its commits then track these MMAs). The K-step advances both start
// addresses by 256 bytes (+16 in descriptor units).
template <uint32_t kIdescT, bool kFirst>
CQ_DEVI void tc_mma_i8_k128(uint32_t dtmem, uint32_t alo, uint32_t blo) {
    asm volatile(
        "{\n.reg .pred q0, q1;\n.reg .b64 da, db;\n.reg .b32 a1, b1;\n"
        "setp.ne.b32 q0, %3, 0;\n"
        "setp.eq.b32 q1, %3, %3;\n"
        "mov.b64 da, {%1, %4};\nmov.b64 db, {%2, %4};\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], da, db, %5, q0;\n"
        "add.u32 a1, %1, 16;\nadd.u32 b1, %2, 16;\nmov.b64 da, {a1, %4};\nmov.b64 db, {b1, %4};\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], da, db, %5, q1;\n"
        "add.u32 a1, %1, 32;\nadd.u32 b1, %2, 32;\nmov.b64 da, {a1, %4};\nmov.b64 db, {b1, %4};\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], da, db, %5, q1;\n"
        "add.u32 a1, %1, 48;\nadd.u32 b1, %2, 48;\nmov.b64 da, {a1, %4};\nmov.b64 db, {b1, %4};\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], da, db, %5, q1;\n}\n" ::"r"(dtmem),
        "r"(alo), "r"(blo), "n"(kFirst ? 0 : 1), "n"(kDescHi), "n"(kIdescT)
        : "memory");
}
CQ_DEVI uint32_t elect_one() {
    uint32_t pred = 0;
    asm volatile(
        "{\n.reg .b32 rx;\n.reg .pred px;\n"
        "elect.sync rx|px, 0xffffffff;\n"
        "@px mov.s32 %0, 1;\n}\n"
        : "+r"(pred));
    return pred;
}
CQ_DEVI void tmem_ld8(uint32_t taddr, uint32_t (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr)
                 : "memory");
}
CQ_DEVI void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }

// ---------------------------------------------------------------------------
// the update: cout[:, j] = cin[:, col(j)] - X_b U_b,j   (j < ncols)
// ---------------------------------------------------------------------------
struct UpdArgs {
    int64_t m, ncols;
    int npanels, ntn;
    const int8_t *aslc;
    const double *rscale;  // 2^e_i per row (NaN: non-finite row)
    const int8_t *bslc;
    const double *cscale;  // 2^(f_j - 12) per column (NaN: non-finite column)
    const double *cin;
    int64_t ldin;
    const int64_t *cols_in;  // nullptr: column j of cin is j
    double *cout;
    int64_t ldout;
};

__global__ void __launch_bounds__(kUpdThreads, 1) oz_update_kernel(UpdArgs P) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t sbase = smem_u32(smem);
    const uint32_t sA = sbase + kSmemA, sB = sbase + kSmemB;
    const uint32_t bar = sbase + kSmemBar;
    const uint32_t a_full = bar, a_empty = bar + 8;
    auto b_full = [&](int s) { return bar + 16 + 8u * s; };
    auto b_empty = [&](int s) { return bar + 16 + 8u * (kBStages + s); };
    auto acc_full = [&](int q) { return bar + 16 + 8u * (2 * kBStages + q); };
    auto acc_empty = [&](int q) { return bar + 16 + 8u * (2 * kBStages + 2 + q); };
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + kSmemBar + 192);

    if (tid == 0) {
        mb_init(a_full, 1);
        mb_init(a_empty, 1);
        for (int s = 0; s < kBStages; ++s) {
            mb_init(b_full(s), 1);
            mb_init(b_empty(s), 1);
        }
        for (int q = 0; q < 2; ++q) {
            mb_init(acc_full(q), 1);
            mb_init(acc_empty(q), kEpiWarps * 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                     "n"(kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    // all 512 columns of the SM's TMEM (one CTA per SM): the allocation
    // starts at lane 0, column 0, so addresses are compile-time constants and
    // the MMA operands stay in uniform registers
    if (*tmem_slot != 0u) __trap();
    constexpr uint32_t tmem = 0u;

    if (warp == 0) {
        if (lane == 0) {  // ---------------- producer
            int bs = 0;
            uint32_t bfill = 0;
            int pi = 0;
            for (int p = blockIdx.x; p < P.npanels; p += gridDim.x, ++pi) {
                if (pi) mb_wait(a_empty, (uint32_t)(pi - 1) & 1u);
                mb_expect_tx(a_full, kPanelBytes);
                const int8_t *ga = P.aslc + (int64_t)p * kPanelBytes;
                for (int s = 0; s < kDig; ++s) bulk_g2s(sA + s * kSliceA, ga + s * kSliceA, kSliceA, a_full);
                for (int nt = 0; nt < P.ntn; ++nt) {
                    if (bfill) mb_wait(b_empty(bs), (bfill - 1u) & 1u);
                    mb_expect_tx(b_full(bs), kTileBBytes);
                    bulk_g2s(sB + bs * kTileBBytes, P.bslc + (int64_t)nt * kTileBBytes, kTileBBytes, b_full(bs));
                    if (++bs == kBStages) bs = 0, ++bfill;
                }
            }
        }
    } else if (warp == 1) {
        {  // ---------------- MMA issuer (whole warp, warp-uniform loop)
            int bs = 0;
            uint32_t buse = 0;
            uint32_t tc = 0;  // tiles issued: accumulator buffer tc & 1, its use tc >> 1
            int pi = 0;
            const uint32_t alo0 = desc_lo(sA);
            for (int p = blockIdx.x; p < P.npanels; p += gridDim.x, ++pi) {
                mb_wait_warp(a_full, (uint32_t)pi & 1u);
                tc_fence_after();
                for (int nt = 0; nt < P.ntn; ++nt) {
                    mb_wait_warp(b_full(bs), buse & 1u);
                    const int q = (int)(tc & 1u);
                    if (tc >= 2u) mb_wait_warp(acc_empty(q), ((tc >> 1) - 1u) & 1u);
                    tc_fence_after();
                    const uint32_t blo0 = desc_lo(sB + bs * kTileBBytes);
                    const uint32_t d0 = tmem + (uint32_t)(q * kGroups * kBN);
                    // digit pairs (s, t) with s + t = g, group by group
                    if (elect_one()) {
#pragma unroll
                    for (int g = 0; g < kGroups; ++g) {
#pragma unroll
                        for (int s = 0; s < kDig; ++s) {
                            const int t = g - s;
                            if (t < 0 || t >= kDig) continue;
                            const uint32_t d = d0 + (uint32_t)(g * kBN);
                            const uint32_t alo = alo0 + (uint32_t)(s * (kSliceA >> 4));
                            const uint32_t blo = blo0 + (uint32_t)(t * (kSliceB >> 4));
                            if (s == (g > kDig - 1 ? g - (kDig - 1) : 0))
                                tc_mma_i8_k128<kIdesc, true>(d, alo, blo);
                            else
                                tc_mma_i8_k128<kIdesc, false>(d, alo, blo);
                        }
                    }
                    tc_commit(b_empty(bs));
                    tc_commit(acc_full(q));
                    }
                    __syncwarp();
                    ++tc;
                    if (++bs == kBStages) bs = 0, ++buse;
                }
                if (elect_one()) tc_commit(a_empty);
                __syncwarp();
            }
        }
    } else {  // ---------------- epilogue warps: lane quadrant warp % 4, 16 columns each
        const int quad = warp & 3, half = (warp - 2) >> 2;
        const int rloc = quad * 32 + lane;
        const uint32_t taddr0 = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(half * 16);
        uint32_t tc = 0;
        for (int p = blockIdx.x; p < P.npanels; p += gridDim.x) {
            const int64_t row = (int64_t)p * kBM + rloc;
            const bool valid = row < P.m;
            const int64_t rowc = valid ? row : 0;  // rows past m load row 0 and store nothing
            const double rs = P.rscale[row];       // rscale covers the padded panel
            for (int nt = 0; nt < P.ntn; ++nt, ++tc) {
                const int64_t j0 = (int64_t)nt * kBN + half * 16;
                const int64_t rem = P.ncols - j0;
                const int nc = rem >= 16 ? 16 : (rem > 0 ? (int)rem : 0);
                // this tile's right-hand side and column scales: loads in
                // flight while the MMAs run
                double cv[16], cs[16];
                if (nc == 16) {
                    if (P.cols_in) {
#pragma unroll
                        for (int c = 0; c < 16; ++c) cv[c] = P.cin[__ldg(P.cols_in + j0 + c) * P.ldin + rowc];
                    } else {
                        const double *pc = P.cin + j0 * P.ldin + rowc;
#pragma unroll
                        for (int c = 0; c < 16; ++c) cv[c] = pc[c * P.ldin];
                    }
#pragma unroll
                    for (int c = 0; c < 16; ++c) cs[c] = __ldg(P.cscale + j0 + c);
                } else {
#pragma unroll
                    for (int c = 0; c < 16; ++c) {
                        cv[c] = 0.0;
                        cs[c] = 0.0;
                        if (c < nc) {
                            const int64_t cj = P.cols_in ? __ldg(P.cols_in + j0 + c) : j0 + c;
                            cv[c] = P.cin[cj * P.ldin + rowc];
                            cs[c] = __ldg(P.cscale + j0 + c);
                        }
                    }
                }
                const int q = (int)(tc & 1u);
                mb_wait(acc_full(q), (tc >> 1) & 1u);
                tc_fence_after();
                const uint32_t ta = taddr0 + (uint32_t)(q * kGroups * kBN);
                double *po = P.cout + j0 * P.ldout + rowc;
#pragma unroll
                for (int h = 0; h < 16; h += 8) {
                    uint32_t v[kGroups][8];
#pragma unroll
                    for (int g = 0; g < kGroups; ++g) tmem_ld8(ta + (uint32_t)(g * kBN + h), v[g]);
                    tmem_wait_ld();
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        // exact integer recombination of groups 0-3 and 4-7
                        // (|.| < 2^50), converted with the scales 2^-24 and
                        // 2^-56 folded into the magic constants
                        const long long hi = (long long)(int)v[0][c] * 16777216ll + (long long)(int)v[1][c] * 65536ll +
                                             (long long)(int)v[2][c] * 256ll + (long long)(int)v[3][c];
                        const long long lo = (long long)(int)v[4][c] * 16777216ll + (long long)(int)v[5][c] * 65536ll +
                                             (long long)(int)v[6][c] * 256ll + (long long)(int)v[7][c];
                        const double hs = __longlong_as_double(hi + 0x41B8000000000000ll) - 402653184.0;  // hi 2^-24
                        const double ls = __longlong_as_double(lo + 0x3FB8000000000000ll) - 0.09375;      // lo 2^-56
                        const double prod = hs + ls;
                        if (valid && h + c < nc) po[(h + c) * P.ldout] = fma(-prod, rs * cs[h + c], cv[h + c]);
                    }
                }
                tc_fence_before();
                mb_arrive(acc_empty(q));
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(kTmemCols) : "memory");
    }
}

int launch_update(const UpdArgs &P, cudaStream_t st) {
    static thread_local int attr_dev = -1;
    const int dev = current_device();
    if (attr_dev != dev) {
        CQ_CUDA(cudaFuncSetAttribute(oz_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kUpdSmem),
                "oz update smem attr");
        attr_dev = dev;
    }
    const int grid = std::min(P.npanels, num_sms());
    oz_update_kernel<<<grid, kUpdThreads, kUpdSmem, st>>>(P);
    note_launch();
    return check_launch("oz_update_kernel");
}

}  // namespace

// Engine choice for trsm_right: CQRRPT_GPU_TRSM=oz | dmma forces one; by
// default the INT8 engine from m >= 65536 rows and k >= 256 columns.
bool trsm_use_ozaki(int64_t m, int64_t k) {
    const char *env = getenv("CQRRPT_GPU_TRSM");
    if (env && env[0] == 'd') return false;
    if (env && env[0] == 'o') return k > 0 && m > 0;
    return m >= 65536 && k >= 256;
}

int trsm_right_oz(int64_t m, int64_t k, const double *b, int64_t ldb, const int64_t *cols, const double *u,
                  int64_t ldu, double *x, int64_t ldx, cudaStream_t st, const BlockSink *sink, const double *dinv,
                  const cudaEvent_t *block_ev) {
    constexpr int64_t NB = 64;
    Workspace &ws = workspace();
    const int64_t npanels = (m + kBM - 1) / kBM;
    const int64_t ntn_max = (std::max<int64_t>(k - kW, 1) + kBN - 1) / kBN;
    int8_t *aslc = ws.get<int8_t>("oz.trsm.a", (size_t)(npanels * kPanelBytes));
    double *rexp = ws.get<double>("oz.trsm.rs", (size_t)(npanels * kBM));
    int8_t *bslc = ws.get<int8_t>("oz.trsm.b", (size_t)(ntn_max * kTileBBytes));
    double *cexp = ws.get<double>("oz.trsm.cs", (size_t)(ntn_max * kBN));
    if (!aslc || !rexp || !bslc || !cexp) return fail_nomem("oz trsm workspace");
    if (npanels > INT_MAX) return fail_internal("oz trsm: too many rows");
    cudaEvent_t *evs = nullptr;
    if (sink) CQ_TRY(cached_events("trsm.sink", (size_t)((k + NB - 1) / NB), &evs));
    for (int64_t b0 = 0; b0 < k; b0 += kW) {
        const int64_t b1 = std::min(k, b0 + kW), w = b1 - b0;
        const bool first = b0 == 0;
        // X_b = T_b U_bb^{-1}: the DMMA block kernel on the view starting at b0
        // (T_b is the gathered input for the first block, else X's own
        // columns, updated in place by the previous steps)
        const double *sview = first ? (cols ? b : b + b0 * ldb) : x + b0 * ldx;
        const int64_t lds = first ? ldb : ldx;
        const int64_t *cview = (first && cols) ? cols + b0 : nullptr;
        for (int64_t c0 = 0; c0 < w; c0 += NB) {
            CQ_TRY(trsm_block(m, k - b0, c0, sview, lds, cview, u + b0 * ldu + b0, ldu,
                              dinv + ((b0 + c0) / NB) * NB * NB, x + b0 * ldx, ldx, st));
            const int64_t cb = (b0 + c0) / NB;
            if (block_ev) CQ_CUDA(cudaEventRecord(block_ev[cb], st), "oz trsm block event");
            if (sink) {
                CQ_CUDA(cudaEventRecord(evs[cb], st), "oz trsm sink record");
                CQ_CUDA(cudaStreamWaitEvent(sink->copy, evs[cb], 0), "oz trsm sink wait");
                const int64_t nb = std::min<int64_t>(NB, k - (b0 + c0));
                CQ_CUDA(cudaMemcpy2DAsync(sink->host + (b0 + c0) * sink->ldh, sizeof(double) * sink->ldh,
                                          x + (b0 + c0) * ldx, sizeof(double) * ldx, sizeof(double) * m, nb,
                                          cudaMemcpyDeviceToHost, sink->copy),
                        "oz trsm sink copy");
            }
        }
        if (b1 >= k) break;
        // T_>b -= X_b U_b,>b on the INT8 tensor cores
        const int64_t ncols = k - b1;
        const int ntn = (int)((ncols + kBN - 1) / kBN);
        oz_slice_rows_kernel<<<(unsigned)npanels, kBM, 0, st>>>(m, (int)w, x + b0 * ldx, ldx, aslc, rexp);
        note_launch();
        CQ_TRY(check_launch("oz_slice_rows_kernel"));
        oz_slice_cols_kernel<<<(unsigned)((ntn * kBN + 127) / 128), 128, 0, st>>>(ncols, (int)w, u + b1 * ldu + b0,
                                                                                   ldu, bslc, cexp);
        note_launch();
        CQ_TRY(check_launch("oz_slice_cols_kernel"));
        UpdArgs P;
        P.m = m;
        P.ncols = ncols;
        P.npanels = (int)npanels;
        P.ntn = ntn;
        P.aslc = aslc;
        P.rscale = rexp;
        P.bslc = bslc;
        P.cscale = cexp;
        if (first) {
            P.cin = cols ? b : b + b1 * ldb;
            P.cols_in = cols ? cols + b1 : nullptr;
            P.ldin = ldb;
        } else {
            P.cin = x + b1 * ldx;
            P.cols_in = nullptr;
            P.ldin = ldx;
        }
        P.cout = x + b1 * ldx;
        P.ldout = ldx;
        CQ_TRY(launch_update(P, st));
    }
    return 0;
}

}  // namespace cqg

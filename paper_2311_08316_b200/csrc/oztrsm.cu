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
// 8 pairs * 128 * 2^14 = 2^24) into TMEM group g; the drain recombines groups
// 0-3 and 4-7 exactly in int64 (|.| < 2^50), converts each with the scale
// 2^-24 / 2^-56 folded into a magic constant, adds them (one rounding) and
// applies T - p 2^(e_i + f_j) with one more. Dropped pairs (g >= 8) and the
// 54-bit rounding bound the error by ~2^-54 max|X_i,:| max|U_:,j| per term --
// the FP64 GEMM's normwise bound (the parity tests compare with the DMMA
// engine and the oracle).
//
// oz_update_kernel: persistent, one CTA per SM (225 KB shared memory, all 512
// TMEM columns), tiles of 128 rows x 16 columns:
//   warp 0    producer (TMA engine): the panel's 7 digit slices (128 rows x 128
//             K each, pre-tiled in the UMMA canonical K-major layout) through a
//             2-slice ring, a ring of U's N tiles (16 x 128 x 7 = 14 KB, staged
//             with an all-zero 8th slice), and per tile the right-hand side
//             into a ring of 16 KB stages (eight 32 x 8 tensor-map boxes, one
//             per drain warp; the gathered first step is read from global
//             memory by the drain warps instead);
//   warp 1    TMEM allocator + MMA issuer (one elected thread, operands in
//             uniform registers): tcgen05.cp of the A slices into TMEM columns
//             0..223 once per panel, then per N tile and K-step ONE
//             tcgen05.mma per digit slice s of X covering all its partner
//             slices t of U at once: U's slices are consecutive 16-row blocks
//             of the canonical layout, so B = slices 0.. with N = 16 * count
//             and D = group s lands every pair (s, t) in group s + t (28 MMAs
//             of N = 32..128 per tile, issued K-step by K-step in chunks of 7
//             that are committed to a chunk barrier with at most two chunks in
//             flight: the issuing thread sleeps on the barrier instead of
//             sitting throttled on the tensor pipe, which starved the drain
//             warps of its scheduler). Two accumulator buffers (columns
//             256..383, 384..511) alternate between tiles, so a tile's MMAs
//             run while the previous tile is drained;
//   warps 2-17 drain + update, two sets of 8 (set = accumulator buffer = tile
//             parity): tcgen05.ld of all 8 groups of the warp's 32 rows x 8
//             columns in one batch, the buffer released at once (this
//             hand-off is the tile period's critical path), then the exact
//             recombination, T - p 2^(e_i + f_j) in place in the staged tile,
//             the warp's own TMA store of its 32 x 8 box.
// Even m only: TMA applies the box's row bound at 16-byte granularity.
#include <cuda.h>

#include <climits>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "internal.hh"

namespace cqg {
namespace {

constexpr int kW = 128;                    // column block = K of each update
constexpr int kDig = 7;                    // base-256 digits per value
constexpr int kGroups = 8;                 // digit-pair groups g = s + t <= 7
constexpr int kBM = 128;                   // panel rows = MMA M = TMEM lanes
constexpr int kBN = 16;                    // N tile
constexpr int kSliceA = kBM * kW;          // 16384 B per digit slice of a panel
constexpr int kSliceB = kBN * kW;          // 2048 B per digit slice of an N tile
constexpr int kPanelBytes = kDig * kSliceA;  // 114688
constexpr int kTileBBytes = kDig * kSliceB;  // 14336 in global memory
constexpr int kTileBSmem = (kDig + 1) * kSliceB;  // staged with an all-zero 8th slice (group 7 of digit 0)
constexpr int kSets = 2;                   // accumulator buffers = drain sets (tile parity)
constexpr int kEpiWarps = 8;               // per drain set: two per TMEM lane quadrant, 8 columns each
constexpr int kDC = kBN / 2;               // columns per drain warp
constexpr int kUpdThreads = 64 + 32 * kEpiWarps * kSets;  // producer, MMA, drain sets
constexpr int kTmemCols = 512;             // A digit slices (7 x 32) | 2 x accumulators (8 x 16)
constexpr uint32_t kTmemAcc = 256;         // first accumulator column
constexpr uint32_t kAccCols = kGroups * kBN;  // 128 columns per buffer

constexpr int kAStages = 2;                // digit slices staged on their way to TMEM
constexpr uint32_t kTileCBytes = kBM * kBN * 8;  // 16384: box (half h, quadrant q) = 32 rows x 8 columns at (4 h + q) * 2048, column c at c * 256
constexpr uint32_t kSmemA = 0;
constexpr uint32_t kSmemB = kAStages * kSliceA;
// ring depths: kBStages staged U tiles (16 KB), kCStages right-hand-side tiles (16 KB)
__host__ __device__ constexpr uint32_t upd_smem(int bst, int cst) {
    return kSmemB + (uint32_t)bst * kTileBSmem + (uint32_t)cst * kTileCBytes + 512u;
}

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

// A operand: rows of X_b (m x w, column-major). CTA = 32 rows: the 32 x 128
// tile is staged through shared memory with coalesced 256-byte column runs
// (X_b is read once), then thread (row, 16-column chunk) forms the row
// maximum's exponent (shared-memory reduction over the chunks) and the 7
// digit slices of its chunk in the canonical layout (16-byte stores: 8
// consecutive rows write one 128-byte core matrix).
constexpr int kSR = 32;
constexpr int kSLd = kW + 1;  // 129: conflict-free row reads
__global__ void __launch_bounds__(256) oz_slice_rows_kernel(int64_t m, int w, const double *__restrict__ x,
                                                            int64_t ldx, int8_t *__restrict__ slices,
                                                            double *__restrict__ rscale) {
    __shared__ double ts[kSR * kSLd];
    __shared__ double mx8[8 * kSR];
    const int r = threadIdx.x & (kSR - 1), q = threadIdx.x >> 5;  // row, 16-column chunk
    const int64_t row = (int64_t)blockIdx.x * kSR + r;
    const bool valid = row < m;
    const double *xr = x + (valid ? row : 0);
#pragma unroll 4
    for (int c = q; c < kW; c += 8) ts[r * kSLd + c] = (valid && c < w) ? xr[(int64_t)c * ldx] : 0.0;
    __syncthreads();
    double mx = 0.0;
    bool bad = false;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const double a = fabs(ts[r * kSLd + q * 16 + j]);
        bad |= !(a <= 1.79769313486231570e308);
        mx = fmax(mx, a);
    }
    mx8[q * kSR + r] = bad ? __longlong_as_double(0x7ff8000000000000ll) : mx;
    __syncthreads();
    mx = 0.0;
    bad = false;
#pragma unroll
    for (int qq = 0; qq < 8; ++qq) {
        const double v = mx8[qq * kSR + r];
        bad |= !(v == v);
        mx = fmax(mx, v);
    }
    int e = 0;
    if (mx > 0.0) frexp(mx, &e);  // mx < 2^e
    if (q == 0) rscale[row] = bad ? __longlong_as_double(0x7ff8000000000000ll) : ldexp(1.0, e);
    const int sh = 54 - e;
    uint32_t wd[4][kDig];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int s2 = 0; s2 < kDig; ++s2) wd[a][s2] = 0u;
    if (valid && !bad) {
#pragma unroll
        for (int j = 0; j < 16; ++j) digits7(ts[r * kSLd + q * 16 + j], sh, wd[j >> 2], j & 3);
    }
    uint8_t *base = reinterpret_cast<uint8_t *>(slices) + (row / kBM) * (int64_t)kPanelBytes;
    const int rp = (int)(row % kBM);
#pragma unroll
    for (int s2 = 0; s2 < kDig; ++s2)
        *reinterpret_cast<uint4 *>(base + s2 * kSliceA + canon_off(rp, q * 16)) =
            make_uint4(wd[0][s2], wd[1][s2], wd[2][s2], wd[3][s2]);
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
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
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
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
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
// 2-D tensor-map load (TMA) of a box at (x = row, y = column) into shared memory
CQ_DEVI void tma_load_2d(uint32_t dst, const CUtensorMap *map, int x, int y, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar)
        : "memory");
}
CQ_DEVI void tma_store_2d(const CUtensorMap *map, int x, int y, uint32_t src) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];\n" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(x), "r"(y), "r"(src)
                 : "memory");
}
CQ_DEVI void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
CQ_DEVI void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
CQ_DEVI void tc_commit(uint32_t bar) {  // by the MMA-issuing thread
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(bar)
                 : "memory");
}
// instruction descriptor: s32 accumulate, s8 x s8, both K-major, N columns, M = 128
__host__ __device__ constexpr uint32_t idesc_n(int n) {
    return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(kBM >> 4) << 24);
}

// Shared-memory matrix descriptor (no swizzle, K-major core matrices): low
// word = start address >> 4 | (LBO = 128) >> 4 << 16, high word = (SBO =
// 1024) >> 4 | version 1 << 14.
CQ_DEVI uint32_t desc_lo(uint32_t addr) { return ((addr >> 4) & 0x3FFFu) | ((128u >> 4) << 16); }
constexpr uint32_t kDescHi = (1024u >> 4) | (1u << 14);

// D[tmem] (+)= A[tmem] * B[smem]^T over the 4 K-steps (K = 128) of one digit
// pair, int8 x int8 -> int32, issued by the single elected thread of the MMA
// warp (its commits then track these MMAs). A's K-step is 8 TMEM columns;
// B's advances its start address by 256 bytes (+16 in descriptor units).
template <uint32_t kIdescT, bool kFirst>
CQ_DEVI void tc_mma_i8_k128(uint32_t dtmem, uint32_t atmem, uint32_t blo) {
    asm volatile(
        "{\n.reg .pred q0, q1;\n.reg .b64 db;\n.reg .b32 a1, b1;\n"
        "setp.ne.b32 q0, %3, 0;\n"
        "setp.eq.b32 q1, %3, %3;\n"
        "mov.b64 db, {%2, %4};\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], db, %5, q0;\n"
        "add.u32 a1, %1, 8;\nadd.u32 b1, %2, 16;\nmov.b64 db, {b1, %4};\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], [a1], db, %5, q1;\n"
        "add.u32 a1, %1, 16;\nadd.u32 b1, %2, 32;\nmov.b64 db, {b1, %4};\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], [a1], db, %5, q1;\n"
        "add.u32 a1, %1, 24;\nadd.u32 b1, %2, 48;\nmov.b64 db, {b1, %4};\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], [a1], db, %5, q1;\n}\n" ::"r"(dtmem),
        "r"(atmem), "r"(blo), "n"(kFirst ? 0 : 1), "n"(kDescHi), "n"(kIdescT)
        : "memory");
}
// one K-step (K = 32) of the same; accumulate = 0 overwrites D
template <uint32_t kIdescT>
CQ_DEVI void tc_mma_i8_k32(uint32_t dtmem, uint32_t atmem, uint32_t blo, uint32_t accumulate) {
    asm volatile(
        "{\n.reg .pred q0;\n.reg .b64 db;\n"
        "setp.ne.b32 q0, %3, 0;\n"
        "mov.b64 db, {%2, %4};\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], db, %5, q0;\n}\n" ::"r"(dtmem),
        "r"(atmem), "r"(blo), "r"(accumulate), "n"(kDescHi), "n"(kIdescT)
        : "memory");
}
// smem (128 rows x 32 bytes, canonical layout) -> TMEM (128 lanes x 8 columns)
CQ_DEVI void tc_cp_128x256b(uint32_t tmem_dst, uint32_t slo) {
    asm volatile(
        "{\n.reg .b64 sd;\n"
        "mov.b64 sd, {%1, %2};\n"
        "tcgen05.cp.cta_group::1.128x256b [%0], sd;\n}\n" ::"r"(tmem_dst),
        "r"(slo), "n"(kDescHi)
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
CQ_DEVI double lds_f64(uint32_t a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(a) : "memory");
    return v;
}
CQ_DEVI void sts_f64(uint32_t a, double v) { asm volatile("st.shared.f64 [%0], %1;\n" ::"r"(a), "d"(v) : "memory"); }
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

template <int kBStages, int kCStages>
__global__ void __launch_bounds__(kUpdThreads, 1)
    oz_update_kernel(const __grid_constant__ CUtensorMap tm_in, const __grid_constant__ CUtensorMap tm_out, UpdArgs P) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t sbase = smem_u32(smem);
    constexpr uint32_t kSmemC = kSmemB + kBStages * kTileBSmem;
    constexpr uint32_t kSmemBar = kSmemC + kCStages * kTileCBytes;
    const uint32_t sA = sbase + kSmemA, sB = sbase + kSmemB, sC = sbase + kSmemC;
    const uint32_t bar = sbase + kSmemBar;
    // a_*: digit-slice staging ring (smem -> TMEM); b_*: U-slice N tiles;
    // c_*: right-hand-side tiles; acc_full / acc_free: accumulator buffer
    // (tile parity) accumulated / read by its drain set
    auto a_full = [&](int s) { return bar + 8u * s; };
    auto a_empty = [&](int s) { return bar + 8u * (kAStages + s); };
    auto b_full = [&](int s) { return bar + 8u * (2 * kAStages + s); };
    auto b_empty = [&](int s) { return bar + 8u * (2 * kAStages + kBStages + s); };
    auto c_full = [&](int s) { return bar + 8u * (2 * kAStages + 2 * kBStages + s); };
    auto c_empty = [&](int s) { return bar + 8u * (2 * kAStages + 2 * kBStages + kCStages + s); };
    auto acc_full = [&](uint32_t s) { return bar + 8u * (2 * (kAStages + kBStages + kCStages) + s); };
    auto acc_free = [&](uint32_t s) { return bar + 8u * (2 * (kAStages + kBStages + kCStages) + kSets + s); };
    const uint32_t chunk_bar = bar + 8u * (2 * (kAStages + kBStages + kCStages) + 2 * kSets);  // two barriers
    static_assert(8 * (2 * (kAStages + kBStages + kCStages) + 2 * kSets + 2) <= 504, "barrier block");
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + kSmemBar + 504);

    if (tid == 0) {
        for (int s = 0; s < kAStages; ++s) {
            mb_init(a_full(s), 1);
            mb_init(a_empty(s), 1);
        }
        for (int s = 0; s < kBStages; ++s) {
            mb_init(b_full(s), 1);
            mb_init(b_empty(s), 1);
        }
        for (int s = 0; s < kCStages; ++s) {
            mb_init(c_full(s), 1);
            mb_init(c_empty(s), kEpiWarps);  // one store per drain warp
        }
        for (int s = 0; s < kSets; ++s) {
            mb_init(acc_full(s), 1);
            mb_init(acc_free(s), kEpiWarps);  // one arrival per drain warp of the set
        }
        mb_init(chunk_bar, 1);
        mb_init(chunk_bar + 8u, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    // the all-zero 8th slice of every staged U tile (the bulk copies write the first 7)
    for (int i = tid; i < kBStages * (kSliceB / 16); i += kUpdThreads) {
        const int st = i / (kSliceB / 16), o = i % (kSliceB / 16);
        *reinterpret_cast<uint4 *>(smem + kSmemB + st * kTileBSmem + kDig * kSliceB + o * 16) = make_uint4(0u, 0u, 0u, 0u);
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
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
        if (lane == 0) {  // ---------------- producer (TMA bulk copies)
            int as = 0, bs = 0, cs = 0;
            uint32_t afill = 0, bfill = 0, cfill = 0;
            for (int p = blockIdx.x; p < P.npanels; p += gridDim.x) {
                const int8_t *ga = P.aslc + (int64_t)p * kPanelBytes;
                for (int s = 0; s < kDig; ++s) {
                    if (afill) mb_wait(a_empty(as), (afill - 1u) & 1u);
                    mb_expect_tx(a_full(as), kSliceA);
                    bulk_g2s(sA + as * kSliceA, ga + s * kSliceA, kSliceA, a_full(as));
                    if (++as == kAStages) as = 0, ++afill;
                }
                const int64_t r0 = (int64_t)p * kBM;
                for (int nt = 0; nt < P.ntn; ++nt) {
                    if (bfill) mb_wait(b_empty(bs), (bfill - 1u) & 1u);
                    mb_expect_tx(b_full(bs), kTileBBytes);
                    bulk_g2s(sB + bs * kTileBSmem, P.bslc + (int64_t)nt * kTileBBytes, kTileBBytes, b_full(bs));
                    if (++bs == kBStages) bs = 0, ++bfill;
                    const int64_t j0 = (int64_t)nt * kBN;
                    if (cfill) mb_wait(c_empty(cs), (cfill - 1u) & 1u);
                    if (!P.cols_in) {  // 8 boxes of 32 rows x 8 columns, one per drain warp (zeros past the ends)
                        mb_expect_tx(c_full(cs), kTileCBytes);
                        for (int sb = 0; sb < 8; ++sb)
                            tma_load_2d(sC + cs * kTileCBytes + (uint32_t)sb * 2048u, &tm_in, (int)(r0 + (sb & 3) * 32),
                                        (int)(j0 + (sb >> 2) * kDC), c_full(cs));
                    } else {  // gathered columns: the drain warps read them from global memory
                        mb_arrive(c_full(cs));
                    }
                    if (++cs == kCStages) cs = 0, ++cfill;
                }
            }
        }
    } else if (warp == 1) {
        {  // ---------------- MMA issuer (whole warp waits; one elected thread issues)
            int as = 0, bs = 0;
            uint32_t ause = 0, buse = 0;
            uint32_t tc = 0;  // tiles issued
            uint32_t nchunk = 0;  // MMA chunks committed before this tile
            const uint32_t alo0 = desc_lo(sA);
            for (int p = blockIdx.x; p < P.npanels; p += gridDim.x) {
                // the panel's digit slices: smem -> TMEM columns [0, 224),
                // ordered after the previous panel's MMAs (same thread)
                for (int s = 0; s < kDig; ++s) {
                    mb_wait_warp(a_full(as), ause & 1u);
                    tc_fence_after();
                    if (elect_one()) {
#pragma unroll
                        for (int ks = 0; ks < kW / 32; ++ks)
                            tc_cp_128x256b(tmem + (uint32_t)(s * 32 + ks * 8),
                                           alo0 + (uint32_t)((as * kSliceA + ks * 256) >> 4));
                        tc_commit(a_empty(as));
                    }
                    __syncwarp();
                    if (++as == kAStages) as = 0, ++ause;
                }
                for (int nt = 0; nt < P.ntn; ++nt, ++tc) {
                    mb_wait_warp(b_full(bs), buse & 1u);
                    const uint32_t blo0 = desc_lo(sB + bs * kTileBSmem);
                    const uint32_t buf = tc & 1u;
                    const uint32_t d0 = tmem + kTmemAcc + buf * kAccCols;
                    // this buffer's previous tile (tc - 2) has been read by its drain set
                    if (tc >= 2) mb_wait_warp(acc_free(buf), ((tc >> 1) - 1u) & 1u);
                    tc_fence_after();
                    if (elect_one()) {
                        // Digit slice s of X against ALL its partner slices t = 0 ..
                        // min(6, 7 - s) of U in one MMA per K-step: U's slices are
                        // consecutive 16-row blocks of the canonical layout, so N =
                        // 16 (count) columns starting at group s land pair (s, t) in
                        // group s + t. Slice 0 runs over the zero 8th slice too: its
                        // first K-step overwrites all 8 groups, the rest accumulate.
                        // K-step-major chunks of 7 MMAs, each committed to a chunk
                        // barrier (chunk c uses barrier c % 2, whose previous arrival
                        // was chunk c - 2); at most two chunks are in flight, so the
                        // issuing thread sleeps on a barrier instead of sitting
                        // throttled on the tensor pipe, which starved the drain warps
                        // of its scheduler (lane quadrant 1) and delayed their release
                        // of the accumulator buffer by a whole tile's issue time
#pragma unroll
                        for (int ks = 0; ks < kW / 32; ++ks) {
                            const uint32_t cb = chunk_bar + 8u * ((nchunk + ks) & 1u);
                            if (nchunk + ks >= 2) mb_wait(cb, (((nchunk + ks) >> 1) - 1u) & 1u);
                            const uint32_t ao = tmem + 8u * ks, bo = blo0 + 16u * ks;
                            tc_mma_i8_k32<idesc_n(128)>(d0 + 0 * kBN, ao + 0 * 32, bo, ks ? 1u : 0u);
                            tc_mma_i8_k32<idesc_n(112)>(d0 + 1 * kBN, ao + 1 * 32, bo, 1u);
                            tc_mma_i8_k32<idesc_n(96)>(d0 + 2 * kBN, ao + 2 * 32, bo, 1u);
                            tc_mma_i8_k32<idesc_n(80)>(d0 + 3 * kBN, ao + 3 * 32, bo, 1u);
                            tc_mma_i8_k32<idesc_n(64)>(d0 + 4 * kBN, ao + 4 * 32, bo, 1u);
                            tc_mma_i8_k32<idesc_n(48)>(d0 + 5 * kBN, ao + 5 * 32, bo, 1u);
                            tc_mma_i8_k32<idesc_n(32)>(d0 + 6 * kBN, ao + 6 * 32, bo, 1u);
                            tc_commit(cb);
                        }
                        tc_commit(b_empty(bs));
                        tc_commit(acc_full(buf));
                    }
                    __syncwarp();
                    nchunk += kW / 32;
                    if (++bs == kBStages) bs = 0, ++buse;
                }
            }
        }
    } else {  // ---------------- drain warps: set (warp - 2) / 8 takes tiles set, set + 2, ...
              // (accumulator buffer = set); lane quadrant warp % 4, 8 columns each
        const int quad = warp & 3, half = ((warp - 2) >> 2) & 1, set = (warp - 2) >> 3;
        const int rloc = quad * 32 + lane;
        const uint32_t taddr0 =
            tmem + kTmemAcc + (uint32_t)set * kAccCols + ((uint32_t)(quad * 32) << 16) + (uint32_t)(half * kDC);
        // tiles of this CTA in issue order: panel blockIdx.x + pcur * gridDim.x, N tile nt
        // (the host bounds npanels * ntn / gridDim.x below 2^31)
        const int npan = P.npanels > (int)blockIdx.x ? (P.npanels - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
        const int ntiles = npan * P.ntn;
        int pi = -1;  // panel index (of this CTA) whose row scale is loaded
        double rs = 0.0;
        int64_t row = 0;
        bool valid = false;
        for (int tc = set; tc < ntiles; tc += kSets) {
            const int pcur = tc / P.ntn;
            const int nt = tc - pcur * P.ntn;
            const int64_t p = (int64_t)blockIdx.x + (int64_t)pcur * gridDim.x;
            if (pcur != pi) {
                pi = pcur;
                row = p * kBM + rloc;
                valid = row < P.m;
                rs = P.rscale[row];  // rscale covers the padded panel
            }
            const uint32_t par = (uint32_t)(tc / kSets) & 1u;
            const int cs = tc % kCStages;
            const uint32_t cpar = (uint32_t)(tc / kCStages) & 1u;
            const int64_t j0 = (int64_t)nt * kBN + half * kDC;
            const int64_t rem = P.ncols - j0;
            const int nc = rem >= kDC ? kDC : (rem > 0 ? (int)rem : 0);
            mb_wait(acc_full(set), par);
            tc_fence_after();
            // all 8 groups of this warp's 8 columns in one batch of TMEM loads,
            // then the buffer is released (the hand-off is the tile period's
            // critical path; the arithmetic comes after it)
            uint32_t v[kGroups][kDC];
#pragma unroll
            for (int g = 0; g < kGroups; ++g) tmem_ld8(taddr0 + (uint32_t)(g * kBN), v[g]);
            tmem_wait_ld();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mb_arrive(acc_free(set));
            // groups 0-3 -> hi (exact, |hi| < 2^50), groups 4-7 -> lo;
            // converted with the scales 2^-24 / 2^-56 folded into the magic
            // constants and added (one rounding)
            double hs[kDC];
#pragma unroll
            for (int c = 0; c < kDC; ++c) {
                const long long hi = (long long)(int)v[0][c] * 16777216ll + (long long)(int)v[1][c] * 65536ll +
                                     (long long)(int)v[2][c] * 256ll + (long long)(int)v[3][c];
                const long long lo = (long long)(int)v[4][c] * 16777216ll + (long long)(int)v[5][c] * 65536ll +
                                     (long long)(int)v[6][c] * 256ll + (long long)(int)v[7][c];
                hs[c] = (__longlong_as_double(hi + 0x41B8000000000000ll) - 402653184.0) +
                        (__longlong_as_double(lo + 0x3FB8000000000000ll) - 0.09375);
            }
            // out = T - prod 2^(e_i + f_j): T from the staged tile, the result
            // written back in place and stored by this warp's own TMA store
            // (the other set drains the next tile meanwhile)
            double wsc[kDC], t[kDC];
#pragma unroll
            for (int c = 0; c < kDC; ++c) wsc[c] = __ldg(P.cscale + j0 + c);  // padded to whole N tiles
            mb_wait(c_full(cs), cpar);
            // this warp's 32 x 8 box of the staged tile (column c at c * 256
            // bytes), shared-memory addresses explicitly; the gathered first
            // step reads its right-hand side from global memory instead
            const uint32_t ct = sC + cs * kTileCBytes + (uint32_t)((half * 4 + quad) * 2048 + lane * 8);
            if (!P.cols_in) {
#pragma unroll
                for (int c = 0; c < kDC; ++c) t[c] = lds_f64(ct + (uint32_t)(c * 256));
            } else {
#pragma unroll
                for (int c = 0; c < kDC; ++c)
                    t[c] = (valid && c < nc) ? P.cin[__ldg(P.cols_in + j0 + c) * P.ldin + row] : 0.0;
            }
#pragma unroll
            for (int c = 0; c < kDC; ++c) sts_f64(ct + (uint32_t)(c * 256), fma(-hs[c], wsc[c] * rs, t[c]));
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            __syncwarp();
            if (lane == 0) {
                // the stage gets this warp's release once the store has read its box
                tma_store_2d(&tm_out, (int)(p * kBM + quad * 32), (int)j0,
                             sC + cs * kTileCBytes + (uint32_t)((half * 4 + quad) * 2048));
                asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
                asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
                mb_arrive(c_empty(cs));
            }
            __syncwarp();
        }
    }
    if (warp >= 2 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(kTmemCols) : "memory");
    }
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link)
using EncodeTiledFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                   const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

// column-major m x n FP64 matrix, 128 x 32 boxes
int make_map(CUtensorMap *map, const double *base, int64_t m, int64_t n, int64_t ld, uint32_t box_cols = kBN) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return fail_internal("cuTensorMapEncodeTiled unavailable");
    const cuuint64_t dims[2] = {(cuuint64_t)m, (cuuint64_t)n};
    const cuuint64_t strides[1] = {(cuuint64_t)ld * 8u};
    const cuuint32_t box[2] = {32, box_cols};  // one epilogue warp's rows
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double *>(base), dims, strides, box, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail_internal("cuTensorMapEncodeTiled failed");
    return 0;
}

int launch_update(const UpdArgs &P, cudaStream_t st) {
    alignas(64) CUtensorMap tm_in, tm_out;
    std::memset(&tm_in, 0, sizeof(tm_in));
    if (!P.cols_in) CQ_TRY(make_map(&tm_in, P.cin, P.m, P.ncols, P.ldin, kDC));
    CQ_TRY(make_map(&tm_out, P.cout, P.m, P.ncols, P.ldout, kDC));  // 32 x 8 boxes
    const int grid = std::min(P.npanels, num_sms());
    if (((int64_t)P.npanels / grid + 1) * P.ntn > INT_MAX / 2) return fail_internal("oz update: too many tiles per CTA");
    const char *sv = getenv("CQRRPT_OZ_STAGES");  // experiments: ring depths "BC" (48 default, 38, 66)
    const int variant = sv ? atoi(sv) : 48;
#define OZ_LAUNCH(BST, CST)                                                                                          \
    do {                                                                                                             \
        auto kern = oz_update_kernel<BST, CST>;                                                                      \
        CQ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)upd_smem(BST, CST)),    \
                "oz update smem attr");                                                                              \
        kern<<<grid, kUpdThreads, upd_smem(BST, CST), st>>>(tm_in, tm_out, P);                                       \
    } while (0)
    switch (variant) {
        case 38: OZ_LAUNCH(3, 8); break;
        case 66: OZ_LAUNCH(6, 6); break;
        default: OZ_LAUNCH(4, 8); break;
    }
#undef OZ_LAUNCH
    note_launch();
    return check_launch("oz_update_kernel");
}

}  // namespace

// Engine choice for trsm_right: CQRRPT_GPU_TRSM=oz | dmma forces one; by
// default the INT8 engine from m >= 131072 rows and k >= 768 columns, where it
// measured faster than the DMMA engine (tools/oz_probe.py, one B200: 131072 x
// 1024 4.37 vs 4.53 ms, 524288 x 768 9.89 vs 10.10, 262144 x 2048 26.3 vs
// 33.4, 2097152 x 1024 63.4 vs 68.0, 1048576 x 2048 107 vs 131); at k = 512
// it was slower (1048576 x 512: 10.3 vs 9.5 ms).
bool trsm_use_ozaki(int64_t m, int64_t k) {
    const char *env = getenv("CQRRPT_GPU_TRSM");
    if (env && env[0] == 'd') return false;
    if (env && env[0] == 'o') return k > 0 && m > 0;
    return m >= 131072 && k >= 768;
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
                              dinv + ((b0 + c0) / NB) * NB * NB, x + b0 * ldx, ldx, st, /*pdl=*/c0 > 0 && !block_ev && !sink));
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
        oz_slice_rows_kernel<<<(unsigned)(npanels * (kBM / kSR)), 256, 0, st>>>(m, (int)w, x + b0 * ldx, ldx, aslc,
                                                                              rexp);
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

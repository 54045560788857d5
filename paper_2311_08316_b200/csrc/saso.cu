// SASO sketch on device: plan (K1), per-tile CSR, apply (K2), partial reduce.
//
// Reference: sample_sketch SASO branch (sketch.cc:73-99) and apply
// (sketch.cc:131-146). The plan is generated from the same counter RNG
// streams (rng.hh:18-53, stream mix_seed(seed, 0x7361736f + c) for GLOBAL
// column c of S), so S is bit-identical to the reference's for the same seed.
//
// Data layout in HBM
//   plan   uint32[m_local * nnz]      row | sign<<31 (sign 1 = +1/sqrt(d))
//   tinfo  uint2[ntiles * nbs]        per 256-row tile, 32 slots per CTA row block
//                                     (slot w < 28: consumer warp w's A rows):
//                                     (first entry index, mask of its rows that
//                                     have entries in the tile)
//   tent   uint32[ntiles * entw]      per tile, entries sorted by (row, c):
//                                     byte offset of A(c_local, 0) in the staged
//                                     tile (c * 264) << 15 | last-of-row << 8 |
//                                     negative (-1/sqrt(d)) << 0
//   part   double[S][d][n]            per c-split partial sketches, row-major
//   Msk    double d x n column-major  fixed-order sum of the partials
//
// Apply kernel: one CTA = 32 columns (lane = column) x 28*A sketch rows x a
// contiguous range of 256-row tiles. Warps 0..27 own A sketch rows each (A
// register accumulators per lane); warps 28..31 (one per SM sub-partition)
// only stage: each 256 x 32 tile of A ([c][33] padded: conflict-free 8-byte
// cp.async writes of a 256-byte column run, conflict-free warp reads of a
// 256-byte row), the tile's entry list and the CTA's 32 block words go through
// a ring of up to 3 stages driven by mbarriers ("full": cp.async arrivals of
// the producer lanes; "empty": one arrival per consumer warp). Consumers never
// wait for each other, only for data, so the per-tile imbalance of their entry
// counts (Poisson per warp and tile) averages out over the ring.
//
// Entry word: byte offset of A(c, 0) in the staged tile << 15 | last-of-row
// << 8 | negative. Per entry a consumer issues LDS (next word, broadcast),
// LEA.HI (x address), LDS.64 x, IMAD (adds sign * 2^31 to x's hi word: x -> -x
// exactly), DFMA with the constant 1/sqrt(d), flag test + branch; the loop is
// unrolled by two so no word rotates between registers. Rows with no entry in
// the tile cost one test of a warp-uniform mask (REDUX). acc = fma(+-v, A(c,
// j), acc) per entry in c order is the reference's own FMA chain per output
// entry (sketch.cc:137-143), so one c-split is bit-identical.
//
// Bound: per entry two shared-memory wavefronts for x (256 B row read) and
// one for the word; per tile 528 for the staging writes, repeated by every
// row block. The x reads alone are 8 bytes of shared-memory traffic per FMA,
// nnz = 8 times the HBM bytes of A, against ~5.5x more shared-memory than HBM
// bandwidth: this kernel cannot reach the HBM roofline whatever its issue
// efficiency.
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "internal.hh"

namespace cqg {

constexpr int kTileRows = 256;  // rows of A per tile (one entry list per tile)
constexpr int kApplyWarps = 32;  // 1024 threads: 8 warps per scheduler hide the shared-memory latency of each entry
constexpr int kApplyThreads = kApplyWarps * 32;
constexpr int kProducers = 4;  // warps 28..31 (one per SM sub-partition) stage the tiles
constexpr int kConsumers = kApplyWarps - kProducers;  // warps 0..27 own sketch rows
constexpr int kXLD = 33;        // staged tile row stride (doubles)
constexpr uint32_t kEntLast = 0x100u;  // entry flag: last entry of its row in the tile
constexpr uint64_t kSasoSalt = 0x7361736fULL;  // sketch.cc:19

// ---------------------------------------------------------------------------
// K1: plan. One thread per column c of S (= row c of the local A shard).
// ---------------------------------------------------------------------------
__global__ void saso_plan_kernel(int64_t d, int64_t c0, int64_t count, int nnz, uint64_t seed,
                                 uint32_t *__restrict__ plan) {
    int64_t cc = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (cc >= count) return;
    const uint64_t cs = mix_seed(seed, kSasoSalt + (uint64_t)(c0 + cc));  // sketch.cc:81
    uint64_t ctr = 0;
    uint32_t *out = plan + cc * nnz;
    uint32_t local[16];
    for (int t = 0; t < nnz; ++t) {
        uint32_t r;
        bool fresh;
        do {  // rejection until distinct, sketch.cc:88-93
            r = (uint32_t)rng_below(cs, ctr++, (uint64_t)d);
            fresh = true;
            for (int u = 0; u < t; ++u) {
                uint32_t prev = (u < 16) ? local[u] : (out[u] & 0x7fffffffu);
                if (prev == r) {
                    fresh = false;
                    break;
                }
            }
        } while (!fresh);
        uint32_t sign = (uint32_t)(rng_bits(cs, ctr++) & 1ULL);  // sketch.cc:95
        if (t < 16) local[t] = r;
        out[t] = r | (sign << 31);
    }
}

// ---------------------------------------------------------------------------
// Per-tile entry lists by sketch row (stable: c ascending within a row) and
// the per-block words. One CTA per tile; histogram + scan by the block,
// ordered scatter by warp 0.
// ---------------------------------------------------------------------------
// xrow: bytes between consecutive rows c of one column in the staged tile
// (264 for the padded row-major LDGSTS layout, 8 for the column segments the
// bulk copies write)
// S: row slots per consumer warp (32 / W lanes-per-row groups of W columns)
__global__ void __launch_bounds__(256) saso_tile_csr_kernel(int64_t m, int64_t d, int nnz, int A, int S, int nbs, int entw,
                                                            uint32_t xrow, const uint32_t *__restrict__ plan,
                                                            uint2 *__restrict__ tinfo, uint32_t *__restrict__ tent) {
    extern __shared__ int32_t s_beg[];  // d + 1 counters -> row begins (s_beg[d] = entries)
    int32_t *s_cur = s_beg + (d + 1);   // d scatter cursors
    __shared__ int32_t s_part[256 / 32 + 1];
    const int64_t tile = blockIdx.x;
    const int64_t row0 = tile * kTileRows;
    const int rows = (int)cmin<int64_t>(kTileRows, m - row0);
    const int nent = rows * nnz;
    const uint32_t *tp = plan + row0 * nnz;

    for (int64_t r = threadIdx.x; r <= d; r += blockDim.x) s_beg[r] = 0;
    __syncthreads();
    for (int e = threadIdx.x; e < nent; e += blockDim.x) atomicAdd(&s_beg[tp[e] & 0x7fffffffu], 1);
    __syncthreads();
    // exclusive scan over d counters: each thread scans a contiguous chunk
    const int64_t per = (d + blockDim.x - 1) / blockDim.x;
    const int64_t lo = threadIdx.x * per, hi = cmin<int64_t>(lo + per, d);
    int32_t run = 0;
    for (int64_t r = lo; r < hi; ++r) run += s_beg[r];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int32_t incl = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) s_part[wid] = incl;
    __syncthreads();
    if (threadIdx.x == 0) {
        int32_t acc = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            int32_t t = s_part[w];
            s_part[w] = acc;
            acc += t;
        }
    }
    __syncthreads();
    int32_t base = s_part[wid] + incl - run;
    for (int64_t r = lo; r < hi; ++r) {
        const int32_t c = s_beg[r];
        s_beg[r] = base;
        s_cur[r] = base;
        base += c;
    }
    if (threadIdx.x == 0) s_beg[d] = nent;
    __syncthreads();
    // block words: (first entry, rows of the block that have entries)
    uint2 *oinfo = tinfo + tile * (int64_t)nbs;
    for (int sl = threadIdx.x; sl < nbs; sl += blockDim.x) {  // slot = (CTA row block * 32 + warp) * S + sub-slot
        const int h = sl % S, w = (sl / S) % kApplyWarps;
        const int64_t rb = (((int64_t)(sl / (S * kApplyWarps)) * kConsumers + w) * S + h) * A;
        uint2 word = make_uint2((uint32_t)nent, 0u);
        if (w < kConsumers && rb < d) {
            uint32_t mask = 0;
            for (int q = 0; q < A && rb + q < d; ++q)
                if (s_beg[rb + q + 1] > s_beg[rb + q]) mask |= 1u << q;
            word = make_uint2((uint32_t)s_beg[rb], mask);
        }
        oinfo[sl] = word;
    }
    uint32_t *oent = tent + tile * (int64_t)entw;
    for (int e = nent + threadIdx.x; e < entw; e += blockDim.x) oent[e] = 0;  // prefetch overrun pad
    // ordered scatter: entry e = c_local*nnz + t, processed in ascending e
    if (wid == 0) {
        const unsigned lt = (1u << lane) - 1u;
        for (int b = 0; b < nent; b += 32) {
            int e = b + lane;
            bool valid = e < nent;
            uint32_t w = valid ? tp[e] : 0xffffffffu;
            uint32_t r = w & 0x7fffffffu;
            unsigned act = __ballot_sync(0xffffffffu, valid);
            unsigned grp = __match_any_sync(0xffffffffu, valid ? r : 0xffffffffu);
            int rank = __popc(grp & lt);
            int pos = valid ? s_cur[r] + rank : 0;
            __syncwarp();
            if (valid) {
                const uint32_t c_local = (uint32_t)(e / nnz);
                const uint32_t neg = (~w >> 31) & 1u;  // plan bit 31 clear: -1/sqrt(d)
                const uint32_t last = (pos == s_beg[r + 1] - 1) ? kEntLast : 0u;
                oent[pos] = ((c_local * xrow) << 15) | last | neg;
                // highest-ranked member advances the cursor
                if (rank == __popc(grp & act) - 1) s_cur[r] += __popc(grp & act);
            }
            __syncwarp();
        }
    }
}

// ---------------------------------------------------------------------------
// mbarrier helpers (CTA scope)
// ---------------------------------------------------------------------------
CQ_DEVI void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}
CQ_DEVI void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
// arrives when every cp.async this thread issued before it has landed
CQ_DEVI void cp_async_mbar_arrive(uint32_t bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(bar) : "memory");
}
// blocking wait: the suspend-time hint lets the thread sleep until the phase
// completes instead of spinning on issue slots
CQ_DEVI void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "MBAR_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 1000000;\n"
        "@!p bra MBAR_WAIT_%=;\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
CQ_DEVI void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
// 1-D bulk copy global -> shared (TMA engine), completion counted on `bar`
CQ_DEVI void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
CQ_DEVI void sts_f64(uint32_t a, double v) { asm volatile("st.shared.f64 [%0], %1;\n" ::"r"(a), "d"(v) : "memory"); }
CQ_DEVI uint32_t lds_u32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];\n" : "=r"(v) : "r"(a) : "memory");
    return v;
}
CQ_DEVI uint2 lds_u32x2(uint32_t a) {
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];\n" : "=r"(v.x), "=r"(v.y) : "r"(a) : "memory");
    return v;
}
CQ_DEVI double lds_f64(uint32_t a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(a) : "memory");
    return v;
}
CQ_DEVI void cp_async8_s(uint32_t s, const void *gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
}

// ---------------------------------------------------------------------------
// K2: apply (see the header). Writes part[split][r][j] (row-major).
// ---------------------------------------------------------------------------
struct ApplyArgs {
    int64_t m, n, lda, d;
    const double *a;
    double val;
    int nnz;
    int entw;    // 32-bit entry words per tile (16-byte multiple, >= kTileRows*nnz + 2)
    int nbs;     // block words per tile (whole CTAs of kApplyWarps)
    int stages;  // ring depth (2..4, as many as fit)
    int64_t ntiles, tiles_per_split;
    int64_t tile_lo, tile_hi;  // tile_hi > 0: this launch takes tiles [tile_lo, tile_hi) (one split)
    int carry;                 // start the chains from part (a previous launch's tiles)
    const uint2 *tinfo;
    const uint32_t *tent;
    double *part;
};

constexpr uint32_t kColB = kTileRows * 8 + 16;          // 2064: one column segment + 16-byte pad (bulk staging)
constexpr uint32_t kTileBytesT = 32 * kColB;            // 66048
// LDGSTS staging: [c][W + 1] padded rows (W = 32: 67584 bytes); one (start,
// mask) word pair per warp and row slot
__host__ __device__ constexpr uint32_t tile_bytes(int W) { return kTileRows * (uint32_t)(W + 1) * 8u; }
__host__ __device__ constexpr uint32_t info_bytes(int W) { return kApplyWarps * (uint32_t)(32 / W) * 8u; }

// TMA = true: one producer thread stages each tile as 32 column segments with
// cp.async.bulk (the TMA engine writes shared memory; no LDGSTS issue slots),
// completion counted on the stage's mbarrier; x of (c, column lane) sits at
// lane * 2064 + 8 c (16-byte aligned segments: a 4-way bank conflict on the
// x reads instead of the padded layout's none, for staging that no longer
// costs 8 cycles per 256-byte warp operation). Needs A 16-byte aligned, lda
// even. TMA = false: the four producer warps' 8-byte LDGSTS into [c][33].
//
// W < 32 (narrow n: too few 32-column groups to fill the GPU, and each CTA's
// staging of its whole column group is the bound): a CTA takes W columns, and
// a consumer warp S = 32 / W row slots at once -- lanes [h W, (h + 1) W) walk
// the entry lists of the A rows of slot h over the same W columns. The slots
// of a warp diverge (different list lengths); every chain is still the
// reference's, so the result is bit-identical. LDGSTS staging only.
template <int A, bool TMA, int W>
__global__ void __launch_bounds__(kApplyThreads, 1) saso_apply_kernel(ApplyArgs P) {
    static_assert(!TMA || W == 32, "bulk staging takes whole 32-column groups");
    constexpr int SL = 32 / W;  // row slots per consumer warp
    constexpr int RB = kConsumers * SL * A;
    constexpr uint32_t kInfoBytes = info_bytes(W);
    constexpr uint32_t kXLDB = (uint32_t)(W + 1) * 8u;  // staged row stride in bytes
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    // grid (row blocks, column groups): the row blocks of one column group
    // are adjacent in launch order, so they are co-resident and march through
    // the same tiles together -- A is read from HBM once, the other row
    // blocks' copies hit L2
    const int64_t j0 = (int64_t)blockIdx.y * W;
    const int64_t r0 = (int64_t)blockIdx.x * RB;
    const int64_t split = blockIdx.z;
    const int64_t t_begin = P.tile_hi ? P.tile_lo : split * P.tiles_per_split;
    const int64_t t_end = P.tile_hi ? P.tile_hi : cmin<int64_t>(t_begin + P.tiles_per_split, P.ntiles);
    const int rows_here = (int)cmin<int64_t>(RB, P.d - r0);  // valid sketch rows in this block
    const int S = P.stages;

    // shared layout: S tiles | S entry lists | S info blocks | S full + S empty mbarriers
    constexpr uint32_t TB = TMA ? kTileBytesT : tile_bytes(W);
    const uint32_t s_tiles = smem_u32(smem_raw);
    const uint32_t ent_bytes = (uint32_t)P.entw * 4u;
    const uint32_t s_ents = s_tiles + (uint32_t)S * TB;
    const uint32_t s_info = s_ents + (uint32_t)S * ent_bytes;
    const uint32_t s_full = s_info + (uint32_t)S * kInfoBytes;
    const uint32_t s_empty = s_full + (uint32_t)S * 8u;
    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(s_full + 8u * s, TMA ? 1 : 32 * kProducers);  // TMA: one arrive.expect_tx
            mbar_init(s_empty + 8u * s, kConsumers);  // one arrival per consumer warp
        }
    }
    if (TMA && tid == 0) asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    __syncthreads();
    const int64_t ntl = t_end - t_begin;

    if (TMA && wid >= kConsumers) {
        if (wid != kConsumers || lane != 0) return;
        const int ncols = (int)cmin<int64_t>(32, P.n - j0);
        const uint32_t *g_ent = P.tent + t_begin * (int64_t)P.entw;
        const uint2 *g_info = P.tinfo + t_begin * P.nbs + (int64_t)blockIdx.x * (kApplyWarps * SL);
        int stg = 0;
        uint32_t use = 0;
        for (int64_t i = 0; i < ntl; ++i) {
            const int64_t t = t_begin + i;
            if (use) mbar_wait(s_empty + 8u * stg, (use - 1u) & 1u);
            const uint32_t sb = s_tiles + (uint32_t)stg * TB;
            const int rows = (int)cmin<int64_t>(kTileRows, P.m - t * kTileRows);
            const uint32_t cb = (uint32_t)(rows & ~1) * 8u;  // bulk part (16-byte multiple)
            const double *a0 = P.a + j0 * P.lda + t * kTileRows;
            if (rows & 1)  // odd tail row of a ragged last tile: plain loads, ordered by the arrive
                for (int jj = 0; jj < ncols; ++jj)
                    sts_f64(sb + (uint32_t)jj * kColB + (uint32_t)(rows - 1) * 8u, a0[jj * P.lda + rows - 1]);
            const uint32_t full = s_full + 8u * stg;
            mbar_arrive_expect_tx(full, (uint32_t)ncols * cb + ent_bytes + kInfoBytes);
            if (cb)
                for (int jj = 0; jj < ncols; ++jj) bulk_g2s(sb + (uint32_t)jj * kColB, a0 + jj * P.lda, cb, full);
            bulk_g2s(s_ents + (uint32_t)stg * ent_bytes, g_ent, ent_bytes, full);
            bulk_g2s(s_info + (uint32_t)stg * kInfoBytes, g_info, kInfoBytes, full);
            g_ent += P.entw;
            g_info += P.nbs;
            if (++stg == S) stg = 0, ++use;
        }
        return;
    }
    if (!TMA && wid >= kConsumers) {
        // ---------------- producer warps: stage tile after tile, up to S ahead.
        // Producer p copies columns p, p+4, ..., lane l rows l + 32k (k = 0..7):
        // 256-byte coalesced runs, immediate offsets, one pointer step per column
        const int pw = wid - kConsumers;
        const int ncols = (int)cmin<int64_t>(W, P.n - j0);
        const int64_t lda4 = kProducers * P.lda;
        const int nent16 = P.entw / 4;
        const double *a_tile = P.a + (j0 + pw) * P.lda + t_begin * kTileRows + lane;
        const uint32_t *g_ent = P.tent + t_begin * (int64_t)P.entw;
        const uint32_t *g_info =
            reinterpret_cast<const uint32_t *>(P.tinfo + t_begin * P.nbs + (int64_t)blockIdx.x * (kApplyWarps * SL));
        const int64_t full_tiles = P.m / kTileRows;  // tiles without rows past m
        const int pl = pw * 32 + lane;                // producer lane 0..127
        int stg = 0;
        uint32_t use = 0;
        for (int64_t i = 0; i < ntl; ++i) {
            if (use) mbar_wait(s_empty + 8u * stg, (use - 1u) & 1u);  // consumers done with the stage's last tile
            const uint32_t sb = s_tiles + (uint32_t)stg * TB + (uint32_t)lane * kXLDB;
            const double *pa = a_tile;
            if (t_begin + i < full_tiles) {
                for (int j = pw; j < ncols; j += kProducers) {
#pragma unroll
                    for (int k = 0; k < kTileRows / 32; ++k)
                        cp_async8_s(sb + 8u * (uint32_t)j + (uint32_t)k * (32u * kXLDB), pa + 32 * k);
                    pa += lda4;
                }
            } else {  // the ragged last tile
                const int64_t rem = P.m - (t_begin + i) * kTileRows;
                for (int j = pw; j < ncols; j += kProducers) {
#pragma unroll
                    for (int k = 0; k < kTileRows / 32; ++k)
                        if (lane + 32 * k < rem)
                            cp_async8_s(sb + 8u * (uint32_t)j + (uint32_t)k * (32u * kXLDB), pa + 32 * k);
                    pa += lda4;
                }
            }
            if (pl < (int)(kInfoBytes / 16)) cp_async16_s(s_info + (uint32_t)stg * kInfoBytes + 16u * pl, g_info + 4 * pl);
            const uint32_t se = s_ents + (uint32_t)stg * ent_bytes;
            for (int w = pl; w < nent16; w += 32 * kProducers) cp_async16_s(se + 16u * (uint32_t)w, g_ent + 4 * w);
            cp_async_mbar_arrive(s_full + 8u * stg);
            a_tile += kTileRows;
            g_ent += P.entw;
            g_info += 2 * P.nbs;
            if (++stg == S) stg = 0, ++use;
        }
        return;
    }

    // ---------------- consumer warps
    const int slot = wid * SL + lane / W, cl = lane % W;  // row slot of the CTA, column of the group
    const int wr0 = slot * A;
    const int64_t col = j0 + cl;
    double acc[A];
#pragma unroll
    for (int q = 0; q < A; ++q) acc[q] = 0.0;
    if (P.carry && col < P.n) {  // carried chains continue bit for bit (one split)
        const double *pp = P.part + (r0 + wr0) * P.n + col;
#pragma unroll
        for (int q = 0; q < A; ++q)
            if (wr0 + q < rows_here) acc[q] = pp[(int64_t)q * P.n];
    }
    int stg = 0;
    uint32_t use = 0;  // how many times this stage has been filled before the current tile
    const double v = P.val;
    const uint32_t lane_x = s_tiles + (TMA ? kColB : 8u) * (uint32_t)cl;
    // x with the entry's sign applied: bit 0 of the entry is 1 for -1/sqrt(d);
    // adding cur * 2^31 flips bit 63 of x exactly when it is set, and
    // fma(v, -x, s) == fma(-v, x, s) bit for bit
    auto signed_x = [](double x, uint32_t cur) {
        return __hiloint2double((int)((uint32_t)__double2hiint(x) + cur * 0x80000000u), __double2loint(x));
    };
    for (int64_t i = 0; i < ntl; ++i) {
        mbar_wait(s_full + 8u * stg, use & 1u);
        const uint2 info = lds_u32x2(s_info + (uint32_t)stg * kInfoBytes + 8u * (uint32_t)slot);
        // one slot per warp: warp-uniform; several: the slots of a warp diverge
        const uint32_t mask = SL == 1 ? __reduce_or_sync(0xffffffffu, info.y) : info.y;
        if (mask) {
            // The warp's entries: rows ascending, c ascending within a row,
            // the last entry of each row flagged. The loop is unrolled by two
            // (cur / nxt swap roles) so no word rotates between registers.
            uint32_t pe = s_ents + (uint32_t)stg * ent_bytes + 4u * info.x;
            const uint32_t xb = lane_x + (uint32_t)stg * TB;
            uint32_t cur = lds_u32(pe);
            pe += 4u;
#pragma unroll
            for (int q = 0; q < A; ++q) {  // row wr0+q: its entries in c order (sketch.cc:137-143)
                if (mask & (1u << q)) {
                    double sq = acc[q];
                    for (;;) {
                        const uint32_t nxt = lds_u32(pe);  // may be past the list: zero pad, in bounds
                        sq = fma(v, signed_x(lds_f64(xb + (cur >> 15)), cur), sq);  // sketch.cc:142
                        if (cur & kEntLast) {
                            cur = nxt;
                            pe += 4u;
                            break;
                        }
                        cur = lds_u32(pe + 4u);
                        pe += 8u;
                        sq = fma(v, signed_x(lds_f64(xb + (nxt >> 15)), nxt), sq);
                        if (nxt & kEntLast) break;
                    }
                    acc[q] = sq;
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(s_empty + 8u * stg);
        if (++stg == S) stg = 0, ++use;
    }
    // write the partial: part[split][r][j]
    if (col < P.n) {
        double *pp = P.part + split * P.d * P.n;
#pragma unroll
        for (int q = 0; q < A; ++q)
            if (wr0 + q < rows_here) pp[(r0 + wr0 + q) * P.n + col] = acc[q];
    }
}

// Msk(r, j) = sum_s part[s][r][j] in split order; 32x32 transposing tiles.
__global__ void saso_reduce_kernel(int64_t d, int64_t n, int64_t nsplit, const double *__restrict__ part,
                                   double *__restrict__ msk, int64_t ldm) {
    __shared__ double t[32][33];
    const int64_t rb = (int64_t)blockIdx.y * 32, jb = (int64_t)blockIdx.x * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
    for (int yy = ty; yy < 32; yy += 8) {
        int64_t r = rb + yy, j = jb + tx;
        double s = 0.0;
        if (r < d && j < n)
            for (int64_t k = 0; k < nsplit; ++k) s += part[k * d * n + r * n + j];
        t[yy][tx] = s;
    }
    __syncthreads();
    for (int yy = ty; yy < 32; yy += 8) {
        int64_t j = jb + yy, r = rb + tx;
        if (r < d && j < n) msk[j * ldm + r] = t[tx][yy];
    }
}

// ---------------------------------------------------------------------------
// host wrappers
// ---------------------------------------------------------------------------
int saso_plan(int64_t d, int64_t c0, int64_t count, int64_t nnz, uint64_t seed, uint32_t *plan,
              cudaStream_t st) {
    if (count <= 0) return 0;
    const int threads = 256;
    saso_plan_kernel<<<(unsigned)((count + threads - 1) / threads), threads, 0, st>>>(d, c0, count, (int)nnz,
                                                                                       seed, plan);
    note_launch();
    return check_launch("saso_plan_kernel");
}

static size_t apply_smem(int nnz, int *entw, int *nbs, int *stages, int64_t d, int A, bool tma, int W) {
    const int S = 32 / W;                    // row slots per consumer warp
    *entw = (kTileRows * nnz + 2 + 3) & ~3;  // u32 entries + two prefetch overrun words, 16-byte multiple
    const int64_t nb = (d + (int64_t)A * S - 1) / ((int64_t)A * S);  // consumer warps needed, kConsumers per CTA
    *nbs = (int)(((nb + kConsumers - 1) / kConsumers) * kApplyWarps * S);  // 32 S slots per CTA row block
    const size_t per = (tma ? kTileBytesT : tile_bytes(W)) + 4 * (size_t)*entw + info_bytes(W) + 16;
    *stages = (int)std::min<size_t>(6, (227 * 1024) / per);
    return per * (size_t)*stages;
}

template <int A, bool TMA, int W = 32>
static int launch_apply(ApplyArgs P, dim3 grid, size_t smem, cudaStream_t st) {
    auto kern = saso_apply_kernel<A, TMA, W>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return fail_cuda("saso_apply smem attr");
    kern<<<grid, kApplyThreads, smem, st>>>(P);
    note_launch();
    return check_launch("saso_apply_kernel");
}

int saso_sketch(int64_t m, int64_t n, const double *a, int64_t lda, int64_t d, int64_t nnz, uint64_t seed,
                int64_t c0, double *msk, int64_t ldm, Workspace &ws, cudaStream_t st, bool allow_split,
                const InputChunks *chunks) {
    const bool follow = chunks && chunks->count > 1 && !allow_split;
    if (chunks && !follow)
        for (int c = 0; c < chunks->count; ++c)
            if (cudaStreamWaitEvent(st, chunks->ev[c], 0) != cudaSuccess) return fail_cuda("sketch wait input");
    if (m <= 0 || n <= 0) {
        // empty shard contributes zeros
        for (int64_t j = 0; j < n; ++j)
            if (cudaMemsetAsync(msk + j * ldm, 0, sizeof(double) * d, st) != cudaSuccess) return fail_cuda("memset");
        return 0;
    }
    if (d > 32767 || nnz * kTileRows > 65535) return fail_internal("saso_sketch: d or nnz too large for the CSR");
    const int64_t ntiles = (m + kTileRows - 1) / kTileRows;
    uint32_t *plan = ws.get<uint32_t>("saso.plan", (size_t)(m * nnz));
    if (!plan) return fail_nomem("saso workspace");
    int rc = saso_plan(d, c0, m, nnz, seed, plan, st);
    if (rc) return rc;
    // Decomposition: RB = 28*A sketch rows per CTA (A register accumulators
    // per lane of each of the 28 consumer warps). Exact order needs one pass over all
    // tiles per CTA, so parallelism comes from row blocks. Cost per 256-row
    // tile and CTA (cycles) is the larger of the shared-memory wavefronts (528
    // for the tile writes, three per entry: word + x, the entry list) and the
    // issue slots (per consumer warp ~30 per tile and ~5 per row, ~7.5 per
    // entry, ~500 for the producer warps, over 4 schedulers); minimise
    // waves * that.
    const int sms = num_sms();
    // Narrow n (at most 512 columns: fewer than 16 column groups of 32, each
    // CTA's LDGSTS staging of its whole column group is the bound, 8 cycles
    // per 256-byte warp copy = 64 W cycles per tile): W = 16 or 8 columns per
    // CTA, a consumer warp walks 32 / W row slots at once (divergent, its
    // iterations ~ the longest of the slots' Poisson entry lists).
    int A = 12, W = 32;
    if (!allow_split) {
        const int candA[] = {16, 12, 8, 6, 4, 2, 1};
        const int candW[] = {32, 16, 8};
        const double lam = (double)kTileRows * (double)nnz / (double)d;  // entries per sketch row and tile
        double best = 1e300;
        for (int w : candW) {
            if (w < 32 && n > 512) continue;
            const int S = 32 / w;
            const double spread = S == 1 ? 0.0 : (S == 2 ? 0.56 : 1.03);  // E[max of S] - mean, in sigmas
            for (int a : candA) {
                if (w < 32 && a == 6) continue;  // not instantiated
                const int64_t rb = (int64_t)kConsumers * S * a;
                const int64_t ctas = ((n + w - 1) / w) * ((d + rb - 1) / rb);
                const double ents = (double)kTileRows * (double)nnz * (double)std::min<int64_t>(rb, d) / (double)d;
                // warp iterations of the CTA per tile: one entry each (S = 1) or one entry per slot
                const double iters =
                    S == 1 ? ents : (double)std::min<int64_t>(rb, d) / S * (lam + spread * std::sqrt(lam));
                const double smem_c = 16.5 * w + 3.0 * iters + (double)kTileRows * (double)nnz / 32.0;
                const double issue_c = (kConsumers * (30.0 + 5.0 * a) + 7.5 * iters + 500.0 * w / 32.0) / 4.0;
                const double stage_c = n <= 512 ? 64.0 * w : 0.0;  // LDGSTS issue (wide n: the choice of A is unchanged)
                const double cost = (double)((ctas + sms - 1) / sms) * std::max(std::max(smem_c, issue_c), stage_c);
                if (cost < best * 0.999) {
                    best = cost;
                    A = a;
                    W = w;
                }
            }
        }
    }
    if (const char *ev = getenv("CQRRPT_SASO_A")) {  // experiments: force the row-block width
        const int fa = atoi(ev);
        if (fa == 1 || fa == 2 || fa == 4 || fa == 6 || fa == 8 || fa == 12 || fa == 16) A = fa;
    }
    if (const char *ev = getenv("CQRRPT_SASO_W")) {  // experiments / tests: force the column-group width
        const int fw = atoi(ev);
        if (fw == 8 || fw == 16 || fw == 32) W = fw;
    }
    if (W < 32 && A == 6) A = 4;  // not instantiated
    const int SL = 32 / W;
    const int64_t cgroups = (n + W - 1) / W;
    const int64_t rblocks = (d + (int64_t)kConsumers * SL * A - 1) / ((int64_t)kConsumers * SL * A);
    // Tile staging: bulk copies (TMA engine: no LDGSTS issue slots, but x
    // reads from 16-byte aligned column segments take 4 instead of 2
    // wavefronts) when A's segments are 16-byte aligned and few row blocks
    // share each tile; else the four producer warps' 8-byte LDGSTS into the
    // padded rows. Measured (tools/sketch_sweep.sh): bulk copies win up to 6
    // row blocks (C2 1.04 -> 0.89 ms, C5-1024 33.1 -> 26.6 ms at 4; C3 5.13 ->
    // 4.94 ms, C5-2048 84.0 -> 77.7 ms at 6 with A = 16) and lose at 12 (C4
    // 55.2 -> 65.8 ms, C5-256 19.7 -> 22.2 ms). CQRRPT_SASO_LDGSTS=1 /
    // CQRRPT_SASO_TMA=1 force either path.
    const bool tma = W == 32 && (reinterpret_cast<uintptr_t>(a) & 15) == 0 && (lda & 1) == 0 &&
                     (rblocks <= 6 || getenv("CQRRPT_SASO_TMA") != nullptr) && getenv("CQRRPT_SASO_LDGSTS") == nullptr;
    int entw = 0, nbs = 0, stages = 0;
    const size_t smem = apply_smem((int)nnz, &entw, &nbs, &stages, d, A, tma, W);
    if (stages < 2) return fail_internal("saso_apply: nnz too large for the staged entry lists");
    uint2 *tinfo = ws.get<uint2>("saso.tinfo", (size_t)(ntiles * nbs) + 32);
    uint32_t *tent = ws.get<uint32_t>("saso.tent", (size_t)(ntiles * entw) + 4);
    if (!tinfo || !tent) return fail_nomem("saso workspace");
    size_t csr_smem = sizeof(int32_t) * (size_t)(2 * d + 2);
    if (csr_smem > 48 * 1024 &&
        cudaFuncSetAttribute(saso_tile_csr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csr_smem) !=
            cudaSuccess)
        return fail_cuda("csr smem attr");
    saso_tile_csr_kernel<<<(unsigned)ntiles, 256, csr_smem, st>>>(m, d, (int)nnz, A, SL, nbs, entw, tma ? 8u : (uint32_t)(W + 1) * 8u,
                                                                  plan, tinfo, tent);
    note_launch();
    if ((rc = check_launch("saso_tile_csr_kernel"))) return rc;

    // allow_split (CQRRPT_GPU_FAST_SKETCH): fewest row blocks (least re-reading
    // of A) and a c-split to fill the GPU. Deterministic (partials summed in
    // split order) but not the reference's single FMA chain per entry.
    int64_t nsplit = 1;
    if (allow_split && ntiles >= 32) {
        const int64_t base = cgroups * rblocks;
        double best = (double)((base + sms - 1) / sms);  // waves per unit of work, nsplit = 1
        for (int64_t ns = 2; ns <= 64 && ns <= ntiles / 8; ++ns) {
            const double t = (double)((base * ns + sms - 1) / sms) / (double)ns;
            if (t < best * 0.95) {
                best = t;
                nsplit = ns;
            }
        }
    }
    int64_t tps = (ntiles + nsplit - 1) / nsplit;
    nsplit = (ntiles + tps - 1) / tps;
    double *part = ws.get<double>("saso.part", (size_t)(nsplit * d * n));
    if (!part) return fail_nomem("saso partials");

    ApplyArgs P;
    P.m = m;
    P.n = n;
    P.lda = lda;
    P.d = d;
    P.a = a;
    P.val = 1.0 / sqrt((double)d);  // sketch.cc:79
    P.nnz = (int)nnz;
    P.entw = entw;
    P.nbs = nbs;
    P.stages = stages;
    P.ntiles = ntiles;
    P.tiles_per_split = tps;
    P.tinfo = tinfo;
    P.tent = tent;
    P.part = part;
    P.tile_lo = 0;
    P.tile_hi = 0;
    P.carry = 0;
    dim3 grid((unsigned)rblocks, (unsigned)cgroups, (unsigned)nsplit);
    auto launch_A = [&](dim3 gr) -> int {
        if (W == 16) {
            switch (A) {
                case 1: return launch_apply<1, false, 16>(P, gr, smem, st);
                case 2: return launch_apply<2, false, 16>(P, gr, smem, st);
                case 4: return launch_apply<4, false, 16>(P, gr, smem, st);
                case 8: return launch_apply<8, false, 16>(P, gr, smem, st);
                case 12: return launch_apply<12, false, 16>(P, gr, smem, st);
                default: return launch_apply<16, false, 16>(P, gr, smem, st);
            }
        }
        if (W == 8) {
            switch (A) {
                case 1: return launch_apply<1, false, 8>(P, gr, smem, st);
                case 2: return launch_apply<2, false, 8>(P, gr, smem, st);
                case 4: return launch_apply<4, false, 8>(P, gr, smem, st);
                case 8: return launch_apply<8, false, 8>(P, gr, smem, st);
                case 12: return launch_apply<12, false, 8>(P, gr, smem, st);
                default: return launch_apply<16, false, 8>(P, gr, smem, st);
            }
        }
        switch (A) {
            case 1: return tma ? launch_apply<1, true>(P, gr, smem, st) : launch_apply<1, false>(P, gr, smem, st);
            case 2: return tma ? launch_apply<2, true>(P, gr, smem, st) : launch_apply<2, false>(P, gr, smem, st);
            case 4: return tma ? launch_apply<4, true>(P, gr, smem, st) : launch_apply<4, false>(P, gr, smem, st);
            case 6: return tma ? launch_apply<6, true>(P, gr, smem, st) : launch_apply<6, false>(P, gr, smem, st);
            case 8: return tma ? launch_apply<8, true>(P, gr, smem, st) : launch_apply<8, false>(P, gr, smem, st);
            case 12: return tma ? launch_apply<12, true>(P, gr, smem, st) : launch_apply<12, false>(P, gr, smem, st);
            default: return tma ? launch_apply<16, true>(P, gr, smem, st) : launch_apply<16, false>(P, gr, smem, st);
        }
    };
    if (follow) {  // one launch per arrived chunk of rows, chains carried through `part`
        int64_t lo = 0;
        for (int c = 0; c < chunks->count; ++c) {
            const int64_t hi = std::min<int64_t>(ntiles, (chunks->row_end[c] + kTileRows - 1) / kTileRows);
            if (cudaStreamWaitEvent(st, chunks->ev[c], 0) != cudaSuccess) return fail_cuda("sketch wait chunk");
            if (hi <= lo) continue;
            P.tile_lo = lo;
            P.tile_hi = hi;
            if ((rc = launch_A(dim3((unsigned)rblocks, (unsigned)cgroups, 1)))) return rc;
            P.carry = 1;
            lo = hi;
        }
        P.tile_lo = P.tile_hi = 0;
        P.carry = 0;
        nsplit = 1;
    } else {
        rc = launch_A(grid);
    }
    if (rc) return rc;
    dim3 g((unsigned)((n + 31) / 32), (unsigned)((d + 31) / 32));
    saso_reduce_kernel<<<g, 256, 0, st>>>(d, n, nsplit, part, msk, ldm);
    note_launch();
    return check_launch("saso_reduce_kernel");
}

}  // namespace cqg

// SASO sketch on device: plan (K1), per-tile CSR, apply (K2), partial reduce.
//
// Reference: sample_sketch SASO branch (sketch.cc:73-99) and apply
// (sketch.cc:131-146). The plan is generated from the same counter RNG
// streams (rng.hh:18-53, stream mix_seed(seed, 0x7361736f + c) for GLOBAL
// column c of S), so S is bit-identical to the reference's for the same seed.
//
// Data layout in HBM
//   plan   uint32[m_local * nnz]      row | sign<<31 (sign 1 = +1/sqrt(d))
//   tptr   uint16[ntiles * (d+1)]     per 128-row tile: entry offsets by sketch row
//   tent   uint32[ntiles * 128*nnz]   per tile, entries sorted by (row, c):
//                                     negative<<31 | row<<16 | byte offset of
//                                     A(c_local, 0) in the staged tile (c*264)
//   part   double[S][d][n]            per c-split partial sketches, row-major
//   Msk    double d x n column-major  fixed-order sum of the partials
//
// Apply kernel: one CTA = 32 columns (lane = column) x a block of RB sketch
// rows x a contiguous range of row tiles. The CTA's RB x 32 accumulators live
// in shared memory; each 128 x 32 tile of A is staged ([c][33] padded:
// conflict-free warp reads of a 256-byte row) through a 3-stage cp.async
// pipeline with the tile's CSR slice. Warp w walks the entries of its RB/16
// sketch rows as one flat, row-sorted list: acc(r, j) = fma(v, A(c, j),
// acc(r, j)) with c ascending, so every output entry is the reference's own
// FMA chain (sketch.cc:137-143) -> bit-identical with one c-split.
#include "common.cuh"
#include "internal.hh"

namespace cqg {

constexpr int kTileRows = 128;  // rows of A per CSR tile
constexpr int kApplyWarps = 16;
constexpr int kApplyThreads = kApplyWarps * 32;
constexpr int kApplyStages = 3;
constexpr int kXLD = 33;        // staged tile row stride (doubles)
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
// Per-tile CSR by sketch row (stable: c ascending within a row).
// One CTA per tile; histogram + scan by the block, ordered scatter by warp 0.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) saso_tile_csr_kernel(int64_t m, int64_t d, int nnz,
                                                            const uint32_t *__restrict__ plan,
                                                            uint16_t *__restrict__ tptr,
                                                            uint32_t *__restrict__ tent) {
    extern __shared__ int32_t s_cnt[];  // d + 1 counters, then d cursors
    int32_t *s_cur = s_cnt + (d + 1);
    __shared__ int32_t s_part[256 / 32 + 1];
    const int64_t tile = blockIdx.x;
    const int64_t row0 = tile * kTileRows;
    const int rows = (int)cmin<int64_t>(kTileRows, m - row0);
    const int nent = rows * nnz;
    const uint32_t *tp = plan + row0 * nnz;

    for (int64_t r = threadIdx.x; r <= d; r += blockDim.x) s_cnt[r] = 0;
    __syncthreads();
    for (int e = threadIdx.x; e < nent; e += blockDim.x) atomicAdd(&s_cnt[tp[e] & 0x7fffffffu], 1);
    __syncthreads();
    // exclusive scan over d counters: each thread scans a contiguous chunk
    const int64_t per = (d + blockDim.x - 1) / blockDim.x;
    const int64_t lo = threadIdx.x * per, hi = cmin<int64_t>(lo + per, d);
    int32_t run = 0;
    for (int64_t r = lo; r < hi; ++r) run += s_cnt[r];
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
    uint16_t *optr = tptr + tile * (d + 1);
    for (int64_t r = lo; r < hi; ++r) {
        int32_t c = s_cnt[r];
        s_cur[r] = base;
        optr[r] = (uint16_t)base;
        base += c;
    }
    if (threadIdx.x == 0) optr[d] = (uint16_t)nent;
    __syncthreads();
    // ordered scatter: entry e = c_local*nnz + t, processed in ascending e
    if (wid == 0) {
        uint32_t *oent = tent + tile * (int64_t)(kTileRows * nnz);
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
                oent[pos] = (~w & 0x80000000u) | (r << 16) | (c_local * kXLD * 8u);  // bit 31: -1/sqrt(d)
                // highest-ranked member advances the cursor
                if (rank == __popc(grp & act) - 1) s_cur[r] += __popc(grp & act);
            }
            __syncwarp();
        }
    }
}

// ---------------------------------------------------------------------------
// K2: apply (see the header). Writes part[split][r][j] (row-major).
// ---------------------------------------------------------------------------
struct ApplyArgs {
    int64_t m, n, lda, d;
    const double *a;
    double val;
    int nnz, rb;            // entries per column of S, sketch rows per CTA (multiple of 16)
    int ptrw, entw;         // 32-bit words per stage for pointers / entries
    int64_t ntiles, tiles_per_split;
    const uint16_t *tptr;
    const uint32_t *tent;
    double *part;
};

__global__ void __launch_bounds__(kApplyThreads, 1) saso_apply_kernel(ApplyArgs P) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int RB = P.rb, A = RB / kApplyWarps;
    double *acc = reinterpret_cast<double *>(smem_raw);  // [RB][32]
    const int stage_words = 2 * kTileRows * kXLD + P.ptrw + P.entw;  // 32-bit words per stage
    uint32_t *stage0 = reinterpret_cast<uint32_t *>(acc + (size_t)RB * 32);

    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int64_t j0 = (int64_t)blockIdx.x * 32;
    const int64_t r0 = (int64_t)blockIdx.y * RB;
    const int64_t split = blockIdx.z;
    const int64_t t_begin = split * P.tiles_per_split;
    const int64_t t_end = cmin<int64_t>(t_begin + P.tiles_per_split, P.ntiles);
    const int rows_here = (int)cmin<int64_t>(RB, P.d - r0);  // valid sketch rows in this block

    for (int q = tid; q < RB * 32; q += kApplyThreads) acc[q] = 0.0;

    // staging map: thread -> tile row cc, columns jj0 + 4*it
    const int cc = tid % kTileRows, jj0 = tid / kTileRows;
    constexpr int kIters = kTileRows * 32 / kApplyThreads;  // 8
    auto issue = [&](int64_t tile, int stg) {
        uint32_t *sw = stage0 + (size_t)stg * stage_words;
        double *dt = reinterpret_cast<double *>(sw);
        const int64_t row = tile * kTileRows + cc;
        const bool rok = row < P.m;
        const double *src = P.a + (j0 + jj0) * P.lda + row;
#pragma unroll
        for (int it = 0; it < kIters; ++it) {
            const int jj = jj0 + 4 * it;
            const bool ok = rok && (j0 + jj < P.n);
            cp_async8_zfill(dt + cc * kXLD + jj, ok ? src + (int64_t)(4 * it) * P.lda : P.a, ok ? 8 : 0);
        }
        // tile pointers tptr[tile][r0 .. r0+rows_here] (4-byte words from the aligned start)
        uint32_t *sp = sw + 2 * kTileRows * kXLD;
        const uint16_t *gp = P.tptr + tile * (P.d + 1) + r0;
        const uint32_t *gpw = reinterpret_cast<const uint32_t *>(reinterpret_cast<uintptr_t>(gp) & ~(uintptr_t)3);
        const int nw = (int)(((reinterpret_cast<uintptr_t>(gp + rows_here + 1) + 3) - reinterpret_cast<uintptr_t>(gpw)) / 4);
        for (int w = tid; w < nw; w += kApplyThreads) cp_async4(sp + w, gpw + w);
        // all entries of the tile (16-byte copies; the array is padded to whole tiles)
        uint32_t *se = sp + P.ptrw;
        const uint32_t *ge = P.tent + tile * (int64_t)(kTileRows * P.nnz);
        for (int w = 4 * tid; w < kTileRows * P.nnz; w += 4 * kApplyThreads) cp_async16(se + w, ge + w);
    };
    for (int s = 0; s < kApplyStages - 1; ++s) {
        if (t_begin + s < t_end) issue(t_begin + s, s);
        cp_async_commit();
    }
    // x with the entry's sign bit (bit 31 = negative) XORed into its sign
    auto flip = [](double x, uint32_t w) {
        return __hiloint2double(__double2hiint(x) ^ (int)(w & 0x80000000u), __double2loint(x));
    };
    // acc row r (absolute) of this lane at accb + r * 256 bytes
    char *accb = reinterpret_cast<char *>(acc + lane) - r0 * 256;
    const int wr0 = wid * A, wr1 = min((wid + 1) * A, rows_here);  // this warp's rows (local)
    for (int64_t tile = t_begin; tile < t_end; ++tile) {
        const int stg = (int)((tile - t_begin) % kApplyStages);
        cp_async_wait<kApplyStages - 2>();
        __syncthreads();  // tile visible to all; stage (tile-1) fully consumed
        {
            const int64_t nt = tile + kApplyStages - 1;
            if (nt < t_end) issue(nt, (int)((nt - t_begin) % kApplyStages));
            cp_async_commit();
        }
        const uint32_t *sw = stage0 + (size_t)stg * stage_words;
        const double *xt = reinterpret_cast<const double *>(sw) + lane;
        const uint16_t *sp = reinterpret_cast<const uint16_t *>(sw + 2 * kTileRows * kXLD) +
                             ((reinterpret_cast<uintptr_t>(P.tptr + tile * (P.d + 1) + r0) >> 1) & 1);
        const uint32_t *se = sw + 2 * kTileRows * kXLD + P.ptrw;
        if (wr0 >= wr1) continue;
        const int eb = sp[wr0], ee = sp[wr1];
        if (eb >= ee) continue;
        // flat walk over this warp's entries (row-sorted, c ascending per row):
        // the running sum of the current row stays in a register; a row
        // change stores it and loads the next row's sum.
        const char *xb = reinterpret_cast<const char *>(xt);
        uint32_t curb = se[eb] & 0x7fff0000u;  // row << 16
        double *cura = reinterpret_cast<double *>(accb + (curb >> 8));
        double sacc = *cura;
        auto step = [&](uint32_t w, double x) {
            if ((w & 0x7fff0000u) != curb) {
                *cura = sacc;
                curb = w & 0x7fff0000u;
                cura = reinterpret_cast<double *>(accb + (curb >> 8));
                sacc = *cura;
            }
            sacc = fma(P.val, flip(x, w), sacc);  // sketch.cc:142; fma(v, x) == fma(|v|, +-x) exactly
        };
        int e = eb;
        for (; e + 2 <= ee; e += 2) {
            const uint32_t w0 = se[e], w1 = se[e + 1];
            const double x0 = *reinterpret_cast<const double *>(xb + (w0 & 0xffffu));
            const double x1 = *reinterpret_cast<const double *>(xb + (w1 & 0xffffu));
            step(w0, x0);
            step(w1, x1);
        }
        if (e < ee) {
            const uint32_t w0 = se[e];
            step(w0, *reinterpret_cast<const double *>(xb + (w0 & 0xffffu)));
        }
        *cura = sacc;
    }
    cp_async_wait<0>();
    __syncthreads();
    // write the partial: part[split][r][j]
    const int64_t col = j0 + lane;
    if (col < P.n) {
        double *pp = P.part + split * P.d * P.n;
        for (int rl = wid; rl < rows_here; rl += kApplyWarps) pp[(r0 + rl) * P.n + col] = acc[rl * 32 + lane];
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

static size_t apply_smem(int rb, int nnz, int *ptrw, int *entw) {
    *ptrw = ((rb + 2) / 2 + 1 + 3) & ~3;                // u16 pointers rb+1 from a 4-byte aligned start
    *entw = (kTileRows * nnz + 3) & ~3;                 // u32 entries, 16-byte multiple
    const size_t stage = sizeof(uint32_t) * (size_t)(2 * kTileRows * kXLD + *ptrw + *entw);
    return sizeof(double) * (size_t)rb * 32 + kApplyStages * stage;
}

int saso_sketch(int64_t m, int64_t n, const double *a, int64_t lda, int64_t d, int64_t nnz, uint64_t seed,
                int64_t c0, double *msk, int64_t ldm, Workspace &ws, cudaStream_t st, bool allow_split) {
    if (m <= 0 || n <= 0) {
        // empty shard contributes zeros
        for (int64_t j = 0; j < n; ++j)
            if (cudaMemsetAsync(msk + j * ldm, 0, sizeof(double) * d, st) != cudaSuccess) return fail_cuda("memset");
        return 0;
    }
    if (d > 32767 || nnz * kTileRows > 65535) return fail_internal("saso_sketch: d or nnz too large for the CSR");
    const int64_t ntiles = (m + kTileRows - 1) / kTileRows;
    uint32_t *plan = ws.get<uint32_t>("saso.plan", (size_t)(m * nnz));
    uint16_t *tptr = ws.get<uint16_t>("saso.tptr", (size_t)(ntiles * (d + 1)) + 2);
    uint32_t *tent = ws.get<uint32_t>("saso.tent", (size_t)(ntiles * kTileRows * nnz) + 4);
    if (!plan || !tptr || !tent) return fail_nomem("saso workspace");
    int rc = saso_plan(d, c0, m, nnz, seed, plan, st);
    if (rc) return rc;
    size_t csr_smem = sizeof(int32_t) * (size_t)(2 * d + 2);
    if (csr_smem > 48 * 1024 &&
        cudaFuncSetAttribute(saso_tile_csr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csr_smem) !=
            cudaSuccess)
        return fail_cuda("csr smem attr");
    saso_tile_csr_kernel<<<(unsigned)ntiles, 256, csr_smem, st>>>(m, d, (int)nnz, plan, tptr, tent);
    note_launch();
    if ((rc = check_launch("saso_tile_csr_kernel"))) return rc;

    // Decomposition. Sketch rows per CTA (RB) are bounded by shared memory;
    // exact order needs one pass over all rows per CTA, so parallelism comes
    // from row blocks: minimise waves * (staging + RB) over the row-block count.
    const int64_t cgroups = (n + 31) / 32;
    const int sms = num_sms();
    const size_t smem_max = 227 * 1024;
    int ptrw = 0, entw = 0;
    int rb_max = 16;
    while (rb_max + 16 <= 4096 && apply_smem(rb_max + 16, (int)nnz, &ptrw, &entw) <= smem_max) rb_max += 16;
    const int64_t min_blocks = (d + rb_max - 1) / rb_max;
    int64_t rblocks = min_blocks;
    {
        double best = 1e300;
        for (int64_t b = min_blocks; b <= std::max<int64_t>(min_blocks, std::min<int64_t>(d / 16, 4 * min_blocks + 8));
             ++b) {
            const int64_t rb = ((d + b - 1) / b + 15) / 16 * 16;
            const int64_t ctas = cgroups * b;
            const double cost = (double)((ctas + sms - 1) / sms) * (128.0 + (double)std::min<int64_t>(rb, d));
            if (cost < best) {
                best = cost;
                rblocks = b;
            }
        }
    }
    // allow_split (CQRRPT_GPU_FAST_SKETCH): fewest row blocks (least re-reading
    // of A) and a c-split to fill the GPU. Deterministic (partials summed in
    // split order) but not the reference's single FMA chain per entry.
    int64_t nsplit = 1;
    if (allow_split && ntiles >= 32) {
        rblocks = min_blocks;
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
    const int rb = (int)(((d + rblocks - 1) / rblocks + 15) / 16 * 16);
    rblocks = (d + rb - 1) / rb;
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
    P.rb = rb;
    const size_t smem = apply_smem(rb, (int)nnz, &P.ptrw, &P.entw);
    P.ntiles = ntiles;
    P.tiles_per_split = tps;
    P.tptr = tptr;
    P.tent = tent;
    P.part = part;
    if (cudaFuncSetAttribute(saso_apply_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
        return fail_cuda("saso_apply smem attr");
    dim3 grid((unsigned)cgroups, (unsigned)rblocks, (unsigned)nsplit);
    saso_apply_kernel<<<grid, kApplyThreads, smem, st>>>(P);
    note_launch();
    if ((rc = check_launch("saso_apply_kernel"))) return rc;
    dim3 g((unsigned)((n + 31) / 32), (unsigned)((d + 31) / 32));
    saso_reduce_kernel<<<g, 256, 0, st>>>(d, n, nsplit, part, msk, ldm);
    note_launch();
    return check_launch("saso_reduce_kernel");
}

}  // namespace cqg

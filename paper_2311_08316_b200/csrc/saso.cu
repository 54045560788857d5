// SASO sketch on device: plan (K1), per-tile CSR, apply (K2), partial reduce.
//
// Reference: sample_sketch SASO branch (sketch.cc:73-99) and apply
// (sketch.cc:131-146). The plan is generated from the same counter RNG
// streams (rng.hh:18-53, stream mix_seed(seed, 0x7361736f + c) for GLOBAL
// column c of S), so S is bit-identical to the reference's for the same seed.
//
// Data layout in HBM
//   plan   uint32[m_local * nnz]      row | sign<<31 (sign 1 = +1/sqrt(d))
//   tptr   uint16[ntiles * tstride]   per 128-row tile: entry offsets by sketch row
//                                     (tstride = d+1 rounded up to even: 4-byte aligned slices)
//   tent   uint32[ntiles * 128*nnz]   per tile, entries sorted by (row, c):
//                                     negative<<31 | (row % A)<<16 | byte offset
//                                     of A(c_local, 0) in the staged tile (c*264)
//   part   double[S][d][n]            per c-split partial sketches, row-major
//   Msk    double d x n column-major  fixed-order sum of the partials
//
// Apply kernel: one CTA = 32 columns (lane = column) x 32*A sketch rows (A
// register accumulators per lane; warp w owns rows w*A .. w*A+A-1) x a
// contiguous range of row tiles. Each 128 x 32 tile of A is staged ([c][33]
// padded: conflict-free warp reads of a 256-byte row) through a 5-stage
// cp.async pipeline with the tile's CSR slice. A warp walks its rows' entries
// (contiguous, row-sorted, c ascending per row) once and sends each to its
// row's accumulator through a jump table on the row % A stored in the entry:
// acc = fma(v, A(c, j), acc) per entry in c order is the reference's own FMA
// chain per output entry (sketch.cc:137-143), so one c-split is bit-identical.
#include <cstdlib>

#include "common.cuh"
#include "internal.hh"

namespace cqg {

constexpr int kTileRows = 128;  // rows of A per CSR tile
constexpr int kApplyWarps = 32;  // 1024 threads: short per-warp entry chains, 8 warps per scheduler
constexpr int kApplyThreads = kApplyWarps * 32;
constexpr int kApplyStages = 5;
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
__global__ void __launch_bounds__(256) saso_tile_csr_kernel(int64_t m, int64_t d, int64_t tstride, int nnz, int A,
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
    uint16_t *optr = tptr + tile * tstride;
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
                oent[pos] = (~w & 0x80000000u) | ((r % (uint32_t)A) << 16) | (c_local * kXLD * 8u);  // bit 31: -1/sqrt(d)
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
    int nnz;
    int ptrw, entw;         // 32-bit words per stage for pointers / entries
    int64_t tstride;        // tptr elements per tile (even)
    int64_t ntiles, tiles_per_split;
    const uint16_t *tptr;
    const uint32_t *tent;
    double *part;
};

template <int A>
__global__ void __launch_bounds__(kApplyThreads, 1) saso_apply_kernel(ApplyArgs P) {
    constexpr int RB = kApplyWarps * A;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int stage_words = 2 * kTileRows * kXLD + P.ptrw + P.entw;  // 32-bit words per stage
    uint32_t *stage0 = reinterpret_cast<uint32_t *>(smem_raw);

    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int64_t j0 = (int64_t)blockIdx.x * 32;
    const int64_t r0 = (int64_t)blockIdx.y * RB;
    const int64_t split = blockIdx.z;
    const int64_t t_begin = split * P.tiles_per_split;
    const int64_t t_end = cmin<int64_t>(t_begin + P.tiles_per_split, P.ntiles);
    const int rows_here = (int)cmin<int64_t>(RB, P.d - r0);  // valid sketch rows in this block

    double acc[A];
#pragma unroll
    for (int q = 0; q < A; ++q) acc[q] = 0.0;

    // staging map: thread -> tile row cc, columns jj0 + kCS*it. Addresses and
    // column bounds are fixed per thread; a tile only moves the row.
    constexpr int kCS = kApplyThreads / kTileRows;         // column stride (8)
    constexpr int kIters = kTileRows * 32 / kApplyThreads;  // copies per thread (4)
    static_assert(kCS * kIters == 32, "staging covers the 32 columns");
    const int cc = tid % kTileRows, jj0 = tid / kTileRows;
    const int64_t ldas = kCS * P.lda;
    unsigned colok = 0;
#pragma unroll
    for (int it = 0; it < kIters; ++it) colok |= (j0 + jj0 + kCS * it < P.n) ? (1u << it) : 0u;
    const double *src0 = P.a + (j0 + jj0) * P.lda + cc;  // column j0+jj0, row cc of tile 0
    const int ent_words = kTileRows * P.nnz;
    // shared byte addresses within a stage, fixed per thread
    const uint32_t s_stage0 = smem_u32(stage0), stage_bytes = (uint32_t)stage_words * 4u;
    const uint32_t a_off = (uint32_t)(cc * kXLD + jj0) * 8u;
    const uint32_t ptr_off = (uint32_t)(2 * kTileRows * kXLD) * 4u, ent_off = ptr_off + (uint32_t)P.ptrw * 4u;
    const int nwp = (rows_here + 2) / 2;  // words holding tptr[tile][r0 .. r0 + rows_here] (r0 even)
    const uint32_t *tpw = reinterpret_cast<const uint32_t *>(P.tptr + r0);
    const int64_t tsw = P.tstride / 2;
    const int nent16 = ent_words / 4;     // 16-byte copies of the tile's entries
    const double *srcA[kIters];  // row cc of tile 0 in this thread's columns (A itself if out of range)
#pragma unroll
    for (int it = 0; it < kIters; ++it) srcA[it] = ((colok >> it) & 1u) ? src0 + it * ldas : P.a;
    auto issue = [&](int64_t tile, int stg) {
        const uint32_t sb = s_stage0 + (uint32_t)stg * stage_bytes;
        const int64_t row0 = tile * kTileRows;
        const unsigned ok = (row0 + cc < P.m) ? colok : 0u;  // zero fill past m / n
#pragma unroll
        for (int it = 0; it < kIters; ++it)
            cp_async8_zfill_s(sb + a_off + (uint32_t)(it * kCS * 8), srcA[it] + (ok ? row0 : 0),
                              ((ok >> it) & 1u) ? 8 : 0);
        if (tid < nwp) cp_async4_s(sb + ptr_off + 4u * (uint32_t)tid, tpw + tile * tsw + tid);
        const uint32_t *ge = P.tent + tile * (int64_t)ent_words;
        if (nent16 <= kApplyThreads) {  // nnz <= 32: one 16-byte copy per thread at most
            if (tid < nent16) cp_async16_s(sb + ent_off + 16u * (uint32_t)tid, ge + 4 * tid);
        } else {
            for (int w = tid; w < nent16; w += kApplyThreads)
                cp_async16_s(sb + ent_off + 16u * (uint32_t)w, ge + 4 * w);
        }
    };
    // Two tiles per CTA barrier (a warp's share of entries varies tile to
    // tile; pairing halves the barriers and averages the imbalance), three
    // more in flight: stages hold tiles modulo kApplyStages.
    constexpr int kPair = 2, kAhead = kApplyStages - kPair;
    for (int s = 0; s < kAhead; ++s) {
        if (t_begin + s < t_end) issue(t_begin + s, s);
        cp_async_commit();
    }
    int stg_next = kAhead % kApplyStages, stg_cur = 0;  // stage of the next tile to issue / to process
    // x with the entry's sign bit (bit 31 = negative) XORed into its sign:
    // fma(v, x, s) == fma(|v|, +-x, s) exactly
    auto flip = [](double x, uint32_t w) {
        return __hiloint2double(__double2hiint(x) ^ (int)(w & 0x80000000u), __double2loint(x));
    };
    const int wr0 = wid * A;  // this warp's first row (local)
    for (int64_t t0 = t_begin; t0 < t_end; t0 += kPair) {
        cp_async_wait<kAhead - kPair>();
        __syncthreads();  // tiles t0, t0+1 visible; the previous pair's stages are free
#pragma unroll
        for (int u = 0; u < kPair; ++u) {
            const int64_t nt = t0 + kAhead + u;
            if (nt < t_end) issue(nt, stg_next);
            cp_async_commit();
            stg_next = (stg_next + 1 == kApplyStages) ? 0 : stg_next + 1;
        }
        const int stg_pair = stg_cur;
        stg_cur = (stg_cur + kPair) % kApplyStages;
        if (wr0 >= rows_here) continue;
#pragma unroll
        for (int u = 0; u < kPair; ++u) {
            const int64_t tile = t0 + u;
            if (tile >= t_end) break;
            const int stg = (stg_pair + u >= kApplyStages) ? stg_pair + u - kApplyStages : stg_pair + u;
            const uint32_t *sw = stage0 + (size_t)stg * stage_words;
            const char *xb = reinterpret_cast<const char *>(reinterpret_cast<const double *>(sw) + lane);
            const uint16_t *sp = reinterpret_cast<const uint16_t *>(sw + 2 * kTileRows * kXLD);
            const uint32_t *se = sw + 2 * kTileRows * kXLD + P.ptrw;
            // the warp's entries: contiguous, row-sorted (row % A in bits 16..20),
            // c ascending within a row. The next entry's word is always in a
            // register, so an empty row costs a compare.
            const int ee = sp[min(wr0 + A, rows_here)];
            int e = sp[wr0];
            constexpr uint32_t kEnd = 31u << 16;  // sentinel: matches no row
            uint32_t w = e < ee ? se[e] : kEnd;
#pragma unroll
            for (int q = 0; q < A; ++q) {  // row wr0+q: its entries in c order (sketch.cc:137-143)
                double sq = acc[q];
                while (((w >> 16) & 31u) == (uint32_t)q) {
                    const double x = flip(*reinterpret_cast<const double *>(xb + (w & 0xffffu)), w);
                    ++e;
                    w = e < ee ? se[e] : kEnd;
                    sq = fma(P.val, x, sq);  // sketch.cc:142
                }
                acc[q] = sq;
            }
        }
    }
    cp_async_wait<0>();
    // write the partial: part[split][r][j]
    const int64_t col = j0 + lane;
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

static size_t apply_smem(int rb, int nnz, int *ptrw, int *entw) {
    *ptrw = ((rb + 2) / 2 + 1 + 3) & ~3;                // u16 pointers rb+1 from a 4-byte aligned start
    *entw = (kTileRows * nnz + 3) & ~3;                 // u32 entries, 16-byte multiple
    return sizeof(uint32_t) * (size_t)(2 * kTileRows * kXLD + *ptrw + *entw) * kApplyStages;
}

template <int A>
static int launch_apply(ApplyArgs P, dim3 grid, size_t smem, cudaStream_t st) {
    auto kern = saso_apply_kernel<A>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return fail_cuda("saso_apply smem attr");
    kern<<<grid, kApplyThreads, smem, st>>>(P);
    note_launch();
    return check_launch("saso_apply_kernel");
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
    const int64_t tstride = (d + 2) & ~(int64_t)1;  // d + 1 rounded up to even
    uint16_t *tptr = ws.get<uint16_t>("saso.tptr", (size_t)(ntiles * tstride) + 2);
    uint32_t *tent = ws.get<uint32_t>("saso.tent", (size_t)(ntiles * kTileRows * nnz) + 4);
    if (!plan || !tptr || !tent) return fail_nomem("saso workspace");
    int rc = saso_plan(d, c0, m, nnz, seed, plan, st);
    if (rc) return rc;
    // Decomposition: RB = 32*A sketch rows per CTA (A register accumulators
    // per lane). Exact order needs one pass over all rows per CTA, so
    // parallelism comes from row blocks: minimise waves * (staging + RB).
    const int64_t cgroups = (n + 31) / 32;
    const int sms = num_sms();
    int A = 10;
    if (!allow_split) {
        const int cand[] = {10, 8, 6, 4, 2, 1};
        double best = 1e300;
        for (int a : cand) {
            const int64_t rb = (int64_t)kApplyWarps * a;
            const int64_t ctas = cgroups * ((d + rb - 1) / rb);
            const double cost = (double)((ctas + sms - 1) / sms) * (128.0 + (double)std::min<int64_t>(rb, d));
            if (cost < best) {
                best = cost;
                A = a;
            }
        }
    }
    if (const char *ev = getenv("CQRRPT_SASO_A")) {  // experiments: force the row-block width
        const int fa = atoi(ev);
        if (fa == 1 || fa == 2 || fa == 4 || fa == 6 || fa == 8 || fa == 10) A = fa;
    }
    const int64_t rblocks = (d + (int64_t)kApplyWarps * A - 1) / ((int64_t)kApplyWarps * A);
    size_t csr_smem = sizeof(int32_t) * (size_t)(2 * d + 2);
    if (csr_smem > 48 * 1024 &&
        cudaFuncSetAttribute(saso_tile_csr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csr_smem) !=
            cudaSuccess)
        return fail_cuda("csr smem attr");
    saso_tile_csr_kernel<<<(unsigned)ntiles, 256, csr_smem, st>>>(m, d, tstride, (int)nnz, A, plan, tptr, tent);
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
    const size_t smem = apply_smem(kApplyWarps * A, (int)nnz, &P.ptrw, &P.entw);
    if (smem > 227 * 1024) return fail_internal("saso_apply: nnz too large for the staged CSR");
    P.ntiles = ntiles;
    P.tiles_per_split = tps;
    P.tptr = tptr;
    P.tstride = tstride;
    P.tent = tent;
    P.part = part;
    dim3 grid((unsigned)cgroups, (unsigned)rblocks, (unsigned)nsplit);
    switch (A) {
        case 1: rc = launch_apply<1>(P, grid, smem, st); break;
        case 2: rc = launch_apply<2>(P, grid, smem, st); break;
        case 4: rc = launch_apply<4>(P, grid, smem, st); break;
        case 6: rc = launch_apply<6>(P, grid, smem, st); break;
        case 8: rc = launch_apply<8>(P, grid, smem, st); break;
        default: rc = launch_apply<10>(P, grid, smem, st); break;
    }
    if (rc) return rc;
    dim3 g((unsigned)((n + 31) / 32), (unsigned)((d + 31) / 32));
    saso_reduce_kernel<<<g, 256, 0, st>>>(d, n, nsplit, part, msk, ldm);
    note_launch();
    return check_launch("saso_reduce_kernel");
}

}  // namespace cqg

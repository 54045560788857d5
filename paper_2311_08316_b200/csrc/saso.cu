// SASO sketch on device: plan (K1), per-tile CSR, apply (K2), partial reduce.
//
// Reference: sample_sketch SASO branch (sketch.cc:73-99) and apply
// (sketch.cc:131-146). The plan is generated from the same counter RNG
// streams (rng.hh:18-53, stream mix_seed(seed, 0x7361736f + c) for GLOBAL
// column c of S), so S is bit-identical to the reference's for the same seed.
//
// Data layout in HBM
//   plan   uint32[m_local * nnz]      row | sign<<31 (sign 1 = +1/sqrt(d))
//   tptr   uint16[ntiles * (d+1)]     per 256-row tile: entry offsets by sketch row
//   tent   uint16[ntiles * 256*nnz]   per tile, entries sorted by (row, c):
//                                     c_local | sign<<15
//   part   double[S][d][n]            per c-split partial sketches, row-major
//   Msk    double d x n column-major  fixed-order sum of the partials
//
// Apply kernel: one CTA = 32 columns (lane = column) x a block of sketch rows
// (register accumulators, 16 warps x A rows) x a contiguous range of row
// tiles. Each 256x32 tile of A is staged once in shared memory ([c][33]
// padded: conflict-free transposed stores and conflict-free warp reads of a
// 256-byte row), then every warp walks the CSR entries of its sketch rows and
// FMAs val * A(c, j) into its accumulators. Sum order: tile-major, c
// ascending within a tile, then splits in fixed order -> deterministic.
#include "common.cuh"
#include "internal.hh"

namespace cqg {

constexpr int kTileRows = 256;  // rows of A per CSR tile
constexpr int kApplyWarps = 16;
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
                                                            uint16_t *__restrict__ tent) {
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
    // block exclusive scan of `run`
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
        uint16_t *oent = tent + tile * (int64_t)(kTileRows * nnz);
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
                int c_local = e / nnz;
                oent[pos] = (uint16_t)(c_local | ((w >> 31) << 15));
                // highest-ranked member advances the cursor
                if (rank == __popc(grp & act) - 1) s_cur[r] += __popc(grp & act);
            }
            __syncwarp();
        }
    }
}

// ---------------------------------------------------------------------------
// K2: apply. A accumulators per lane (template), 16 warps -> 16*A sketch rows
// per CTA. Tiles of 256 rows x 32 columns of A plus the tile's CSR slice are
// double-buffered in shared memory with cp.async (the copy of tile t+1 runs
// under the FMAs of tile t). Writes part[split][r][j] (row-major).
// ---------------------------------------------------------------------------
template <int A>
__global__ void __launch_bounds__(kApplyWarps * 32, 1)
    saso_apply_kernel(int64_t m, int64_t n, const double *__restrict__ a, int64_t lda, int64_t d,
                      double val, int nnz, int64_t ntiles, int64_t tiles_per_split,
                      const uint16_t *__restrict__ tptr, const uint16_t *__restrict__ tent,
                      double *__restrict__ part) {
    constexpr int RB = kApplyWarps * A;
    constexpr int LD = 33;
    constexpr int NT = kApplyWarps * 32;
    constexpr int PTRW = ((RB + 1 + 1) / 2 + 1 + 3) & ~3;  // 32-bit words per ptr buffer (16B multiple)
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double *s_tile = reinterpret_cast<double *>(smem_raw);                     // [2][256][33]
    uint32_t *s_ptrw = reinterpret_cast<uint32_t *>(s_tile + 2 * kTileRows * LD);  // [2][PTRW]
    const int entw = ((kTileRows * nnz + 1) / 2 + 3) & ~3;                    // words per entry buffer
    uint32_t *s_entw = s_ptrw + 2 * PTRW;                                      // [2][entw]

    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t j0 = (int64_t)blockIdx.x * 32;
    const int64_t r0 = (int64_t)blockIdx.y * RB;
    const int64_t split = blockIdx.z;
    const int64_t t_begin = split * tiles_per_split;
    const int64_t t_end = cmin<int64_t>(t_begin + tiles_per_split, ntiles);
    const int rows_here = (int)cmin<int64_t>(RB, d - r0);  // valid sketch rows in this block

    double acc[A];
#pragma unroll
    for (int i = 0; i < A; ++i) acc[i] = 0.0;

    // async copy of tile `tile` into buffer `bf`:
    //   A rows [256*tile, +256) x cols [j0, j0+32) -> s_tile[bf][row][col] (8-byte copies,
    //   a warp covers 256 contiguous bytes of one column)
    //   tptr[tile][r0 .. r0+rows_here] (absolute offsets) -> ptr buffer (4-byte copies from
    //   the 4-byte aligned start; odd start recorded by the parity of the address)
    //   tent[tile][0 .. 256*nnz) -> entry buffer (4-byte copies)
    auto issue = [&](int64_t tile, int bf) {
        const int64_t row0 = tile * kTileRows;
        double *dt = s_tile + bf * kTileRows * LD;
#pragma unroll 4
        for (int it = 0; it < kTileRows * 32 / NT; ++it) {
            int e = it * NT + threadIdx.x;
            int jj = e / kTileRows, cc = e % kTileRows;
            int64_t row = row0 + cc, col = j0 + jj;
            bool ok = row < m && col < n;
            cp_async8_zfill(dt + cc * LD + jj, a + (ok ? col * lda + row : 0), ok ? 8 : 0);
        }
        const uint16_t *gp = tptr + tile * (d + 1) + r0;
        const uint32_t *gpw = reinterpret_cast<const uint32_t *>(reinterpret_cast<uintptr_t>(gp) & ~(uintptr_t)3);
        const int nw = (int)(((reinterpret_cast<uintptr_t>(gp + rows_here + 1) + 3) - reinterpret_cast<uintptr_t>(gpw)) / 4);
        for (int w = threadIdx.x; w < nw; w += NT) cp_async4(s_ptrw + bf * PTRW + w, gpw + w);
        const uint32_t *gew = reinterpret_cast<const uint32_t *>(tent + tile * (int64_t)(kTileRows * nnz));
        const int nent_w = (kTileRows * nnz + 1) / 2;  // tile entry arrays start 4-byte aligned (256*nnz even)
        for (int w = threadIdx.x; w < nent_w; w += NT) cp_async4(s_entw + bf * entw + w, gew + w);
        cp_async_commit();
    };
    if (t_begin < t_end) issue(t_begin, 0);

    for (int64_t tile = t_begin; tile < t_end; ++tile) {
        const int bf = (int)((tile - t_begin) & 1);
        if (tile + 1 < t_end) {
            issue(tile + 1, bf ^ 1);  // buffer bf^1 was released by the barrier below (previous iteration)
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const double *st = s_tile + bf * kTileRows * LD;
        const uint16_t *sp = reinterpret_cast<const uint16_t *>(s_ptrw + bf * PTRW) +
                             ((reinterpret_cast<uintptr_t>(tptr + tile * (d + 1) + r0) >> 1) & 1);
        const uint16_t *se = reinterpret_cast<const uint16_t *>(s_entw + bf * entw);

        // Each sketch row's entries in c order (sketch.cc:137-143); IL rows
        // interleaved for instruction-level parallelism.
        constexpr int IL = A < 4 ? A : 4;
#pragma unroll
        for (int i0 = 0; i0 < A; i0 += IL) {
            int beg[IL], end[IL];
            double s[IL];
            int nmax = 0;
#pragma unroll
            for (int q = 0; q < IL; ++q) {
                const int rl = min(wid * A + i0 + q, rows_here);
                beg[q] = sp[rl];
                end[q] = sp[min(rl + 1, rows_here)];
                s[q] = acc[i0 + q];
                nmax = max(nmax, end[q] - beg[q]);
            }
            for (int jj = 0; jj < nmax; ++jj) {
#pragma unroll
                for (int q = 0; q < IL; ++q) {
                    const int e = beg[q] + jj;
                    if (e < end[q]) {
                        const uint32_t w = se[e];
                        const double v = (w & 0x8000u) ? val : -val;
                        s[q] = fma(v, st[(w & 0x7fffu) * LD + lane], s[q]);  // sketch.cc:142
                    }
                }
            }
#pragma unroll
            for (int q = 0; q < IL; ++q) acc[i0 + q] = s[q];
        }
        __syncthreads();  // buffer bf fully consumed before it is refilled
    }
    // write the partial: part[split][r][j]
    const int64_t col = j0 + lane;
    if (col < n) {
        double *pp = part + split * d * n;
#pragma unroll
        for (int i = 0; i < A; ++i) {
            int64_t r = r0 + wid * A + i;
            if (r < d) pp[r * n + col] = acc[i];
        }
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

template <int A>
static int launch_apply(int64_t m, int64_t n, const double *a, int64_t lda, int64_t d, double val, int nnz,
                        int64_t ntiles, const uint16_t *tptr, const uint16_t *tent, double *part,
                        int64_t nsplit, int64_t tps, int64_t rblocks, cudaStream_t st) {
    constexpr int RB = kApplyWarps * A;
    constexpr int PTRW = ((RB + 1 + 1) / 2 + 1 + 3) & ~3;
    const int entw = ((kTileRows * nnz + 1) / 2 + 3) & ~3;
    size_t smem = sizeof(double) * 2 * kTileRows * 33 + sizeof(uint32_t) * 2 * (PTRW + entw);
    if (smem > 220 * 1024) return fail_internal("saso_apply: nnz too large for the shared-memory CSR");
    auto kern = saso_apply_kernel<A>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return fail_cuda("saso_apply smem attr");
    dim3 grid((unsigned)((n + 31) / 32), (unsigned)rblocks, (unsigned)nsplit);
    kern<<<grid, kApplyWarps * 32, smem, st>>>(m, n, a, lda, d, val, nnz, ntiles, tps, tptr, tent, part);
    note_launch();
    return check_launch("saso_apply_kernel");
}

int saso_sketch(int64_t m, int64_t n, const double *a, int64_t lda, int64_t d, int64_t nnz, uint64_t seed,
                int64_t c0, double *msk, int64_t ldm, Workspace &ws, cudaStream_t st, bool exact_order) {
    if (m <= 0 || n <= 0) {
        // empty shard contributes zeros
        for (int64_t j = 0; j < n; ++j)
            if (cudaMemsetAsync(msk + j * ldm, 0, sizeof(double) * d, st) != cudaSuccess) return fail_cuda("memset");
        return 0;
    }
    if (d > 65535 || nnz * kTileRows > 65535) return fail_internal("saso_sketch: d or nnz too large for uint16 CSR");
    const int64_t ntiles = (m + kTileRows - 1) / kTileRows;
    uint32_t *plan = ws.get<uint32_t>("saso.plan", (size_t)(m * nnz));
    uint16_t *tptr = ws.get<uint16_t>("saso.tptr", (size_t)(ntiles * (d + 1)));
    uint16_t *tent = ws.get<uint16_t>("saso.tent", (size_t)(ntiles * kTileRows * nnz));
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

    const int64_t cgroups = (n + 31) / 32;
    const int sms = num_sms();
    int A = 20;
    int64_t nsplit = 1;
    if (exact_order) {
        // One pass over all rows per CTA keeps the reference's per-entry sum
        // order (c ascending, sketch.cc:137-143) -> bit-identical sketch.
        // Parallelism comes from finer sketch-row blocks instead.
        // Every CTA streams all m rows of its 32 columns (a fixed staging cost,
        // ~ the entry work of 256 sketch rows) plus work proportional to its
        // row-block height 16*A; CTAs run one per SM: minimise
        // waves(A) * (256 + 16*A).
        const int cand[] = {20, 16, 12, 8, 4, 2, 1};
        double best = 1e300;
        for (int a : cand) {
            const int64_t ctas = cgroups * ((d + 16 * a - 1) / (16 * a));
            const int64_t waves = (ctas + sms - 1) / sms;
            const double cost = (double)waves * (256.0 + (double)std::min<int64_t>(16 * a, d));
            if (cost < best) {
                best = cost;
                A = a;
            }
        }
    } else {
        if (d <= 16 * 8) A = 8;
        else if (d <= 16 * 12) A = 12;
        else if (d <= 16 * 16) A = 16;
        int64_t base = cgroups * ((d + 16 * A - 1) / (16 * A));
        nsplit = std::max<int64_t>(1, std::min<int64_t>(ntiles, (2 * sms + base - 1) / base));
    }
    const int64_t RB = 16 * A;
    const int64_t rblocks = (d + RB - 1) / RB;
    int64_t tps = (ntiles + nsplit - 1) / nsplit;
    nsplit = (ntiles + tps - 1) / tps;
    double *part = ws.get<double>("saso.part", (size_t)(nsplit * d * n));
    if (!part) return fail_nomem("saso partials");
    const double val = 1.0 / sqrt((double)d);  // sketch.cc:79
#define CQ_APPLY(AA) \
    case AA: rc = launch_apply<AA>(m, n, a, lda, d, val, (int)nnz, ntiles, tptr, tent, part, nsplit, tps, rblocks, st); break;
    switch (A) {
        CQ_APPLY(1) CQ_APPLY(2) CQ_APPLY(4) CQ_APPLY(8) CQ_APPLY(12) CQ_APPLY(16) CQ_APPLY(20)
        default: return fail_internal("saso: bad A");
    }
#undef CQ_APPLY
    if (rc) return rc;
    dim3 g((unsigned)((n + 31) / 32), (unsigned)((d + 31) / 32));
    saso_reduce_kernel<<<g, 256, 0, st>>>(d, n, nsplit, part, msk, ldm);
    note_launch();
    return check_launch("saso_reduce_kernel");
}

}  // namespace cqg

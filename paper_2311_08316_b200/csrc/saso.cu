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
// per CTA. Writes part[split][r][j] (row-major, coalesced over lanes).
// ---------------------------------------------------------------------------
template <int A>
__global__ void __launch_bounds__(kApplyWarps * 32, 1)
    saso_apply_kernel(int64_t m, int64_t n, const double *__restrict__ a, int64_t lda, int64_t d,
                      double val, int nnz, int64_t ntiles, int64_t tiles_per_split,
                      const uint16_t *__restrict__ tptr, const uint16_t *__restrict__ tent,
                      double *__restrict__ part) {
    constexpr int RB = kApplyWarps * A;
    constexpr int LD = 33;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double *s_tile = reinterpret_cast<double *>(smem_raw);                       // [256][33]
    uint16_t *s_ptr = reinterpret_cast<uint16_t *>(s_tile + kTileRows * LD);     // [RB+1]
    uint16_t *s_ent = s_ptr + ((RB + 1 + 7) & ~7);                                // [256*nnz]

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

    // register prefetch of one 256x32 tile: element e = it*512 + tid ->
    // column e/256, row e%256 (a warp reads 256 contiguous bytes of a column)
    constexpr int PER = kTileRows * 32 / (kApplyWarps * 32);  // 16
    double pre[PER];
    auto load_tile = [&](int64_t tile) {
        const int64_t row0 = tile * kTileRows;
#pragma unroll
        for (int it = 0; it < PER; ++it) {
            int e = it * (kApplyWarps * 32) + threadIdx.x;
            int jj = e / kTileRows, cc = e % kTileRows;
            int64_t row = row0 + cc, col = j0 + jj;
            pre[it] = (row < m && col < n) ? __ldg(a + col * lda + row) : 0.0;
        }
    };
    if (t_begin < t_end) load_tile(t_begin);

    for (int64_t tile = t_begin; tile < t_end; ++tile) {
        __syncthreads();  // previous tile fully consumed
#pragma unroll
        for (int it = 0; it < PER; ++it) {
            int e = it * (kApplyWarps * 32) + threadIdx.x;
            s_tile[(e % kTileRows) * LD + e / kTileRows] = pre[it];
        }
        const uint16_t *gp = tptr + tile * (d + 1);
        const int e_lo = gp[r0];
        const int e_hi = gp[r0 + rows_here];
        for (int i = threadIdx.x; i <= RB; i += blockDim.x)
            s_ptr[i] = (uint16_t)((i <= rows_here ? gp[r0 + i] : e_hi) - e_lo);
        const uint16_t *ge = tent + tile * (int64_t)(kTileRows * nnz) + e_lo;
        for (int i = threadIdx.x; i < e_hi - e_lo; i += blockDim.x) s_ent[i] = ge[i];
        __syncthreads();
        if (tile + 1 < t_end) load_tile(tile + 1);  // overlaps the compute below

#pragma unroll
        for (int i = 0; i < A; ++i) {
            const int rl = wid * A + i;
            const int beg = s_ptr[rl], end = s_ptr[rl + 1];
            double s = acc[i];
            for (int e = beg; e < end; ++e) {
                const uint32_t w = s_ent[e];
                const double v = (w & 0x8000u) ? val : -val;
                s = fma(v, s_tile[(w & 0x7fffu) * LD + lane], s);  // sketch.cc:142
            }
            acc[i] = s;
        }
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
    size_t smem = sizeof(double) * kTileRows * 33 + sizeof(uint16_t) * (((RB + 1 + 7) & ~7) + kTileRows * nnz);
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
        const int cand[] = {20, 16, 12, 8, 4, 2, 1};
        A = 1;
        for (int a : cand)
            if (cgroups * ((d + 16 * a - 1) / (16 * a)) >= sms) {
                A = a;
                break;
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

// K5b on the INT8 tensor cores: the Gram G = X^T X (reference gram,
// linalg.cc:298-307) emulated exactly in modular integer arithmetic
// (Ozaki scheme II: error-free integer products, Chinese remainder theorem).
//
// B200 has ~4.5 POPS of dense INT8 tensor throughput against ~37 TFLOP/s of
// FP64 (DMMA): an FP64 product reassembled from NMOD int8 GEMMs runs several
// times faster than the DMMA SYRK while keeping FP64-level accuracy.
//
//   1. scale: every column j of X gets a power of two 2^{s_j} so that
//      |X(i,j)| 2^{s_j} < 2^beta; t_ij = trunc(X(i,j) 2^{s_j}) is an integer
//      (exact in a double: for |t| >= 2^53 the scaled double already is one).
//      beta is the largest with m 2^{2 beta} < P/2, P = prod p_l, so the
//      integer Gram T^T T is exactly representable by its residues.
//   2. per K-chunk of <= 131072 rows and per modulus p_l <= 255 (pairwise
//      coprime): the symmetric residues t mod p_l fit int8 (|r| <= 127), and
//      the chunk's R_l^T R_l is exact in int32 (131072 * 127^2 < 2^31) --
//      a plain INT8 GEMM (cuBLASLt IMMA on sm_100a). Residues of the chunk
//      sums accumulate mod p_l.
//   3. CRT (Garner, symmetric mixed radix, exact int32 arithmetic) gives the
//      integer (T^T T)_ij as sum_l v_l W_l (W_l = p_1..p_{l-1}), evaluated in
//      double-double, then scaled by 2^{-s_i - s_j}.
// The only roundings are the truncation of X to beta bits (relative 2^-beta
// of the column max) and the final double-double -> double rounding, so the
// result is at least as accurate as an FP64 GEMM; it is deterministic,
// bitwise symmetric, and G_ij depends only on columns i and j (the leading
// block of G is gram(X[:, :j]) bitwise: the Cholesky-retry property of
// cqrrpt.cc:162-164 holds).
#include <dlfcn.h>

#include <cmath>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>

#include <cublasLt.h>

#include "common.cuh"
#include "internal.hh"

namespace cqg {

namespace {

constexpr int kMaxMod = 24;
constexpr int kModList[kMaxMod] = {255, 254, 253, 251, 247, 241, 239, 233, 229, 227, 223, 217,
                                   211, 199, 197, 193, 191, 181, 179, 173, 167, 163, 157, 151};
constexpr int64_t kChunk = 131072;  // rows per int8 GEMM: 131072 * 127^2 < 2^31
constexpr double kResidueBytes = 10e9;  // cap of the residue double buffer
constexpr int kBeta = 53;           // bits kept per column (relative to its max): t < 2^53 is an exact double

struct OzConst {
    int nmod;
    int p[kMaxMod];
    double pinv[kMaxMod];           // 1 / p (for the residue quotient estimate)
    int inv[kMaxMod][kMaxMod];      // inv[i][j] = p_j^{-1} mod p_i (j < i)
    double whi[kMaxMod], wlo[kMaxMod];  // W_l = p_0 .. p_{l-1} as double-double
};
__constant__ OzConst c_oz;

// ---- cuBLASLt (dlopen'ed: no link-time dependency) ---------------------------
struct LtApi {
    bool tried = false, ok = false;
    decltype(&cublasLtCreate) create = nullptr;
    decltype(&cublasLtMatmulDescCreate) desc_create = nullptr;
    decltype(&cublasLtMatmulDescSetAttribute) desc_set = nullptr;
    decltype(&cublasLtMatrixLayoutCreate) layout_create = nullptr;
    decltype(&cublasLtMatmulPreferenceCreate) pref_create = nullptr;
    decltype(&cublasLtMatmulPreferenceSetAttribute) pref_set = nullptr;
    decltype(&cublasLtMatmulAlgoGetHeuristic) heuristic = nullptr;
    decltype(&cublasLtMatmul) matmul = nullptr;
    decltype(&cublasLtMatrixLayoutSetAttribute) layout_set = nullptr;
};
LtApi &lt_api() {
    static LtApi api;
    static std::mutex mu;
    std::lock_guard<std::mutex> g(mu);
    if (api.tried) return api;
    api.tried = true;
    const char *names[] = {"libcublasLt.so.12", "/usr/local/cuda/lib64/libcublasLt.so.12", "libcublasLt.so"};
    void *h = nullptr;
    for (const char *nm : names)
        if ((h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL))) break;
    if (!h) return api;
    api.create = (decltype(api.create))dlsym(h, "cublasLtCreate");
    api.desc_create = (decltype(api.desc_create))dlsym(h, "cublasLtMatmulDescCreate");
    api.desc_set = (decltype(api.desc_set))dlsym(h, "cublasLtMatmulDescSetAttribute");
    api.layout_create = (decltype(api.layout_create))dlsym(h, "cublasLtMatrixLayoutCreate");
    api.pref_create = (decltype(api.pref_create))dlsym(h, "cublasLtMatmulPreferenceCreate");
    api.pref_set = (decltype(api.pref_set))dlsym(h, "cublasLtMatmulPreferenceSetAttribute");
    api.heuristic = (decltype(api.heuristic))dlsym(h, "cublasLtMatmulAlgoGetHeuristic");
    api.matmul = (decltype(api.matmul))dlsym(h, "cublasLtMatmul");
    api.layout_set = (decltype(api.layout_set))dlsym(h, "cublasLtMatrixLayoutSetAttribute");
    api.ok = api.create && api.desc_create && api.desc_set && api.layout_create && api.pref_create && api.pref_set &&
             api.heuristic && api.matmul;
    return api;
}

constexpr size_t kLtWorkspace = size_t(32) << 20;
decltype(&cublasLtMatrixLayoutSetAttribute) lt_api_layout_set() { return lt_api().layout_set; }

// C (M x N int32, ldc) = A^T B with A (K x M) and B (K x N) column-major int8.
struct LtPlan {
    cublasLtMatmulDesc_t desc = nullptr;
    cublasLtMatrixLayout_t la = nullptr, lb = nullptr, lc = nullptr;
    cublasLtMatmulAlgo_t algo;
};
int lt_plan(int dev, int64_t M, int64_t N, int64_t K, int64_t lda, int64_t ldb, int64_t ldc, int batch, int64_t sa,
            int64_t sc, LtPlan **out, cublasLtHandle_t *handle_out) {
    LtApi &api = lt_api();
    if (!api.ok) return set_error("libcublasLt.so.12 not loadable"), CQRRPT_GPU_ERR_INTERNAL;
    static std::mutex mu;
    static std::map<int, cublasLtHandle_t> handles;
    static std::map<std::tuple<int, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, int, int64_t, int64_t>, LtPlan>
        plans;
    std::lock_guard<std::mutex> g(mu);
    if (!handles.count(dev)) {
        cublasLtHandle_t h;
        if (api.create(&h) != CUBLAS_STATUS_SUCCESS) return set_error("cublasLtCreate failed"), CQRRPT_GPU_ERR_INTERNAL;
        handles[dev] = h;
    }
    *handle_out = handles[dev];
    auto key = std::make_tuple(dev, M, N, K, lda, ldb, ldc, batch, sa, sc);
    auto it = plans.find(key);
    if (it != plans.end()) {
        *out = &it->second;
        return 0;
    }
    LtPlan p;
    bool ok = api.desc_create(&p.desc, CUBLAS_COMPUTE_32I, CUDA_R_32I) == CUBLAS_STATUS_SUCCESS;
    const cublasOperation_t ta = CUBLAS_OP_T, tb = CUBLAS_OP_N;
    ok = ok && api.desc_set(p.desc, CUBLASLT_MATMUL_DESC_TRANSA, &ta, sizeof(ta)) == CUBLAS_STATUS_SUCCESS;
    ok = ok && api.desc_set(p.desc, CUBLASLT_MATMUL_DESC_TRANSB, &tb, sizeof(tb)) == CUBLAS_STATUS_SUCCESS;
    ok = ok && api.layout_create(&p.la, CUDA_R_8I, K, M, lda) == CUBLAS_STATUS_SUCCESS;
    ok = ok && api.layout_create(&p.lb, CUDA_R_8I, K, N, ldb) == CUBLAS_STATUS_SUCCESS;
    ok = ok && api.layout_create(&p.lc, CUDA_R_32I, M, N, ldc) == CUBLAS_STATUS_SUCCESS;
    if (ok && batch > 1) {  // strided batch: one problem per modulus
        auto lset = lt_api_layout_set();
        const int32_t bc = batch;
        ok = lset && lset(p.la, CUBLASLT_MATRIX_LAYOUT_BATCH_COUNT, &bc, sizeof(bc)) == CUBLAS_STATUS_SUCCESS &&
             lset(p.lb, CUBLASLT_MATRIX_LAYOUT_BATCH_COUNT, &bc, sizeof(bc)) == CUBLAS_STATUS_SUCCESS &&
             lset(p.lc, CUBLASLT_MATRIX_LAYOUT_BATCH_COUNT, &bc, sizeof(bc)) == CUBLAS_STATUS_SUCCESS &&
             lset(p.la, CUBLASLT_MATRIX_LAYOUT_STRIDED_BATCH_OFFSET, &sa, sizeof(sa)) == CUBLAS_STATUS_SUCCESS &&
             lset(p.lb, CUBLASLT_MATRIX_LAYOUT_STRIDED_BATCH_OFFSET, &sa, sizeof(sa)) == CUBLAS_STATUS_SUCCESS &&
             lset(p.lc, CUBLASLT_MATRIX_LAYOUT_STRIDED_BATCH_OFFSET, &sc, sizeof(sc)) == CUBLAS_STATUS_SUCCESS;
    }
    cublasLtMatmulPreference_t pref = nullptr;
    ok = ok && api.pref_create(&pref) == CUBLAS_STATUS_SUCCESS;
    const size_t wsb = kLtWorkspace;
    ok = ok && api.pref_set(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &wsb, sizeof(wsb)) == CUBLAS_STATUS_SUCCESS;
    cublasLtMatmulHeuristicResult_t res;
    int nres = 0;
    ok = ok && api.heuristic(handles[dev], p.desc, p.la, p.lb, p.lc, p.lc, pref, 1, &res, &nres) ==
                   CUBLAS_STATUS_SUCCESS && nres > 0;
    if (!ok) return set_error("cuBLASLt int8 GEMM: no algorithm for this shape"), CQRRPT_GPU_ERR_INTERNAL;
    p.algo = res.algo;
    *out = &(plans[key] = p);
    return 0;
}

// batch > 1: `batch` problems with A/B strides sa (elements) and C stride sc
int lt_gemm_tn(int64_t M, int64_t N, int64_t K, const int8_t *a, int64_t lda, const int8_t *b, int64_t ldb,
               int32_t *c, int64_t ldc, int batch, int64_t sa, int64_t sc, void *lt_ws, cudaStream_t st) {
    LtPlan *p = nullptr;
    cublasLtHandle_t h = nullptr;
    CQ_TRY(lt_plan(current_device(), M, N, K, lda, ldb, ldc, batch, sa, sc, &p, &h));
    const int32_t one = 1, zero = 0;
    if (lt_api().matmul(h, p->desc, &one, a, p->la, b, p->lb, &zero, c, p->lc, c, p->lc, &p->algo, lt_ws,
                        kLtWorkspace, st) != CUBLAS_STATUS_SUCCESS)
        return set_error("cublasLtMatmul (int8) failed"), CQRRPT_GPU_ERR_INTERNAL;
    note_launch();
    return 0;
}

// ---- host constants ------------------------------------------------------------
int64_t modinv(int64_t a, int64_t m) {  // a^{-1} mod m (gcd 1)
    int64_t t = 0, nt = 1, r = m, nr = ((a % m) + m) % m;
    while (nr) {
        const int64_t q = r / nr;
        std::tie(t, nt) = std::make_tuple(nt, t - q * nt);
        std::tie(r, nr) = std::make_tuple(nr, r - q * nr);
    }
    return (t % m + m) % m;
}

// moduli count for m rows: the fewest with m 2^{2 kBeta} < P/8 (|G_int| < P/2
// with margin for the even modulus' slightly asymmetric digit range)
int choose_nmod(int64_t m, int *beta) {
    const double lk = std::log2((double)std::max<int64_t>(m, 1));
    double lp = 0.0;
    *beta = kBeta;
    for (int l = 0; l < kMaxMod; ++l) {
        lp += std::log2((double)kModList[l]);
        if (lp - 3.0 - lk >= 2.0 * kBeta + 1e-9) return l + 1;
    }
    *beta = (int)std::floor((lp - 3.0 - lk) / 2.0 - 1e-9);  // m beyond 2^44 rows: fewer bits
    return kMaxMod;
}

int upload_constants(int nmod) {
    static int uploaded[64] = {0};
    const int dev = current_device() & 63;
    if (uploaded[dev] == nmod) return 0;
    OzConst h{};
    h.nmod = nmod;
    for (int l = 0; l < nmod; ++l) {
        h.p[l] = kModList[l];
        h.pinv[l] = 1.0 / (double)kModList[l];
        for (int j = 0; j < l; ++j) h.inv[l][j] = (int)modinv(kModList[j], kModList[l]);
    }
    // W_l = p_0 .. p_{l-1} exactly in 32-bit limbs, split into a double-double
    // (hi = W rounded, lo = the exact remainder W - hi rounded)
    {
        uint32_t limbs[8] = {1, 0, 0, 0, 0, 0, 0, 0};
        for (int l = 0; l < nmod; ++l) {
            // to double-double: take the top 106 bits
            int top = 7;
            while (top > 0 && limbs[top] == 0) --top;
            double hi = 0.0;
            for (int q = top; q >= 0; --q) hi = hi * 4294967296.0 + (double)limbs[q];  // rounded once per step
            // exact remainder W - hi, computed limb-wise with the integer value of hi
            // (hi is an integer; represent it in limbs)
            uint32_t hl[8] = {0};
            {
                int e = 0;
                double f = std::frexp(hi, &e);  // hi = f 2^e, f in [0.5, 1)
                const uint64_t mant = (uint64_t)std::ldexp(f, 53);  // 53-bit integer, hi = mant 2^(e-53)
                const int sh = e - 53;
                if (sh >= 0) {
                    const int w0 = sh / 32, b0 = sh % 32;
                    const unsigned __int128 v = (unsigned __int128)mant << b0;
                    for (int q = 0; q < 4 && w0 + q < 8; ++q) hl[w0 + q] = (uint32_t)(v >> (32 * q));
                } else {
                    hl[0] = (uint32_t)(mant >> (-sh));
                    hl[1] = (uint32_t)((mant >> (-sh)) >> 32);
                }
            }
            // diff = limbs - hl (signed), to double
            int64_t borrow = 0;
            uint32_t dl[8];
            bool neg = false;
            {
                // compare
                int cmp = 0;
                for (int q = 7; q >= 0 && !cmp; --q) cmp = (limbs[q] > hl[q]) - (limbs[q] < hl[q]);
                const uint32_t *x = cmp >= 0 ? limbs : hl, *y = cmp >= 0 ? hl : limbs;
                neg = cmp < 0;
                for (int q = 0; q < 8; ++q) {
                    int64_t d = (int64_t)x[q] - (int64_t)y[q] - borrow;
                    borrow = d < 0;
                    dl[q] = (uint32_t)(d + (borrow ? ((int64_t)1 << 32) : 0));
                }
            }
            double lo = 0.0;
            for (int q = 7; q >= 0; --q) lo = lo * 4294967296.0 + (double)dl[q];
            h.whi[l] = hi;
            h.wlo[l] = neg ? -lo : lo;
            // limbs *= p_l
            uint64_t carry = 0;
            for (int q = 0; q < 8; ++q) {
                const uint64_t v = (uint64_t)limbs[q] * (uint64_t)kModList[l] + carry;
                limbs[q] = (uint32_t)v;
                carry = v >> 32;
            }
        }
    }
    CQ_CUDA(cudaMemcpyToSymbol(c_oz, &h, sizeof(h)), "ozaki constants");
    uploaded[dev] = nmod;
    return 0;
}

// ---- kernels -----------------------------------------------------------------------
// s_j = beta - E_j with max_i |X(i,j)| = f 2^{E_j}, f in [0.5, 1) (0 for a zero column)
__global__ void oz_colscale_kernel(int64_t m, const double *__restrict__ x, int64_t ldx, int beta,
                                   int *__restrict__ sexp) {
    __shared__ double red[32];
    const int64_t j = blockIdx.x;
    const double *xj = x + j * ldx;
    double mx = 0.0;
    for (int64_t i = threadIdx.x; i < m; i += blockDim.x) mx = fmax(mx, fabs(xj[i]));
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x < 32) {
        mx = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : 0.0;
        for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (threadIdx.x == 0) {
            int e = 0;
            if (mx > 0.0) frexp(mx, &e);
            sexp[j] = (mx > 0.0) ? beta - e : 0;
        }
    }
}

// residues of rows [r0, r0 + rows) (rows padded to ldr with zeros), all columns:
// out[l][j * ldr + i] = sym(trunc(X(r0+i, j) 2^{s_j}) mod p_l). Thread = 4 rows of a column.
__global__ void oz_residue_kernel(int64_t m, int64_t k, const double *__restrict__ x, int64_t ldx, int64_t r0,
                                  int64_t rows, int64_t ldr, const int *__restrict__ sexp, int8_t *__restrict__ out,
                                  int64_t lstride) {
    const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;  // 4-row group
    const int64_t groups = ldr / 4;
    const int64_t j = blockIdx.y;  // j in [k, kp): zero padding columns
    if (q >= groups) return;
    const int s = (j < k) ? sexp[j] : 0;
    double t[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int64_t i = q * 4 + u;
        t[u] = (j < k && i < rows && r0 + i < m) ? trunc(ldexp(x[j * ldx + r0 + i], s)) : 0.0;
    }
    // |t| < 2^53. q = t/p rounded to the nearest integer through the 1.5 2^52
    // shifter (one DFMA + one DADD, no FRND), exact remainder by fma, the
    // integer read from the shifted double's low word (no F2I), one
    // symmetric fixup in int32 for the rare quotient that rounds the other way
    const double kShift = 6755399441055744.0;  // 1.5 * 2^52
    const int nmod = c_oz.nmod;
#pragma unroll
    for (int l = 0; l < kMaxMod; ++l) {
        if (l >= nmod) break;
        const double p = (double)c_oz.p[l], pi = c_oz.pinv[l];
        const int pint = c_oz.p[l], hp = pint >> 1;
        char4 o;
        int8_t *ov = reinterpret_cast<int8_t *>(&o);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const double qq = __dsub_rn(__fma_rn(t[u], pi, kShift), kShift);
            const double r = __fma_rn(-qq, p, t[u]);  // exact
            int ri = __double2loint(__dadd_rn(r, kShift));
            ri = (ri > hp) ? ri - pint : ri;
            ri = (ri < -hp) ? ri + pint : ri;  // p = 254: [-127, 127]; odd p: [-(p-1)/2, (p-1)/2]
            ov[u] = (int8_t)ri;
        }
        *reinterpret_cast<char4 *>(out + l * lstride + j * ldr + q * 4) = o;
    }
}

// acc[l][e] = (acc[l][e] + c[l][e]) mod p_l, acc in [0, p_l)
// Product layout. FULL: one k x k block per modulus (region l, ld ldc).
// SPLIT (the integer Gram is symmetric, so only 3 of the 2 x 2 half blocks
// are multiplied): regions 2l + b = diagonal block b of modulus l, regions
// 2 nmod + l = the upper off-diagonal block of modulus l; every region is
// kh x kh (ld kh).
struct OzLayout {
    int split;
    int64_t kh, region;  // SPLIT: half size and region size; FULL: region = ldc * k
    int64_t ldc;
};
CQ_DEVI int region_mod(const OzLayout &L, int b, int nmod) {
    return L.split ? (b < 2 * nmod ? (b >> 1) : b - 2 * nmod) : b;
}

// acc[b][e] = (acc[b][e] + c[b][e]) mod p, acc in [0, p)
__global__ void oz_accum_kernel(OzLayout L, const int32_t *__restrict__ c, int32_t *__restrict__ acc, int first) {
    const int b = blockIdx.y;
    const int p = c_oz.p[region_mod(L, b, c_oz.nmod)];
    const int64_t nelem = L.region;
    const int32_t *cl = c + (int64_t)b * nelem;
    int32_t *al = acc + (int64_t)b * nelem;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nelem; e += (int64_t)gridDim.x * blockDim.x) {
        int r = cl[e] % p;
        if (r < 0) r += p;
        if (!first) {
            r += al[e];
            if (r >= p) r -= p;
        }
        al[e] = r;
    }
}

// double-double helpers
CQ_DEVI void two_sum(double a, double b, double &s, double &e) {
    s = __dadd_rn(a, b);
    const double bb = __dsub_rn(s, a);
    e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
}

// Garner (symmetric digits) + double-double evaluation + 2^{-s_i-s_j}; G is k x k (ldg)
__global__ void oz_crt_kernel(int64_t k, OzLayout L, const int32_t *__restrict__ acc, const int *__restrict__ sexp,
                              double *__restrict__ g, int64_t ldg) {
    const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= k * k) return;
    const int64_t i = q % k, j = q / k;
    // the integer Gram is exactly symmetric: read (min, max) so G is bitwise
    // symmetric whatever the GEMMs wrote
    const int64_t ii = i < j ? i : j, jj = i < j ? j : i;
    int64_t base, stride;  // element of modulus l at acc[base + l * stride]
    if (!L.split) {
        base = jj * L.ldc + ii;
        stride = L.region;
    } else {
        const int64_t kh = L.kh;
        const int bi = ii >= kh, bj = jj >= kh;
        if (bi == bj) {  // diagonal block b: region 2l + b
            base = (int64_t)bi * L.region + (jj - bj * kh) * kh + (ii - bi * kh);
            stride = 2 * L.region;
        } else {         // upper off-diagonal block: region 2 nmod + l
            base = 2 * (int64_t)c_oz.nmod * L.region + (jj - kh) * kh + ii;
            stride = L.region;
        }
    }
    const int nmod = c_oz.nmod;
    int v[kMaxMod];
    for (int l = 0; l < nmod; ++l) {
        const int p = c_oz.p[l];
        // t = (r_l - (v_0 + v_1 W_1 + ... + v_{l-1} W_{l-1})) / W_l  mod p_l, by Garner's
        // recurrence: t = (((r - v_0) inv_0 - v_1) inv_1 - ...) mod p
        int t = acc[base + (int64_t)l * stride];
        for (int q = 0; q < l; ++q) {
            t = (t - v[q]) % p;
            if (t < 0) t += p;
            t = (int)(((int64_t)t * c_oz.inv[l][q]) % p);
        }
        if (t > p / 2) t -= p;  // symmetric digit: the sum spans (-P/2, P/2]
        v[l] = t;
    }
    // sum v_l W_l from the top digit down, in double-double
    double sh = 0.0, sl = 0.0;
    for (int l = nmod - 1; l >= 0; --l) {
        const double d = (double)v[l];
        const double ph = __dmul_rn(d, c_oz.whi[l]);
        const double pe = fma(d, c_oz.whi[l], -ph);  // exact product error
        const double pl = fma(d, c_oz.wlo[l], pe);
        double s, err;
        two_sum(sh, ph, s, err);
        sl = __dadd_rn(sl, __dadd_rn(err, pl));
        two_sum(s, sl, sh, sl);
    }
    const double val = __dadd_rn(sh, sl);
    g[j * ldg + i] = ldexp(val, -(sexp[i] + sexp[j]));
}

}  // namespace

bool gram_ozaki_available() { return lt_api().ok; }

int gram_ozaki(int64_t m, int64_t k, const double *x, int64_t ldx, double *gmat, int64_t ldg, Workspace &ws,
               cudaStream_t st) {
    if (k <= 0) return 0;
    if (m <= 0) {
        for (int64_t j = 0; j < k; ++j) CQ_CUDA(cudaMemsetAsync(gmat + j * ldg, 0, sizeof(double) * k, st), "gram 0");
        return 0;
    }
    int beta = 0;
    const int nmod = choose_nmod(m, &beta);
    CQ_TRY(upload_constants(nmod));
    OzLayout L;
    // the int8 GEMMs run on kp = k rounded up to 16 columns (zero residues in
    // the padding), which every IMMA algorithm accepts
    const int64_t kp = ((k + 15) / 16) * 16;
    L.split = (kp >= 1024) ? 1 : 0;
    L.kh = kp / 2;
    L.ldc = L.split ? L.kh : kp;  // int32 output rows
    L.region = L.split ? L.kh * L.kh : L.ldc * kp;
    const int64_t nregions = L.split ? 3 * (int64_t)nmod : nmod;
    const int64_t nelem = L.region * nregions / nmod;  // int32 entries per modulus
    // Workspace (cached, grow-only like every other buffer): the residue
    // double buffer is capped at kResidueBytes and at half of what is free
    // beyond the buffers this Gram already holds; chunks shrink to fit, and
    // below 4096 rows the DMMA Gram takes over.
    size_t free_b = 0, total_b = 0;
    CQ_CUDA(cudaMemGetInfo(&free_b, &total_b), "oz meminfo");
    const double held = (double)ws_bytes("oz.res") + (double)ws_bytes("oz.c") + (double)ws_bytes("oz.acc");
    const double budget = std::min(kResidueBytes, 0.5 * ((double)free_b + held) - 2.0 * nmod * (double)nelem * 4.0);
    int64_t chunk = std::min<int64_t>(kChunk, ((m + 15) / 16) * 16);
    chunk = std::min<int64_t>(chunk, (int64_t)(budget / (2.0 * nmod * (double)kp)) / 16 * 16);
    if (chunk < 4096 && chunk < m) return gram_dmma(m, k, x, ldx, gmat, ldg, ws, st);
    const int64_t lstride = chunk * kp;
    int *sexp = ws.get<int>("oz.sexp", (size_t)k);
    void *ltws = ws.raw("oz.ltws", kLtWorkspace);
    if (!sexp || !ltws) return fail_nomem("ozaki gram workspace");
    int8_t *res = ws.get<int8_t>("oz.res", (size_t)(2 * nmod * lstride));  // double buffer
    int32_t *cbuf = ws.get<int32_t>("oz.c", (size_t)(nmod * nelem));
    int32_t *acc = ws.get<int32_t>("oz.acc", (size_t)(nmod * nelem));
    if (!res || !cbuf || !acc) return gram_dmma(m, k, x, ldx, gmat, ldg, ws, st);
    cudaStream_t aux = nullptr;
    cudaEvent_t *ev = nullptr;  // [0] start, [1..2] residues ready, [3..4] buffer free
    CQ_TRY(cached_stream("oz.aux", 0, &aux));
    CQ_TRY(cached_events("oz.ev", 5, &ev));
    oz_colscale_kernel<<<(unsigned)k, 256, 0, st>>>(m, x, ldx, beta, sexp);
    note_launch();
    CQ_TRY(check_launch("oz_colscale_kernel"));
    CQ_CUDA(cudaEventRecord(ev[0], st), "oz start");
    CQ_CUDA(cudaStreamWaitEvent(aux, ev[0], 0), "oz start wait");
    // residues of chunk c+1 (CUDA cores, aux stream) overlap the int8 GEMMs
    // of chunk c (tensor cores, st)
    int64_t c = 0;
    for (int64_t r0 = 0; r0 < m; r0 += chunk, ++c) {
        const int64_t rows = std::min<int64_t>(chunk, m - r0);
        const int64_t ldr = ((rows + 15) / 16) * 16;
        const int64_t cls = ldr * kp;  // this chunk's residue stride between moduli (<= lstride)
        const int b = (int)(c & 1);
        int8_t *rb = res + (int64_t)b * nmod * lstride;
        if (c >= 2) CQ_CUDA(cudaStreamWaitEvent(aux, ev[3 + b], 0), "oz buffer wait");
        dim3 grid((unsigned)((ldr / 4 + 255) / 256), (unsigned)kp);
        oz_residue_kernel<<<grid, 256, 0, aux>>>(m, k, x, ldx, r0, rows, ldr, sexp, rb, cls);
        note_launch();
        CQ_TRY(check_launch("oz_residue_kernel"));
        CQ_CUDA(cudaEventRecord(ev[1 + b], aux), "oz residues ready");
        CQ_CUDA(cudaStreamWaitEvent(st, ev[1 + b], 0), "oz residues wait");
        if (!L.split) {  // one strided-batched int8 GEMM per chunk: batch = moduli
            CQ_TRY(lt_gemm_tn(kp, kp, ldr, rb, ldr, rb, ldr, cbuf, L.ldc, nmod, cls, L.region, ltws, st));
        } else {
            // diagonal half blocks of every modulus (batch 2 nmod: column half
            // b of modulus l starts at (2l + b) kh ldr) and the upper
            // off-diagonal half block (batch nmod)
            const int64_t kh = L.kh;
            CQ_TRY(lt_gemm_tn(kh, kh, ldr, rb, ldr, rb, ldr, cbuf, kh, 2 * nmod, kh * ldr, L.region, ltws, st));
            CQ_TRY(lt_gemm_tn(kh, kh, ldr, rb, ldr, rb + kh * ldr, ldr, cbuf + 2 * nmod * L.region, kh, nmod, cls,
                              L.region, ltws, st));
        }
        CQ_CUDA(cudaEventRecord(ev[3 + b], st), "oz buffer free");
        const unsigned gx = (unsigned)std::min<int64_t>((L.region + 255) / 256, 2048);
        oz_accum_kernel<<<dim3(gx, (unsigned)nregions), 256, 0, st>>>(L, cbuf, acc, r0 == 0 ? 1 : 0);
        note_launch();
        CQ_TRY(check_launch("oz_accum_kernel"));
    }
    oz_crt_kernel<<<(unsigned)((k * k + 255) / 256), 256, 0, st>>>(k, L, acc, sexp, gmat, ldg);
    note_launch();
    return check_launch("oz_crt_kernel");
}

}  // namespace cqg

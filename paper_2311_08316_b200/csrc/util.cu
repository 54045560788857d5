// Small device utilities + the host runtime (errors, launch accounting,
// workspace cache).
#include <cstdio>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "internal.hh"

namespace cqg {

// ---------------------------------------------------------------------------
// runtime
// ---------------------------------------------------------------------------
static thread_local std::string g_err = "";
static thread_local int64_t g_launches = 0;

void set_error(const std::string &msg) { g_err = msg; }
int fail_cuda(const char *what) {
    cudaError_t e = cudaGetLastError();
    g_err = std::string(what) + ": " + cudaGetErrorString(e);
    return CQRRPT_GPU_ERR_CUDA;
}
int fail_nomem(const char *what) {
    cudaGetLastError();
    g_err = std::string("out of device memory: ") + what;
    return CQRRPT_GPU_ERR_NOMEM;
}
int fail_internal(const char *what) {
    g_err = what;
    return CQRRPT_GPU_ERR_INTERNAL;
}
int check_launch(const char *kernel) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        g_err = std::string(kernel) + ": " + cudaGetErrorString(e);
        return CQRRPT_GPU_ERR_CUDA;
    }
    return 0;
}
void note_launch() { ++g_launches; }
int64_t launch_count(bool reset) {
    int64_t v = g_launches;
    if (reset) g_launches = 0;
    return v;
}
const char *last_error() { return g_err.c_str(); }

int num_sms() {
    static int cached[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && cached[dev]) return cached[dev];
    int v = 148;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    if (dev < 64) cached[dev] = v;
    return v;
}

struct Buf {
    void *p = nullptr;
    size_t bytes = 0;
};
static thread_local std::map<std::pair<int, std::string>, Buf> g_ws;

void *Workspace::raw(const char *name, size_t bytes) {
    int dev = 0;
    cudaGetDevice(&dev);
    Buf &b = g_ws[{dev, name}];
    if (b.bytes < bytes) {
        if (b.p) {
            cudaDeviceSynchronize();  // a previous call may still use it
            cudaFree(b.p);
            b.p = nullptr;
            b.bytes = 0;
        }
        size_t want = bytes + bytes / 8;  // headroom for slowly growing sizes
        if (cudaMalloc(&b.p, want) != cudaSuccess) {
            cudaGetLastError();
            if (cudaMalloc(&b.p, bytes) != cudaSuccess) {
                cudaGetLastError();
                b.p = nullptr;
                return nullptr;
            }
            want = bytes;
        }
        b.bytes = want;
    }
    return b.p;
}

// ---- per-device streams, events and one-time attributes -------------------
// Streams and events belong to the device that was current when they were
// created, so the library caches them per (host thread, device): a thread
// that later calls on another device gets that device's own objects.
namespace {
struct DevObjs {
    std::map<std::string, cudaStream_t> streams;
    std::map<std::string, std::vector<cudaEvent_t>> events;
};
thread_local std::map<int, DevObjs> g_objs;
std::mutex g_once_mu;
std::map<std::pair<int, const void *>, bool> g_once;
}  // namespace

int current_device() {
    int dev = 0;
    cudaGetDevice(&dev);
    return dev;
}

int cached_stream(const char *name, int prio, cudaStream_t *out) {
    DevObjs &o = g_objs[current_device()];
    auto it = o.streams.find(name);
    if (it != o.streams.end()) {
        *out = it->second;
        return 0;
    }
    int least = 0, greatest = 0;
    CQ_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest), "stream priorities");
    int p = least;  // prio 0: default priority
    if (prio == 1) p = greatest;
    if (prio == 2) p = greatest < least ? greatest + 1 : least;
    cudaStream_t s = nullptr;
    CQ_CUDA(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, p), name);
    o.streams[name] = s;
    *out = s;
    return 0;
}

int cached_events(const char *name, size_t count, cudaEvent_t **out) {
    std::vector<cudaEvent_t> &v = g_objs[current_device()].events[name];
    while (v.size() < count) {
        cudaEvent_t e;
        CQ_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), name);
        v.push_back(e);
    }
    *out = v.data();
    return 0;
}

bool first_on_device(const void *key) {
    std::lock_guard<std::mutex> g(g_once_mu);
    bool &done = g_once[{current_device(), key}];
    if (done) return false;
    done = true;
    return true;
}

size_t ws_bytes(const char *name) {
    int dev = 0;
    cudaGetDevice(&dev);
    auto it = g_ws.find({dev, name});
    return it == g_ws.end() ? 0 : it->second.bytes;
}

Workspace &workspace() {
    static thread_local Workspace ws;
    return ws;
}

void release_workspace() {
    cudaDeviceSynchronize();
    for (auto &kv : g_ws)
        if (kv.second.p) cudaFree(kv.second.p);
    g_ws.clear();
}

// ---------------------------------------------------------------------------
// device utilities
// ---------------------------------------------------------------------------
__global__ void fill_identity_kernel(int64_t n, double *a, int64_t lda) {
    int64_t j = blockIdx.x;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) a[j * lda + i] = (i == j) ? 1.0 : 0.0;
}
int fill_identity(int64_t n, double *a, int64_t lda, cudaStream_t st) {
    if (n <= 0) return 0;
    fill_identity_kernel<<<(unsigned)n, 256, 0, st>>>(n, a, lda);
    note_launch();
    return check_launch("fill_identity");
}

__global__ void copy_matrix_kernel(int64_t m, int64_t n, const double *src, int64_t lds, double *dst, int64_t ldd) {
    int64_t j = blockIdx.y;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        dst[j * ldd + i] = src[j * lds + i];
}
int copy_matrix(int64_t m, int64_t n, const double *src, int64_t lds, double *dst, int64_t ldd, cudaStream_t st) {
    if (m <= 0 || n <= 0) return 0;
    unsigned gx = (unsigned)std::min<int64_t>((m + 255) / 256, 64);
    copy_matrix_kernel<<<dim3(gx, (unsigned)n), 256, 0, st>>>(m, n, src, lds, dst, ldd);
    note_launch();
    return check_launch("copy_matrix");
}

// per-column sums of squares of the upper triangle (rows <= j), then a fixed-order total
__global__ void colsq_upper_kernel(int64_t n, const double *a, int64_t lda, double *colsq) {
    __shared__ double sc[32];
    int64_t j = blockIdx.x;
    double s = 0.0;
    for (int64_t i = threadIdx.x; i <= j && i < n; i += blockDim.x) {
        double v = a[j * lda + i];
        s = fma(v, v, s);
    }
    s = block_sum(s, sc);
    if (threadIdx.x == 0) colsq[j] = s;
}
__global__ void sum_kernel(int64_t n, const double *v, double *out) {
    __shared__ double sc[32];
    double s = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += v[i];
    s = block_sum(s, sc);
    if (threadIdx.x == 0) out[0] = s;
}
int frob_norm_upper(int64_t n, const double *a, int64_t lda, double *out_host, Workspace &ws, cudaStream_t st) {
    if (n <= 0) {
        *out_host = 0.0;
        return 0;
    }
    double *colsq = ws.get<double>("frob.col", n);
    double *tot = ws.get<double>("frob.tot", 1);
    colsq_upper_kernel<<<(unsigned)n, 256, 0, st>>>(n, a, lda, colsq);
    note_launch();
    sum_kernel<<<1, 1024, 0, st>>>(n, colsq, tot);
    note_launch();
    CQ_TRY(check_launch("frob_norm_upper"));
    double h = 0.0;
    CQ_CUDA(cudaMemcpyAsync(&h, tot, sizeof(double), cudaMemcpyDeviceToHost, st), "frob d2h");
    CQ_CUDA(cudaStreamSynchronize(st), "frob sync");
    *out_host = sqrt(h);
    return 0;
}

}  // namespace cqg

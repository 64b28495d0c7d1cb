// capi.cu -- the extern "C" boundary (include/questkv_b200.h): argument validation with
// the reference's error semantics, cache allocation, and dispatch to the kernels.
// No exception crosses this boundary; every failure is a status code plus a
// thread-local message.
#include <cmath>
#include <chrono>
#include <cstring>
#include <map>
#include <mutex>
#include <new>
#include <string>
#include <utility>

#include "qk_internal.cuh"

namespace qk {

namespace {
thread_local std::string g_last_error;
}

int set_error(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

int cuda_check(cudaError_t err, const char* what) {
    if (err == cudaSuccess) return QK_OK;
    return set_error(QK_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(err));
}

int ensure_func_attrs(const void* func, size_t smem, int device, bool nonportable_cluster,
                      const char* what) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, size_t> configured;  // (func, device) -> smem
    std::lock_guard<std::mutex> lock(mu);
    size_t& have = configured[{func, device}];
    if (have >= smem && have != 0) return QK_OK;
    if (int rc = cuda_check(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 int(smem)), what))
        return rc;
    if (nonportable_cluster)
        if (int rc = cuda_check(cudaFuncSetAttribute(func, cudaFuncAttributeNonPortableClusterSizeAllowed, 1),
                                what))
            return rc;
    have = smem ? smem : 1;
    return QK_OK;
}

namespace {

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

inline cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

int check_layer_batch(const qk_cache* c, uint32_t layer, uint32_t batch, const char* fn) {
    if (layer >= c->L)
        return set_error(QK_ERR_OUT_OF_RANGE, std::string(fn) + ": layer out of range");
    if (batch == 0 || batch > c->B)
        return set_error(QK_ERR_INVALID_ARGUMENT,
                         std::string(fn) + ": batch must be in 1..max_batch");
    return QK_OK;
}

uint32_t pages_of(const qk_cache* c, uint32_t tokens) { return (tokens + c->S - 1) / c->S; }

// Max page count over sequences [0, batch) of a layer (host shadow); 0 if any is empty
// and `require_nonempty`.
uint32_t max_pages(const qk_cache* c, uint32_t layer, uint32_t batch, bool* any_empty) {
    uint32_t m = 0;
    *any_empty = false;
    for (uint32_t b = 0; b < batch; ++b) {
        const uint32_t t = c->h_len[size_t(layer) * c->B + b];
        if (t == 0) *any_empty = true;
        const uint32_t p = pages_of(c, t);
        m = p > m ? p : m;
    }
    return m;
}

template <typename T>
int dmalloc(qk_cache* c, T** p, size_t count) {
    const size_t bytes = count * sizeof(T);
    const cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), bytes ? bytes : 16);
    if (e != cudaSuccess) return cuda_check(e, "cudaMalloc");
    c->device_bytes += bytes;
    return cuda_check(cudaMemset(*p, 0, bytes ? bytes : 16), "cudaMemset");
}

// Pinned, mapped blocks handed out by qk_host_alloc: [host address, (bytes, device view)].
// Caller buffers inside one of them are read and written by the host step's kernel in place;
// a registry lookup costs ~50 ns where cudaPointerGetAttributes costs ~1 us per pointer.
struct HostBlock {
    size_t bytes;
    unsigned char* dev;
};
std::mutex g_host_mu;
std::map<uintptr_t, HostBlock> g_host_blocks;

template <typename T>
T* mapped_host(T* p, size_t bytes) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(p);
    std::lock_guard<std::mutex> lock(g_host_mu);
    auto it = g_host_blocks.upper_bound(a);
    if (it == g_host_blocks.begin()) return nullptr;
    --it;
    if (a + bytes > it->first + it->second.bytes) return nullptr;
    return reinterpret_cast<T*>(it->second.dev + (a - it->first));
}

void free_cache(qk_cache* c) {
    void* ptrs[] = {c->k_pool,    c->v_pool,    c->meta,      c->d_len,     c->ws_partial,
                    c->ws_ticket, c->d_status,  c->ws_scores, c->ws_pages,  c->ws_counts,
                    c->ws_io,     c->ws_out,    c->len_ticket, c->probe,     c->ws_lse,
                    c->prange,    c->done_counter, c->ws_wsum};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    if (c->host_stage) cudaFreeHost(c->host_stage);
    for (auto& hg : c->host_graphs)
        if (hg.exec) cudaGraphExecDestroy(hg.exec);
    if (c->capture_stream) cudaStreamDestroy(c->capture_stream);
    delete c;
}

}  // namespace
}  // namespace qk

using namespace qk;

extern "C" {

const char* qk_last_error(void) { return g_last_error.c_str(); }
int qk_abi_version(void) { return QK_ABI_VERSION; }

int qk_cache_create(const qk_cache_desc* desc, qk_cache** out) {
    if (!desc || !out) return set_error(QK_ERR_INVALID_ARGUMENT, "qk_cache_create: null argument");
    *out = nullptr;
    // CacheConfig::validate, kv_store.cpp:8-13 (same messages).
    if (desc->head_dim == 0)
        return set_error(QK_ERR_INVALID_ARGUMENT, "CacheConfig: head_dim must be >= 1");
    if (desc->page_size == 0)
        return set_error(QK_ERR_INVALID_ARGUMENT, "CacheConfig: page_size must be >= 1");
    if (desc->bytes_per_element == 0)
        return set_error(QK_ERR_INVALID_ARGUMENT, "CacheConfig: bytes_per_element must be >= 1");
    if (desc->bytes_per_element != 2)
        return set_error(QK_ERR_UNSUPPORTED, "qk_cache_create: pools are fp16 (bytes_per_element 2)");
    if (desc->head_dim > 256)
        return set_error(QK_ERR_UNSUPPORTED, "qk_cache_create: head_dim > 256");
    if (desc->page_size > 64)
        return set_error(QK_ERR_UNSUPPORTED, "qk_cache_create: page_size > 64");
    if (desc->num_layers == 0 || desc->max_batch == 0 || desc->num_q_heads == 0 ||
        desc->num_kv_heads == 0 || desc->max_tokens == 0)
        return set_error(QK_ERR_INVALID_ARGUMENT, "qk_cache_create: zero dimension");
    if (desc->num_q_heads % desc->num_kv_heads != 0)
        return set_error(QK_ERR_INVALID_ARGUMENT,
                         "qk_cache_create: num_q_heads must be a multiple of num_kv_heads");
    const uint32_t G = desc->num_q_heads / desc->num_kv_heads;
    if (G != 1 && G != 2 && G != 4 && G != 8)
        return set_error(QK_ERR_UNSUPPORTED, "qk_cache_create: GQA group must be 1, 2, 4 or 8");
    const uint64_t pmax = (uint64_t(desc->max_tokens) + desc->page_size - 1) / desc->page_size;
    if (pmax > kMaxPages)
        return set_error(QK_ERR_UNSUPPORTED, "qk_cache_create: more than 16384 pages per slice");

    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return set_error(QK_ERR_CUDA, "qk_cache_create: no CUDA device (this library has no CPU path)");
    if (desc->device < 0 || desc->device >= ndev)
        return set_error(QK_ERR_INVALID_ARGUMENT, "qk_cache_create: bad device ordinal");
    DeviceGuard guard(desc->device);

    qk_cache* c = new (std::nothrow) qk_cache;
    if (!c) return set_error(QK_ERR_CUDA, "qk_cache_create: out of host memory");
    c->desc = *desc;
    c->D = desc->head_dim <= 64 ? 64 : (desc->head_dim <= 128 ? 128 : 256);
    c->S = desc->page_size;
    c->L = desc->num_layers;
    c->B = desc->max_batch;
    c->Hq = desc->num_q_heads;
    c->Hkv = desc->num_kv_heads;
    c->G = G;
    c->Pmax = uint32_t(pmax);
    c->Mrow = (c->Pmax + kMetaAlign - 1) / kMetaAlign * kMetaAlign;
    c->slice_kv = size_t(c->Pmax) * c->S * c->D;
    c->slice_meta = size_t(2) * c->D * c->Mrow;
    const size_t slices = size_t(c->L) * c->B * c->Hkv;
    c->h_len.assign(size_t(c->L) * c->B, 0);
    int rc = QK_OK;
    if (!rc) rc = dmalloc(c, &c->k_pool, slices * c->slice_kv);
    if (!rc) rc = dmalloc(c, &c->v_pool, slices * c->slice_kv);
    if (!rc) rc = dmalloc(c, &c->meta, slices * c->slice_meta);
    if (!rc) rc = dmalloc(c, &c->prange, slices * c->Mrow);
    if (!rc) rc = dmalloc(c, &c->d_len, size_t(c->L) * c->B);
    if (!rc) rc = dmalloc(c, &c->ws_partial, size_t(c->B) * c->Hq * kMaxSplits * (c->D + 2));
    if (!rc) rc = dmalloc(c, &c->ws_ticket, size_t(c->B) * c->Hq);
    if (!rc) rc = dmalloc(c, &c->d_status, 1);
    if (!rc) rc = dmalloc(c, &c->len_ticket, size_t(c->L) * c->B);
    if (!rc && getenv("QK_PROBE")) rc = dmalloc(c, &c->probe, size_t(c->L) * c->B * c->Hkv * kMaxClusterCtas * kProbeSlots);
    if (!rc) rc = dmalloc(c, &c->ws_scores, size_t(c->B) * c->Hq * c->Pmax);
    if (!rc) rc = dmalloc(c, &c->ws_pages, size_t(c->B) * c->Hq * c->Pmax);
    if (!rc) rc = dmalloc(c, &c->ws_counts, size_t(c->B) * c->Hq);
    if (!rc) rc = dmalloc(c, &c->ws_io, size_t(c->B) * (c->Hq + 2 * c->Hkv) * desc->head_dim);
    if (!rc) rc = dmalloc(c, &c->ws_out, size_t(c->B) * c->Hq * desc->head_dim);
    if (!rc) rc = dmalloc(c, &c->ws_lse, size_t(c->B) * c->Hq);
    if (!rc) rc = dmalloc(c, &c->ws_wsum, size_t(c->B) * c->Hq);
    if (!rc) rc = cuda_check(cudaDeviceSynchronize(), "qk_cache_create");
    if (rc) {
        free_cache(c);
        return rc;
    }
    *out = c;
    return QK_OK;
}

int qk_cache_destroy(qk_cache* c) {
    if (!c) return QK_OK;
    DeviceGuard guard(c->desc.device);
    cudaDeviceSynchronize();
    free_cache(c);
    return QK_OK;
}

int qk_cache_describe(const qk_cache* c, qk_cache_desc* out) {
    if (!c || !out) return set_error(QK_ERR_INVALID_ARGUMENT, "qk_cache_describe: null argument");
    *out = c->desc;
    return QK_OK;
}

int qk_cache_reserve(qk_cache* c, uint32_t max_tokens) {
    if (!c) return set_error(QK_ERR_INVALID_ARGUMENT, "qk_cache_reserve: null cache");
    if (max_tokens <= c->desc.max_tokens) return QK_OK;
    const uint64_t pmax = (uint64_t(max_tokens) + c->S - 1) / c->S;
    if (pmax > kMaxPages)
        return set_error(QK_ERR_UNSUPPORTED, "qk_cache_reserve: more than 16384 pages per slice");
    DeviceGuard guard(c->desc.device);
    if (int rc = cuda_check(cudaDeviceSynchronize(), "qk_cache_reserve")) return rc;
    if (uint32_t(pmax) == c->Pmax) {  // the last page already has room
        c->desc.max_tokens = max_tokens;
        return QK_OK;
    }
    const uint32_t Pn = uint32_t(pmax);
    const uint32_t Mn = (Pn + kMetaAlign - 1) / kMetaAlign * kMetaAlign;
    const size_t kv_n = size_t(Pn) * c->S * c->D, meta_n = size_t(2) * c->D * Mn;
    const size_t slices = size_t(c->L) * c->B * c->Hkv;
    const size_t ws_n = size_t(c->B) * c->Hq * Pn;
    // New buffers, zero-filled like qk_cache_create's; on failure the cache is untouched.
    struct Buf {
        void** slot;
        size_t bytes;
        void* p;
    } bufs[] = {{reinterpret_cast<void**>(&c->k_pool), slices * kv_n * 2, nullptr},
                {reinterpret_cast<void**>(&c->v_pool), slices * kv_n * 2, nullptr},
                {reinterpret_cast<void**>(&c->meta), slices * meta_n * 2, nullptr},
                {reinterpret_cast<void**>(&c->prange), slices * Mn * 4, nullptr},
                {reinterpret_cast<void**>(&c->ws_scores), ws_n * 8, nullptr},
                {reinterpret_cast<void**>(&c->ws_pages), ws_n * 4, nullptr}};
    int rc = QK_OK;
    for (Buf& b : bufs) {
        if (!rc) rc = cuda_check(cudaMalloc(&b.p, b.bytes), "qk_cache_reserve: cudaMalloc");
        if (!rc) rc = cuda_check(cudaMemset(b.p, 0, b.bytes), "qk_cache_reserve: cudaMemset");
    }
    // Per slice: the cached pages ([Pmax][S][D] contiguous), every metadata row ([2][D] rows
    // of Mrow pages) and the page records keep their offsets inside the longer rows.
    if (!rc) rc = cuda_check(cudaMemcpy2D(bufs[0].p, kv_n * 2, c->k_pool, c->slice_kv * 2,
                                          c->slice_kv * 2, slices, cudaMemcpyDeviceToDevice),
                             "qk_cache_reserve: copy K");
    if (!rc) rc = cuda_check(cudaMemcpy2D(bufs[1].p, kv_n * 2, c->v_pool, c->slice_kv * 2,
                                          c->slice_kv * 2, slices, cudaMemcpyDeviceToDevice),
                             "qk_cache_reserve: copy V");
    if (!rc) rc = cuda_check(cudaMemcpy2D(bufs[2].p, size_t(Mn) * 2, c->meta, size_t(c->Mrow) * 2,
                                          size_t(c->Mrow) * 2, slices * 2 * c->D,
                                          cudaMemcpyDeviceToDevice),
                             "qk_cache_reserve: copy metadata");
    if (!rc) rc = cuda_check(cudaMemcpy2D(bufs[3].p, size_t(Mn) * 4, c->prange, size_t(c->Mrow) * 4,
                                          size_t(c->Mrow) * 4, slices, cudaMemcpyDeviceToDevice),
                             "qk_cache_reserve: copy page records");
    if (!rc) rc = cuda_check(cudaDeviceSynchronize(), "qk_cache_reserve");
    if (rc) {
        for (Buf& b : bufs)
            if (b.p) cudaFree(b.p);
        return rc;
    }
    for (Buf& b : bufs) {
        cudaFree(*b.slot);
        *b.slot = b.p;
    }
    c->device_bytes += (bufs[0].bytes + bufs[1].bytes + bufs[2].bytes + bufs[3].bytes +
                        bufs[4].bytes + bufs[5].bytes) -
                       (slices * (2 * c->slice_kv * 2 + c->slice_meta * 2 + size_t(c->Mrow) * 4) +
                        size_t(c->B) * c->Hq * c->Pmax * 12);
    c->desc.max_tokens = max_tokens;
    c->Pmax = Pn;
    c->Mrow = Mn;
    c->slice_kv = kv_n;
    c->slice_meta = meta_n;
    // The host step's graphs hold the old pool pointers.
    for (auto& hg : c->host_graphs) {
        if (hg.exec) cudaGraphExecDestroy(hg.exec);
        hg.exec = nullptr;
        hg.key.clear();
    }
    return QK_OK;
}

uint64_t qk_cache_device_bytes(const qk_cache* c) { return c ? c->device_bytes : 0; }
uint32_t qk_cache_max_pages(const qk_cache* c) { return c ? c->Pmax : 0; }
uint64_t qk_kernel_launches(const qk_cache* c) { return c ? c->launches.load() : 0; }

int qk_token_count(const qk_cache* c, uint32_t layer, uint32_t seq, uint32_t* count) {
    if (!c || !count) return set_error(QK_ERR_INVALID_ARGUMENT, "qk_token_count: null argument");
    if (layer >= c->L || seq >= c->B)
        return set_error(QK_ERR_OUT_OF_RANGE, "qk_token_count: slice out of range");
    *count = c->h_len[size_t(layer) * c->B + seq];
    return QK_OK;
}

int qk_page_count(const qk_cache* c, uint32_t layer, uint32_t seq, uint32_t* count) {
    uint32_t t = 0;
    const int rc = qk_token_count(c, layer, seq, &t);
    if (rc) return rc;
    *count = pages_of(c, t);
    return QK_OK;
}

int qk_reset(qk_cache* c, uint32_t layer, void* stream) {
    if (!c) return set_error(QK_ERR_INVALID_ARGUMENT, "qk_reset: null cache");
    DeviceGuard guard(c->desc.device);
    if (layer == UINT32_MAX) {
        std::fill(c->h_len.begin(), c->h_len.end(), 0u);
        return cuda_check(cudaMemsetAsync(c->d_len, 0, sizeof(int32_t) * c->L * c->B,
                                          as_stream(stream)),
                          "qk_reset");
    }
    if (layer >= c->L) return set_error(QK_ERR_OUT_OF_RANGE, "qk_reset: layer out of range");
    std::fill(c->h_len.begin() + size_t(layer) * c->B, c->h_len.begin() + size_t(layer + 1) * c->B, 0u);
    return cuda_check(cudaMemsetAsync(c->d_len + size_t(layer) * c->B, 0, sizeof(int32_t) * c->B,
                                      as_stream(stream)),
                      "qk_reset");
}

int qk_append(qk_cache* c, uint32_t layer, const uint16_t* k, const uint16_t* v,
              uint32_t batch, void* stream) {
    if (!c || !k || !v) return set_error(QK_ERR_INVALID_ARGUMENT, "KvCache::append: null argument");
    if (int rc = check_layer_batch(c, layer, batch, "KvCache::append")) return rc;
    for (uint32_t b = 0; b < batch; ++b)
        if (c->h_len[size_t(layer) * c->B + b] >= c->desc.max_tokens)
            return set_error(QK_ERR_OUT_OF_RANGE, "KvCache::append: cache slice is full");
    DeviceGuard guard(c->desc.device);
    const int rc = launch_append(c, layer, reinterpret_cast<const __half*>(k),
                                 reinterpret_cast<const __half*>(v), batch, as_stream(stream));
    if (rc) return rc;
    for (uint32_t b = 0; b < batch; ++b) c->h_len[size_t(layer) * c->B + b] += 1;
    return QK_OK;
}

int qk_prefill(qk_cache* c, uint32_t layer, uint32_t seq, const uint16_t* k, const uint16_t* v,
               uint32_t n_tokens, void* stream) {
    if (!c || !k || !v) return set_error(QK_ERR_INVALID_ARGUMENT, "qk_prefill: null argument");
    if (layer >= c->L || seq >= c->B)
        return set_error(QK_ERR_OUT_OF_RANGE, "qk_prefill: slice out of range");
    if (n_tokens == 0) return QK_OK;
    uint32_t& t = c->h_len[size_t(layer) * c->B + seq];
    if (uint64_t(t) + n_tokens > c->desc.max_tokens)
        return set_error(QK_ERR_OUT_OF_RANGE, "qk_prefill: exceeds cache capacity");
    DeviceGuard guard(c->desc.device);
    const int rc = launch_prefill(c, layer, seq, reinterpret_cast<const __half*>(k),
                                  reinterpret_cast<const __half*>(v), n_tokens, t,
                                  as_stream(stream));
    if (rc) return rc;
    t += n_tokens;
    return QK_OK;
}

}  // extern "C"

namespace qk {
namespace readback {

__global__ void gather_meta_kernel(const __half* __restrict__ meta, __half* __restrict__ mn,
                                   __half* __restrict__ mx, size_t slice_meta, uint32_t mrow,
                                   size_t s, uint32_t page0, uint32_t n, int D,
                                   uint32_t head_dim) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n * head_dim) return;
    const uint32_t p = page0 + i / head_dim, ch = i % head_dim;
    mn[i] = meta[meta_offset(slice_meta, mrow, s, p, D, 0, int(ch))];
    mx[i] = meta[meta_offset(slice_meta, mrow, s, p, D, 1, int(ch))];
}

__global__ void gather_kv_kernel(const __half* __restrict__ kp, const __half* __restrict__ vp,
                                 __half* __restrict__ ko, __half* __restrict__ vo, size_t base,
                                 uint32_t t0, uint32_t n, int D, uint32_t head_dim) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n * head_dim) return;
    const uint32_t t = t0 + i / head_dim, ch = i % head_dim;
    const size_t off = base + size_t(t) * D + ch;  // token t = page*S + row
    ko[i] = kp[off];
    vo[i] = vp[off];
}

int read_back(qk_cache* c, __half* d0, __half* d1, uint16_t* h0, uint16_t* h1, size_t n,
              cudaStream_t st) {
    int rc = cuda_check(cudaMemcpyAsync(h0, d0, n * 2, cudaMemcpyDeviceToHost, st), "read");
    if (!rc) rc = cuda_check(cudaMemcpyAsync(h1, d1, n * 2, cudaMemcpyDeviceToHost, st), "read");
    if (!rc) rc = cuda_check(cudaStreamSynchronize(st), "read");
    return rc;
}

// out / lse / weights_sum device workspaces -> host (asynchronous on st).
int copy_results(qk_cache* c, float* out_host, float* lse_host, double* wsum_host, size_t rows,
                 size_t nq, cudaStream_t st) {
    int rc = cuda_check(cudaMemcpyAsync(out_host, c->ws_out, nq * 4, cudaMemcpyDeviceToHost, st), "d2h out");
    if (!rc && lse_host)
        rc = cuda_check(cudaMemcpyAsync(lse_host, c->ws_lse, rows * 4, cudaMemcpyDeviceToHost, st), "d2h lse");
    if (!rc && wsum_host)
        rc = cuda_check(cudaMemcpyAsync(wsum_host, c->ws_wsum, rows * 8, cudaMemcpyDeviceToHost, st), "d2h wsum");
    return rc;
}

// check_token_set (attention.cpp:19-30) on host lists, same errors and messages.
int check_token_sets(const qk_cache* c, uint32_t layer, const int32_t* tokens, uint32_t stride,
                     const int32_t* counts, size_t rows) {
    for (size_t r = 0; r < rows; ++r) {
        const uint32_t L = c->h_len[size_t(layer) * c->B + r / c->Hq];
        const int32_t n = counts[r];
        if (n <= 0) return set_error(QK_ERR_INVALID_ARGUMENT, "attention: empty token set");
        if (uint32_t(n) > stride)
            return set_error(QK_ERR_INVALID_ARGUMENT, "attention: token count above tokens_stride");
        const int32_t* tl = tokens + r * stride;
        for (int32_t i = 0; i < n; ++i) {
            if (tl[i] < 0 || uint32_t(tl[i]) >= L)
                return set_error(QK_ERR_OUT_OF_RANGE, "attention: token index out of range");
            if (i > 0 && tl[i] <= tl[i - 1])
                return set_error(QK_ERR_INVALID_ARGUMENT, "attention: token set must be strictly ascending");
        }
    }
    return QK_OK;
}

}  // namespace readback
}  // namespace qk

using namespace qk::readback;

extern "C" {

int qk_read_metadata(const qk_cache* cc, uint32_t layer, uint32_t seq, uint32_t kv_head,
                     uint32_t page0, uint32_t n_pages, uint16_t* min_host, uint16_t* max_host,
                     void* stream) {
    qk_cache* c = const_cast<qk_cache*>(cc);
    if (!c || !min_host || !max_host)
        return set_error(QK_ERR_INVALID_ARGUMENT, "KvCache::page_metadata: null argument");
    if (layer >= c->L || seq >= c->B || kv_head >= c->Hkv)
        return set_error(QK_ERR_OUT_OF_RANGE, "KvCache::page_metadata: slice out of range");
    const uint32_t P = pages_of(c, c->h_len[size_t(layer) * c->B + seq]);
    if (uint64_t(page0) + n_pages > P)
        return set_error(QK_ERR_OUT_OF_RANGE, "KvCache::page_metadata: page index " +
                                                  std::to_string(page0 + n_pages - 1) +
                                                  " out of range");
    if (n_pages == 0) return QK_OK;
    DeviceGuard guard(c->desc.device);
    cudaStream_t st = as_stream(stream);
    const size_t n = size_t(n_pages) * c->desc.head_dim;
    __half* tmp = nullptr;
    int rc = cuda_check(cudaMalloc(&tmp, 2 * n * sizeof(__half)), "qk_read_metadata");
    if (rc) return rc;
    gather_meta_kernel<<<unsigned((n + 255) / 256), 256, 0, st>>>(
        c->meta, tmp, tmp + n, c->slice_meta, c->Mrow, c->slice(layer, seq, kv_head), page0,
        n_pages, c->D, c->desc.head_dim);
    c->launches++;
    rc = cuda_check(cudaGetLastError(), "gather_meta_kernel");
    if (!rc) rc = read_back(c, tmp, tmp + n, min_host, max_host, n, st);
    cudaFree(tmp);
    return rc;
}

int qk_read_kv(const qk_cache* cc, uint32_t layer, uint32_t seq, uint32_t kv_head,
               uint32_t token0, uint32_t n_tokens, uint16_t* k_host, uint16_t* v_host,
               void* stream) {
    qk_cache* c = const_cast<qk_cache*>(cc);
    if (!c || !k_host || !v_host)
        return set_error(QK_ERR_INVALID_ARGUMENT, "KvCache::key: null argument");
    if (layer >= c->L || seq >= c->B || kv_head >= c->Hkv)
        return set_error(QK_ERR_OUT_OF_RANGE, "KvCache::key: slice out of range");
    if (uint64_t(token0) + n_tokens > c->h_len[size_t(layer) * c->B + seq])
        return set_error(QK_ERR_OUT_OF_RANGE, "KvCache::key: token " +
                                                  std::to_string(token0 + n_tokens - 1) +
                                                  " out of range");
    if (n_tokens == 0) return QK_OK;
    DeviceGuard guard(c->desc.device);
    cudaStream_t st = as_stream(stream);
    const size_t n = size_t(n_tokens) * c->desc.head_dim;
    __half* tmp = nullptr;
    int rc = cuda_check(cudaMalloc(&tmp, 2 * n * sizeof(__half)), "qk_read_kv");
    if (rc) return rc;
    gather_kv_kernel<<<unsigned((n + 255) / 256), 256, 0, st>>>(
        c->k_pool, c->v_pool, tmp, tmp + n, c->slice(layer, seq, kv_head) * c->slice_kv, token0,
        n_tokens, c->D, c->desc.head_dim);
    c->launches++;
    rc = cuda_check(cudaGetLastError(), "gather_kv_kernel");
    if (!rc) rc = read_back(c, tmp, tmp + n, k_host, v_host, n, st);
    cudaFree(tmp);
    return rc;
}

int qk_estimate(const qk_cache* c, uint32_t layer, const uint16_t* q, uint32_t batch,
                double* scores, uint32_t scores_stride, void* stream) {
    if (!c || !q || !scores) return set_error(QK_ERR_INVALID_ARGUMENT, "estimate_all: null argument");
    if (int rc = check_layer_batch(c, layer, batch, "estimate_all")) return rc;
    bool empty = false;
    const uint32_t mp = max_pages(c, layer, batch, &empty);
    if (empty) return set_error(QK_ERR_INVALID_ARGUMENT, "estimate_all: empty cache");
    if (scores_stride < mp)
        return set_error(QK_ERR_INVALID_ARGUMENT, "estimate_all: scores_stride below page count");
    DeviceGuard guard(c->desc.device);
    return launch_estimate(c, layer, reinterpret_cast<const __half*>(q), batch, scores,
                           scores_stride, c->Pmax, as_stream(stream));
}

int qk_select_topk(const qk_cache* c, uint32_t layer, const double* scores,
                   uint32_t scores_stride, uint32_t batch, const qk_selection_cfg* cfg,
                   int32_t* pages, uint32_t pages_stride, int32_t* counts, void* stream) {
    if (!c || !scores || !cfg || !pages || !counts)
        return set_error(QK_ERR_INVALID_ARGUMENT, "select_top_k: null argument");
    if (int rc = check_layer_batch(c, layer, batch, "select_top_k")) return rc;
    bool empty = false;
    const uint32_t mp = max_pages(c, layer, batch, &empty);
    qk_selection_cfg eff = *cfg;
    if (!cfg->per_layer_enabled) {
        eff.token_budget = UINT32_MAX;  // every page (criticality.cpp:47)
    } else {
        if (cfg->token_budget < c->S)
            return set_error(QK_ERR_INVALID_ARGUMENT, "select_top_k: token_budget below page_size");
        if (empty) return set_error(QK_ERR_INVALID_ARGUMENT, "select_top_k: no scores");
    }
    const uint32_t k = eff.token_budget / c->S;
    const uint32_t need = k < mp ? k : mp;
    if (pages_stride < need)
        return set_error(QK_ERR_INVALID_ARGUMENT, "select_top_k: pages_stride below selection size");
    if (scores_stride < mp)
        return set_error(QK_ERR_INVALID_ARGUMENT, "select_top_k: scores_stride below page count");
    DeviceGuard guard(c->desc.device);
    return launch_topk(c, layer, scores, scores_stride, batch, eff, pages, pages_stride, counts,
                       c->Pmax, as_stream(stream));
}

int qk_select_topk_pairs(qk_cache* c, uint32_t layer, uint32_t seq, const uint32_t* page_index,
                         const double* scores, uint32_t n, const qk_selection_cfg* cfg,
                         int32_t* pages, uint32_t pages_capacity, int32_t* count, void* stream) {
    if (!c || !cfg || !pages || !count || (n && (!page_index || !scores)))
        return set_error(QK_ERR_INVALID_ARGUMENT, "select_top_k: null argument");
    if (layer >= c->L || seq >= c->B)
        return set_error(QK_ERR_OUT_OF_RANGE, "select_top_k: slice out of range");
    // criticality.cpp:46-59, in the reference's order.
    int all_pages = 0;
    uint32_t k = 0;
    if (!cfg->per_layer_enabled) {
        all_pages = 2;
    } else {
        if (cfg->token_budget < c->S)
            return set_error(QK_ERR_INVALID_ARGUMENT, "select_top_k: token_budget below page_size");
        if (n == 0) return set_error(QK_ERR_INVALID_ARGUMENT, "select_top_k: no scores");
        if (n > kMaxPages)
            return set_error(QK_ERR_UNSUPPORTED, "select_top_k: more than 16384 scores");
        k = cfg->token_budget / c->S;
        if (k >= n) all_pages = 1;
        else if (pages_capacity < k)
            return set_error(QK_ERR_INVALID_ARGUMENT, "select_top_k: pages capacity below K");
    }
    if (all_pages && pages_capacity < pages_of(c, c->h_len[size_t(layer) * c->B + seq]))
        return set_error(QK_ERR_INVALID_ARGUMENT, "select_top_k: pages capacity below page count");
    DeviceGuard guard(c->desc.device);
    return launch_topk_pairs(c, layer, seq, page_index, scores, all_pages == 2 ? 0 : n, k,
                             cfg->force_include_recent ? 1 : 0, all_pages, pages_capacity, pages,
                             count, as_stream(stream));
}

int qk_select_topk_pairs_host(qk_cache* c, uint32_t layer, uint32_t seq,
                              const uint32_t* page_index_host, const double* scores_host,
                              uint32_t n, const qk_selection_cfg* cfg, int32_t* pages_host,
                              uint32_t pages_capacity, int32_t* count_host, void* stream) {
    if (!c || !cfg || !pages_host || !count_host || (n && (!page_index_host || !scores_host)))
        return set_error(QK_ERR_INVALID_ARGUMENT, "select_top_k: null argument");
    if (layer >= c->L || seq >= c->B)
        return set_error(QK_ERR_OUT_OF_RANGE, "select_top_k: slice out of range");
    if (cfg->per_layer_enabled) {  // the reference's checks, host side first (same order)
        if (cfg->token_budget < c->S)
            return set_error(QK_ERR_INVALID_ARGUMENT, "select_top_k: token_budget below page_size");
        if (n == 0) return set_error(QK_ERR_INVALID_ARGUMENT, "select_top_k: no scores");
        const uint32_t P = pages_of(c, c->h_len[size_t(layer) * c->B + seq]);
        for (uint32_t i = 0; i < n; ++i)
            if (page_index_host[i] >= P)
                return set_error(QK_ERR_OUT_OF_RANGE, "select_top_k: score for nonexistent page");
    }
    DeviceGuard guard(c->desc.device);
    cudaStream_t st = as_stream(stream);
    void* buf = nullptr;
    const size_t nb = size_t(n) * 12 + size_t(pages_capacity) * 4 + 16;
    int rc = cuda_check(cudaMalloc(&buf, nb), "select_top_k");
    if (rc) return rc;
    double* dsc = static_cast<double*>(buf);
    uint32_t* dpi = reinterpret_cast<uint32_t*>(dsc + n);
    int32_t* dpages = reinterpret_cast<int32_t*>(dpi + n);
    int32_t* dcount = dpages + pages_capacity;
    if (n) rc = cuda_check(cudaMemcpyAsync(dsc, scores_host, size_t(n) * 8, cudaMemcpyHostToDevice, st), "h2d");
    if (!rc && n) rc = cuda_check(cudaMemcpyAsync(dpi, page_index_host, size_t(n) * 4, cudaMemcpyHostToDevice, st), "h2d");
    if (!rc) rc = qk_select_topk_pairs(c, layer, seq, dpi, dsc, n, cfg, dpages, pages_capacity, dcount, stream);
    if (!rc) rc = cuda_check(cudaMemcpyAsync(count_host, dcount, 4, cudaMemcpyDeviceToHost, st), "d2h");
    if (!rc) rc = cuda_check(cudaStreamSynchronize(st), "select_top_k");
    if (!rc && *count_host > 0)
        rc = cuda_check(cudaMemcpy(pages_host, dpages, size_t(*count_host) * 4, cudaMemcpyDeviceToHost), "d2h");
    cudaFree(buf);
    if (!rc) rc = qk_check_status(c, stream);
    return rc;
}

int qk_sparse_attend(const qk_cache* c, uint32_t layer, const uint16_t* q, uint32_t batch,
                     const int32_t* pages, uint32_t pages_stride, const int32_t* counts,
                     void* out, int32_t out_dtype, float* lse, double* weights_sum,
                     void* stream) {
    if (!c || !q || !pages || !counts || !out)
        return set_error(QK_ERR_INVALID_ARGUMENT, "sparse_attention: null argument");
    if (int rc = check_layer_batch(c, layer, batch, "sparse_attention")) return rc;
    if (out_dtype != QK_DTYPE_F32 && out_dtype != QK_DTYPE_F16)
        return set_error(QK_ERR_INVALID_ARGUMENT, "sparse_attention: bad out_dtype");
    bool empty = false;
    const uint32_t mp = max_pages(c, layer, batch, &empty);
    if (empty) return set_error(QK_ERR_INVALID_ARGUMENT, "sparse_attention: empty cache");
    const uint32_t max_list = pages_stride < c->Pmax ? pages_stride : c->Pmax;
    DeviceGuard guard(c->desc.device);
    return launch_attend(c, layer, reinterpret_cast<const __half*>(q), batch, pages, pages_stride,
                         counts, kModePages, max_list, out, out_dtype, lse, weights_sum,
                         as_stream(stream));
}

int qk_dense_attend(const qk_cache* c, uint32_t layer, const uint16_t* q, uint32_t batch,
                    void* out, int32_t out_dtype, float* lse, double* weights_sum, void* stream) {
    if (!c || !q || !out) return set_error(QK_ERR_INVALID_ARGUMENT, "full_attention: null argument");
    if (int rc = check_layer_batch(c, layer, batch, "full_attention")) return rc;
    if (out_dtype != QK_DTYPE_F32 && out_dtype != QK_DTYPE_F16)
        return set_error(QK_ERR_INVALID_ARGUMENT, "full_attention: bad out_dtype");
    bool empty = false;
    const uint32_t mp = max_pages(c, layer, batch, &empty);
    if (empty) return set_error(QK_ERR_INVALID_ARGUMENT, "full_attention: empty cache");
    DeviceGuard guard(c->desc.device);
    return launch_attend(c, layer, reinterpret_cast<const __half*>(q), batch, nullptr, 0, nullptr,
                         kModeDense, c->Pmax, out, out_dtype, lse, weights_sum, as_stream(stream));
}

int qk_attend_tokens(const qk_cache* c, uint32_t layer, const uint16_t* q, uint32_t batch,
                     const int32_t* tokens, uint32_t tokens_stride, const int32_t* counts,
                     void* out, int32_t out_dtype, float* lse, double* weights_sum,
                     void* stream) {
    if (!c || !q || !tokens || !counts || !out)
        return set_error(QK_ERR_INVALID_ARGUMENT, "attend_tokens: null argument");
    if (int rc = check_layer_batch(c, layer, batch, "attend_tokens")) return rc;
    if (out_dtype != QK_DTYPE_F32 && out_dtype != QK_DTYPE_F16)
        return set_error(QK_ERR_INVALID_ARGUMENT, "attend_tokens: bad out_dtype");
    if (tokens_stride == 0) return set_error(QK_ERR_INVALID_ARGUMENT, "attention: empty token set");
    const uint64_t cap = uint64_t(c->Pmax) * c->S;
    const uint32_t max_list = uint32_t(tokens_stride < cap ? tokens_stride : cap);
    DeviceGuard guard(c->desc.device);
    return launch_attend(c, layer, reinterpret_cast<const __half*>(q), batch, tokens, tokens_stride,
                         counts, kModeTokens, max_list, out, out_dtype, lse, weights_sum,
                         as_stream(stream));
}

int qk_attention_logits(const qk_cache* c, uint32_t layer, const uint16_t* q, uint32_t batch,
                        const int32_t* tokens, uint32_t tokens_stride, const int32_t* counts,
                        double* logits, uint32_t logits_stride, void* stream) {
    if (!c || !q || !logits || (tokens && !counts))
        return set_error(QK_ERR_INVALID_ARGUMENT, "attention_logits: null argument");
    if (int rc = check_layer_batch(c, layer, batch, "attention_logits")) return rc;
    uint32_t max_list = 0;
    if (tokens) {
        if (tokens_stride == 0) return set_error(QK_ERR_INVALID_ARGUMENT, "attention: empty token set");
        max_list = tokens_stride;
    } else {
        for (uint32_t b = 0; b < batch; ++b) {
            const uint32_t t = c->h_len[size_t(layer) * c->B + b];
            if (t == 0) return set_error(QK_ERR_INVALID_ARGUMENT, "attention: empty token set");
            max_list = t > max_list ? t : max_list;
        }
        // Sized for the capacity: the device length decides (graph replays may grow it).
        max_list = c->desc.max_tokens;
    }
    if (logits_stride < (tokens ? tokens_stride : 1))
        return set_error(QK_ERR_INVALID_ARGUMENT, "attention_logits: logits_stride below the list");
    DeviceGuard guard(c->desc.device);
    return launch_logits(c, layer, reinterpret_cast<const __half*>(q), batch, tokens, tokens_stride,
                         counts, max_list, logits, logits_stride, as_stream(stream));
}

int qk_softmax_weights(qk_cache* c, const double* logits, const int32_t* counts, uint32_t n,
                       uint32_t stride, uint32_t rows, double* weights, void* stream) {
    if (!c || !logits || !weights)
        return set_error(QK_ERR_INVALID_ARGUMENT, "softmax_weights: null argument");
    if (!counts && n == 0) return set_error(QK_ERR_INVALID_ARGUMENT, "softmax_weights: empty logits");
    if (!counts && n > stride)
        return set_error(QK_ERR_INVALID_ARGUMENT, "softmax_weights: n above stride");
    DeviceGuard guard(c->desc.device);
    return launch_softmax(logits, counts, n, stride, rows, weights, c->d_status, as_stream(stream));
}

int qk_decode_step(qk_cache* c, uint32_t layer, const uint16_t* q, const uint16_t* k,
                   const uint16_t* v, uint32_t batch, const qk_selection_cfg* cfg, void* out,
                   int32_t out_dtype, int32_t* pages_out, uint32_t pages_stride,
                   int32_t* counts_out, void* stream) {
    if (!c || !q || !cfg || !out) return set_error(QK_ERR_INVALID_ARGUMENT, "qk_decode_step: null argument");
    if (int rc = check_layer_batch(c, layer, batch, "qk_decode_step")) return rc;
    if ((k == nullptr) != (v == nullptr))
        return set_error(QK_ERR_INVALID_ARGUMENT, "qk_decode_step: k and v must both be given");
    if (out_dtype != QK_DTYPE_F32 && out_dtype != QK_DTYPE_F16)
        return set_error(QK_ERR_INVALID_ARGUMENT, "qk_decode_step: bad out_dtype");
    if (cfg->per_layer_enabled && cfg->token_budget < c->S)
        return set_error(QK_ERR_INVALID_ARGUMENT, "select_top_k: token_budget below page_size");
    const uint32_t add = k ? 1 : 0;
    bool empty = false;
    for (uint32_t b = 0; b < batch; ++b) {
        const uint32_t t = c->h_len[size_t(layer) * c->B + b];
        if (t + add > c->desc.max_tokens)
            return set_error(QK_ERR_OUT_OF_RANGE, "KvCache::append: cache slice is full");
        if (t + add == 0) empty = true;
    }
    if (empty) return set_error(QK_ERR_INVALID_ARGUMENT, "estimate_all: empty cache");
    uint32_t mp = 0;
    for (uint32_t b = 0; b < batch; ++b) {
        const uint32_t p = pages_of(c, c->h_len[size_t(layer) * c->B + b] + add);
        mp = p > mp ? p : mp;
    }
    if (pages_out) {
        const uint32_t kk = cfg->per_layer_enabled ? cfg->token_budget / c->S : UINT32_MAX;
        const uint32_t need = kk < mp ? kk : mp;
        if (pages_stride < need)
            return set_error(QK_ERR_INVALID_ARGUMENT, "qk_decode_step: pages_stride below selection size");
    }
    DeviceGuard guard(c->desc.device);
    const int rc = launch_decode(c, layer, reinterpret_cast<const __half*>(q),
                                 reinterpret_cast<const __half*>(k),
                                 reinterpret_cast<const __half*>(v), batch, *cfg, mp, out,
                                 out_dtype, pages_out, pages_stride, counts_out,
                                 as_stream(stream));
    if (rc) return rc;
    if (add)
        for (uint32_t b = 0; b < batch; ++b) c->h_len[size_t(layer) * c->B + b] += 1;
    return QK_OK;
}

int qk_select_topk_grouped(const qk_cache* c, uint32_t layer, const double* scores,
                           uint32_t scores_stride, uint32_t batch, const qk_selection_cfg* cfg,
                           int32_t group_reduce, int32_t* pages, uint32_t pages_stride,
                           int32_t* counts, void* stream) {
    if (!c || !scores || !cfg || !pages || !counts)
        return set_error(QK_ERR_INVALID_ARGUMENT, "select_top_k: null argument");
    if (int rc = check_layer_batch(c, layer, batch, "select_top_k")) return rc;
    if (group_reduce != QK_GROUP_MAX && group_reduce != QK_GROUP_SUM)
        return set_error(QK_ERR_INVALID_ARGUMENT, "select_top_k: bad group_reduce");
    bool empty = false;
    const uint32_t mp = max_pages(c, layer, batch, &empty);
    uint32_t kk = UINT32_MAX;  // every page (criticality.cpp:47)
    if (cfg->per_layer_enabled) {
        if (cfg->token_budget < c->S)
            return set_error(QK_ERR_INVALID_ARGUMENT, "select_top_k: token_budget below page_size");
        if (empty) return set_error(QK_ERR_INVALID_ARGUMENT, "select_top_k: no scores");
        kk = cfg->token_budget / c->S;
    }
    const uint32_t need = kk < mp ? kk : mp;
    if (pages_stride < need)
        return set_error(QK_ERR_INVALID_ARGUMENT, "select_top_k: pages_stride below selection size");
    if (scores_stride < mp)
        return set_error(QK_ERR_INVALID_ARGUMENT, "select_top_k: scores_stride below page count");
    if (c->G > 8 || (c->G & (c->G - 1)))
        return set_error(QK_ERR_UNSUPPORTED, "grouped decode: GQA group must be 1, 2, 4 or 8");
    DeviceGuard guard(c->desc.device);
    return launch_group_topk(c, layer, scores, scores_stride, batch, kk,
                             cfg->force_include_recent ? 1 : 0, group_reduce, pages,
                             pages_stride, counts, as_stream(stream));
}

int qk_sparse_attend_grouped(const qk_cache* c, uint32_t layer, const uint16_t* q, uint32_t batch,
                             const int32_t* pages, uint32_t pages_stride, const int32_t* counts,
                             void* out, int32_t out_dtype, void* stream) {
    if (!c || !q || !pages || !counts || !out)
        return set_error(QK_ERR_INVALID_ARGUMENT, "sparse_attention: null argument");
    if (int rc = check_layer_batch(c, layer, batch, "sparse_attention")) return rc;
    if (out_dtype != QK_DTYPE_F32 && out_dtype != QK_DTYPE_F16)
        return set_error(QK_ERR_INVALID_ARGUMENT, "sparse_attention: bad out_dtype");
    if (pages_stride == 0)
        return set_error(QK_ERR_INVALID_ARGUMENT, "sparse_attention: pages_stride is 0");
    DeviceGuard guard(c->desc.device);
    const uint32_t max_list = pages_stride < c->Pmax ? pages_stride : c->Pmax;
    return launch_group_attend(c, layer, reinterpret_cast<const __half*>(q), batch, pages,
                               pages_stride, counts, max_list, out, out_dtype, as_stream(stream));
}

int qk_decode_step_grouped(qk_cache* c, uint32_t layer, const uint16_t* q, const uint16_t* k,
                           const uint16_t* v, uint32_t batch, const qk_selection_cfg* cfg,
                           int32_t group_reduce, void* out, int32_t out_dtype, int32_t* pages_out,
                           uint32_t pages_stride, int32_t* counts_out, void* stream) {
    if (!c || !q || !cfg || !out)
        return set_error(QK_ERR_INVALID_ARGUMENT, "qk_decode_step_grouped: null argument");
    if (int rc = check_layer_batch(c, layer, batch, "qk_decode_step_grouped")) return rc;
    if ((k == nullptr) != (v == nullptr))
        return set_error(QK_ERR_INVALID_ARGUMENT, "qk_decode_step_grouped: k and v must both be given");
    if (out_dtype != QK_DTYPE_F32 && out_dtype != QK_DTYPE_F16)
        return set_error(QK_ERR_INVALID_ARGUMENT, "qk_decode_step_grouped: bad out_dtype");
    if (group_reduce != QK_GROUP_MAX && group_reduce != QK_GROUP_SUM)
        return set_error(QK_ERR_INVALID_ARGUMENT, "qk_decode_step_grouped: bad group_reduce");
    if (cfg->per_layer_enabled && cfg->token_budget < c->S)
        return set_error(QK_ERR_INVALID_ARGUMENT, "select_top_k: token_budget below page_size");
    if (c->G > 8 || (c->G & (c->G - 1)) || c->D > 128)
        return set_error(QK_ERR_UNSUPPORTED,
                         "grouped decode: GQA group must be 1, 2, 4 or 8 and head_dim <= 128");
    const uint32_t add = k ? 1 : 0;
    uint32_t mp = 0;
    for (uint32_t b = 0; b < batch; ++b) {
        const uint32_t t = c->h_len[size_t(layer) * c->B + b];
        if (t + add > c->desc.max_tokens)
            return set_error(QK_ERR_OUT_OF_RANGE, "KvCache::append: cache slice is full");
        if (t + add == 0) return set_error(QK_ERR_INVALID_ARGUMENT, "estimate_all: empty cache");
        const uint32_t p = pages_of(c, t + add);
        mp = p > mp ? p : mp;
    }
    const uint32_t kk = cfg->per_layer_enabled ? cfg->token_budget / c->S : UINT32_MAX;
    const uint32_t need = kk < mp ? kk : mp;
    if (pages_out) {
        if (pages_stride < need || (kk >= c->Pmax && pages_stride < c->Pmax))
            return set_error(QK_ERR_INVALID_ARGUMENT,
                             "qk_decode_step_grouped: pages_stride below selection size");
    }
    DeviceGuard guard(c->desc.device);
    const int rc = launch_decode_grouped(c, layer, reinterpret_cast<const __half*>(q),
                                         reinterpret_cast<const __half*>(k),
                                         reinterpret_cast<const __half*>(v), batch, *cfg,
                                         group_reduce, mp, out, out_dtype, pages_out, pages_stride,
                                         counts_out, as_stream(stream));
    if (rc) return rc;
    if (add)
        for (uint32_t b = 0; b < batch; ++b) c->h_len[size_t(layer) * c->B + b] += 1;
    return QK_OK;
}

int qk_decode_step_host(qk_cache* c, uint32_t layer, const uint16_t* q_host,
                        const uint16_t* k_host, const uint16_t* v_host, uint32_t batch,
                        const qk_selection_cfg* cfg, float* out_host, void* stream) {
    if (!c || !q_host || !cfg || !out_host)
        return set_error(QK_ERR_INVALID_ARGUMENT, "qk_decode_step_host: null argument");
    if (int rc = check_layer_batch(c, layer, batch, "qk_decode_step_host")) return rc;
    if ((k_host == nullptr) != (v_host == nullptr))
        return set_error(QK_ERR_INVALID_ARGUMENT, "qk_decode_step_host: k and v must both be given");
    DeviceGuard guard(c->desc.device);
    cudaStream_t st = as_stream(stream);
    const size_t hd = c->desc.head_dim;
    const size_t nq = size_t(batch) * c->Hq * hd, nkv = size_t(batch) * c->Hkv * hd;
    // Inputs and output go through a pinned, device-mapped staging buffer that the fused
    // kernel reads and writes directly (zero-copy): one launch and one synchronisation per
    // call instead of three host-to-device copies, the kernel and a device-to-host copy.
    // Regions rounded to 64 bytes: the kernel does 4-byte output stores and the completion
    // word is a 4-byte atomic (an odd head_dim would otherwise misalign both).
    const size_t in_max = (size_t(c->B) * (c->Hq + 2 * c->Hkv) * hd * 2 + 63) & ~size_t(63);
    const size_t out_max = (size_t(c->B) * c->Hq * hd * 4 + 63) & ~size_t(63);
    if (!c->host_stage) {
        void* h = nullptr;
        int rc = cuda_check(cudaHostAlloc(&h, in_max + out_max + 64, cudaHostAllocMapped), "cudaHostAlloc");
        if (rc) return rc;
        void* d = nullptr;
        rc = cuda_check(cudaHostGetDevicePointer(&d, h, 0), "cudaHostGetDevicePointer");
        if (!rc) rc = cuda_check(cudaMalloc(&c->done_counter, 2 * sizeof(uint32_t)), "cudaMalloc done");
        if (!rc) rc = cuda_check(cudaMemset(c->done_counter, 0, 2 * sizeof(uint32_t)), "cudaMemset done");
        if (rc) {
            cudaFreeHost(h);
            return rc;
        }
        c->host_stage = static_cast<unsigned char*>(h);
        c->host_stage_dev = static_cast<unsigned char*>(d);
        c->done_flag_dev = reinterpret_cast<uint32_t*>(c->host_stage_dev + in_max + out_max);
        *reinterpret_cast<volatile uint32_t*>(c->host_stage + in_max + out_max) = 0;
    }
    // Caller buffers that are already pinned and device-mapped (cudaHostAlloc, torch
    // pin_memory, cudaHostRegister) are read and written by the kernel in place; pageable
    // ones go through the staging buffer.
    uint16_t* hq = reinterpret_cast<uint16_t*>(c->host_stage);
    const uint16_t* dq = mapped_host(q_host, nq * 2);
    const uint16_t* dk = k_host ? mapped_host(k_host, nkv * 2) : nullptr;
    const uint16_t* dv = k_host ? mapped_host(v_host, nkv * 2) : nullptr;
    if (!dq) {
        std::memcpy(hq, q_host, nq * 2);
        dq = reinterpret_cast<const uint16_t*>(c->host_stage_dev);
    }
    if (k_host && !dk) {
        std::memcpy(hq + nq, k_host, nkv * 2);
        dk = reinterpret_cast<const uint16_t*>(c->host_stage_dev) + nq;
    }
    if (k_host && !dv) {
        std::memcpy(hq + nq + nkv, v_host, nkv * 2);
        dv = reinterpret_cast<const uint16_t*>(c->host_stage_dev) + nq + nkv;
    }
    float* mapped_out = mapped_host(out_host, size_t(batch) * c->Hq * hd * 4);
    float* dout = mapped_out ? mapped_out : reinterpret_cast<float*>(c->host_stage_dev + in_max);
    // Completion: the fused kernel's last unit publishes `seq` in the mapped word, so the host
    // spins on it (~1 us after the last output lands) instead of synchronising the stream.
    // Paths that do not consume the request (unfused fallback) synchronise as before.
    // The kernel publishes the device's count of completed host steps: the host expects one
    // more than the last value it saw (advanced only when a fused launch consumed the request).
    const uint32_t seq = c->done_seq + 1u;
    c->pending_done_flag = c->done_flag_dev;
    if (c->host_graphs.size() != c->L) c->host_graphs.resize(c->L);
    static const int no_graph = getenv("QK_NO_HOST_GRAPH") ? 1 : 0;  // read once
    c->host_graph_mode = !no_graph;
    int rc = qk_decode_step(c, layer, dq, dk, dv, batch, cfg, dout, QK_DTYPE_F32, nullptr, 0,
                            nullptr, stream);
    c->host_graph_mode = false;
    const bool signalled = c->pending_done_flag == nullptr;  // consumed by a fused launch
    c->pending_done_flag = nullptr;
    if (signalled && !rc) c->done_seq = seq;
    if (!rc && signalled) {
        const volatile uint32_t* word = reinterpret_cast<volatile uint32_t*>(c->host_stage + in_max + out_max);
        const auto t0 = std::chrono::steady_clock::now();
        while (__atomic_load_n(const_cast<const uint32_t*>(word), __ATOMIC_ACQUIRE) != seq) {
            // A kernel that faults never signals: after a generous wait, let the stream
            // synchronisation report the error.
            if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(2)) {
                rc = cuda_check(cudaStreamSynchronize(st), "qk_decode_step_host");
                if (!rc && __atomic_load_n(const_cast<const uint32_t*>(word), __ATOMIC_ACQUIRE) != seq)
                    rc = set_error(QK_ERR_CUDA, "qk_decode_step_host: completion not signalled");
                break;
            }
        }
    } else if (!rc) {
        rc = cuda_check(cudaStreamSynchronize(st), "qk_decode_step_host");
    }
    if (!rc && !mapped_out) std::memcpy(out_host, c->host_stage + in_max, size_t(batch) * c->Hq * hd * 4);
    return rc;
}

void* qk_host_alloc(size_t bytes) {
    void* p = nullptr;
    void* d = nullptr;
    if (bytes == 0) bytes = 16;
    if (cudaHostAlloc(&p, bytes, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess ||
        cudaHostGetDevicePointer(&d, p, 0) != cudaSuccess) {
        cudaGetLastError();
        if (p) cudaFreeHost(p);
        set_error(QK_ERR_CUDA, "qk_host_alloc: cudaHostAlloc failed");
        return nullptr;
    }
    std::lock_guard<std::mutex> lock(g_host_mu);
    g_host_blocks[reinterpret_cast<uintptr_t>(p)] = HostBlock{bytes, static_cast<unsigned char*>(d)};
    return p;
}

void qk_host_free(void* p) {
    if (!p) return;
    {
        std::lock_guard<std::mutex> lock(g_host_mu);
        if (g_host_blocks.erase(reinterpret_cast<uintptr_t>(p)) == 0) return;  // not ours
    }
    cudaFreeHost(p);
}

// ---- host-buffer variants (the questkv:: C++ layer, include/questkv_b200.hpp) ----------
// Each stages its inputs into the cache's device workspaces, runs the device entry point
// on `stream` and copies the result back; synchronous.

int qk_append_host(qk_cache* c, uint32_t layer, const uint16_t* k_host, const uint16_t* v_host,
                   uint32_t batch, void* stream) {
    if (!c || !k_host || !v_host)
        return set_error(QK_ERR_INVALID_ARGUMENT, "KvCache::append: null argument");
    if (int rc = check_layer_batch(c, layer, batch, "KvCache::append")) return rc;
    DeviceGuard guard(c->desc.device);
    cudaStream_t st = as_stream(stream);
    const size_t nkv = size_t(batch) * c->Hkv * c->desc.head_dim;
    uint16_t* dk = c->ws_io;
    uint16_t* dv = dk + nkv;
    int rc = cuda_check(cudaMemcpyAsync(dk, k_host, nkv * 2, cudaMemcpyHostToDevice, st), "h2d k");
    if (!rc) rc = cuda_check(cudaMemcpyAsync(dv, v_host, nkv * 2, cudaMemcpyHostToDevice, st), "h2d v");
    if (!rc) rc = qk_append(c, layer, dk, dv, batch, stream);
    if (!rc) rc = cuda_check(cudaStreamSynchronize(st), "qk_append_host");
    return rc;
}

int qk_prefill_host(qk_cache* c, uint32_t layer, uint32_t seq, const uint16_t* k_host,
                    const uint16_t* v_host, uint32_t n_tokens, void* stream) {
    if (!c || !k_host || !v_host)
        return set_error(QK_ERR_INVALID_ARGUMENT, "qk_prefill: null argument");
    if (n_tokens == 0) return QK_OK;
    DeviceGuard guard(c->desc.device);
    cudaStream_t st = as_stream(stream);
    const size_t n = size_t(c->Hkv) * n_tokens * c->desc.head_dim;
    uint16_t* tmp = nullptr;
    int rc = cuda_check(cudaMalloc(&tmp, 2 * n * sizeof(uint16_t)), "qk_prefill_host");
    if (rc) return rc;
    rc = cuda_check(cudaMemcpyAsync(tmp, k_host, n * 2, cudaMemcpyHostToDevice, st), "h2d k");
    if (!rc) rc = cuda_check(cudaMemcpyAsync(tmp + n, v_host, n * 2, cudaMemcpyHostToDevice, st), "h2d v");
    if (!rc) rc = qk_prefill(c, layer, seq, tmp, tmp + n, n_tokens, stream);
    const int rs = cuda_check(cudaStreamSynchronize(st), "qk_prefill_host");
    cudaFree(tmp);
    return rc ? rc : rs;
}

int qk_estimate_host(const qk_cache* cc, uint32_t layer, const uint16_t* q_host, uint32_t batch,
                     double* scores_host, uint32_t scores_stride, void* stream) {
    qk_cache* c = const_cast<qk_cache*>(cc);
    if (!c || !q_host || !scores_host)
        return set_error(QK_ERR_INVALID_ARGUMENT, "estimate_all: null argument");
    if (int rc = check_layer_batch(c, layer, batch, "estimate_all")) return rc;
    if (scores_stride > c->Pmax)
        return set_error(QK_ERR_INVALID_ARGUMENT, "estimate_all: scores_stride above max_pages");
    DeviceGuard guard(c->desc.device);
    cudaStream_t st = as_stream(stream);
    const size_t nq = size_t(batch) * c->Hq * c->desc.head_dim;
    int rc = cuda_check(cudaMemcpyAsync(c->ws_io, q_host, nq * 2, cudaMemcpyHostToDevice, st), "h2d q");
    if (!rc) rc = qk_estimate(c, layer, c->ws_io, batch, c->ws_scores, c->Pmax, stream);
    if (!rc && scores_stride > 0)
        rc = cuda_check(cudaMemcpy2DAsync(scores_host, size_t(scores_stride) * 8, c->ws_scores,
                                          size_t(c->Pmax) * 8, size_t(scores_stride) * 8,
                                          size_t(batch) * c->Hq, cudaMemcpyDeviceToHost, st),
                        "d2h scores");
    if (!rc) rc = cuda_check(cudaStreamSynchronize(st), "qk_estimate_host");
    return rc;
}

int qk_select_topk_host(const qk_cache* cc, uint32_t layer, const double* scores_host,
                        uint32_t scores_stride, uint32_t batch, const qk_selection_cfg* cfg,
                        int32_t* pages_host, uint32_t pages_stride, int32_t* counts_host,
                        void* stream) {
    qk_cache* c = const_cast<qk_cache*>(cc);
    if (!c || !scores_host || !cfg || !pages_host || !counts_host)
        return set_error(QK_ERR_INVALID_ARGUMENT, "select_top_k: null argument");
    if (int rc = check_layer_batch(c, layer, batch, "select_top_k")) return rc;
    if (scores_stride > c->Pmax || pages_stride > c->Pmax)
        return set_error(QK_ERR_INVALID_ARGUMENT, "select_top_k: stride above max_pages");
    DeviceGuard guard(c->desc.device);
    cudaStream_t st = as_stream(stream);
    const size_t rows = size_t(batch) * c->Hq;
    int rc = QK_OK;
    if (scores_stride > 0)
        rc = cuda_check(cudaMemcpy2DAsync(c->ws_scores, size_t(c->Pmax) * 8, scores_host,
                                          size_t(scores_stride) * 8, size_t(scores_stride) * 8, rows,
                                          cudaMemcpyHostToDevice, st),
                        "h2d scores");
    if (!rc)
        rc = qk_select_topk(c, layer, c->ws_scores, c->Pmax, batch, cfg, c->ws_pages, c->Pmax,
                            c->ws_counts, stream);
    if (!rc && pages_stride > 0)
        rc = cuda_check(cudaMemcpy2DAsync(pages_host, size_t(pages_stride) * 4, c->ws_pages,
                                          size_t(c->Pmax) * 4, size_t(pages_stride) * 4, rows,
                                          cudaMemcpyDeviceToHost, st),
                        "d2h pages");
    if (!rc)
        rc = cuda_check(cudaMemcpyAsync(counts_host, c->ws_counts, rows * 4, cudaMemcpyDeviceToHost, st),
                        "d2h counts");
    if (!rc) rc = cuda_check(cudaStreamSynchronize(st), "qk_select_topk_host");
    return rc;
}

int qk_sparse_attend_host(const qk_cache* cc, uint32_t layer, const uint16_t* q_host,
                          uint32_t batch, const int32_t* pages_host, uint32_t pages_stride,
                          const int32_t* counts_host, float* out_host, float* lse_host,
                          double* wsum_host, void* stream) {
    qk_cache* c = const_cast<qk_cache*>(cc);
    if (!c || !q_host || !pages_host || !counts_host || !out_host)
        return set_error(QK_ERR_INVALID_ARGUMENT, "sparse_attention: null argument");
    if (int rc = check_layer_batch(c, layer, batch, "sparse_attention")) return rc;
    if (pages_stride == 0 || pages_stride > c->Pmax)
        return set_error(QK_ERR_INVALID_ARGUMENT, "sparse_attention: pages_stride must be in 1..max_pages");
    const size_t rows = size_t(batch) * c->Hq;
    // The reference's page-list validation (attention.cpp:99-106), host side, before any
    // device work: empty -> invalid_argument, out of range -> out_of_range, duplicates
    // -> invalid_argument.  Lists must be given ascending (qk_sparse_attend's form).
    for (size_t r = 0; r < rows; ++r) {
        const uint32_t P = pages_of(c, c->h_len[size_t(layer) * c->B + r / c->Hq]);
        const int32_t n = counts_host[r];
        if (n <= 0) return set_error(QK_ERR_INVALID_ARGUMENT, "sparse_attention: empty page selection");
        if (uint32_t(n) > pages_stride)
            return set_error(QK_ERR_INVALID_ARGUMENT, "sparse_attention: count above pages_stride");
        const int32_t* pl = pages_host + r * pages_stride;
        for (int32_t i = 0; i < n; ++i) {
            if (pl[i] < 0 || uint32_t(pl[i]) >= P)
                return set_error(QK_ERR_OUT_OF_RANGE, "sparse_attention: page index out of range");
            if (i > 0 && pl[i] <= pl[i - 1])
                return set_error(QK_ERR_INVALID_ARGUMENT,
                                 pl[i] == pl[i - 1] ? "sparse_attention: duplicate page index"
                                                    : "sparse_attention: page list not ascending");
        }
    }
    DeviceGuard guard(c->desc.device);
    cudaStream_t st = as_stream(stream);
    const size_t nq = rows * c->desc.head_dim;
    float* dlse = lse_host ? c->ws_lse : nullptr;
    int rc = cuda_check(cudaMemcpyAsync(c->ws_io, q_host, nq * 2, cudaMemcpyHostToDevice, st), "h2d q");
    if (!rc)
        rc = cuda_check(cudaMemcpy2DAsync(c->ws_pages, size_t(c->Pmax) * 4, pages_host,
                                          size_t(pages_stride) * 4, size_t(pages_stride) * 4, rows,
                                          cudaMemcpyHostToDevice, st),
                        "h2d pages");
    if (!rc) rc = cuda_check(cudaMemcpyAsync(c->ws_counts, counts_host, rows * 4, cudaMemcpyHostToDevice, st),
                             "h2d counts");
    double* dws = wsum_host ? c->ws_wsum : nullptr;
    if (!rc)
        rc = qk_sparse_attend(c, layer, c->ws_io, batch, c->ws_pages, c->Pmax, c->ws_counts, c->ws_out,
                              QK_DTYPE_F32, dlse, dws, stream);
    if (!rc) rc = copy_results(c, out_host, lse_host, wsum_host, rows, nq, st);
    if (!rc) rc = cuda_check(cudaStreamSynchronize(st), "qk_sparse_attend_host");
    if (!rc) rc = qk_check_status(c, stream);
    return rc;
}

int qk_attend_tokens_host(const qk_cache* cc, uint32_t layer, const uint16_t* q_host,
                          uint32_t batch, const int32_t* tokens_host, uint32_t tokens_stride,
                          const int32_t* counts_host, float* out_host, float* lse_host,
                          double* wsum_host, void* stream) {
    qk_cache* c = const_cast<qk_cache*>(cc);
    if (!c || !q_host || !tokens_host || !counts_host || !out_host)
        return set_error(QK_ERR_INVALID_ARGUMENT, "attend_tokens: null argument");
    if (int rc = check_layer_batch(c, layer, batch, "attend_tokens")) return rc;
    const size_t rows = size_t(batch) * c->Hq;
    if (int rc = check_token_sets(c, layer, tokens_host, tokens_stride, counts_host, rows)) return rc;
    DeviceGuard guard(c->desc.device);
    cudaStream_t st = as_stream(stream);
    const size_t nq = rows * c->desc.head_dim;
    int32_t* dtok = nullptr;
    int rc = cuda_check(cudaMalloc(&dtok, (rows * tokens_stride + rows) * sizeof(int32_t)), "attend_tokens");
    if (rc) return rc;
    int32_t* dcnt = dtok + rows * tokens_stride;
    rc = cuda_check(cudaMemcpyAsync(c->ws_io, q_host, nq * 2, cudaMemcpyHostToDevice, st), "h2d q");
    if (!rc) rc = cuda_check(cudaMemcpyAsync(dtok, tokens_host, rows * tokens_stride * 4, cudaMemcpyHostToDevice, st), "h2d tokens");
    if (!rc) rc = cuda_check(cudaMemcpyAsync(dcnt, counts_host, rows * 4, cudaMemcpyHostToDevice, st), "h2d counts");
    if (!rc)
        rc = qk_attend_tokens(c, layer, c->ws_io, batch, dtok, tokens_stride, dcnt, c->ws_out,
                              QK_DTYPE_F32, lse_host ? c->ws_lse : nullptr,
                              wsum_host ? c->ws_wsum : nullptr, stream);
    if (!rc) rc = copy_results(c, out_host, lse_host, wsum_host, rows, nq, st);
    const int rs = cuda_check(cudaStreamSynchronize(st), "qk_attend_tokens_host");
    cudaFree(dtok);
    if (!rc) rc = rs;
    if (!rc) rc = qk_check_status(c, stream);
    return rc;
}

int qk_attention_logits_host(const qk_cache* cc, uint32_t layer, const uint16_t* q_host,
                             uint32_t batch, const int32_t* tokens_host, uint32_t tokens_stride,
                             const int32_t* counts_host, double* logits_host,
                             uint32_t logits_stride, void* stream) {
    qk_cache* c = const_cast<qk_cache*>(cc);
    if (!c || !q_host || !logits_host || (tokens_host && !counts_host))
        return set_error(QK_ERR_INVALID_ARGUMENT, "attention_logits: null argument");
    if (int rc = check_layer_batch(c, layer, batch, "attention_logits")) return rc;
    const size_t rows = size_t(batch) * c->Hq;
    if (tokens_host) {
        if (int rc = check_token_sets(c, layer, tokens_host, tokens_stride, counts_host, rows)) return rc;
    } else {
        for (uint32_t b = 0; b < batch; ++b) {
            const uint32_t t = c->h_len[size_t(layer) * c->B + b];
            if (t == 0) return set_error(QK_ERR_INVALID_ARGUMENT, "attention: empty token set");
            if (t > logits_stride)
                return set_error(QK_ERR_INVALID_ARGUMENT, "attention_logits: logits_stride below the token count");
        }
    }
    if (tokens_host && logits_stride < tokens_stride)
        return set_error(QK_ERR_INVALID_ARGUMENT, "attention_logits: logits_stride below the list");
    DeviceGuard guard(c->desc.device);
    cudaStream_t st = as_stream(stream);
    const size_t nq = rows * c->desc.head_dim;
    const size_t ntok = tokens_host ? rows * tokens_stride + rows : 0;
    int32_t* dtok = nullptr;
    double* dlog = nullptr;
    int rc = cuda_check(cudaMalloc(&dlog, rows * logits_stride * sizeof(double) + ntok * 4), "attention_logits");
    if (rc) return rc;
    if (tokens_host) dtok = reinterpret_cast<int32_t*>(dlog + rows * logits_stride);
    rc = cuda_check(cudaMemcpyAsync(c->ws_io, q_host, nq * 2, cudaMemcpyHostToDevice, st), "h2d q");
    if (!rc && dtok)
        rc = cuda_check(cudaMemcpyAsync(dtok, tokens_host, rows * tokens_stride * 4, cudaMemcpyHostToDevice, st), "h2d tokens");
    if (!rc && dtok)
        rc = cuda_check(cudaMemcpyAsync(dtok + rows * tokens_stride, counts_host, rows * 4, cudaMemcpyHostToDevice, st), "h2d counts");
    if (!rc)
        rc = qk_attention_logits(c, layer, c->ws_io, batch, dtok, tokens_stride,
                                 dtok ? dtok + rows * tokens_stride : nullptr, dlog, logits_stride, stream);
    if (!rc)
        rc = cuda_check(cudaMemcpyAsync(logits_host, dlog, rows * logits_stride * sizeof(double),
                                        cudaMemcpyDeviceToHost, st), "d2h logits");
    const int rs = cuda_check(cudaStreamSynchronize(st), "qk_attention_logits_host");
    cudaFree(dlog);
    if (!rc) rc = rs;
    if (!rc) rc = qk_check_status(c, stream);
    return rc;
}

int qk_estimate_metadata_host(const uint16_t* q_host, const uint16_t* min_host,
                              const uint16_t* max_host, uint32_t n_pages, uint32_t head_dim,
                              double* scores_host, int32_t device) {
    if (!q_host || (n_pages && (!min_host || !max_host || !scores_host)))
        return set_error(QK_ERR_INVALID_ARGUMENT, "estimate_page_score: null argument");
    if (head_dim == 0) return set_error(QK_ERR_INVALID_ARGUMENT, "estimate_page_score: dimension mismatch");
    if (n_pages == 0) return QK_OK;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return set_error(QK_ERR_CUDA, "estimate_page_score: no CUDA device (this library has no CPU path)");
    if (device < 0 || device >= ndev) return set_error(QK_ERR_INVALID_ARGUMENT, "estimate_page_score: bad device");
    DeviceGuard guard(device);
    // Per-device grow-only scratch (no allocation per call once warm).
    static std::mutex mu;
    static std::map<int, std::pair<void*, size_t>> scratch;
    std::lock_guard<std::mutex> lock(mu);
    const size_t halves = size_t(head_dim) * (1 + 2 * size_t(n_pages));
    const size_t need = ((halves * 2 + 15) & ~size_t(15)) + size_t(n_pages) * 8;
    auto& sl = scratch[device];
    if (sl.second < need) {
        if (sl.first) cudaFree(sl.first);
        sl = {nullptr, 0};
        void* p = nullptr;
        if (int rc = cuda_check(cudaMalloc(&p, need), "estimate_page_score")) return rc;
        sl = {p, need};
    }
    __half* dq = static_cast<__half*>(sl.first);
    __half* dmn = dq + head_dim;
    __half* dmx = dmn + size_t(n_pages) * head_dim;
    double* dout = reinterpret_cast<double*>(static_cast<unsigned char*>(sl.first) +
                                             ((halves * 2 + 15) & ~size_t(15)));
    const size_t nb = size_t(n_pages) * head_dim * 2;
    int rc = cuda_check(cudaMemcpy(dq, q_host, head_dim * 2, cudaMemcpyHostToDevice), "h2d q");
    if (!rc) rc = cuda_check(cudaMemcpy(dmn, min_host, nb, cudaMemcpyHostToDevice), "h2d min");
    if (!rc) rc = cuda_check(cudaMemcpy(dmx, max_host, nb, cudaMemcpyHostToDevice), "h2d max");
    if (!rc) rc = launch_page_scores(dq, dmn, dmx, n_pages, head_dim, dout, nullptr);
    if (!rc) rc = cuda_check(cudaMemcpy(scores_host, dout, size_t(n_pages) * 8, cudaMemcpyDeviceToHost), "d2h");
    return rc;
}

int qk_softmax_weights_host(const double* logits_host, uint32_t n, double* weights_host,
                            int32_t device) {
    if (!logits_host || !weights_host)
        return set_error(QK_ERR_INVALID_ARGUMENT, "softmax_weights: null argument");
    if (n == 0) return set_error(QK_ERR_INVALID_ARGUMENT, "softmax_weights: empty logits");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return set_error(QK_ERR_CUDA, "softmax_weights: no CUDA device (this library has no CPU path)");
    if (device < 0 || device >= ndev) return set_error(QK_ERR_INVALID_ARGUMENT, "softmax_weights: bad device");
    DeviceGuard guard(device);
    double* d = nullptr;
    int rc = cuda_check(cudaMalloc(&d, size_t(n) * 2 * sizeof(double)), "softmax_weights");
    if (rc) return rc;
    rc = cuda_check(cudaMemcpy(d, logits_host, size_t(n) * 8, cudaMemcpyHostToDevice), "h2d logits");
    if (!rc) rc = launch_softmax(d, nullptr, n, n, 1, d + n, nullptr, nullptr);
    if (!rc) rc = cuda_check(cudaMemcpy(weights_host, d + n, size_t(n) * 8, cudaMemcpyDeviceToHost), "d2h weights");
    cudaFree(d);
    return rc;
}

int qk_dense_attend_host(const qk_cache* cc, uint32_t layer, const uint16_t* q_host,
                         uint32_t batch, float* out_host, float* lse_host, double* wsum_host,
                         void* stream) {
    qk_cache* c = const_cast<qk_cache*>(cc);
    if (!c || !q_host || !out_host)
        return set_error(QK_ERR_INVALID_ARGUMENT, "full_attention: null argument");
    if (int rc = check_layer_batch(c, layer, batch, "full_attention")) return rc;
    DeviceGuard guard(c->desc.device);
    cudaStream_t st = as_stream(stream);
    const size_t rows = size_t(batch) * c->Hq;
    const size_t nq = rows * c->desc.head_dim;
    float* dlse = lse_host ? c->ws_lse : nullptr;
    int rc = cuda_check(cudaMemcpyAsync(c->ws_io, q_host, nq * 2, cudaMemcpyHostToDevice, st), "h2d q");
    if (!rc)
        rc = qk_dense_attend(c, layer, c->ws_io, batch, c->ws_out, QK_DTYPE_F32, dlse,
                             wsum_host ? c->ws_wsum : nullptr, stream);
    if (!rc) rc = copy_results(c, out_host, lse_host, wsum_host, rows, nq, st);
    if (!rc) rc = cuda_check(cudaStreamSynchronize(st), "qk_dense_attend_host");
    return rc;
}

int qk_debug_probe(qk_cache* c, uint64_t* host, uint32_t n, void* stream) {
    if (!c || !host) return set_error(QK_ERR_INVALID_ARGUMENT, "qk_debug_probe: null argument");
    if (!c->probe) return set_error(QK_ERR_INVALID_ARGUMENT, "qk_debug_probe: set QK_PROBE=1 before qk_cache_create");
    const size_t cap = size_t(c->L) * c->B * c->Hkv * kMaxClusterCtas * kProbeSlots;
    const size_t cnt = n < cap ? n : cap;
    DeviceGuard guard(c->desc.device);
    cudaStream_t st = as_stream(stream);
    int rc = cuda_check(cudaMemcpyAsync(host, c->probe, cnt * 8, cudaMemcpyDeviceToHost, st), "probe");
    if (!rc) rc = cuda_check(cudaMemsetAsync(c->probe, 0, cap * 8, st), "probe");  // re-arm
    if (!rc) rc = cuda_check(cudaStreamSynchronize(st), "probe");
    return rc;
}

int qk_debug_step_scores(qk_cache* c, uint32_t seq, uint32_t q_head, double* host, uint32_t n,
                         void* stream) {
    if (!c || !host) return set_error(QK_ERR_INVALID_ARGUMENT, "qk_debug_step_scores: null argument");
    if (seq >= c->B || q_head >= c->Hq || n > c->Pmax)
        return set_error(QK_ERR_OUT_OF_RANGE, "qk_debug_step_scores: out of range");
    DeviceGuard guard(c->desc.device);
    cudaStream_t st = as_stream(stream);
    int rc = cuda_check(cudaMemcpyAsync(host, c->ws_scores + (size_t(seq) * c->Hq + q_head) * c->Pmax,
                                        size_t(n) * 8, cudaMemcpyDeviceToHost, st), "scores");
    if (!rc) rc = cuda_check(cudaStreamSynchronize(st), "scores");
    return rc;
}

int qk_debug_keep_scores(qk_cache* c, int32_t on) {
    if (!c) return set_error(QK_ERR_INVALID_ARGUMENT, "qk_debug_keep_scores: null cache");
    c->keep_scores = on != 0;
    return QK_OK;
}

int qk_sync_lengths(qk_cache* c, void* stream) {
    if (!c) return set_error(QK_ERR_INVALID_ARGUMENT, "qk_sync_lengths: null cache");
    DeviceGuard guard(c->desc.device);
    cudaStream_t st = as_stream(stream);
    std::vector<int32_t> tmp(size_t(c->L) * c->B);
    int rc = cuda_check(cudaMemcpyAsync(tmp.data(), c->d_len, tmp.size() * 4,
                                        cudaMemcpyDeviceToHost, st), "qk_sync_lengths");
    if (!rc) rc = cuda_check(cudaStreamSynchronize(st), "qk_sync_lengths");
    if (rc) return rc;
    for (size_t i = 0; i < tmp.size(); ++i) c->h_len[i] = uint32_t(tmp[i]);
    return QK_OK;
}

int qk_check_status(qk_cache* c, void* stream) {
    if (!c) return set_error(QK_ERR_INVALID_ARGUMENT, "qk_check_status: null cache");
    DeviceGuard guard(c->desc.device);
    cudaStream_t st = as_stream(stream);
    int32_t code = 0;
    int rc = cuda_check(cudaMemcpyAsync(&code, c->d_status, 4, cudaMemcpyDeviceToHost, st), "status");
    if (!rc) rc = cuda_check(cudaMemsetAsync(c->d_status, 0, 4, st), "status");
    if (!rc) rc = cuda_check(cudaStreamSynchronize(st), "status");
    if (rc) return rc;
    switch (code) {
        case QK_DEV_OK: return QK_OK;
        case QK_DEV_PAGE_OUT_OF_RANGE:
            return set_error(QK_ERR_OUT_OF_RANGE, "sparse_attention: page index out of range");
        case QK_DEV_PAGE_NOT_ASCENDING:
            return set_error(QK_ERR_INVALID_ARGUMENT,
                             "sparse_attention: page list not strictly ascending (duplicate page index)");
        case QK_DEV_EMPTY_SELECTION:
            return set_error(QK_ERR_INVALID_ARGUMENT, "sparse_attention: empty page selection");
        case QK_DEV_CAPACITY:
            return set_error(QK_ERR_OUT_OF_RANGE, "KvCache::append: cache slice is full");
        case QK_DEV_TOKEN_OUT_OF_RANGE:
            return set_error(QK_ERR_OUT_OF_RANGE, "attention: token index out of range");
        case QK_DEV_TOKEN_NOT_ASCENDING:
            return set_error(QK_ERR_INVALID_ARGUMENT, "attention: token set must be strictly ascending");
        case QK_DEV_EMPTY_TOKENS:
            return set_error(QK_ERR_INVALID_ARGUMENT, "attention: empty token set");
        case QK_DEV_SCORE_PAGE_OUT_OF_RANGE:
            return set_error(QK_ERR_OUT_OF_RANGE, "select_top_k: score for nonexistent page");
        case QK_DEV_BAD_COUNT:
            return set_error(QK_ERR_INVALID_ARGUMENT,
                             "sparse_attention: page count exceeds the page list (pages_stride)");
        default: return set_error(QK_ERR_CUDA, "unknown device status");
    }
}

}  // extern "C"

// qk_internal.cuh -- shared state and helpers of the B200 Quest decode library.
//
// Device layout (all fp16 unless noted), per cache slice s = (layer * max_batch + seq) *
// num_kv_heads + kv_head, D = head_dim padded up to 64/128/256 with zero channels:
//   K pool   k_pool[s][Pmax][S][D]           one page = S*D*2 contiguous bytes (4 KiB at
//   V pool   v_pool[s][Pmax][S][D]           S=16, D=128), the unit of a page fetch
//   metadata meta[s][2][D][Mrow]              channel-major: row (minmax, c) holds channel
//                                            c of every page of the slice (Mrow = Pmax
//                                            rounded up to 64), so a CTA estimating a page
//                                            range reads, per channel, one contiguous run
//                                            of the row the query's sign selects
//   prange   prange[s][Mrow] u32              per-page magnitude record of the metadata
//                                            (page_record below), the certificate that
//                                            lets the fused estimate split its fp64 chain
//   lengths  len[layer][seq]                 int32 token counts (device copy; the host
//                                            keeps a shadow for validation / grid sizing)
// Zero padding channels never change a result: padded q is 0, so every estimate term
// and every logit term they add is +-0.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>
#include <vector>

#include "questkv_b200.h"

namespace qk {

constexpr int kMetaAlign = 64;      // metadata rows are padded to a multiple of 64 pages
constexpr int kMaxSplits = 64;      // split-KV partitions per (sequence, query head)
constexpr int kMinPagesPerSplit = 8;
constexpr uint32_t kMaxClusterCtas = 16;  // fused decode: CTAs per (sequence, KV head)
constexpr int kProbeSlots = 32;           // QK_PROBE globaltimer stamps per fused CTA
constexpr uint32_t kMaxPages = 16384;  // top-K keeps one slice's scores in shared memory

struct Status {
    int code = QK_OK;
    std::string msg;
};

int set_error(int code, const std::string& msg);
int cuda_check(cudaError_t err, const char* what);
// Kernel attributes are per device: raise `func`'s dynamic shared-memory limit to at least
// `smem` bytes (and allow non-portable cluster sizes when asked) on `device`, once per
// (function, device, size); thread-safe.
int ensure_func_attrs(const void* func, size_t smem, int device, bool nonportable_cluster,
                      const char* what);

}  // namespace qk

struct qk_cache {
    qk_cache_desc desc{};
    int D = 0;               // padded head dim
    uint32_t S = 0, L = 0, B = 0, Hq = 0, Hkv = 0, G = 0;
    uint32_t Pmax = 0;       // logical pages per slice
    uint32_t Mrow = 0;       // pages per metadata row (Pmax rounded up to kMetaAlign)
    size_t slice_kv = 0;     // halves per slice in k_pool / v_pool
    size_t slice_meta = 0;   // halves per slice in meta
    __half* k_pool = nullptr;
    __half* v_pool = nullptr;
    __half* meta = nullptr;
    uint32_t* prange = nullptr;          // [slices][Mrow] per-page magnitude records
    int32_t* d_len = nullptr;            // [L][B]
    std::vector<uint32_t> h_len;         // host shadow [L][B]
    float* ws_partial = nullptr;         // [B][Hq][kMaxSplits][D + 2]
    int32_t* ws_ticket = nullptr;        // [B][Hq]
    int32_t* d_status = nullptr;         // first device-side error code
    int32_t* len_ticket = nullptr;       // [L][B] CTAs done with this step's length
    double* ws_scores = nullptr;         // [B][Hq][Pmax]  (fused step)
    int32_t* ws_pages = nullptr;         // [B][Hq][Pmax]
    int32_t* ws_counts = nullptr;        // [B][Hq]
    uint16_t* ws_io = nullptr;           // staging for qk_decode_step_host
    float* ws_out = nullptr;             // [B][Hq][head_dim] fp32
    float* ws_lse = nullptr;             // [B][Hq] fp32 (host-buffer entry points)
    double* ws_wsum = nullptr;           // [B][Hq] f64 weights_sum_check (host-buffer entry points)
    unsigned char* host_stage = nullptr; // pinned, device-mapped staging of the host step
    unsigned char* host_stage_dev = nullptr;  // (q, k, v in; fp32 out), allocated lazily
    // Host-step completion: the last unit of a fused launch writes `seq` into the mapped word
    // (the host spins on it instead of a stream synchronisation).
    uint32_t* done_counter = nullptr;    // device [2]: units finished in the current launch,
                                         // completed host steps (the published sequence)
    uint32_t* done_flag_dev = nullptr;   // device view of the mapped completion word
    uint32_t done_seq = 0;
    uint32_t* pending_done_flag = nullptr;  // set by the host step for the next fused launch;
                                            // launch_decode clears it when it consumes it
    unsigned long long* probe = nullptr; // phase timestamps of the fused kernel (QK_PROBE)
    // Host step: one instantiated CUDA graph per layer holding its fused launch, replayed while
    // the launch (parameters, grid, cluster, shared memory) is unchanged -- a graph launch costs
    // ~1.5 us less host-to-GPU round trip than cudaLaunchKernelEx with cluster attributes.
    struct HostGraph {
        cudaGraphExec_t exec = nullptr;
        std::vector<unsigned char> key;  // bytes of the launch it replays
    };
    std::vector<HostGraph> host_graphs;  // [L]
    cudaStream_t capture_stream = nullptr;
    bool host_graph_mode = false;        // set by qk_decode_step_host around its launch
    bool keep_scores = false;            // fused step: estimate every page, keep scores
    uint64_t device_bytes = 0;
    std::atomic<uint64_t> launches{0};

    size_t slice(uint32_t layer, uint32_t seq, uint32_t h) const {
        return (size_t(layer) * B + seq) * Hkv + h;
    }
};

// Device-side error codes recorded in qk_cache::d_status.
enum : int32_t {
    QK_DEV_OK = 0,
    QK_DEV_PAGE_OUT_OF_RANGE = 1,
    QK_DEV_PAGE_NOT_ASCENDING = 2,
    QK_DEV_EMPTY_SELECTION = 3,
    QK_DEV_CAPACITY = 4,
    QK_DEV_BAD_COUNT = 5,  // a page/token count past its list row or the launched splits
    QK_DEV_TOKEN_OUT_OF_RANGE = 6,   // attend_tokens / attention_logits (check_token_set)
    QK_DEV_TOKEN_NOT_ASCENDING = 7,
    QK_DEV_EMPTY_TOKENS = 8,
    QK_DEV_SCORE_PAGE_OUT_OF_RANGE = 9,  // select_top_k: score for a nonexistent page
};

// launch_attend list modes.
enum : int { kModePages = 0, kModeDense = 1, kModeTokens = 2 };

// Kernel launchers (one translation unit each).
namespace qk {
int launch_append(qk_cache* c, uint32_t layer, const __half* k, const __half* v,
                  uint32_t batch, cudaStream_t st);
int launch_prefill(qk_cache* c, uint32_t layer, uint32_t seq, const __half* k,
                   const __half* v, uint32_t n, uint32_t t0, cudaStream_t st);
int launch_estimate(const qk_cache* c, uint32_t layer, const __half* q, uint32_t batch,
                    double* scores, uint32_t stride, uint32_t max_pages, cudaStream_t st);
int launch_topk(const qk_cache* c, uint32_t layer, const double* scores, uint32_t sstride,
                uint32_t batch, const qk_selection_cfg& cfg, int32_t* pages,
                uint32_t pstride, int32_t* counts, uint32_t max_pages, cudaStream_t st);
int launch_attend(const qk_cache* c, uint32_t layer, const __half* q, uint32_t batch,
                  const int32_t* pages, uint32_t pstride, const int32_t* counts,
                  int mode, uint32_t max_list, void* out, int out_dtype, float* lse,
                  double* weights_sum, cudaStream_t st);
int launch_topk_pairs(const qk_cache* c, uint32_t layer, uint32_t seq, const uint32_t* page_index,
                      const double* score, uint32_t n, uint32_t k, int force, int all_pages,
                      uint32_t capacity, int32_t* pages, int32_t* count, cudaStream_t st);
int launch_logits(const qk_cache* c, uint32_t layer, const __half* q, uint32_t batch,
                  const int32_t* tokens, uint32_t tstride, const int32_t* counts,
                  uint32_t max_list, double* logits, uint32_t lstride, cudaStream_t st);
int launch_page_scores(const __half* q, const __half* mn, const __half* mx, uint32_t n,
                       uint32_t d, double* out, cudaStream_t st);
int launch_softmax(const double* logits, const int32_t* counts, uint32_t n, uint32_t stride,
                   uint32_t rows, double* weights, int32_t* status, cudaStream_t st);
int launch_group_topk(const qk_cache* c, uint32_t layer, const double* scores, uint32_t sstride,
                      uint32_t batch, uint32_t k_budget, int force, int reduce, int32_t* pages,
                      uint32_t pstride, int32_t* counts, cudaStream_t st);
int launch_group_attend(const qk_cache* c, uint32_t layer, const __half* q, uint32_t batch,
                        const int32_t* pages, uint32_t pstride, const int32_t* counts,
                        uint32_t max_list, void* out, int out_dtype, cudaStream_t st);
int launch_decode_grouped(qk_cache* c, uint32_t layer, const __half* q, const __half* k,
                          const __half* v, uint32_t batch, const qk_selection_cfg& cfg,
                          int reduce, uint32_t max_pages_after, void* out, int out_dtype,
                          int32_t* pages, uint32_t pstride, int32_t* counts, cudaStream_t st);
int launch_decode(qk_cache* c, uint32_t layer, const __half* q, const __half* k,
                  const __half* v, uint32_t batch, const qk_selection_cfg& cfg,
                  uint32_t max_pages_after, void* out, int out_dtype, int32_t* pages,
                  uint32_t pstride, int32_t* counts, cudaStream_t st);
}  // namespace qk

// ---- device helpers ------------------------------------------------------------------

namespace qk {

// Offset (halves) of channel c of page `page` in the min (minmax 0) or max (1) row of
// slice s: meta[s][minmax][D][mrow].
__host__ __device__ __forceinline__ size_t meta_offset(size_t slice_meta, uint32_t mrow, size_t s,
                                                       uint32_t page, int D, int minmax, int c) {
    return s * slice_meta + (size_t(minmax) * D + c) * mrow + page;
}

// Per-page magnitude record: bits 0..14 = the largest |x| (fp16 magnitude bits) over the
// page's min and max rows, bits 16..20 = the smallest ulp code over their nonzero values
// (ulp(x) = 2^(code - 24)), 31 when every value is zero.  Computed from the final min/max
// rows by every writer of metadata (append, prefill, the fused step's append).
__device__ __forceinline__ uint32_t ulp_code(uint16_t h) {
    const uint32_t m = h & 0x7fffu;
    if (m == 0) return 31u;
    const uint32_t e = m >> 10;
    return e == 0 ? 0u : e - 1u;
}

// Reduction of the record over the NT threads [0, NT) holding one channel's (min, max)
// each; `scratch` holds NT/32 words; barrier `bar` spans those threads.  Returns the record
// in every participating thread.
template <int NT>
__device__ __forceinline__ uint32_t page_record(__half mn, __half mx, uint32_t* scratch, int bar) {
    const uint16_t a = __half_as_ushort(mn), b = __half_as_ushort(mx);
    const uint32_t mag = max(uint32_t(a & 0x7fffu), uint32_t(b & 0x7fffu));
    const uint32_t code = min(ulp_code(a), ulp_code(b));
    const uint32_t wmag = __reduce_max_sync(0xffffffffu, mag);
    const uint32_t wcode = __reduce_min_sync(0xffffffffu, code);
    if ((threadIdx.x & 31) == 0) scratch[threadIdx.x >> 5] = wmag | (wcode << 16);
    asm volatile("bar.sync %0, %1;" ::"r"(bar), "n"(NT) : "memory");
    uint32_t m = 0, c = 31u;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) {
        const uint32_t r = scratch[w];
        m = max(m, r & 0xffffu);
        c = min(c, r >> 16);
    }
    asm volatile("bar.sync %0, %1;" ::"r"(bar), "n"(NT) : "memory");  // scratch reusable
    return m | (c << 16);
}

__device__ __forceinline__ void record_status(int32_t* status, int32_t code) {
    atomicCAS(status, QK_DEV_OK, code);
}

// Ordered unsigned key of a double: larger double <-> larger key (no NaNs expected).
__device__ __forceinline__ unsigned long long order_key(double x) {
    unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(x));
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

__device__ __forceinline__ int4 ld_nc_v4(const void* p) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N));
}
// cp.async.wait_group with a run-time count (0..7).
__device__ __forceinline__ void cp_async_wait_n(int n) {
    switch (n) {
        case 0: cp_async_wait<0>(); break;
        case 1: cp_async_wait<1>(); break;
        case 2: cp_async_wait<2>(); break;
        case 3: cp_async_wait<3>(); break;
        case 4: cp_async_wait<4>(); break;
        case 5: cp_async_wait<5>(); break;
        case 6: cp_async_wait<6>(); break;
        default: cp_async_wait<7>(); break;
    }
}

}  // namespace qk

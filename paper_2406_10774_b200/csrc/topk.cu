// topk.cu -- per-(sequence, query head) top-K page selection (K3), bit-exact.
//
// Reference: select_top_k, /root/reference/proj/core/src/criticality.cpp:36-81.
//   (1) !per_layer_enabled -> every page (:47)          [host-decided: K = UINT32_MAX]
//   (2) token_budget < page_size -> invalid_argument   [host-checked before launch]
//   (3) K = budget / page_size; K >= page_count -> every page (:58-59)
//   (4) order by (score desc, page asc), take K (:62-71)
//   (5) force_include_recent: if page P-1 is not taken, it replaces the K-th pick (:73-77)
//   (6) ascending output (:79)
// (4)+(5) equal "{P-1} plus the best K-1 of pages [0, P-1)": if P-1 is among the best K,
// the other K-1 picks are the best K-1 of the rest; if it is not, it is not among the
// best K-1 either.  So the kernel selects the best `target` of the candidate pages
// exactly (select.cuh) and appends P-1, the largest index, keeping the output ascending.
#include "topk_rows.cuh"

namespace qk {
namespace {

constexpr int kThreads = 256;

__global__ void __launch_bounds__(kThreads)
topk_kernel(const double* __restrict__ scores, uint32_t sstride, const int32_t* __restrict__ len,
            uint32_t layer, uint32_t B, uint32_t Hq, uint32_t S, uint32_t k_budget, int force,
            int32_t* __restrict__ pages, uint32_t pstride, int32_t* __restrict__ counts) {
    extern __shared__ __align__(16) unsigned long long keys[];  // kThreads * (kpt + 1)
    __shared__ SelectScratch<kThreads> sc;

    const uint32_t bh = blockIdx.x;
    const uint32_t b = bh / Hq;
    const uint32_t n_tok = static_cast<uint32_t>(len[layer * B + b]);
    const uint32_t P = (n_tok + S - 1) / S;
    int32_t* out = pages + size_t(bh) * pstride;

    if (k_budget >= P) {  // (3): every page
        for (uint32_t p = threadIdx.x; p < P && p < pstride; p += kThreads) out[p] = int32_t(p);
        if (threadIdx.x == 0) counts[bh] = int32_t(P);
        return;
    }
    if (P > sstride || k_budget > pstride) return;  // host-checked; never write out of bounds
    const uint32_t n_cand = force ? P - 1 : P;  // pages competing on score
    const uint32_t target = force ? k_budget - 1 : k_budget;
    if (target > 0) {
        unsigned long long kmax, kmin;
        const int kpt = load_keys<kThreads>(scores + size_t(bh) * sstride, n_cand, keys, sc,
                                            &kmax, &kmin);
        block_select<kThreads>(keys, kpt, n_cand, target, kmax, kmin, out, sc);
    }
    if (threadIdx.x == 0) {
        if (force) out[target] = int32_t(P - 1);
        counts[bh] = int32_t(k_budget);
    }
}

}  // namespace

int launch_topk(const qk_cache* c, uint32_t layer, const double* scores, uint32_t sstride,
                uint32_t batch, const qk_selection_cfg& cfg, int32_t* pages,
                uint32_t pstride, int32_t* counts, uint32_t max_pages, cudaStream_t st) {
    const uint32_t k = cfg.token_budget / c->S;
    // Keys of up to max_pages pages per CTA; callers pass the cache capacity so that a CUDA
    // graph captured now stays in bounds when replays grow the context.
    if (max_pages < c->Pmax) max_pages = c->Pmax;
    if (max_pages <= kRowMaxPages) {  // keys in registers (topk_rows.cuh)
        launch_topk_rows<1>(batch * c->Hq, max_pages, scores, sstride, c->d_len, layer, c->B,
                            c->Hq, c->S, k, cfg.force_include_recent, QK_GROUP_MAX, pages,
                            pstride, counts, st);
        const_cast<qk_cache*>(c)->launches++;
        return cuda_check(cudaGetLastError(), "topk_rows_kernel");
    }
    const uint32_t kpt = (max_pages + kThreads - 1) / kThreads;
    const size_t smem = size_t(kThreads) * (kpt + 1) * sizeof(unsigned long long);
    if (int rc = ensure_func_attrs(reinterpret_cast<const void*>(topk_kernel), smem, c->desc.device,
                                   false, "topk_kernel attributes"))
        return rc;
    topk_kernel<<<batch * c->Hq, kThreads, smem, st>>>(scores, sstride, c->d_len, layer, c->B,
                                                       c->Hq, c->S, k, cfg.force_include_recent,
                                                       pages, pstride, counts);
    const_cast<qk_cache*>(c)->launches++;
    return cuda_check(cudaGetLastError(), "topk_kernel");
}

}  // namespace qk

// ---- select_top_k on an arbitrary PageScore vector ----------------------------------------
// criticality.cpp:36-81 applied literally to (page_index, score) pairs in any order, with
// repeated page indices allowed: order by (score desc, page asc) -- one bitonic sort of
// (key, page) in shared memory -- take the first K, apply force_include_recent (the K-th
// pick is replaced by page P-1 when P-1 is not among the K) and sort the K ascending.  The
// caller has handled the early exits (disabled, budget < S, no scores, K >= n).
namespace qk {
namespace {

constexpr int kPairThreads = 1024;

__device__ __forceinline__ bool pair_before(unsigned long long ka, uint32_t pa,
                                            unsigned long long kb, uint32_t pb) {
    return ka > kb || (ka == kb && pa < pb);
}

__global__ void __launch_bounds__(kPairThreads)
topk_pairs_kernel(const uint32_t* __restrict__ page_index, const double* __restrict__ score,
                  uint32_t n, uint32_t npad, const int32_t* __restrict__ len, uint32_t layer,
                  uint32_t B, uint32_t seq, uint32_t S, uint32_t k, int force, int all_pages,
                  uint32_t capacity, int32_t* __restrict__ pages_out,
                  int32_t* __restrict__ count_out, int32_t* __restrict__ status) {
    extern __shared__ __align__(16) unsigned char smem[];
    unsigned long long* key = reinterpret_cast<unsigned long long*>(smem);  // [npad]
    uint32_t* pg = reinterpret_cast<uint32_t*>(key + npad);                 // [npad]
    __shared__ int s_bad, s_has_last;
    const uint32_t P = (uint32_t(len[layer * B + seq]) + S - 1) / S;
    if (threadIdx.x == 0) {
        s_bad = 0;
        s_has_last = 0;
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < npad; i += kPairThreads) {
        if (i < n) {
            const uint32_t p = page_index[i];
            if (p >= P) s_bad = 1;
            key[i] = order_key(__dadd_rn(score[i], 0.0));  // -0 ties +0, as the reference
            pg[i] = p;
        } else {
            key[i] = 0ull;  // below every real key: sorts last
            pg[i] = 0xffffffffu;
        }
    }
    __syncthreads();
    if (s_bad && all_pages != 2) {  // criticality.cpp:54-56 (not checked when disabled, :47)
        if (threadIdx.x == 0) record_status(status, QK_DEV_SCORE_PAGE_OUT_OF_RANGE);
        return;
    }
    if (all_pages) {  // disabled (:47) or K >= #scores (:58-59): every page of the cache
        if (P > capacity) {
            if (threadIdx.x == 0) record_status(status, QK_DEV_BAD_COUNT);
            return;
        }
        for (uint32_t i = threadIdx.x; i < P; i += kPairThreads) pages_out[i] = int32_t(i);
        if (threadIdx.x == 0) *count_out = int32_t(P);
        return;
    }
    // Bitonic sort, "before" first: (key desc, page asc).
    for (uint32_t size = 2; size <= npad; size <<= 1) {
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (uint32_t t = threadIdx.x; t < npad / 2; t += kPairThreads) {
                const uint32_t i = 2 * t - (t & (stride - 1));
                const uint32_t j = i + stride;
                const bool up = (i & size) == 0;  // this run sorts "before"-first
                const unsigned long long ki = key[i], kj = key[j];
                const uint32_t pi = pg[i], pj = pg[j];
                if (pair_before(kj, pj, ki, pi) == up) {
                    key[i] = kj;
                    key[j] = ki;
                    pg[i] = pj;
                    pg[j] = pi;
                }
            }
            __syncthreads();
        }
    }
    // The first k picks; force_include_recent (criticality.cpp:73-77).
    for (uint32_t i = threadIdx.x; i < k; i += kPairThreads)
        if (pg[i] == P - 1) s_has_last = 1;
    __syncthreads();
    if (force && !s_has_last && threadIdx.x == 0) pg[k - 1] = P - 1;
    // Ascending order of the k picks (criticality.cpp:79): sort pg[0..kpad) ascending.
    uint32_t kpad = 1;
    while (kpad < k) kpad <<= 1;
    for (uint32_t i = k + threadIdx.x; i < kpad; i += kPairThreads) pg[i] = 0xffffffffu;
    __syncthreads();
    for (uint32_t size = 2; size <= kpad; size <<= 1) {
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (uint32_t t = threadIdx.x; t < kpad / 2; t += kPairThreads) {
                const uint32_t i = 2 * t - (t & (stride - 1));
                const uint32_t j = i + stride;
                const bool up = (i & size) == 0;
                const uint32_t pi = pg[i], pj = pg[j];
                if ((pj < pi) == up) {
                    pg[i] = pj;
                    pg[j] = pi;
                }
            }
            __syncthreads();
        }
    }
    for (uint32_t i = threadIdx.x; i < k; i += kPairThreads) pages_out[i] = int32_t(pg[i]);
    if (threadIdx.x == 0) *count_out = int32_t(k);
}

}  // namespace

int launch_topk_pairs(const qk_cache* c, uint32_t layer, uint32_t seq, const uint32_t* page_index,
                      const double* score, uint32_t n, uint32_t k, int force, int all_pages,
                      uint32_t capacity, int32_t* pages, int32_t* count, cudaStream_t st) {
    uint32_t npad = 1;
    while (npad < n) npad <<= 1;
    const size_t smem = size_t(npad) * (sizeof(unsigned long long) + sizeof(uint32_t));
    if (int rc = ensure_func_attrs(reinterpret_cast<const void*>(topk_pairs_kernel), smem,
                                   c->desc.device, false, "topk_pairs_kernel attributes"))
        return rc;
    topk_pairs_kernel<<<1, kPairThreads, smem, st>>>(page_index, score, n, npad, c->d_len, layer,
                                                     c->B, seq, c->S, k, force, all_pages,
                                                     capacity, pages, count, c->d_status);
    const_cast<qk_cache*>(c)->launches++;
    return cuda_check(cudaGetLastError(), "topk_pairs_kernel");
}

}  // namespace qk

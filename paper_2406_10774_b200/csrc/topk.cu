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
#include "select.cuh"

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

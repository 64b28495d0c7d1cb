// topk_rows.cuh -- select_top_k over rows of scores, one CTA per row, keys in registers.
//
// Reference: select_top_k, /root/reference/proj/core/src/criticality.cpp:36-81 (see topk.cu
// for the early-exit order and the force_include_recent identity).  Row r of the grid is
// (sequence b = r / rows_per_seq, row h = r % rows_per_seq); its scores are the G score
// rows starting at scores + (b * rows_per_seq + h) * G * sstride, combined per page by
// `reduce` (G = 1: the row itself; G > 1: the GQA group score of grouped.cu -- max, or the
// fp64 sum in head order).  Thread t of the NT-thread CTA holds the keys of candidates
// [16t, 16t + 16) in registers and block_select_reg (select.cuh) selects exactly: one
// 11-bit radix pass on the 32-bit word past the keys' common prefix, the threshold bin
// ranked by (key desc, page asc), heavy ties falling back to the 64-bit multi-pass routine.
// NT * 16 >= the cache capacity, chosen on the host, so a captured graph stays valid.
#pragma once

#include "select.cuh"

namespace qk {

constexpr int kRowKpt = 16;
constexpr uint32_t kRowMaxPages = 512u * kRowKpt;

// The 512 x 16 form serves only wide launches (more rows than SMs): two CTAs per SM at 64
// registers (some spills) beat one at 125 (cfg4: -4 us per layer step).
template <int NT, int G, int KPT = kRowKpt>
__global__ void __launch_bounds__(NT, (NT >= 512 && KPT >= 16) ? 2 : 1)
topk_rows_kernel(const double* __restrict__ scores, uint32_t sstride,
                 const int32_t* __restrict__ len, uint32_t layer, uint32_t B,
                 uint32_t rows_per_seq, uint32_t S, uint32_t k_budget, int force, int reduce,
                 int32_t* __restrict__ pages, uint32_t pstride, int32_t* __restrict__ counts) {
    __shared__ SelectScratch<NT> sc;
    const uint32_t row = blockIdx.x;
    const uint32_t b = row / rows_per_seq;
    const uint32_t n_tok = static_cast<uint32_t>(len[layer * B + b]);
    const uint32_t P = (n_tok + S - 1) / S;
    int32_t* out = pages + size_t(row) * pstride;

    if (k_budget >= P) {  // criticality.cpp:58-59: every page
        for (uint32_t p = threadIdx.x; p < P && p < pstride; p += NT) out[p] = int32_t(p);
        if (threadIdx.x == 0) counts[row] = int32_t(P);
        return;
    }
    if (P > sstride || k_budget > pstride || P > uint32_t(NT) * KPT) return;  // host-checked
    const uint32_t n_cand = force ? P - 1 : P;  // pages competing on score
    const uint32_t target = force ? k_budget - 1 : k_budget;
    const double* src = scores + size_t(row) * G * sstride;
    auto score = [&](uint32_t i) {
        double x = __ldcg(src + i);
#pragma unroll
        for (int g = 1; g < G; ++g) {
            const double y = __ldcg(src + size_t(g) * sstride + i);
            x = reduce == QK_GROUP_SUM ? __dadd_rn(x, y) : (y > x ? y : x);
        }
        // -0 and +0 tie in the reference's sort (criticality.cpp:64-67): canonicalise.
        return order_key(__dadd_rn(x, 0.0));
    };
    if (target > 0) {
        const int t = threadIdx.x;
        const uint32_t i0 = uint32_t(t) * KPT;
        unsigned long long key[KPT];
        if (G == 1 && i0 + KPT <= n_cand && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
            // a full, aligned run: 16-byte loads
            const double2* s2 = reinterpret_cast<const double2*>(src + i0);
#pragma unroll
            for (int j = 0; j < KPT / 2; ++j) {
                const double2 v = __ldcg(s2 + j);
                key[2 * j] = order_key(__dadd_rn(v.x, 0.0));
                key[2 * j + 1] = order_key(__dadd_rn(v.y, 0.0));
            }
        } else {
#pragma unroll
            for (int j = 0; j < KPT; ++j) key[j] = i0 + j < n_cand ? score(i0 + j) : 0ull;
        }
        const unsigned long long ref = score(0);
        block_select_reg<NT, KPT>(key, n_cand, target, ref, out, sc, t, 1);
    }
    if (threadIdx.x == 0) {
        if (force) out[target] = int32_t(P - 1);
        counts[row] = int32_t(k_budget);
    }
}

// Launches topk_rows_kernel with the smallest NT whose NT * 16 keys cover `capacity`
// (<= kRowMaxPages; larger caches use topk.cu's shared-memory selection).
template <int G>
inline cudaError_t launch_topk_rows(uint32_t rows, uint32_t capacity, const double* scores,
                                    uint32_t sstride, const int32_t* len, uint32_t layer,
                                    uint32_t B, uint32_t rows_per_seq, uint32_t S,
                                    uint32_t k_budget, int force, int reduce, int32_t* pages,
                                    uint32_t pstride, int32_t* counts, cudaStream_t st) {
#define QK_TOPK_ROWS_K(NT, KPT)                                                                  \
    topk_rows_kernel<NT, G, KPT><<<rows, NT, 0, st>>>(scores, sstride, len, layer, B,            \
                                                      rows_per_seq, S, k_budget, force, reduce,  \
                                                      pages, pstride, counts)
#define QK_TOPK_ROWS(NT) QK_TOPK_ROWS_K(NT, kRowKpt)
    // A launch of at most one row per SM: twice the threads with half the keys each (the
    // per-thread serial work of the radix pass halves; occupancy does not matter).
    if (rows <= 148u && capacity > 128u * 8u && capacity <= 512u * 8u) {
        if (capacity <= 256u * 8u) QK_TOPK_ROWS_K(256, 8);
        else QK_TOPK_ROWS_K(512, 8);
    } else if (capacity <= 128u * kRowKpt) QK_TOPK_ROWS(128);
    else if (capacity <= 256u * kRowKpt) QK_TOPK_ROWS(256);
    else QK_TOPK_ROWS(512);
#undef QK_TOPK_ROWS
#undef QK_TOPK_ROWS_K
    return cudaGetLastError();
}

}  // namespace qk

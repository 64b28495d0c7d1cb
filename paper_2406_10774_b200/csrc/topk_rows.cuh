// topk_rows.cuh -- select_top_k over rows of scores, one CTA per row, keys in registers.
//
// Reference: select_top_k, /root/reference/proj/core/src/criticality.cpp:36-81 (see topk.cu
// for the early-exit order and the force_include_recent identity).  Row r of the grid is
// (sequence b = r / rows_per_seq, row h = r % rows_per_seq); its scores are the G score
// rows starting at scores + (b * rows_per_seq + h) * G * sstride, combined per page by
// `reduce` (G = 1: the row itself; G > 1: the GQA group score of grouped.cu -- max, or the
// fp64 sum in head order).  Thread t of an NT-thread group holds the keys of candidates
// [KPT t, KPT t + KPT) in registers and block_select_reg (select.cuh) selects exactly: one
// 11-bit radix pass on the 32-bit word past the keys' common prefix, the threshold bin
// ranked by (key desc, page asc), heavy ties falling back to the 64-bit multi-pass routine.
// The launch covers the cache capacity (NT * KPT >= capacity, or the row-pair kernel's
// whole-CTA mode), chosen on the host, so a captured graph stays valid as contexts grow.
#pragma once

#include "select.cuh"

namespace qk {

constexpr int kRowKpt = 16;
constexpr uint32_t kRowMaxPages = 512u * kRowKpt;

// One row's select_top_k by a group of NT threads (thread t of the group, named barrier
// `bar` spanning the group): early exits, keys in registers, block_select_reg.
template <int NT, int G, int KPT>
__device__ __forceinline__ void topk_row(uint32_t row, int t, int bar, SelectScratch<NT>& sc,
                                         const double* __restrict__ scores, uint32_t sstride,
                                         const int32_t* __restrict__ len, uint32_t layer,
                                         uint32_t B, uint32_t rows_per_seq, uint32_t S,
                                         uint32_t k_budget, int force, int reduce,
                                         int32_t* __restrict__ pages, uint32_t pstride,
                                         int32_t* __restrict__ counts) {
    const uint32_t b = row / rows_per_seq;
    const uint32_t n_tok = static_cast<uint32_t>(len[layer * B + b]);
    const uint32_t P = (n_tok + S - 1) / S;
    int32_t* out = pages + size_t(row) * pstride;

    if (k_budget >= P) {  // criticality.cpp:58-59: every page
        for (uint32_t p = uint32_t(t); p < P && p < pstride; p += NT) out[p] = int32_t(p);
        if (t == 0) counts[row] = int32_t(P);
        return;
    }
    const uint32_t n_cand = force ? P - 1 : P;  // pages competing on score (the keys)
    if (P > sstride || k_budget > pstride || n_cand > uint32_t(NT) * KPT) return;  // host-checked
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
        block_select_reg<NT, KPT>(key, n_cand, target, ref, out, sc, t, bar);
    }
    if (t == 0) {
        if (force) out[target] = int32_t(P - 1);
        counts[row] = int32_t(k_budget);
    }
}

template <int NT, int G, int KPT = kRowKpt>
__global__ void __launch_bounds__(NT)
topk_rows_kernel(const double* __restrict__ scores, uint32_t sstride,
                 const int32_t* __restrict__ len, uint32_t layer, uint32_t B,
                 uint32_t rows_per_seq, uint32_t S, uint32_t k_budget, int force, int reduce,
                 int32_t* __restrict__ pages, uint32_t pstride, int32_t* __restrict__ counts) {
    __shared__ SelectScratch<NT> sc;
    topk_row<NT, G, KPT>(blockIdx.x, threadIdx.x, 1, sc, scores, sstride, len, layer, B,
                         rows_per_seq, S, k_budget, force, reduce, pages, pstride, counts);
}

// Capacities in (4096, 8192]: a 512-thread CTA per PAIR of rows.  While both rows'
// candidates fit 256 x 16 keys (up to 4096 candidate pages: cfg4's 64K tokens) its halves
// select one row each (half the CTAs of one 512-thread CTA per row, each row with the keys of
// 256 threads); a longer row takes the whole CTA, one row after the other.  The mode is
// uniform over the CTA (both halves read both rows' lengths).  Held to 64 registers (some
// spills) for two CTAs per SM: cfg4 per-head 352 -> 348 us per layer step against one
// 512-thread CTA per row (2-round A/B).
template <int G>
__global__ void __launch_bounds__(512, 2)
topk_row_pairs_kernel(const double* __restrict__ scores, uint32_t sstride,
                      const int32_t* __restrict__ len, uint32_t layer, uint32_t B,
                      uint32_t rows, uint32_t rows_per_seq, uint32_t S, uint32_t k_budget,
                      int force, int reduce, int32_t* __restrict__ pages, uint32_t pstride,
                      int32_t* __restrict__ counts) {
    __shared__ union {
        SelectScratch<256> half[2];
        SelectScratch<512> whole;
    } sc;
    const uint32_t r0 = 2u * blockIdx.x;
    auto cand = [&](uint32_t row) -> uint32_t {
        if (row >= rows) return 0u;
        const uint32_t n_tok = static_cast<uint32_t>(len[layer * B + row / rows_per_seq]);
        const uint32_t P = (n_tok + S - 1) / S;
        return force ? (P ? P - 1 : 0u) : P;
    };
    const int t = threadIdx.x;
    if (cand(r0) <= 256u * kRowKpt && cand(r0 + 1) <= 256u * kRowKpt) {
        const int h = t >> 8;
        if (r0 + h < rows)
            topk_row<256, G, kRowKpt>(r0 + h, t & 255, 1 + h, sc.half[h], scores, sstride, len,
                                      layer, B, rows_per_seq, S, k_budget, force, reduce, pages,
                                      pstride, counts);
    } else {
        for (uint32_t r = r0; r < r0 + 2 && r < rows; ++r) {
            topk_row<512, G, kRowKpt>(r, t, 1, sc.whole, scores, sstride, len, layer, B,
                                      rows_per_seq, S, k_budget, force, reduce, pages, pstride,
                                      counts);
            __syncthreads();  // scratch reuse
        }
    }
}

// Launches the row top-K for `capacity` pages (<= kRowMaxPages; larger caches use topk.cu's
// shared-memory selection): 8 keys per thread for launches of at most one row per SM, else
// the smallest 128/256 x 16 CTA that covers the capacity, else the row-pair kernel.
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
    else
        topk_row_pairs_kernel<G><<<(rows + 1) / 2, 512, 0, st>>>(
            scores, sstride, len, layer, B, rows, rows_per_seq, S, k_budget, force, reduce, pages,
            pstride, counts);
#undef QK_TOPK_ROWS
#undef QK_TOPK_ROWS_K
    return cudaGetLastError();
}

}  // namespace qk

#include <algorithm>
// attend.cu -- split-KV sparse paged decode attention with an LSE merge (K4 + K5), and
// dense attention as the same kernel over every page (K6).
//
// Reference: sparse_attention / attend_tokens / full_attention,
// /root/reference/proj/core/src/attention.cpp:54-116:
//   tokens = rows [0, page.length) of each selected page (partial last page masked,
//   :108-114); logits q.k/sqrt(d) (:34-46); max-subtracted softmax over exactly those
//   tokens (:54-67); out = sum_t w_t v_t (:76-82).  The reference accumulates in fp64;
//   this kernel accumulates in fp32 (tolerance: relative L2 <= 1e-5, the reference's own
//   oracle bar, acceptance_main.cpp:165).
//
// Work split: grid (split, sequence * query head).  A (sequence, head) with `count`
// listed pages is cut into ceil(count / pps) splits of pps = max(8, ceil(count/64)) pages
// -- a function of count only, so dense attention and sparse attention over every page
// run the identical partition and produce bitwise identical outputs (the reference's
// full-budget degeneracy, attention.hpp:34-36).  In a CTA each warp streams whole pages:
// a page is S rows x D fp16 = one contiguous block; lanes cover it with 16-byte
// non-allocating loads (K and V for the page issued together), logits are reduced with
// shuffles inside each row group, and an online softmax (base-2, fp32) folds the page
// into the warp's running (m, l, o).  Warps combine through shared memory in fixed
// order; splits write (m, l, o) partials and the last CTA of a (sequence, head) -- found
// with a ticket counter -- merges them in split order (deterministic) and writes the
// output.
//
// Token mode (attend_tokens, attention.cpp:69-84): the list holds token indices (strictly
// ascending, < token_count, checked on the device like check_token_set, attention.cpp:19-30);
// chunks of page_size consecutive list entries play the role of pages (same split rule over
// ceil(count / S) chunks), so attend_tokens over every token is bitwise full_attention.
//
// weights_sum (optional, AttentionOutput::weights_sum_check, attention.cpp:81): the
// post-softmax mass of the weights the output applied, sum_s l_s*2^(m_s-M) / L, evaluated in
// fp64 from the fp32 partials (1 up to the fp32 rounding of the normaliser L).
#include "attend_warp.cuh"

namespace qk {
namespace {

constexpr int kThreads = 128;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxSplitPages = 256;  // page-list entries of a split staged in shared memory
constexpr uint32_t kSplitTarget = 512;  // CTAs per launch the split rule aims at
constexpr int kMinUnitsPerSplit = 16;     // pages (token mode: S-entry chunks) per split, at least

template <int D>
__global__ void __launch_bounds__(kThreads)
attend_kernel(const __half* __restrict__ kp, const __half* __restrict__ vp,
              const int32_t* __restrict__ len, const __half* __restrict__ q,
              const int32_t* __restrict__ pages, uint32_t pstride,
              const int32_t* __restrict__ counts, int mode, uint32_t layer, uint32_t B,
              uint32_t Hq, uint32_t Hkv, uint32_t S, uint32_t head_dim, size_t slice_kv,
              float scale_log2, float* __restrict__ ws_partial, int32_t* __restrict__ ws_ticket,
              void* __restrict__ out, int out_dtype, float* __restrict__ lse,
              double* __restrict__ wsum, int32_t* __restrict__ status, int max_splits) {
    const bool dense = mode == kModeDense, tokens = mode == kModeTokens;
    constexpr int CPR = D / 8;  // 16-byte chunks per row
    __shared__ float s_o[kWarps][D];
    __shared__ float s_m[kWarps], s_l[kWarps];
    __shared__ int s_last;

    const uint32_t bh = blockIdx.y;
    const uint32_t b = bh / Hq, h = bh % Hq;
    const uint32_t kvh = h / (Hq / Hkv);
    const uint32_t n_tok = static_cast<uint32_t>(len[layer * B + b]);
    const uint32_t P = (n_tok + S - 1) / S;
    const int count = dense ? int(P) : counts[bh];
    if (count < 1) {
        if (blockIdx.x == 0 && threadIdx.x == 0)
            record_status(status, tokens ? QK_DEV_EMPTY_TOKENS : QK_DEV_EMPTY_SELECTION);
        return;
    }
    // Units of the split rule: pages, or chunks of S list entries (token mode).
    const int units = tokens ? int((uint32_t(count) + S - 1) / S) : count;
    const int pps = max(kMinUnitsPerSplit, (units + max_splits - 1) / max_splits);
    const int nsplit = (units + pps - 1) / pps;
    // A count past the list row, or needing more splits than the host launched, would read
    // past the row or never complete the merge ticket: reject it (uniform over the CTAs of
    // this (sequence, head), so no CTA takes the ticket).
    if ((!dense && uint32_t(count) > pstride) || nsplit > int(gridDim.x)) {
        if (blockIdx.x == 0 && threadIdx.x == 0) record_status(status, QK_DEV_BAD_COUNT);
        return;
    }
    const int split = blockIdx.x;
    if (split >= nsplit) return;
    const int first = split * pps;
    const int last = min(units, first + pps);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int chunk = lane % CPR, rgrp = lane / CPR;

    float qf[8];
    load_q8<D>(q + size_t(bh) * head_dim, head_dim, qf);
    const size_t s = (size_t(layer) * B + b) * Hkv + kvh;
    const __half* kslice = kp + s * slice_kv;
    const __half* vslice = vp + s * slice_kv;
    const int32_t* plist = pages + size_t(bh) * pstride;

    float m = -CUDART_INF_F, l = 0.0f;
    float o[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = 0.0f;

    // Page mode: this split's page list, validated once (sparse_attention's checks,
    // attention.cpp:99-106; invalid entries are recorded and become -1, skipped).
    __shared__ int32_t s_pg[kMaxSplitPages];
    const bool list_smem = !dense && !tokens && last - first <= kMaxSplitPages;
    if (list_smem) {
        for (int i = first + tid; i < last; i += kThreads) {
            const int pg = plist[i];
            const bool bad_range = pg < 0 || uint32_t(pg) >= P;
            const bool bad_order = i > 0 && plist[i - 1] >= pg;
            if (bad_range || bad_order)
                record_status(status, bad_range ? QK_DEV_PAGE_OUT_OF_RANGE : QK_DEV_PAGE_NOT_ASCENDING);
            s_pg[i - first] = (bad_range || bad_order) ? -1 : pg;
        }
        __syncthreads();
    }
    for (int i = first + warp; i < last; i += kWarps) {
        if (tokens) {
            // Chunk i: list entries [i*S, min(count, i*S+S)), each checked like
            // check_token_set (attention.cpp:19-30).
            const uint32_t e0 = uint32_t(i) * S;
            const uint32_t n = min(S, uint32_t(count) - e0);
            bool bad_range = false, bad_order = false;
            for (uint32_t r = lane; r < n; r += 32) {
                const int32_t t = plist[e0 + r];
                bad_range |= t < 0 || uint32_t(t) >= n_tok;
                bad_order |= (e0 + r) > 0 && plist[e0 + r - 1] >= t;
            }
            bad_range = __any_sync(0xffffffffu, bad_range);
            bad_order = __any_sync(0xffffffffu, bad_order);
            if (bad_range || bad_order) {
                if (lane == 0)
                    record_status(status, bad_range ? QK_DEV_TOKEN_OUT_OF_RANGE
                                                    : QK_DEV_TOKEN_NOT_ASCENDING);
                continue;
            }
            warp_fold_page<D, false>(kslice, vslice, n, qf, scale_log2, m, l, o, plist + e0);
            continue;
        }
        int pg = i;
        if (list_smem) {
            pg = s_pg[i - first];
            if (pg < 0) continue;
        } else if (!dense) {
            pg = plist[i];
            const bool bad_range = pg < 0 || uint32_t(pg) >= P;
            const bool bad_order = i > 0 && plist[i - 1] >= pg;
            if (bad_range || bad_order) {
                if (lane == 0)
                    record_status(status, bad_range ? QK_DEV_PAGE_OUT_OF_RANGE
                                                    : QK_DEV_PAGE_NOT_ASCENDING);
                continue;
            }
        }
        const uint32_t plen = min(S, n_tok - uint32_t(pg) * S);
        const __half* kpage = kslice + size_t(pg) * S * D;
        const __half* vpage = vslice + size_t(pg) * S * D;
        warp_fold_page<D, false>(kpage, vpage, plen, qf, scale_log2, m, l, o);
    }
    warp_fold_rows<D>(l, o);
    if (rgrp == 0) {
#pragma unroll
        for (int j = 0; j < 8; ++j) s_o[warp][chunk * 8 + j] = o[j];
    }
    if (lane == 0) {
        s_m[warp] = m;
        s_l[warp] = l;
    }
    __syncthreads();

    // CTA combine in warp order.
    float M = -CUDART_INF_F;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) M = fmaxf(M, s_m[w]);
    float L = 0.0f;
    float w_scale[kWarps];
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
        w_scale[w] = (s_m[w] == -CUDART_INF_F) ? 0.0f : exp2f(s_m[w] - M);
        L += s_l[w] * w_scale[w];
    }
    const size_t out_base = size_t(bh) * head_dim;
    if (nsplit == 1) {
        for (int d = tid; d < int(head_dim); d += kThreads) {
            float acc = 0.0f;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) acc += s_o[w][d] * w_scale[w];
            const float r = acc / L;
            if (out_dtype == QK_DTYPE_F32) static_cast<float*>(out)[out_base + d] = r;
            else static_cast<__half*>(out)[out_base + d] = __float2half_rn(r);
        }
        if (lse && tid == 0) lse[bh] = (M + log2f(L)) * 0.69314718055994530942f;
        if (wsum && tid == 0) {
            double mass = 0.0;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) mass += double(s_l[w]) * double(w_scale[w]);
            wsum[bh] = mass / double(L);
        }
        return;
    }

    float* part = ws_partial + (size_t(bh) * kMaxSplits + split) * (D + 2);
    for (int d = tid; d < D; d += kThreads) {
        float acc = 0.0f;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) acc += s_o[w][d] * w_scale[w];
        part[2 + d] = acc;
    }
    if (tid == 0) {
        part[0] = M;
        part[1] = L;
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = (atomicAdd(ws_ticket + bh, 1) == nsplit - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();

    // Last CTA: merge every split in split order.
    const float* parts = ws_partial + size_t(bh) * kMaxSplits * (D + 2);
    float Mg = -CUDART_INF_F;
    for (int sp = 0; sp < nsplit; ++sp) Mg = fmaxf(Mg, __ldcg(parts + size_t(sp) * (D + 2)));
    float Lg = 0.0f;
    for (int sp = 0; sp < nsplit; ++sp) {
        const float ms = __ldcg(parts + size_t(sp) * (D + 2));
        const float ls = __ldcg(parts + size_t(sp) * (D + 2) + 1);
        Lg += (ms == -CUDART_INF_F) ? 0.0f : ls * exp2f(ms - Mg);
    }
    for (int d = tid; d < int(head_dim); d += kThreads) {
        float acc = 0.0f;
        for (int sp = 0; sp < nsplit; ++sp) {
            const float ms = __ldcg(parts + size_t(sp) * (D + 2));
            if (ms == -CUDART_INF_F) continue;
            acc += __ldcg(parts + size_t(sp) * (D + 2) + 2 + d) * exp2f(ms - Mg);
        }
        const float r = acc / Lg;
        if (out_dtype == QK_DTYPE_F32) static_cast<float*>(out)[out_base + d] = r;
        else static_cast<__half*>(out)[out_base + d] = __float2half_rn(r);
    }
    if (lse && tid == 0) lse[bh] = (Mg + log2f(Lg)) * 0.69314718055994530942f;
    if (wsum && tid == 0) {
        double mass = 0.0;
        for (int sp = 0; sp < nsplit; ++sp) {
            const float ms = __ldcg(parts + size_t(sp) * (D + 2));
            const float ls = __ldcg(parts + size_t(sp) * (D + 2) + 1);
            if (ms != -CUDART_INF_F) mass += double(ls) * double(exp2f(ms - Mg));
        }
        wsum[bh] = mass / double(Lg);
    }
    if (tid == 0) ws_ticket[bh] = 0;  // re-arm for the next launch / graph replay
}

template <int D>
int run(const qk_cache* c, uint32_t layer, const __half* q, uint32_t batch,
        const int32_t* pages, uint32_t pstride, const int32_t* counts, int mode,
        uint32_t max_list, void* out, int out_dtype, float* lse, double* wsum, cudaStream_t st) {
    // max_list: the longest list (pages, or tokens in token mode) a row may hold.
    const uint32_t max_units = mode == kModeTokens ? (max_list + c->S - 1) / c->S : max_list;
    // Splits per row: about kSplitTarget CTAs per launch (one wave of a few CTAs per SM; a
    // CTA's fixed costs -- q, page list, combine, partials, merge ticket -- over as many pages
    // as that allows), at least 16 units each (sparse cfg2: 16.3 -> 15.2 us against 8).  Measured (cfg2 unless noted, µs per layer):
    // dense 109 -> 88 (16 splits of 128 pages instead of 64 of 32), cfg4 per-head 366 -> 351
    // (1 split per row instead of 8), cfg5 unfused 111 -> 107 (2 instead of 8), sparse cfg2
    // unchanged (16 splits of 8).  A function of the launch's rows and the row's own count
    // only, so dense, sparse-over-every-page and token-mode calls of one batch share the
    // partition (and stay bitwise equal).
    const uint32_t rows = batch * c->Hq;
    const int max_splits = int(std::min<uint32_t>(kMaxSplits, std::max<uint32_t>(1u, kSplitTarget / rows)));
    const uint32_t splits_needed = std::min<uint32_t>(uint32_t(max_splits),
                                                      (max_units + kMinUnitsPerSplit - 1) / kMinUnitsPerSplit);
    const dim3 grid(splits_needed ? splits_needed : 1, batch * c->Hq);
    const float scale_log2 = float(1.4426950408889634 / sqrt(double(c->desc.head_dim)));
    attend_kernel<D><<<grid, kThreads, 0, st>>>(
        c->k_pool, c->v_pool, c->d_len, q, pages, pstride, counts, mode, layer, c->B,
        c->Hq, c->Hkv, c->S, c->desc.head_dim, c->slice_kv, scale_log2, c->ws_partial,
        c->ws_ticket, out, out_dtype, lse, wsum, c->d_status, max_splits);
    const_cast<qk_cache*>(c)->launches++;
    return cuda_check(cudaGetLastError(), "attend_kernel");
}

}  // namespace

int launch_attend(const qk_cache* c, uint32_t layer, const __half* q, uint32_t batch,
                  const int32_t* pages, uint32_t pstride, const int32_t* counts, int mode,
                  uint32_t max_list, void* out, int out_dtype, float* lse, double* wsum,
                  cudaStream_t st) {
    switch (c->D) {
        case 64: return run<64>(c, layer, q, batch, pages, pstride, counts, mode, max_list, out, out_dtype, lse, wsum, st);
        case 128: return run<128>(c, layer, q, batch, pages, pstride, counts, mode, max_list, out, out_dtype, lse, wsum, st);
        case 256: return run<256>(c, layer, q, batch, pages, pstride, counts, mode, max_list, out, out_dtype, lse, wsum, st);
        default: return set_error(QK_ERR_UNSUPPORTED, "qk_attend: unsupported head_dim");
    }
}

}  // namespace qk

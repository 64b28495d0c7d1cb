// grouped.cu -- GQA group-shared Quest decode: ONE page set per
// (sequence, KV head), chosen from a group score that combines the exact per-query-head
// estimates, and attention of all G query heads of the group over that shared set as a
// real dense contraction on the tensor cores.
//
// This is an OPT-IN variant, not the reference's semantics: the reference selects per
// query head (criticality.cpp:36-81 applied to each head's estimate_all,
// criticality.cpp:25-34).  What stays exact:
//   * per-head scores: estimate_kernel, bitwise the reference's doubles;
//   * the group score of page p: QK_GROUP_MAX -> max_g score_g(p) (exact),
//     QK_GROUP_SUM -> ((score_0 + score_1) + score_2) + ... in head order (fp64 adds);
//   * selection: select_top_k's rule (criticality.cpp:36-81: early exits, (score desc,
//     page asc), force_include_recent) applied to the group scores -- bitwise page sets
//     against the oracle composed from the reference's own functions;
//   * attention of each query head over the shared pages: sparse_attention
//     (attention.cpp:94-116) within the fp32 tolerance (relative L2 <= 1e-5).
//
// Group attention (grouped_attend_kernel): K and V of a selected page are read from HBM
// ONCE for the G query heads (the per-head path reads them G times, from L2 at best).
// Per 16-token chunk of a page a warp computes S = Q K^T and O += P V with
// mma.sync.m16n8k16 (fp16 operands, fp32 accumulate): M = the G query heads (rows >= G
// are zero), N = tokens (S) or channels (PV), K = channels (S) or tokens (PV).
//   * S: the k-slot -> channel map is permuted so that a lane's B fragments are whole
//     16-byte loads of one K row (chunk 4j+c of token r); Q's A fragments follow the same
//     map (a dot product is order-free; the tensor core sums in fp32).
//   * P V: P is the S accumulator re-used as the A fragment (the FlashAttention-2 register
//     identity), split into fp16 hi + lo halves (two MMAs) so the weights keep ~22 bits;
//     the n -> channel map is permuted so a lane's B fragments come from 16-byte loads of
//     its own channel run of 4 V rows (PRMT packs the token pairs).
//   * online softmax per head in the base-2 domain, warps combined in order, splits merged
//     by the last CTA (attend.cu's split rule, ticket and merge).
#include <algorithm>
#include <math_constants.h>

#include "topk_rows.cuh"

namespace qk {
namespace {

// ---- group top-K ------------------------------------------------------------------------

constexpr int kSelThreads = 256;

template <int G>
__global__ void __launch_bounds__(kSelThreads)
group_topk_kernel(const double* __restrict__ scores, uint32_t sstride,
                  const int32_t* __restrict__ len, uint32_t layer, uint32_t B, uint32_t Hkv,
                  uint32_t S, uint32_t k_budget, int force, int reduce,
                  int32_t* __restrict__ pages, uint32_t pstride, int32_t* __restrict__ counts) {
    extern __shared__ __align__(16) unsigned long long keys[];  // kSelThreads * (kpt + 1)
    __shared__ SelectScratch<kSelThreads> sc;

    const uint32_t bk = blockIdx.x;  // (sequence, KV head)
    const uint32_t b = bk / Hkv, kvh = bk % Hkv;
    const uint32_t n_tok = static_cast<uint32_t>(len[layer * B + b]);
    const uint32_t P = (n_tok + S - 1) / S;
    int32_t* out = pages + size_t(bk) * pstride;

    if (k_budget >= P) {  // criticality.cpp:58-59: every page
        for (uint32_t p = threadIdx.x; p < P && p < pstride; p += kSelThreads) out[p] = int32_t(p);
        if (threadIdx.x == 0) counts[bk] = int32_t(P);
        return;
    }
    if (P > sstride || k_budget > pstride) return;  // host-checked
    const uint32_t n_cand = force ? P - 1 : P;
    const uint32_t target = force ? k_budget - 1 : k_budget;
    const double* rows = scores + (size_t(b) * Hkv * G + size_t(kvh) * G) * sstride;
    if (target > 0) {
        unsigned long long kmax, kmin;
        auto group_score = [rows, sstride, reduce](uint32_t i) {
            double x = __ldcg(rows + i);
#pragma unroll
            for (int g = 1; g < G; ++g) {
                const double y = __ldcg(rows + size_t(g) * sstride + i);
                x = reduce == QK_GROUP_SUM ? __dadd_rn(x, y) : (y > x ? y : x);
            }
            return x;
        };
        const int kpt = load_keys_fn<kSelThreads>(group_score, n_cand, keys, sc, &kmax, &kmin);
        block_select<kSelThreads>(keys, kpt, n_cand, target, kmax, kmin, out, sc);
    }
    if (threadIdx.x == 0) {
        if (force) out[target] = int32_t(P - 1);
        counts[bk] = int32_t(k_budget);
    }
}

// ---- group attention on the tensor cores --------------------------------------------------

constexpr int kThreads = 128;
constexpr int kWarps = kThreads / 32;
constexpr int kListCap = 256;  // page-list entries of a split staged in shared memory

__device__ __forceinline__ void mma16816(float (&d)[4], uint32_t a0, uint32_t a2, uint32_t b0,
                                         uint32_t b1) {
    // Rows 8..15 of A (a1, a3) are zero: the group has at most 8 query heads.
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(0u), "r"(a2), "r"(0u), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t word(const int4& v, int i) {
    return i == 0 ? uint32_t(v.x) : i == 1 ? uint32_t(v.y) : i == 2 ? uint32_t(v.z) : uint32_t(v.w);
}

__device__ __forceinline__ uint32_t pack_h2(float lo, float hi) {
    const __half2 h = __floats2half2_rn(lo, hi);
    return *reinterpret_cast<const uint32_t*>(&h);
}

template <int D, int G>
__global__ void __launch_bounds__(kThreads, 3)
grouped_attend_kernel(const __half* __restrict__ kp, const __half* __restrict__ vp,
                      const int32_t* __restrict__ len, const __half* __restrict__ q,
                      const int32_t* __restrict__ pages, uint32_t pstride,
                      const int32_t* __restrict__ counts, uint32_t layer, uint32_t B,
                      uint32_t Hkv, uint32_t S, uint32_t head_dim, size_t slice_kv,
                      float scale_log2, float* __restrict__ ws_partial,
                      int32_t* __restrict__ ws_ticket, void* __restrict__ out, int out_dtype,
                      int32_t* __restrict__ status, int max_splits) {
    static_assert(G >= 1 && G <= 8, "at most 8 query heads per group (MMA rows 0..7)");
    constexpr int KS = D / 16;   // k-steps of S = Q K^T
    constexpr int NT = D / 8;    // n-tiles (8 channels) of O = P V
    constexpr int KCH = D / 32;  // 16-byte chunks of one K row per lane (chunks 4j + c)
    constexpr int VCH = NT / 8;  // 16-byte chunks of a lane's V channel run (NT channels)
    __shared__ float s_o[kWarps][G][D];
    __shared__ float s_m[kWarps][G], s_l[kWarps][G];
    __shared__ int s_last;

    const uint32_t bk = blockIdx.y;
    const uint32_t b = bk / Hkv, kvh = bk % Hkv;
    const uint32_t Hq = Hkv * G;
    const uint32_t n_tok = static_cast<uint32_t>(len[layer * B + b]);
    const uint32_t P = (n_tok + S - 1) / S;
    const int count = counts[bk];
    if (count < 1) {
        if (blockIdx.x == 0 && threadIdx.x == 0) record_status(status, QK_DEV_EMPTY_SELECTION);
        return;
    }
    const int pps = max(kMinPagesPerSplit, (count + max_splits - 1) / max_splits);
    const int nsplit = (count + pps - 1) / pps;
    if (uint32_t(count) > pstride || nsplit > int(gridDim.x)) {
        if (blockIdx.x == 0 && threadIdx.x == 0) record_status(status, QK_DEV_BAD_COUNT);
        return;
    }
    const int split = blockIdx.x;
    if (split >= nsplit) return;
    const int first = split * pps, last = min(count, first + pps);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int r = lane >> 2, c = lane & 3;  // fragment row (head / token / channel) and column pair

    // Q A-fragments of head r: k-step s = 2j + t covers channels 8(4j+c) + 4t + {0,1} (a0) and
    // + {2,3} (a2).
    uint32_t qa[KS][2];
    {
        const __half* qrow = q + (size_t(b) * Hq + size_t(kvh) * G + (r < G ? r : 0)) * head_dim;
#pragma unroll
        for (int j = 0; j < KCH; ++j) {
            uint32_t w[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int ch = 8 * (4 * j + c) + 2 * e;
                __half lo = __float2half(0.0f), hi = __float2half(0.0f);
                if (r < G && ch < int(head_dim)) lo = qrow[ch];
                if (r < G && ch + 1 < int(head_dim)) hi = qrow[ch + 1];
                const __half2 h2 = __halves2half2(lo, hi);
                w[e] = *reinterpret_cast<const uint32_t*>(&h2);
            }
            qa[2 * j][0] = w[0];
            qa[2 * j][1] = w[1];
            qa[2 * j + 1][0] = w[2];
            qa[2 * j + 1][1] = w[3];
        }
    }

    const size_t sl = (size_t(layer) * B + b) * Hkv + kvh;
    const __half* kslice = kp + sl * slice_kv;
    const __half* vslice = vp + sl * slice_kv;
    const int32_t* plist = pages + size_t(bk) * pstride;

    float m = -CUDART_INF_F, l = 0.0f;  // head r's running max (base 2) and this lane's mass
    float o[NT][2];                      // O[r][NT*2c + nt], O[r][NT*(2c+1) + nt]
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) o[nt][0] = o[nt][1] = 0.0f;

    // Chunks (16 tokens of a page) of this warp's pages [first + warp, last; kWarps), walked
    // with the next chunk's K/V loads in flight while the current one is folded.
    struct Chunk {
        int4 ka[KCH], kb[KCH], va[4][VCH];
        uint32_t n;  // valid rows of the chunk (0: nothing to fold)
    };
    // The CTA's page list, validated once (sparse_attention's checks, attention.cpp:99-106):
    // invalid entries are recorded and skipped.
    __shared__ int32_t s_pg[kListCap];
    const bool in_smem = last - first <= kListCap;
    for (int i = first + tid; i < last && in_smem; i += kThreads) {
        const int pg = plist[i];
        const bool bad_range = pg < 0 || uint32_t(pg) >= P;
        const bool bad_order = i > 0 && plist[i - 1] >= pg;
        if (bad_range || bad_order)
            record_status(status, bad_range ? QK_DEV_PAGE_OUT_OF_RANGE : QK_DEV_PAGE_NOT_ASCENDING);
        s_pg[i - first] = (bad_range || bad_order) ? -1 : pg;
    }
    __syncthreads();
    int ci = first + warp;  // page list position of the chunk to load next
    uint32_t ct0 = 0;       // its first row within the page
    auto load = [&](Chunk& ch) {
        ch.n = 0;
        while (ci < last) {
            int pg;
            if (in_smem) {
                pg = s_pg[ci - first];
            } else {
                pg = plist[ci];
                if (pg < 0 || uint32_t(pg) >= P || (ci > 0 && plist[ci - 1] >= pg)) {
                    if (lane == 0)
                        record_status(status, (pg < 0 || uint32_t(pg) >= P) ? QK_DEV_PAGE_OUT_OF_RANGE
                                                                            : QK_DEV_PAGE_NOT_ASCENDING);
                    pg = -1;
                }
            }
            if (pg < 0) {
                ci += kWarps;
                ct0 = 0;
                continue;
            }
            const uint32_t plen = min(S, n_tok - uint32_t(pg) * S);
            const uint32_t t0 = ct0;
            const uint32_t n = min(16u, plen - t0);
            const __half* kpage = kslice + (size_t(pg) * S + t0) * D;
            const __half* vpage = vslice + (size_t(pg) * S + t0) * D;
            // K rows r and r+8 (chunks 4j + c); V rows 2c, 2c+1, 2c+8, 2c+9 (channels NT*r..).
#pragma unroll
            for (int j = 0; j < KCH; ++j) {
                ch.ka[j] = uint32_t(r) < n ? ld_nc_v4(kpage + size_t(r) * D + 8 * (4 * j + c))
                                           : make_int4(0, 0, 0, 0);
                ch.kb[j] = uint32_t(r + 8) < n ? ld_nc_v4(kpage + size_t(r + 8) * D + 8 * (4 * j + c))
                                               : make_int4(0, 0, 0, 0);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t row = 2 * c + (u & 1) + 8 * (u >> 1);
#pragma unroll
                for (int x = 0; x < VCH; ++x)
                    ch.va[u][x] = row < n ? ld_nc_v4(vpage + size_t(row) * D + NT * r + 8 * x)
                                          : make_int4(0, 0, 0, 0);
            }
            ch.n = n;
            if (t0 + 16 < plen) {
                ct0 = t0 + 16;
            } else {
                ci += kWarps;
                ct0 = 0;
            }
            return;
        }
    };
    auto fold = [&](const Chunk& ch) {
        const uint32_t n = ch.n;
        // S = Q K^T: n-tile 0 = tokens 0..7, n-tile 1 = tokens 8..15 of the chunk.
        float s0[4] = {0.f, 0.f, 0.f, 0.f}, s1[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int j = 0; j < KCH; ++j) {
#pragma unroll
            for (int t = 0; t < 2; ++t) {
                mma16816(s0, qa[2 * j + t][0], qa[2 * j + t][1], word(ch.ka[j], 2 * t), word(ch.ka[j], 2 * t + 1));
                mma16816(s1, qa[2 * j + t][0], qa[2 * j + t][1], word(ch.kb[j], 2 * t), word(ch.kb[j], 2 * t + 1));
            }
        }
        // Head r's logits of tokens 2c, 2c+1, 8+2c, 9+2c (base 2, masked past n).
        float x[4];
        x[0] = (uint32_t(2 * c) < n) ? s0[0] * scale_log2 : -CUDART_INF_F;
        x[1] = (uint32_t(2 * c + 1) < n) ? s0[1] * scale_log2 : -CUDART_INF_F;
        x[2] = (uint32_t(2 * c + 8) < n) ? s1[0] * scale_log2 : -CUDART_INF_F;
        x[3] = (uint32_t(2 * c + 9) < n) ? s1[1] * scale_log2 : -CUDART_INF_F;
        float mx = fmaxf(fmaxf(x[0], x[1]), fmaxf(x[2], x[3]));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
        const float m_new = fmaxf(m, mx);  // finite: row 0 of a chunk is always valid
        const float alpha = exp2f(m - m_new);  // 0 on the first chunk
        float p[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) p[e] = exp2f(x[e] - m_new);
        l = l * alpha + ((p[0] + p[1]) + (p[2] + p[3]));
        m = m_new;
        // P as A fragments (k = token 2c.. / 2c+8..), split into fp16 hi + lo.
        const uint32_t ph0 = pack_h2(p[0], p[1]), ph2 = pack_h2(p[2], p[3]);
        const __half2 h0 = *reinterpret_cast<const __half2*>(&ph0);
        const __half2 h2 = *reinterpret_cast<const __half2*>(&ph2);
        const uint32_t pl0 = pack_h2(p[0] - __low2float(h0), p[1] - __high2float(h0));
        const uint32_t pl2 = pack_h2(p[2] - __low2float(h2), p[3] - __high2float(h2));
        // O += P V: n-tile nt = channels NT*n + nt; B fragment = V[2c][ch], V[2c+1][ch] and
        // V[2c+8][ch], V[2c+9][ch] of this lane's channel ch = NT*r + nt.
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            const int x8 = nt / 8, w = (nt % 8) / 2;
            const uint32_t sel = (nt & 1) ? 0x7632u : 0x5410u;
            const uint32_t b0 = __byte_perm(word(ch.va[0][x8], w), word(ch.va[1][x8], w), sel);
            const uint32_t b1 = __byte_perm(word(ch.va[2][x8], w), word(ch.va[3][x8], w), sel);
            float acc[4] = {o[nt][0] * alpha, o[nt][1] * alpha, 0.f, 0.f};
            mma16816(acc, ph0, ph2, b0, b1);
            mma16816(acc, pl0, pl2, b0, b1);
            o[nt][0] = acc[0];
            o[nt][1] = acc[1];
        }
    };
#ifdef QK_GROUPED_DOUBLE_BUFFER
    Chunk c0, c1;  // two buffers, alternating roles (no register copies)
    load(c0);
    while (c0.n) {
        load(c1);  // in flight during the fold
        fold(c0);
        if (!c1.n) break;
        load(c0);
        fold(c1);
    }
#else
    // One chunk in flight per warp; occupancy (3 CTAs per SM) supplies the parallelism (the
    // double-buffered form measured the same at cfg4 with twice the registers).
    Chunk c0;
    for (load(c0); c0.n; load(c0)) fold(c0);
#endif
    // This warp's mass of head r: the four lanes of the row.
    l += __shfl_xor_sync(0xffffffffu, l, 1);
    l += __shfl_xor_sync(0xffffffffu, l, 2);
    if (r < G) {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            s_o[warp][r][NT * (2 * c) + nt] = o[nt][0];
            s_o[warp][r][NT * (2 * c + 1) + nt] = o[nt][1];
        }
        if (c == 0) {
            s_m[warp][r] = m;
            s_l[warp][r] = l;
        }
    }
    __syncthreads();

    // CTA combine per head in warp order, then (multi-split) partials + last-CTA merge.
    __shared__ float s_w[kWarps][G], s_M[G], s_L[G];
    __shared__ float s_sw[kMaxSplits][G];  // merge weights exp2(m_s - M) / L per split
    if (tid < G) {
        const int g = tid;
        float M = -CUDART_INF_F;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) M = fmaxf(M, s_m[w][g]);
        float L = 0.0f;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            const float sc = (s_m[w][g] == -CUDART_INF_F) ? 0.0f : exp2f(s_m[w][g] - M);
            s_w[w][g] = sc;
            L += s_l[w][g] * sc;
        }
        s_M[g] = M;
        s_L[g] = L;
    }
    __syncthreads();
    float* part_base = ws_partial + size_t(bk) * kMaxSplits * G * (D + 2);
    for (int i = tid; i < G * D; i += kThreads) {
        const int g = i / D, d = i % D;
        float acc = 0.0f;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) acc += s_o[w][g][d] * s_w[w][g];
        if (nsplit == 1) {
            if (d < int(head_dim)) {
                const size_t oi = (size_t(b) * Hq + size_t(kvh) * G + g) * head_dim + d;
                if (out_dtype == QK_DTYPE_F32) static_cast<float*>(out)[oi] = acc / s_L[g];
                else static_cast<__half*>(out)[oi] = __float2half_rn(acc / s_L[g]);
            }
        } else {
            float* part = part_base + (size_t(split) * G + g) * (D + 2);
            part[2 + d] = acc;
            if (d == 0) {
                part[0] = s_M[g];
                part[1] = s_L[g];
            }
        }
    }
    if (nsplit == 1) return;
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = (atomicAdd(ws_ticket + bk, 1) == nsplit - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    // Last CTA: every split's (m, l) in parallel, then per-head weights in split order.
    for (int i = tid; i < nsplit * G; i += kThreads) {
        const float* pp = part_base + size_t(i) * (D + 2);  // i = split * G + g
        s_sw[i / G][i % G] = __ldcg(pp);
    }
    __syncthreads();
    if (tid < G) {
        const int g = tid;
        float Mg = -CUDART_INF_F;
        for (int sp = 0; sp < nsplit; ++sp) Mg = fmaxf(Mg, s_sw[sp][g]);
        float Lg = 0.0f;
        for (int sp = 0; sp < nsplit; ++sp) {
            const float ms = s_sw[sp][g];
            const float w = (ms == -CUDART_INF_F) ? 0.0f : exp2f(ms - Mg);
            Lg += __ldcg(part_base + (size_t(sp) * G + g) * (D + 2) + 1) * w;
            s_sw[sp][g] = w;
        }
        s_L[g] = Lg;
    }
    __syncthreads();
    for (int i = tid; i < G * int(head_dim); i += kThreads) {
        const int g = i / int(head_dim), d = i % int(head_dim);
        float acc = 0.0f;
#pragma unroll 8
        for (int sp = 0; sp < nsplit; ++sp)
            acc += __ldcg(part_base + (size_t(sp) * G + g) * (D + 2) + 2 + d) * s_sw[sp][g];
        const size_t oi = (size_t(b) * Hq + size_t(kvh) * G + g) * head_dim + d;
        if (out_dtype == QK_DTYPE_F32) static_cast<float*>(out)[oi] = acc / s_L[g];
        else static_cast<__half*>(out)[oi] = __float2half_rn(acc / s_L[g]);
    }
    if (tid == 0) ws_ticket[bk] = 0;  // re-arm for the next launch / graph replay
}

template <int G>
int run_topk(const qk_cache* c, uint32_t layer, const double* scores, uint32_t sstride,
             uint32_t batch, uint32_t k_budget, int force, int reduce, int32_t* pages,
             uint32_t pstride, int32_t* counts, cudaStream_t st) {
    if (c->Pmax <= kRowMaxPages) {  // keys in registers (topk_rows.cuh)
        launch_topk_rows<G>(batch * c->Hkv, c->Pmax, scores, sstride, c->d_len, layer, c->B,
                            c->Hkv, c->S, k_budget, force, reduce, pages, pstride, counts, st);
        const_cast<qk_cache*>(c)->launches++;
        return cuda_check(cudaGetLastError(), "topk_rows_kernel");
    }
    const uint32_t kpt = (c->Pmax + kSelThreads - 1) / kSelThreads;  // sized for the capacity
    const size_t smem = size_t(kSelThreads) * (kpt + 1) * sizeof(unsigned long long);
    auto kern = group_topk_kernel<G>;
    if (int rc = ensure_func_attrs(reinterpret_cast<const void*>(kern), smem, c->desc.device, false,
                                   "group_topk_kernel attributes"))
        return rc;
    kern<<<batch * c->Hkv, kSelThreads, smem, st>>>(scores, sstride, c->d_len, layer, c->B,
                                                    c->Hkv, c->S, k_budget, force, reduce, pages,
                                                    pstride, counts);
    const_cast<qk_cache*>(c)->launches++;
    return cuda_check(cudaGetLastError(), "group_topk_kernel");
}

template <int D, int G>
int run_attend(const qk_cache* c, uint32_t layer, const __half* q, uint32_t batch,
               const int32_t* pages, uint32_t pstride, const int32_t* counts, uint32_t max_list,
               void* out, int out_dtype, cudaStream_t st) {
    // Splits per (sequence, KV head): about 256 CTAs per launch (this kernel holds 3 CTAs
    // per SM: one wave), at least 8 pages each.  cfg4 group-shared: 283 -> 257 us per layer
    // step (1 split of 128 pages per unit instead of 8 of 16; 2 splits: 278, a 1.15-wave grid).
    const uint32_t units = batch * c->Hkv;
    const int max_splits = int(std::min<uint32_t>(kMaxSplits, std::max<uint32_t>(1u, 256u / units)));
    const uint32_t splits = std::min<uint32_t>(uint32_t(max_splits),
                                               (max_list + kMinPagesPerSplit - 1) / kMinPagesPerSplit);
    const dim3 grid(splits ? splits : 1, batch * c->Hkv);
    const float scale_log2 = float(1.4426950408889634 / sqrt(double(c->desc.head_dim)));
    grouped_attend_kernel<D, G><<<grid, kThreads, 0, st>>>(
        c->k_pool, c->v_pool, c->d_len, q, pages, pstride, counts, layer, c->B, c->Hkv, c->S,
        c->desc.head_dim, c->slice_kv, scale_log2, c->ws_partial, c->ws_ticket, out, out_dtype,
        c->d_status, max_splits);
    const_cast<qk_cache*>(c)->launches++;
    return cuda_check(cudaGetLastError(), "grouped_attend_kernel");
}

template <int D>
int attend_d(const qk_cache* c, uint32_t layer, const __half* q, uint32_t batch,
             const int32_t* pages, uint32_t pstride, const int32_t* counts, uint32_t max_list,
             void* out, int out_dtype, cudaStream_t st) {
    switch (c->G) {
        case 1: return run_attend<D, 1>(c, layer, q, batch, pages, pstride, counts, max_list, out, out_dtype, st);
        case 2: return run_attend<D, 2>(c, layer, q, batch, pages, pstride, counts, max_list, out, out_dtype, st);
        case 4: return run_attend<D, 4>(c, layer, q, batch, pages, pstride, counts, max_list, out, out_dtype, st);
        case 8: return run_attend<D, 8>(c, layer, q, batch, pages, pstride, counts, max_list, out, out_dtype, st);
        default: return set_error(QK_ERR_UNSUPPORTED, "grouped decode: GQA group must be 1, 2, 4 or 8");
    }
}

}  // namespace

int launch_group_topk(const qk_cache* c, uint32_t layer, const double* scores, uint32_t sstride,
                      uint32_t batch, uint32_t k_budget, int force, int reduce, int32_t* pages,
                      uint32_t pstride, int32_t* counts, cudaStream_t st) {
    switch (c->G) {
        case 1: return run_topk<1>(c, layer, scores, sstride, batch, k_budget, force, reduce, pages, pstride, counts, st);
        case 2: return run_topk<2>(c, layer, scores, sstride, batch, k_budget, force, reduce, pages, pstride, counts, st);
        case 4: return run_topk<4>(c, layer, scores, sstride, batch, k_budget, force, reduce, pages, pstride, counts, st);
        case 8: return run_topk<8>(c, layer, scores, sstride, batch, k_budget, force, reduce, pages, pstride, counts, st);
        default: return set_error(QK_ERR_UNSUPPORTED, "grouped decode: GQA group must be 1, 2, 4 or 8");
    }
}

int launch_group_attend(const qk_cache* c, uint32_t layer, const __half* q, uint32_t batch,
                        const int32_t* pages, uint32_t pstride, const int32_t* counts,
                        uint32_t max_list, void* out, int out_dtype, cudaStream_t st) {
    switch (c->D) {
        case 64: return attend_d<64>(c, layer, q, batch, pages, pstride, counts, max_list, out, out_dtype, st);
        case 128: return attend_d<128>(c, layer, q, batch, pages, pstride, counts, max_list, out, out_dtype, st);
        default: return set_error(QK_ERR_UNSUPPORTED, "grouped decode: head_dim must be <= 128");
    }
}

// append -> estimate (per head, exact) -> group top-K -> group attention.
int launch_decode_grouped(qk_cache* c, uint32_t layer, const __half* q, const __half* k,
                          const __half* v, uint32_t batch, const qk_selection_cfg& cfg,
                          int reduce, uint32_t max_pages_after, void* out, int out_dtype,
                          int32_t* pages, uint32_t pstride, int32_t* counts, cudaStream_t st) {
    int rc = QK_OK;
    if (k) rc = launch_append(c, layer, k, v, batch, st);
    if (rc) return rc;
    const uint32_t kk = cfg.per_layer_enabled ? cfg.token_budget / c->S : UINT32_MAX;
    // Grids and shared memory sized for the capacity: a captured graph stays correct as
    // replays grow the context.
    if (kk < c->Pmax) {  // a partial selection is possible: estimate
        rc = launch_estimate(c, layer, q, batch, c->ws_scores, c->Pmax, c->Pmax, st);
        if (rc) return rc;
    }
    int32_t* sel = pages ? pages : c->ws_pages;
    const uint32_t sstride = pages ? pstride : c->Pmax;
    int32_t* cnt = counts ? counts : c->ws_counts;
    rc = launch_group_topk(c, layer, c->ws_scores, c->Pmax, batch, kk,
                           cfg.force_include_recent ? 1 : 0, reduce, sel, sstride, cnt, st);
    if (rc) return rc;
    const uint32_t max_list = kk < c->Pmax ? kk : c->Pmax;
    return launch_group_attend(c, layer, q, batch, sel, sstride, cnt, max_list, out, out_dtype, st);
}

}  // namespace qk

// decode.cu -- one Quest decode step for a layer in ONE kernel launch:
//     KvCache::append (fused metadata update) -> estimate_all -> select_top_k ->
//     sparse_attention with a split-KV log-sum-exp merge
// (R/README.md:151-158 usage; metrics.cpp:90-95 step order; kv_store.cpp:19-47;
//  criticality.cpp:9-81; attention.cpp:54-116).
//
// Work decomposition: one thread-block CLUSTER of C CTAs per (sequence, KV head) unit.
//   phase A  the CTA owning the newest page appends the token's K/V row and updates that
//            page's min/max metadata (strict compares, first-seen kept);
//   phase B  each CTA estimates its contiguous range of pages for all G query heads of
//            the KV head (bitwise fp64 chains, as estimate.cu) and writes the scores to an
//            L2-resident workspace;  -- cluster barrier (release/acquire) --
//   phase C  every CTA reads the unit's scores back and runs the exact selection
//            (select.cuh) itself, so no second exchange is needed;
//   phase D  each CTA attends its share of every query head's selected pages (warps
//            stream pages into an online softmax, as attend.cu) and ships its (m, l, o)
//            partial to rank 0's shared memory over DSMEM;  -- cluster barrier --
//            rank 0 merges the partials in rank order and writes the output.
// With C CTAs per unit the metadata and KV streams of a batch-1 layer are spread over
// 32*C SMs; the two HBM streams are separated only by the selection's dependency.
// The launch uses programmatic dependent launch so its prologue overlaps the previous
// kernel's tail; griddepcontrol.wait precedes every read of data a prior kernel wrote.
#include "attend_warp.cuh"
#include "select.cuh"

namespace qk {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kGroups = 4;
constexpr uint32_t kMaxFusedK = 512;  // selected pages per query head kept in smem

__device__ __forceinline__ double h2d(__half h) {
    double d;
    asm("cvt.f64.f16 %0, %1;" : "=d"(d) : "h"(__half_as_ushort(h)));
    return d;
}

// fp16 bits -> the double sel * 2^-1008, exactly, for every finite fp16 (normal,
// subnormal, +-0): the 15 exponent/mantissa bits land in the double's exponent/mantissa
// fields unbiased (hence the 2^-1008 scale; fp16 subnormals become double subnormals with
// the same scale) and the sign moves from bit 25 to bit 31 (t + 63*s clears bit 25 and
// sets bit 31).  Three integer ops instead of one F2F on the 16-lane/clk XU pipe.
__device__ __forceinline__ double h2d_scaled(unsigned short h) {
    const uint32_t t = uint32_t(h) << 10;
    const uint32_t s = t & 0x02000000u;
    return __hiloint2double(int(t + s * 63u), 0);
}

__device__ __forceinline__ void stamp(unsigned long long* probe, int slot) {
    if (probe != nullptr && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        probe[blockIdx.x * 16 + slot] = t;
    }
}

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cluster_size() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_acqrel() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n"
                 "barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void st_cluster_f32(float* local_addr, uint32_t rank, float v) {
    const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(local_addr));
    uint32_t ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
    asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(ra), "f"(v) : "memory");
}

struct FusedParams {
    __half* k_pool;
    __half* v_pool;
    __half* meta;
    int32_t* len;
    int32_t* len_ticket;
    int32_t* status;
    const __half* q;
    const __half* k_new;  // nullable
    const __half* v_new;
    double* ws_scores;    // [B][Hq][Pmax]
    void* out;
    int32_t* pages_out;   // nullable
    int32_t* counts_out;  // nullable
    size_t slice_kv, slice_meta;
    uint32_t layer, B, Hkv, S, head_dim, Pmax, capacity, pstride;
    uint32_t k_budget;    // pages per query head (UINT32_MAX: selection disabled)
    int force, out_dtype;
    float scale_log2;
    unsigned long long* probe;  // optional [grid][8] globaltimer stamps (phase timing)
};

// Dynamic shared memory: [region A: metadata stage | top-K keys] [dq G*D doubles]
// [selected pages G*kMaxFusedK ints] [partials G*8*(D+2) floats]
template <int D, int G>
struct Layout {
    static constexpr int NROW = (G == 1) ? 1 : 2;
    static constexpr int PPC = (G == 1) ? 256 : 128;  // pages per estimate chunk
    static constexpr size_t stage_bytes = size_t(NROW) * D * PPC * 2;
    static size_t region_a(uint32_t pmax) {
        const size_t kpt = (pmax + kThreads - 1) / kThreads;
        const size_t keys = size_t(kThreads) * (kpt + 1) * 8;
        return stage_bytes > keys ? stage_bytes : keys;
    }
    static size_t bytes(uint32_t pmax) {
        return region_a(pmax) + size_t(G) * D * 8 + size_t(G) * kMaxFusedK * 4 +
               size_t(G) * 8 * (D + 2) * 4;
    }
};

template <int D, int G>
__global__ void __launch_bounds__(kThreads, 2) decode_fused_kernel(const FusedParams p,
                                                                    uint32_t region_a_bytes) {
    using LY = Layout<D, G>;
    constexpr int NROW = LY::NROW, PPC = LY::PPC;
    constexpr int CH_PER_GROUP = D / kGroups;
    constexpr int CPR = D / 8;
    extern __shared__ __align__(16) unsigned char smem[];
    __half* stage = reinterpret_cast<__half*>(smem);                       // [NROW][D][PPC]
    unsigned long long* keys = reinterpret_cast<unsigned long long*>(smem);  // aliases stage
    double* dq = reinterpret_cast<double*>(smem + region_a_bytes);        // [G][D]
    int32_t* sel = reinterpret_cast<int32_t*>(dq + G * D);                 // [G][kMaxFusedK]
    float* parts = reinterpret_cast<float*>(sel + G * kMaxFusedK);        // [G][C][D+2]
    __shared__ SelectScratch<kThreads> sc;
    __shared__ unsigned char need[D];
    __shared__ float s_o[kWarps][D];
    __shared__ float s_m[kWarps], s_l[kWarps];

    const uint32_t C = cluster_size(), rank = cluster_rank();
    const uint32_t unit = blockIdx.x / C;
    const uint32_t b = unit / p.Hkv, kvh = unit % p.Hkv;
    const uint32_t Hq = p.Hkv * G;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool append = p.k_new != nullptr;

    // Everything below reads data earlier kernels wrote.
    stamp(p.probe, 0);
    asm volatile("griddepcontrol.wait;" ::: "memory");
    stamp(p.probe, 1);

    // The length and the query are independent loads: issue both before either is used.
    constexpr int QPT = (G * D + kThreads - 1) / kThreads;
    __half qv[QPT];
#pragma unroll
    for (int j = 0; j < QPT; ++j) {
        const int i = tid + j * kThreads, g = i / D, c = i % D;
        qv[j] = (i < G * D && c < int(p.head_dim))
                    ? p.q[(size_t(b) * Hq + size_t(kvh) * G + g) * p.head_dim + c]
                    : __float2half(0.0f);
    }
    const uint32_t t_old = static_cast<uint32_t>(p.len[p.layer * p.B + b]);
    const uint32_t n_tok = t_old + (append ? 1u : 0u);
    const uint32_t P = (n_tok + p.S - 1) / p.S;
    const size_t s = (size_t(p.layer) * p.B + b) * p.Hkv + kvh;
    if (append && t_old >= p.capacity) {  // host-checked; keep the cache intact
        if (tid == 0 && rank == 0) record_status(p.status, QK_DEV_CAPACITY);
        return;  // uniform over the cluster: no barrier is left waiting
    }

    // Query heads of this KV head widened to double (exact), and the rows they need.
    // MHA: odd channels take the integer fp16 -> f64 path (h2d_scaled), whose operand is
    // scaled by 2^-1008, so their query weight is pre-scaled by 2^1008 (exact: |q| <
    // 2^16 keeps it finite).
#pragma unroll
    for (int j = 0; j < QPT; ++j) {
        const int i = tid + j * kThreads, c = i % D;
        if (i < G * D) {
            const double x = double(__half2float(qv[j]));
            dq[i] = (G == 1 && (c & 1)) ? x * 0x1p1008 : x;
        }
    }
    __syncthreads();
    for (int c = tid; c < D; c += kThreads) {
        unsigned char m = 0;
#pragma unroll
        for (int g = 0; g < G; ++g) m |= (dq[g * D + c] < 0.0) ? 2 : 1;
        need[c] = m;
    }
    __syncthreads();

    // This CTA's page range, tile aligned.
    const uint32_t per = ((P + C - 1) / C + kMetaTile - 1) / kMetaTile * kMetaTile;
    const uint32_t r_begin = min(P, rank * per), r_end = min(P, r_begin + per);

    // ---- phase A: append into the newest page (owner CTA only) ----------------------
    // Done after the first metadata chunk's copies are in flight (see phase B); the staged
    // copy of the newest page is patched with the new min/max before it is used.
    const uint32_t new_page = append ? t_old / p.S : 0xffffffffu;
    const bool owner = append && new_page >= r_begin && new_page < r_end;
    __half new_min = __float2half(0.0f), new_max = __float2half(0.0f);

    // ---- phase B: estimate this CTA's pages -------------------------------------------
    const __half* mslice = p.meta + s * p.slice_meta;
    for (uint32_t c0 = r_begin; c0 < r_end; c0 += PPC) {
        const uint32_t npg = min(uint32_t(PPC), r_end - c0);
        const int ntiles = int((npg + kMetaTile - 1) / kMetaTile);
        constexpr int CHUNKS = kMetaTile * 2 / 16;
#pragma unroll
        for (int grp = 0; grp < kGroups; ++grp) {
            const int n_items = ntiles * CH_PER_GROUP * NROW * CHUNKS;
            for (int i = tid; i < n_items; i += kThreads) {
                const int part = i % CHUNKS;
                int rest = i / CHUNKS;
                const int r = rest % NROW;
                rest /= NROW;
                const int c = grp * CH_PER_GROUP + rest % CH_PER_GROUP;
                const int t = rest / CH_PER_GROUP;
                const int minmax = (G == 1) ? ((need[c] & 2) ? 0 : 1) : r;
                if (G > 1 && !(need[c] & (minmax == 0 ? 2 : 1))) continue;
                const __half* src = mslice + (size_t(c0 / kMetaTile + t) * 2 + minmax) * D * kMetaTile +
                                    size_t(c) * kMetaTile + part * 8;
                __half* dst = stage + (size_t(r) * D + c) * PPC + t * kMetaTile + part * 8;
                cp_async16(dst, src);
            }
            cp_async_commit();
        }
    if (c0 == r_begin && owner && tid < D) {  // phase A, overlapping the copies above
        const uint32_t c = tid, row = t_old % p.S;
        const size_t in = (size_t(b) * p.Hkv + kvh) * p.head_dim + c;
        const __half x = c < p.head_dim ? p.k_new[in] : __float2half(0.0f);
        const __half y = c < p.head_dim ? p.v_new[in] : __float2half(0.0f);
        const size_t kv = s * p.slice_kv + (size_t(new_page) * p.S + row) * D + c;
        p.k_pool[kv] = x;
        p.v_pool[kv] = y;
        const size_t mbase = s * p.slice_meta + size_t(new_page / kMetaTile) * 2 * D * kMetaTile +
                             size_t(c) * kMetaTile + (new_page % kMetaTile);
        __half* mnp = p.meta + mbase;
        __half* mxp = p.meta + mbase + size_t(D) * kMetaTile;
        if (row == 0) {
            new_min = x;
            new_max = x;
        } else {
            new_min = *mnp;
            new_max = *mxp;
            const float xf = __half2float(x);
            if (xf < __half2float(new_min)) new_min = x;
            if (xf > __half2float(new_max)) new_max = x;
        }
        *mnp = new_min;
        *mxp = new_max;
    }
        // Thread -> (page, query-head subset) of this chunk.
        constexpr int TPP = kThreads / PPC;  // threads per page: 1 (MHA) or 2 (GQA)
        constexpr int GPT = (G + TPP - 1) / TPP;
        const int pi = tid % PPC, gsub = tid / PPC;
        const bool active = uint32_t(pi) < npg;
        double acc[GPT];
#pragma unroll
        for (int j = 0; j < GPT; ++j) acc[j] = 0.0;
#pragma unroll
        for (int grp = 0; grp < kGroups; ++grp) {
            if (grp == 0) cp_async_wait<kGroups - 1>();
            if (grp == 1) cp_async_wait<kGroups - 2>();
            if (grp == 2) cp_async_wait<kGroups - 3>();
            if (grp == 3) cp_async_wait<0>();
            __syncthreads();
            if (owner && new_page >= c0 && new_page < c0 + PPC && tid < D &&
                tid / CH_PER_GROUP == grp) {
                // Replace the staged (pre-append) metadata of the newest page.
                const int c = tid;
                const uint32_t col = new_page - c0;
                if (G == 1) {
                    stage[size_t(c) * PPC + col] = (need[c] & 2) ? new_min : new_max;
                } else {
                    stage[size_t(0 * D + c) * PPC + col] = new_min;
                    stage[size_t(1 * D + c) * PPC + col] = new_max;
                }
            }
            if (owner) __syncthreads();
            if (active && G == 1) {
                // Channel pairs: the even one converts on the XU pipe (F2F), the odd one
                // with three integer ops (h2d_scaled), so the two pipes share the work.
                const unsigned short* st16 = reinterpret_cast<const unsigned short*>(stage);
#pragma unroll
                for (int cc = 0; cc < CH_PER_GROUP; cc += 2) {
                    const int c = grp * CH_PER_GROUP + cc;
                    const double2 w = *reinterpret_cast<const double2*>(dq + c);
                    const unsigned short h0 = st16[size_t(c) * PPC + pi];
                    const unsigned short h1 = st16[size_t(c + 1) * PPC + pi];
                    acc[0] = __fma_rn(w.x, h2d(__ushort_as_half(h0)), acc[0]);
                    acc[0] = __fma_rn(w.y, h2d_scaled(h1), acc[0]);
                }
            } else if (active) {
#pragma unroll 4
                for (int cc = 0; cc < CH_PER_GROUP; ++cc) {
                    const int c = grp * CH_PER_GROUP + cc;
                    {
                        const double lo = h2d(stage[size_t(c) * PPC + pi]);
                        const double hi = h2d(stage[size_t(D + c) * PPC + pi]);
#pragma unroll
                        for (int j = 0; j < GPT; ++j) {
                            const int g = gsub * GPT + j;
                            if (g < G) {
                                const double w = dq[g * D + c];
                                acc[j] = __fma_rn(w, (w < 0.0) ? lo : hi, acc[j]);
                            }
                        }
                    }
                }
            }
        }
        if (active) {
#pragma unroll
            for (int j = 0; j < GPT; ++j) {
                const int g = gsub * GPT + j;
                if (g < G)
                    p.ws_scores[(size_t(b) * Hq + size_t(kvh) * G + g) * p.Pmax + c0 + pi] = acc[j];
            }
        }
        __syncthreads();  // stage reused by the next chunk
    }

    // Scores of every CTA of the unit are visible after this barrier (and so is the new
    // K/V row written in phase A).
    stamp(p.probe, 2);
    cluster_sync_acqrel();
    stamp(p.probe, 3);
    if (append && rank == 0 && tid == 0) {
        // Every CTA of this unit has read the old length.  The last unit of the sequence
        // to get here publishes the new length for the next step.
        if (atomicAdd(p.len_ticket + p.layer * p.B + b, 1) == int(p.Hkv) - 1) {
            p.len_ticket[p.layer * p.B + b] = 0;
            p.len[p.layer * p.B + b] = int32_t(n_tok);
        }
    }

    // ---- phase C: selection (redundantly in every CTA of the cluster) ----------------
    const bool all_pages = p.k_budget >= P;
    const uint32_t count = all_pages ? P : p.k_budget;
    if (!all_pages) {
        const uint32_t n_cand = p.force ? P - 1 : P;
        const uint32_t target = p.force ? p.k_budget - 1 : p.k_budget;
        for (int g = 0; g < G; ++g) {
            int32_t* list = sel + g * kMaxFusedK;
            if (target > 0) {
                unsigned long long kmax, kmin;
                const double* src = p.ws_scores + (size_t(b) * Hq + size_t(kvh) * G + g) * p.Pmax;
                const int kpt = load_keys<kThreads>(src, n_cand, keys, sc, &kmax, &kmin);
                sel_stamp(p.probe, 8);
                block_select<kThreads>(keys, kpt, n_cand, target, kmax, kmin, list, sc, p.probe);
            }
            if (tid == 0 && p.force) list[target] = int32_t(P - 1);
        }
        __syncthreads();
    }
    if (rank == 0 && (p.pages_out || p.counts_out)) {
        for (int g = 0; g < G; ++g) {
            const size_t bh = size_t(b) * Hq + size_t(kvh) * G + g;
            if (p.pages_out)
                for (uint32_t i = tid; i < count && i < p.pstride; i += kThreads)
                    p.pages_out[bh * p.pstride + i] = all_pages ? int32_t(i) : sel[g * kMaxFusedK + i];
            if (p.counts_out && tid == 0) p.counts_out[bh] = int32_t(count);
        }
    }

    stamp(p.probe, 4);
    // ---- phase D: attention over this CTA's share of every head's pages ---------------
    const uint32_t i_begin = uint32_t((uint64_t(count) * rank) / C);
    const uint32_t i_end = uint32_t((uint64_t(count) * (rank + 1)) / C);
    const __half* kslice = p.k_pool + s * p.slice_kv;
    const __half* vslice = p.v_pool + s * p.slice_kv;
    const int chunk = lane % CPR, rgrp = lane / CPR;
    for (int g = 0; g < G; ++g) {
        const size_t bh = size_t(b) * Hq + size_t(kvh) * G + g;
        float qf[8];
        load_q8<D>(p.q + bh * p.head_dim, p.head_dim, qf);
        float m = -CUDART_INF_F, l = 0.0f, o[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) o[j] = 0.0f;
        for (uint32_t i = i_begin + warp; i < i_end; i += kWarps) {
            const uint32_t pg = all_pages ? i : uint32_t(sel[g * kMaxFusedK + i]);
            const uint32_t plen = min(p.S, n_tok - pg * p.S);
            warp_fold_page<D, true>(kslice + size_t(pg) * p.S * D, vslice + size_t(pg) * p.S * D,
                                    plen, qf, p.scale_log2, m, l, o);
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
        float M = -CUDART_INF_F;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) M = fmaxf(M, s_m[w]);
        float L = 0.0f, wsc[kWarps];
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            wsc[w] = (s_m[w] == -CUDART_INF_F) ? 0.0f : exp2f(s_m[w] - M);
            L += s_l[w] * wsc[w];
        }
        float* slot = parts + (size_t(g) * 8 + rank) * (D + 2);
        for (int d = tid; d < D; d += kThreads) {
            float acc = 0.0f;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) acc += s_o[w][d] * wsc[w];
            if (C == 1) slot[2 + d] = acc;
            else st_cluster_f32(slot + 2 + d, 0, acc);
        }
        if (tid == 0) {
            if (C == 1) {
                slot[0] = M;
                slot[1] = L;
            } else {
                st_cluster_f32(slot, 0, M);
                st_cluster_f32(slot + 1, 0, L);
            }
        }
        __syncthreads();  // s_o / s_m reused by the next head
    }
    asm volatile("griddepcontrol.launch_dependents;");
    stamp(p.probe, 5);
    if (C > 1) cluster_sync_acqrel();
    stamp(p.probe, 6);
    if (rank != 0) return;

    // Rank 0: merge the C partials of every head in rank order.  One thread per head
    // turns the C maxima into weights w_r = exp2(m_r - M) / L; then every channel is a
    // C-term dot product.
    float* wts = s_o[0];  // [G][8] (s_o is free now)
    if (tid < G) {
        const float* base = parts + size_t(tid) * 8 * (D + 2);
        float Mg = -CUDART_INF_F;
        for (uint32_t r = 0; r < C; ++r) Mg = fmaxf(Mg, base[r * (D + 2)]);
        float Lg = 0.0f;
        for (uint32_t r = 0; r < C; ++r) {
            const float mr = base[r * (D + 2)];
            const float w = (mr == -CUDART_INF_F) ? 0.0f : exp2f(mr - Mg);
            wts[tid * 8 + r] = w;
            Lg += base[r * (D + 2) + 1] * w;
        }
        const float inv = 1.0f / Lg;
        for (uint32_t r = 0; r < C; ++r) wts[tid * 8 + r] *= inv;
    }
    __syncthreads();
    for (int i = tid; i < G * int(p.head_dim); i += kThreads) {
        const int g = i / int(p.head_dim), d = i % int(p.head_dim);
        const size_t bh = size_t(b) * Hq + size_t(kvh) * G + g;
        const float* base = parts + size_t(g) * 8 * (D + 2) + 2 + d;
        float acc = 0.0f;
        for (uint32_t r = 0; r < C; ++r) acc = fmaf(base[r * (D + 2)], wts[g * 8 + r], acc);
        if (p.out_dtype == QK_DTYPE_F32) static_cast<float*>(p.out)[bh * p.head_dim + d] = acc;
        else static_cast<__half*>(p.out)[bh * p.head_dim + d] = __float2half_rn(acc);
    }
    stamp(p.probe, 7);
}

template <int D, int G>
int run_fused(qk_cache* c, const FusedParams& prm, uint32_t batch, uint32_t cluster,
              cudaStream_t st) {
    using LY = Layout<D, G>;
    const size_t region_a = LY::region_a(c->Pmax);
    const size_t smem = LY::bytes(c->Pmax);
    auto kern = decode_fused_kernel<D, G>;
    static size_t configured = 0;
    if (smem > configured) {
        int rc = cuda_check(
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)),
            "decode_fused_kernel smem");
        if (rc) return rc;
        cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        configured = smem;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(batch * c->Hkv * cluster);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attrs[2];
    attrs[0].id = cudaLaunchAttributeClusterDimension;
    attrs[0].val.clusterDim.x = cluster;
    attrs[0].val.clusterDim.y = 1;
    attrs[0].val.clusterDim.z = 1;
    attrs[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attrs[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attrs;
    cfg.numAttrs = 2;
    const int rc = cuda_check(cudaLaunchKernelEx(&cfg, kern, prm, uint32_t(region_a)),
                              "decode_fused_kernel");
    c->launches++;
    return rc;
}

template <int D>
int dispatch_g(qk_cache* c, const FusedParams& prm, uint32_t batch, uint32_t cluster,
               cudaStream_t st) {
    switch (c->G) {
        case 1: return run_fused<D, 1>(c, prm, batch, cluster, st);
        case 2: return run_fused<D, 2>(c, prm, batch, cluster, st);
        case 4: return run_fused<D, 4>(c, prm, batch, cluster, st);
        case 8: return run_fused<D, 8>(c, prm, batch, cluster, st);
        default: return set_error(QK_ERR_UNSUPPORTED, "qk_decode_step: GQA group");
    }
}

// Unfused reference sequence of the same step (used when the fused kernel's limits --
// kMaxFusedK selected pages per head -- are exceeded).
int decode_unfused(qk_cache* c, uint32_t layer, const __half* q, const __half* k,
                   const __half* v, uint32_t batch, const qk_selection_cfg& cfg,
                   uint32_t max_pages, void* out, int out_dtype, int32_t* pages,
                   uint32_t pstride, int32_t* counts, cudaStream_t st) {
    int rc = QK_OK;
    if (k) rc = launch_append(c, layer, k, v, batch, st);
    if (rc) return rc;
    rc = launch_estimate(c, layer, q, batch, c->ws_scores, c->Pmax, max_pages, st);
    if (rc) return rc;
    qk_selection_cfg eff = cfg;
    if (!cfg.per_layer_enabled) eff.token_budget = UINT32_MAX;
    int32_t* sel = pages ? pages : c->ws_pages;
    const uint32_t sstride = pages ? pstride : c->Pmax;
    int32_t* cnt = counts ? counts : c->ws_counts;
    rc = launch_topk(c, layer, c->ws_scores, c->Pmax, batch, eff, sel, sstride, cnt, max_pages, st);
    if (rc) return rc;
    const uint32_t kk = eff.token_budget / c->S;
    const uint32_t max_list = kk < max_pages ? kk : max_pages;
    return launch_attend(c, layer, q, batch, sel, sstride, cnt, false, max_list, out, out_dtype,
                         nullptr, st);
}

}  // namespace

// Cluster size: enough CTAs per unit to put ~2 CTAs on every SM at batch 1, at most 8,
// and never more than the pages warrant (one 64-page tile per CTA minimum).
uint32_t fused_cluster_size(const qk_cache* c, uint32_t batch, uint32_t pages) {
    const uint32_t units = batch * c->Hkv;
    uint32_t cl = 1;
    while (cl < 8 && units * cl * 2 <= 2 * 148 && (pages + cl * 2 * kMetaTile - 1) / (cl * 2 * kMetaTile) >= 1 &&
           pages > cl * kMetaTile)
        cl *= 2;
    return cl;
}

int launch_decode(qk_cache* c, uint32_t layer, const __half* q, const __half* k,
                  const __half* v, uint32_t batch, const qk_selection_cfg& cfg,
                  uint32_t max_pages, void* out, int out_dtype, int32_t* pages,
                  uint32_t pstride, int32_t* counts, cudaStream_t st) {
    const uint32_t kk = cfg.per_layer_enabled ? cfg.token_budget / c->S : UINT32_MAX;
    const bool fits = (kk >= c->Pmax || kk <= kMaxFusedK) && (c->D == 64 || c->D == 128);
    if (!fits)
        return decode_unfused(c, layer, q, k, v, batch, cfg, max_pages, out, out_dtype, pages,
                              pstride, counts, st);
    FusedParams prm{};
    prm.k_pool = c->k_pool;
    prm.v_pool = c->v_pool;
    prm.meta = c->meta;
    prm.len = c->d_len;
    prm.len_ticket = c->len_ticket;
    prm.status = c->d_status;
    prm.q = q;
    prm.k_new = k;
    prm.v_new = v;
    prm.ws_scores = c->ws_scores;
    prm.out = out;
    prm.pages_out = pages;
    prm.counts_out = counts;
    prm.slice_kv = c->slice_kv;
    prm.slice_meta = c->slice_meta;
    prm.layer = layer;
    prm.B = c->B;
    prm.Hkv = c->Hkv;
    prm.S = c->S;
    prm.head_dim = c->desc.head_dim;
    prm.Pmax = c->Pmax;
    prm.capacity = c->desc.max_tokens;
    prm.pstride = pstride;
    prm.k_budget = kk;
    prm.force = cfg.force_include_recent ? 1 : 0;
    prm.out_dtype = out_dtype;
    prm.scale_log2 = float(1.4426950408889634 / sqrt(double(c->desc.head_dim)));
    prm.probe = c->probe;
    const uint32_t cluster = fused_cluster_size(c, batch, max_pages);
    switch (c->D) {
        case 64: return dispatch_g<64>(c, prm, batch, cluster, st);
        case 128: return dispatch_g<128>(c, prm, batch, cluster, st);
        default: return set_error(QK_ERR_UNSUPPORTED, "qk_decode_step: head_dim");
    }
}

}  // namespace qk

// decode.cu -- one Quest decode step for a layer in ONE kernel launch:
//     KvCache::append (fused metadata update) -> estimate_all -> select_top_k ->
//     sparse_attention with a split-KV log-sum-exp merge
// (R/README.md:151-158 usage; metrics.cpp:90-95 step order; kv_store.cpp:19-47;
//  criticality.cpp:9-81; attention.cpp:54-116).
//
// Work decomposition: one thread-block CLUSTER of C CTAs (512 threads, one CTA per SM) per
// (sequence, KV head) unit; C is chosen so the grid fills the 148 SMs in one wave.
//   phase A  the CTA owning the newest page appends the token's K/V row and updates that
//            page's min/max metadata in HBM (strict compares, first-seen kept);
//   phase B  each CTA estimates a contiguous range of the pages that compete on score
//            (bitwise fp64 chains, see estimate.cu) for all G query heads of the KV head;
//            the scores stay in the CTA's shared memory;  -- cluster barrier --
//   phase C  every CTA pulls the unit's scores over DSMEM and runs the exact selection
//            (select.cuh) itself, so no second exchange is needed;
//   phase D  each CTA attends its share of every query head's selected pages (warps
//            stream pages into an online softmax, as attend.cu) and ships its (m, l, o)
//            partial to rank 0's shared memory over DSMEM;  -- cluster barrier --
//            rank 0 merges the partials in rank order and writes the output.
// With force_include_recent the newest page never competes on score (top-(K-1) of pages
// [0, P-1) plus page P-1 == the reference's replace-the-weakest rule, see topk.cu), so its
// metadata is not estimated at all; when K >= P nothing is estimated.  qk_debug_keep_scores
// restores the full estimate_all (every page, scores kept in HBM) for parity tests.
// The launch uses programmatic dependent launch; griddepcontrol.wait precedes every read
// of data a prior kernel wrote.
#include <cstring>
#include <type_traits>
#include <vector>

#include "attend_warp.cuh"
#include "select.cuh"

namespace qk {
namespace {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kMetaGroups = 8;          // channel groups of the metadata pipeline (mbarriers)
constexpr int kSelThreads = 128;        // one selection group: a warp per scheduler
constexpr int kSelGroups = kThreads / kSelThreads;
constexpr int kSelKpt = 16;             // keys per thread of a selection group
constexpr uint32_t kMaxFusedK = 512;    // selected pages per query head kept in smem
constexpr uint32_t kMaxCluster = 16;
// Cluster-exchanged selection keys per CTA (MHA has no metadata stage in shared memory,
// so its budget covers 128K-token contexts).
constexpr size_t keys_budget(int G) { return G == 1 ? 96 * 1024 : 40 * 1024; }
constexpr uint32_t kTail = 64;  // MHA: pages past the 512-page passes staged with cp.async
constexpr size_t kMaxSmem = 227 * 1024 - 8 * 1024;  // opt-in limit minus static smem

__device__ __forceinline__ double h2d(__half h) {
    double d;
    asm("cvt.f64.f16 %0, %1;" : "=d"(d) : "h"(__half_as_ushort(h)));
    return d;
}

// fp16 bits -> the double sel * 2^-1008, exactly, for every finite fp16 (normal,
// subnormal, +-0): the 15 exponent/mantissa bits land in the double's exponent/mantissa
// fields unbiased (hence the 2^-1008 scale; fp16 subnormals become double subnormals with
// the same scale) and the sign moves from bit 25 to bit 31 (t + 63*s clears bit 25 and
// sets bit 31).  Three integer ops instead of one F2F on the XU pipe.
__device__ __forceinline__ double h2d_scaled(unsigned short h) {
    const uint32_t t = uint32_t(h) << 10;
    const uint32_t s = t & 0x02000000u;
    return __hiloint2double(int(t + s * 63u), 0);
}

__device__ __forceinline__ void stamp(unsigned long long* probe, int slot) {
    if (probe != nullptr) {  // (callers are warp-uniform)
        if (threadIdx.x == 0) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            probe[blockIdx.x * kProbeSlots + slot] = t;
        }
        __syncwarp();  // reconverge: a diverged warp would take the collectives' slow path
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
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t map_rank(const void* local_addr, uint32_t rank) {
    uint32_t ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(local_addr)), "r"(rank));
    return ra;
}

// Asynchronous remote shared-memory stores that complete transaction bytes on the
// receiver's mbarrier (the receiver's wait is the only synchronisation they need).
__device__ __forceinline__ void st_async_u64(uint32_t cluster_addr, unsigned long long v, uint32_t cluster_bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(cluster_addr),
                 "l"(v), "r"(cluster_bar)
                 : "memory");
}
__device__ __forceinline__ void st_async_f32(uint32_t cluster_addr, float v, uint32_t cluster_bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f32 [%0], %1, [%2];" ::"r"(cluster_addr),
                 "f"(v), "r"(cluster_bar)
                 : "memory");
}

// mbarrier + bulk-copy (TMA 1D) helpers.
__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx_only(unsigned long long* bar, uint32_t bytes) {
    asm volatile("mbarrier.expect_tx.relaxed.cluster.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "QK_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra QK_WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(unsigned long long* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "QK_WAITC_%=:\n"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra QK_WAITC_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

struct FusedParams {
    __half* k_pool;
    __half* v_pool;
    __half* meta;
    uint32_t* prange;     // [slices][mrow] page magnitude records
    int32_t* len;
    int32_t* len_ticket;
    int32_t* status;
    const __half* q;
    const __half* k_new;  // nullable
    const __half* v_new;
    double* ws_scores;    // [B][Hq][Pmax]: score exchange when keys do not fit smem
    void* out;
    int32_t* pages_out;   // nullable
    int32_t* counts_out;  // nullable
    size_t slice_kv, slice_meta;
    uint32_t mrow;        // pages per metadata row
    uint32_t layer, B, Hkv, S, head_dim, Pmax, capacity, pstride;
    uint32_t k_budget;    // pages per query head (UINT32_MAX: selection disabled)
    uint32_t key_cap;     // key slots per head in the cluster-exchanged key array (0: HBM)
    int force, out_dtype, keep_scores;
    int prefetch;         // L2-prefetch certainly-selected pages during the selection
    float scale_log2;
    unsigned long long* probe;  // optional [grid][kProbeSlots] globaltimer stamps
    uint32_t* done_flag;        // optional host-mapped completion word (host step)
    uint32_t* done_counter;     // [0] units finished in this launch (reset by the last one),
                                // [1] host steps completed (the value published)
};

// Host-step completion (called by thread 0 of a unit's rank-0 CTA once its outputs are
// written and ordered by a CTA barrier): the last unit publishes the sequence number with
// release at system scope, after every unit's fence.
__device__ __forceinline__ void signal_done(const FusedParams& p, uint32_t units) {
    __threadfence_system();
    if (atomicAdd(p.done_counter, 1u) == units - 1) {
        *p.done_counter = 0;  // for the next launch (ordered by the kernel boundary)
        // The sequence lives on the device (a replayed CUDA graph carries fixed parameters):
        // the host expects one more than the last value it saw.
        const uint32_t seq = p.done_counter[1] + 1u;
        p.done_counter[1] = seq;
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p.done_flag), "r"(seq) : "memory");
    }
}

// Dynamic shared memory:
//   [region A: metadata stage | after the estimate: selection scratch + padded keys]
//   [keys: G*key_cap u64, written by every CTA of the cluster]
//   [dq G*D doubles] [selected pages G*kMaxFusedK ints] [partials G*C*(D+2) floats]
//   [kMetaGroups mbarriers]
template <int D, int G>
struct Layout {
    static constexpr int NROW = (G == 1) ? 1 : 2;    // metadata rows staged per channel
    static constexpr int PPC = (G == 1) ? 512 : 256;  // pages per estimate chunk
    // GQA: the metadata stage; MHA: the channel-group partial sums [8][512] (fp64) and the
    // tail rows [D][kTail].
    static constexpr size_t stage_bytes =
        (G == 1) ? size_t(8) * kThreads * 8 + size_t(D) * kTail * 2 : size_t(NROW) * D * PPC * 2;
    static constexpr size_t scratch_bytes =
        kSelGroups * sizeof(SelectScratch<kSelThreads>) + sizeof(SelectScratch<kThreads>);
    static size_t region_a(uint32_t pmax) {
        const size_t kpt = (pmax + kThreads - 1) / kThreads;
        const size_t sel = scratch_bytes + size_t(kThreads) * (kpt + 1) * 8;
        return stage_bytes > sel ? stage_bytes : sel;
    }
    static size_t bytes(uint32_t pmax, uint32_t key_cap, uint32_t cluster) {
        return region_a(pmax) + size_t(G) * key_cap * 8 + size_t(G) * D * 8 +
               size_t(G) * kMaxFusedK * 4 + size_t(G) * cluster * (D + 2) * 4 + kMetaGroups * 8;
    }
};

template <int D, int G>
__global__ void __launch_bounds__(kThreads, 1) decode_fused_kernel(const FusedParams p,
                                                                    uint32_t region_a_bytes) {
    using LY = Layout<D, G>;
    constexpr int NROW = LY::NROW, PPC = LY::PPC;
    constexpr int CH_PER_GROUP = D / kMetaGroups;
    constexpr int CPR = D / 8;
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t C = cluster_size(), rank = cluster_rank();
    __half* stage = reinterpret_cast<__half*>(smem);  // [NROW][D][PPC], region A
    auto* grp_sc = reinterpret_cast<SelectScratch<kSelThreads>*>(smem);  // region A, later
    auto* big_sc = reinterpret_cast<SelectScratch<kThreads>*>(grp_sc + kSelGroups);
    unsigned long long* pkeys = reinterpret_cast<unsigned long long*>(big_sc + 1);  // padded
    unsigned long long* keys = reinterpret_cast<unsigned long long*>(smem + region_a_bytes);
    double* dq = reinterpret_cast<double*>(keys + size_t(G) * p.key_cap);  // [G][D]
    int32_t* sel = reinterpret_cast<int32_t*>(dq + G * D);                 // [G][kMaxFusedK]
    float* parts = reinterpret_cast<float*>(sel + G * kMaxFusedK);        // [G][D+2][C]
    unsigned long long* mbar = reinterpret_cast<unsigned long long*>(
        (reinterpret_cast<uintptr_t>(parts + size_t(G) * C * (D + 2)) + 7) & ~uintptr_t(7));
    __shared__ unsigned char need[D];
    __shared__ float s_o[kWarps][D];
    __shared__ float s_m[kWarps], s_l[kWarps];

    // merge_bar (rank 0): the peers' partials land on it (st.async, transaction bytes).
    // keys_bar (every CTA): every CTA of the cluster arrives once with release after its
    // estimate (its scores, the appended K/V row and its read of the old length are then
    // visible), and the pushed selection keys complete transaction bytes on it.
    __shared__ __align__(8) unsigned long long merge_bar[1], keys_bar[1];
    if (threadIdx.x == 0) {
        mbar_init(merge_bar, 1);
        mbar_init(keys_bar, C);
        if (C > 1 && cluster_rank() == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(merge_bar)),
                         "r"(uint32_t((C - 1) * G * (D + 2) * 4))
                         : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    const uint32_t unit = blockIdx.x / C;
    const uint32_t b = unit / p.Hkv, kvh = unit % p.Hkv;
    const uint32_t Hq = p.Hkv * G;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool append = p.k_new != nullptr;

    // Peers store into this CTA's shared memory during the estimate: the cluster must have
    // started everywhere first (arrive now, wait just before the first remote store).
    __syncwarp();  // thread 0's barrier set-up above: reconverge before the aligned arrive
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
    // Everything below reads data earlier kernels wrote.
    stamp(p.probe, 0);
    if (p.probe) {
        if (tid == 0) p.probe[blockIdx.x * kProbeSlots + 24] = clock64();
        __syncwarp();
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");
    // The next kernel may launch now: its CTAs take idle SMs and block in their own
    // griddepcontrol.wait until this grid has completed (hides the launch latency).
    asm volatile("griddepcontrol.launch_dependents;");
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
        if (p.done_flag && tid == 0 && rank == 0) signal_done(p, gridDim.x / C);
        return;  // uniform over the cluster: no barrier is left waiting
    }

    // Query heads of this KV head widened to double (exact), and the rows they need.
    // MHA: odd channels take the integer fp16 -> f64 path (h2d_scaled), whose operand is
    // scaled by 2^-1008, so their query weight is pre-scaled by 2^1008 (exact: |q| <
    // 2^16 keeps it finite).  Per head also sum|q| and the smallest ulp code of q (the
    // split-estimate certificate, phase B).
    __shared__ double s_qabs[G];
    __shared__ unsigned int s_qcode[G];
    __shared__ double s_qpart[D / 32];
    __shared__ unsigned int s_qcodep[D / 32];
    if constexpr (G == 1) {
        // Thread c < D holds channel c: its weight, its row and its warp's share of the
        // q statistics (per-warp partials: sum|q| of fp16 values is exact in any order).
        if (tid < D) {
            const double x = double(__half2float(qv[0]));
            dq[tid] = (tid & 1) ? x * 0x1p1008 : x;
            need[tid] = (x < 0.0) ? 2 : 1;
            double a = fabs(x);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);  // exact
            const unsigned int code = __reduce_min_sync(0xffffffffu, ulp_code(__half_as_ushort(qv[0])));
            if (lane == 0) {
                s_qpart[warp] = a;
                s_qcodep[warp] = code;
            }
        }
        __syncthreads();
    } else {
    if (tid < G) {
        s_qabs[tid] = 0.0;
        s_qcode[tid] = 31u;
    }
#pragma unroll
    for (int j = 0; j < QPT; ++j) {
        const int i = tid + j * kThreads, c = i % D;
        if (i < G * D) {
            const double x = double(__half2float(qv[j]));
            dq[i] = (G == 1 && (c & 1)) ? x * 0x1p1008 : x;
        }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < QPT; ++j) {
        const int i = tid + j * kThreads;  // warp-uniform head: D is a multiple of 32
        if (i < G * D) {
            double a = fabs(double(__half2float(qv[j])));
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);  // exact
            const unsigned int code = __reduce_min_sync(0xffffffffu, ulp_code(__half_as_ushort(qv[j])));
            if (lane == 0) {
                atomicAdd(&s_qabs[i / D], a);
                atomicMin(&s_qcode[i / D], code);
            }
        }
    }
    for (int c = tid; c < D; c += kThreads) {
        unsigned char m = 0;
#pragma unroll
        for (int g = 0; g < G; ++g) m |= (dq[g * D + c] < 0.0) ? 2 : 1;
        need[c] = m;
    }
    __syncthreads();
    }
    stamp(p.probe, 2);

    // Selection shape (criticality.cpp:47-59): K >= P -> every page; with force-recent
    // the candidates are pages [0, P-1) and target K-1, page P-1 is appended.
    const bool all_pages = p.k_budget >= P;
    const uint32_t count = all_pages ? P : p.k_budget;
    const uint32_t n_cand = all_pages ? 0u : (p.force ? P - 1 : P);
    const uint32_t n_est = p.keep_scores ? P : n_cand;
    // Keys exchanged through the cluster's shared memory only when they fit the key array
    // AND a shared-memory selection tier (phase C: <= kThreads*kSelKpt candidates);
    // otherwise every CTA writes its scores to HBM and the selection reads them there.
    const bool smem_keys = p.key_cap != 0 && key_slots(n_cand) <= p.key_cap &&
                           n_cand <= uint32_t(kThreads * kSelKpt);
    // (A one-CTA cluster exchanges nothing: plain shared stores and a CTA barrier.)
    if (tid == 0 && smem_keys && n_cand > 0 && C > 1)
        mbar_expect_tx_only(keys_bar, uint32_t(G) * n_cand * 8u);
    // This CTA's estimate range: contiguous, a multiple of 8 pages (16-byte metadata
    // pieces), balanced over the cluster.
    const uint32_t per = ((n_est + C - 1) / C + 7) & ~7u;
    const uint32_t r_begin = min(n_est, rank * per), r_end = min(n_est, r_begin + per);

    // ---- phase A: append into the newest page --------------------------------------------
    // Owner: the CTA whose estimate range holds the newest page (it patches its staged
    // copy of that page's metadata), else the last CTA.
    const uint32_t new_page = append ? t_old / p.S : 0xffffffffu;
    const uint32_t owner_rank = (append && new_page < n_est) ? new_page / per : C - 1;
    const bool owner = append && rank == owner_rank;
    const bool patch = owner && new_page < n_est;  // staged copy to patch
    __shared__ __half s_new_min[D], s_new_max[D];
    __shared__ uint32_t s_rec_scratch[D / 32];
    __shared__ uint32_t s_spec_pg[kWarps];  // each warp's speculatively prefetched page (or ~0u)
    if (tid < kWarps) s_spec_pg[tid] = 0xffffffffu;  // (ordered by the barriers below)
    bool appended = false, arrived = false;
    // Each CTA arrives once on every CTA's keys_bar; with release when it wrote data its
    // peers read (the owner's new K/V row, scores through HBM).
    auto arrive_keys = [&](bool release) {
        if (tid == 0) {
            if (release) asm volatile("fence.acq_rel.cluster;" ::: "memory");
            for (uint32_t r = 0; r < C; ++r)
                asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                                 map_rank(keys_bar, r))
                             : "memory");
        }
        arrived = true;
    };
    auto do_append = [&]() {
        if (tid < D) {
            const uint32_t c = tid, row = t_old % p.S;
            const size_t in = (size_t(b) * p.Hkv + kvh) * p.head_dim + c;
            const __half x = c < p.head_dim ? p.k_new[in] : __float2half(0.0f);
            const __half y = c < p.head_dim ? p.v_new[in] : __float2half(0.0f);
            const size_t kv = s * p.slice_kv + (size_t(new_page) * p.S + row) * D + c;
            p.k_pool[kv] = x;
            p.v_pool[kv] = y;
            __half* mnp = p.meta + meta_offset(p.slice_meta, p.mrow, s, new_page, D, 0, int(c));
            __half* mxp = p.meta + meta_offset(p.slice_meta, p.mrow, s, new_page, D, 1, int(c));
            __half new_min = x, new_max = x;
            if (row != 0) {
                new_min = *mnp;
                new_max = *mxp;
                const float xf = __half2float(x);
                if (xf < __half2float(new_min)) new_min = x;
                if (xf > __half2float(new_max)) new_max = x;
            }
            *mnp = new_min;
            *mxp = new_max;
            s_new_min[c] = new_min;
            s_new_max[c] = new_max;
            const uint32_t rec = page_record<D>(new_min, new_max, s_rec_scratch, 6);
            if (tid == 0) p.prange[s * p.mrow + new_page] = rec;
        }
        appended = true;
    };

    // ---- phase B: estimate this CTA's pages --------------------------------------------
    // All threads stage the needed metadata rows of a chunk with 16-byte cp.async in
    // kMetaGroups channel groups, then fold the groups into the fp64 sums as they land.
    //
    // Split chains.  The reference sums the 128 exact products q_i*x_i sequentially in
    // fp64 (criticality.cpp:16-21); one dependent DFMA costs ~34 cycles here, so a
    // sequential chain is ~2.2 us.  Instead each page keeps NACC accumulators over the
    // channel residues mod NACC and adds them pairwise at the end.  That is bitwise the
    // sequential sum whenever no partial sum can round: every product is a multiple of
    // 2^(uq + ux) (uq, ux = the smallest ulp exponents of the query and of the page's
    // metadata), so if sum_i |q_i|*|x_i| < 2^(53 + uq + ux) every partial sum -- in any order
    // -- is an exactly representable multiple of 2^(uq+ux).  The bound uses
    // sum|q| * max|x| from the page's magnitude record; a page that fails it (or the newest
    // page, patched in shared memory) is recomputed with the sequential chain.
    constexpr int NACC = (G == 1) ? 8 : 4;
    const __half* mslice = p.meta + s * p.slice_meta;
    const uint32_t* rslice = p.prange + s * p.mrow;
    stamp(p.probe, 21);
    asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
    stamp(p.probe, 22);
    if constexpr (G == 1) {
        // MHA: metadata straight into registers.  Warp (half, cg) covers pages
        // c0 + 256*half + 8*lane .. +7 over channels [cg*CPG, cg*CPG + CPG): one 16-byte
        // load per channel of its sign-selected row, every load instruction 512 contiguous
        // bytes, all of a pass in flight at once.  The 8 channel-group partial sums of a
        // page are added through shared memory (exact under the certificate; failing pages
        // take the sequential chain).  A remainder of <= kTail pages past the 512-page
        // passes is staged with cp.async at the start and finished after the last pass, so
        // it costs no extra round trip.
        constexpr int CPG = D / 8;  // channels per warp
        const int cg = warp & 7, half = warp >> 3;
        double* part = reinterpret_cast<double*>(smem);               // [8][512] (region A)
        __half* tstage = reinterpret_cast<__half*>(part + 8 * kThreads);  // [D][kTail]
        const uint32_t n_mine = r_end - r_begin;
        const uint32_t rem = n_mine % kThreads;
        const uint32_t tail = (n_mine > kThreads && rem != 0 && rem <= kTail) ? rem : 0u;
        const uint32_t main_end = r_end - tail;
        if (tail) {
            const int pieces = int((tail + 7) / 8);
            for (int i = tid; i < D * pieces; i += kThreads) {
                const int c = i / pieces, pc = i % pieces;
                const int minmax = (need[c] & 2) ? 0 : 1;
                cp_async16(tstage + size_t(c) * kTail + pc * 8,
                           mslice + (size_t(minmax) * D + c) * p.mrow + main_end + pc * 8);
            }
            cp_async_commit();
        }
        const uint32_t tail_rec = (tid < int(tail)) ? __ldg(rslice + main_end + tid) : 0u;
        if (r_begin < r_end) stamp(p.probe, 3);

        // The certificate, the sequential fallback and the hand-off of one page's score.
        auto finish = [&](uint32_t pg, double sc, uint32_t rec) {
            double qabs = 0.0;
            unsigned int qcode = 31u;
#pragma unroll
            for (int w = 0; w < D / 32; ++w) {
                qabs += s_qpart[w];
                qcode = min(qcode, s_qcodep[w]);
            }
            const uint32_t xcode = rec >> 16;
            bool exact = xcode >= 31u || qcode >= 31u;
            if (!exact) {
                const double bound = __dmul_ru(
                    qabs, double(__half2float(__ushort_as_half(uint16_t(rec & 0x7fffu)))));
                const int e = 5 + int(qcode) + int(xcode);
                exact = bound < __longlong_as_double(static_cast<long long>(e + 1023) << 52);
            }
            const bool newest = patch && pg == new_page;
            if (!exact || newest) {
                if (p.probe) atomicAdd(p.probe + blockIdx.x * kProbeSlots + 23, 1ull);
                // The reference's sequential chain (criticality.cpp:16-21).
                double a = 0.0;
                for (int c = 0; c < D; ++c) {
                    const int minmax = (need[c] & 2) ? 0 : 1;
                    const __half x = newest ? (minmax == 0 ? s_new_min[c] : s_new_max[c])
                                            : mslice[(size_t(minmax) * D + c) * p.mrow + pg];
                    const double w = (c & 1) ? dq[c] * 0x1p-1008 : dq[c];
                    a = __fma_rn(w, h2d(x), a);
                }
                sc = a;
            }
            if (smem_keys) {
                if (pg < n_cand) {
                    const unsigned long long k = order_key(sc);
                    if (C == 1) keys[key_slot(pg)] = k;
                    else
                        for (uint32_t r = 0; r < C; ++r) st_async_u64(map_rank(keys + key_slot(pg), r), k, map_rank(keys_bar, r));
                }
            }
            if (!smem_keys || p.keep_scores)
                p.ws_scores[(size_t(b) * Hq + size_t(kvh)) * p.Pmax + pg] = sc;
        };

        for (uint32_t c0 = r_begin; c0 < main_end; c0 += kThreads) {
            const uint32_t pbase = c0 + uint32_t(half) * 256 + uint32_t(lane) * 8;
            const bool act = pbase < main_end;  // pages past main_end: loaded in-bounds, unused
            const uint32_t pg = c0 + uint32_t(tid);  // the page this thread finishes below
            const uint32_t rec = pg < main_end ? __ldg(rslice + pg) : 0u;  // with the rows
            int4 v[CPG];
#pragma unroll
            for (int k = 0; k < CPG; ++k) {
                const int c = cg * CPG + k;
                const int minmax = (need[c] & 2) ? 0 : 1;
                v[k] = act ? ld_nc_v4(mslice + (size_t(minmax) * D + c) * p.mrow + pbase)
                           : make_int4(0, 0, 0, 0);
            }
            // The append overlaps the loads above (s_new_* are read after the barrier below).
            if (owner && !appended) {
                do_append();
                if (smem_keys && C > 1) arrive_keys(true);  // the new K/V row released early
            }
            if (tail && c0 == r_begin) {
                // The staged tail pages (issued first) are finished while this pass's
                // register loads are still in flight.
                cp_async_wait<0>();
                __syncthreads();  // tail rows and s_new_* visible
                if (uint32_t(tid) < tail) {
                    const uint32_t tpg = main_end + tid;
                    double tacc[8];
#pragma unroll
                    for (int j = 0; j < 8; ++j) tacc[j] = 0.0;
                    const unsigned short* t16 = reinterpret_cast<const unsigned short*>(tstage);
#pragma unroll 16
                    for (int c = 0; c < D; ++c) {
                        const unsigned short hh = t16[size_t(c) * kTail + tid];
                        tacc[c & 7] = __fma_rn(dq[c], (c & 1) ? h2d_scaled(hh) : h2d(__ushort_as_half(hh)), tacc[c & 7]);
                    }
                    finish(tpg, ((tacc[0] + tacc[1]) + (tacc[2] + tacc[3])) + ((tacc[4] + tacc[5]) + (tacc[6] + tacc[7])),
                           tail_rec);
                }
            }
            double acc[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[j] = 0.0;
            if (__any_sync(0xffffffffu, act)) {  // short ranges leave whole warps without pages
#pragma unroll
                for (int k = 0; k < CPG; ++k) {
                    const int c = cg * CPG + k;
                    const double w = dq[c];
                    const unsigned short* h = reinterpret_cast<const unsigned short*>(&v[k]);
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        acc[j] = __fma_rn(w, (c & 1) ? h2d_scaled(h[j]) : h2d(__ushort_as_half(h[j])), acc[j]);
                }
            }
            if (c0 == r_begin) stamp(p.probe, 5);
            double2* dst = reinterpret_cast<double2*>(part + cg * kThreads + half * 256 + lane * 8);
#pragma unroll
            for (int j = 0; j < 4; ++j) dst[j] = make_double2(acc[2 * j], acc[2 * j + 1]);
            __syncthreads();
            if (c0 == r_begin) stamp(p.probe, 6);
            double sc_pass = 0.0;
            if (pg < main_end) {
                const double sc = ((part[0 * kThreads + tid] + part[1 * kThreads + tid]) +
                                   (part[2 * kThreads + tid] + part[3 * kThreads + tid])) +
                                  ((part[4 * kThreads + tid] + part[5 * kThreads + tid]) +
                                   (part[6 * kThreads + tid] + part[7 * kThreads + tid]));
                finish(pg, sc, rec);
                sc_pass = sc;
            }
            if (p.prefetch && smem_keys && main_end - r_begin <= uint32_t(kThreads)) {
                // Speculative L2 prefetch of each warp's best page of the pass (the best of 32
                // pages is in the top 127 of 2047 ~86% of the time at cfg2): HBM idles between
                // the metadata stream and the selection, so half the budget's K/V starts early.
                // Only a hint -- the selection's own prefetch and the attention are unchanged.
                // Measured: 20.10 -> 19.35-19.49 us/layer; the best two per warp (the whole
                // budget) gains nothing, the fast CTAs' extra prefetches then slow the slowest
                // CTA's metadata stream -- and for the same reason only single-pass CTAs
                // speculate (with 4 passes per CTA, cfg3 and cfg5 lost 9 and 14 us).
                unsigned long long best = (pg < main_end && pg < n_cand) ? order_key(sc_pass) : 0ull;
                uint32_t bp = pg;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    const unsigned long long ok = __shfl_xor_sync(0xffffffffu, best, o);
                    const uint32_t op = __shfl_xor_sync(0xffffffffu, bp, o);
                    if (ok > best || (ok == best && op < bp)) {
                        best = ok;
                        bp = op;
                    }
                }
                if (lane == 0) s_spec_pg[warp] = best != 0ull ? bp : 0xffffffffu;
                if (lane == 0 && best != 0ull) {
                    const uint32_t pbytes = p.S * D * 2;
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(
                                     p.k_pool + s * p.slice_kv + size_t(bp) * p.S * D),
                                 "r"(pbytes) : "memory");
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(
                                     p.v_pool + s * p.slice_kv + size_t(bp) * p.S * D),
                                 "r"(pbytes) : "memory");
                }
            }
            if (c0 == r_begin) stamp(p.probe, 7);
            __syncthreads();  // part reused by the next pass
        }
        if (r_begin < r_end) stamp(p.probe, 4);
    } else {
    for (uint32_t c0 = r_begin; c0 < r_end; c0 += PPC) {
        const uint32_t npg = min(uint32_t(PPC), r_end - c0);
        const int n8 = int((npg + 7) / 8);  // 16-byte pieces per channel row
        // Thread -> (row, 16-byte piece): piece = tid % PIECES, rows tid / PIECES + k*RSTEP.
        constexpr int PIECES = PPC / 8, RSTEP = kThreads / PIECES;
        constexpr int ROWS = CH_PER_GROUP * NROW;  // staged rows per channel group
        const int my_piece = tid % PIECES;
        const bool piece_ok = my_piece < n8;
#pragma unroll 1
        for (int grp = 0; grp < kMetaGroups; ++grp) {
#pragma unroll
            for (int rr = tid / PIECES; rr < ROWS; rr += RSTEP) {
                const int r = rr % NROW;
                const int c = grp * CH_PER_GROUP + rr / NROW;
                const int minmax = (G == 1) ? ((need[c] & 2) ? 0 : 1) : r;
                const bool needed = (G == 1) || (need[c] & (minmax == 0 ? 2 : 1));
                if (piece_ok && needed)
                    cp_async16(stage + (size_t(r) * D + c) * PPC + my_piece * 8,
                               mslice + (size_t(minmax) * D + c) * p.mrow + c0 + my_piece * 8);
            }
            cp_async_commit();
        }
        if (c0 == r_begin) stamp(p.probe, 3);
        if (owner && !appended) {
            do_append();  // overlaps the copies above
            __syncthreads();  // s_new_min/max for the patch below
        }
        // Thread -> (page, query-head subset) of this chunk.
        constexpr int TPP = kThreads / PPC;  // threads per page: 1 (MHA) or 2 (GQA)
        constexpr int GPT = (G + TPP - 1) / TPP;
        const int pi = tid % PPC, gsub = tid / PPC;
        const uint32_t pg = c0 + pi;
        const bool active = uint32_t(pi) < npg;
        const uint32_t rec = active ? rslice[pg] : 0u;
        double acc[GPT][NACC];
#pragma unroll
        for (int j = 0; j < GPT; ++j)
#pragma unroll
            for (int k = 0; k < NACC; ++k) acc[j][k] = 0.0;
#pragma unroll 1
        for (int grp = 0; grp < kMetaGroups; ++grp) {
            cp_async_wait_n(kMetaGroups - 1 - grp);
            if (patch && new_page >= c0 && new_page < c0 + PPC) {  // CTA-uniform
                // Replace the staged (pre-append) metadata of the newest page.  The column
                // was copied by other threads' cp.async: every thread's copies of this
                // group must have landed before the patch, or a late copy would overwrite
                // it with the pre-append values.
                __syncthreads();
                if (tid < D && tid / CH_PER_GROUP == grp) {
                    const int c = tid;
                    const uint32_t col = new_page - c0;
                    stage[size_t(0 * D + c) * PPC + col] = s_new_min[c];
                    stage[size_t(1 * D + c) * PPC + col] = s_new_max[c];
                }
            }
            __syncthreads();
            if (c0 == r_begin && grp < 4) stamp(p.probe, 4 + grp);
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
                    acc[0][cc % NACC] = __fma_rn(w.x, h2d(__ushort_as_half(h0)), acc[0][cc % NACC]);
                    acc[0][(cc + 1) % NACC] = __fma_rn(w.y, h2d_scaled(h1), acc[0][(cc + 1) % NACC]);
                }
            } else if (active) {
#pragma unroll
                for (int cc = 0; cc < CH_PER_GROUP; ++cc) {
                    const int c = grp * CH_PER_GROUP + cc;
                    const double lo = h2d(stage[size_t(c) * PPC + pi]);
                    const double hi = h2d(stage[size_t(D + c) * PPC + pi]);
#pragma unroll
                    for (int j = 0; j < GPT; ++j) {
                        const int g = gsub * GPT + j;
                        if (g < G) {
                            const double w = dq[g * D + c];
                            acc[j][cc % NACC] = __fma_rn(w, (w < 0.0) ? lo : hi, acc[j][cc % NACC]);
                        }
                    }
                }
            }
        }
        if (active) {
#pragma unroll
            for (int j = 0; j < GPT; ++j) {
                const int g = gsub * GPT + j;
                if (g < G) {
                    double sc;
                    if (NACC == 8)
                        sc = ((acc[j][0] + acc[j][1]) + (acc[j][2] + acc[j][3])) +
                             ((acc[j][4 % NACC] + acc[j][5 % NACC]) + (acc[j][6 % NACC] + acc[j][7 % NACC]));
                    else
                        sc = (acc[j][0] + acc[j][1]) + (acc[j][2] + acc[j][3]);
                    // Certificate: sum|q| * max|x| < 2^(53 + uq + ux), ulp = 2^(code - 24).
                    const uint32_t xcode = rec >> 16, qcode = s_qcode[g];
                    bool exact = xcode >= 31u || qcode >= 31u;  // all-zero operands
                    if (!exact) {
                        const double bound = __dmul_ru(
                            s_qabs[g], double(__half2float(__ushort_as_half(uint16_t(rec & 0x7fffu)))));
                        const int e = 5 + int(qcode) + int(xcode);  // 53 + (qcode-24) + (xcode-24)
                        exact = bound < __longlong_as_double(static_cast<long long>(e + 1023) << 52);
                    }
                    if (!exact || (patch && pg == new_page)) {
                        // The sequential chain of the reference, from the staged rows.
                        double a = 0.0;
                        for (int c = 0; c < D; ++c) {
                            const double w = dq[g * D + c];
                            if (G == 1) {
                                const unsigned short h = reinterpret_cast<const unsigned short*>(stage)[size_t(c) * PPC + pi];
                                a = __fma_rn(w, (c & 1) ? h2d_scaled(h) : h2d(__ushort_as_half(h)), a);
                            } else {
                                const double lo = h2d(stage[size_t(c) * PPC + pi]);
                                const double hi = h2d(stage[size_t(D + c) * PPC + pi]);
                                a = __fma_rn(w, (w < 0.0) ? lo : hi, a);
                            }
                        }
                        sc = a;
                    }
                    if (smem_keys) {
                        if (pg < n_cand) {
                            // Push the key to every CTA of the cluster (padded slot).
                            const unsigned long long k = order_key(sc);
                            unsigned long long* dst = keys + size_t(g) * p.key_cap + key_slot(pg);
                            if (C == 1) *dst = k;
                            else
                                for (uint32_t r = 0; r < C; ++r) st_async_u64(map_rank(dst, r), k, map_rank(keys_bar, r));
                        }
                    }
                    if (!smem_keys || p.keep_scores)
                        p.ws_scores[(size_t(b) * Hq + size_t(kvh) * G + g) * p.Pmax + pg] = sc;
                }
            }
        }
        __syncthreads();  // stage reused by the next chunk
    }
    }  // G > 1
    if (owner && !appended) do_append();  // an empty estimate range

    // Keys of every CTA of the unit are visible after this barrier (and so is the new K/V
    // row written in phase A).
    stamp(p.probe, 8);
    if (C > 1) {
        if (!arrived) arrive_keys(!smem_keys || owner);
        mbar_wait_cluster(keys_bar, 0);
    } else {
        __syncthreads();  // this CTA's keys (or HBM scores) and its appended row
    }
    stamp(p.probe, 9);
    if (append && rank == 0 && tid == kThreads - 1) {  // off the selection warps' path
        // Every CTA of this unit has read the old length.  The last unit of the sequence
        // to get here publishes the new length for the next step.
        if (atomicAdd(p.len_ticket + p.layer * p.B + b, 1) == int(p.Hkv) - 1) {
            p.len_ticket[p.layer * p.B + b] = 0;
            p.len[p.layer * p.B + b] = int32_t(n_tok);
        }
    }

    // ---- phase C: selection (redundantly in every CTA of the cluster) ----------------
    if (!all_pages) {
        const uint32_t target = p.force ? p.k_budget - 1 : p.k_budget;
        if (target > 0) {
            // Groups of NTS threads select one head each (GQA heads in parallel); during an
            // MHA selection the other warps prefetch into L2 the K/V pages the first radix
            // pass proves selected (pages i % C == rank: the cluster requests each once),
            // so HBM streams attention bytes while the boundary is still being resolved.
            auto group_select = [&](auto nts_tag, auto kpt_tag) {
                constexpr int NTS = decltype(nts_tag)::value;
                constexpr int KP = decltype(kpt_tag)::value;
                constexpr int NGRP = kThreads / NTS;
                auto* gsc = reinterpret_cast<SelectScratch<NTS>*>(smem);  // region A
                const int grpi = tid / NTS, gt = tid % NTS;
                if (G == 1 && grpi > 0) {
                    asm volatile("bar.sync %0, %1;" ::"r"(7), "r"(kThreads) : "memory");
                    const bool ok = gsc[0].sig_valid != 0 && p.prefetch;

                    const int shift = gsc[0].sig_shift;
                    const unsigned int bin = gsc[0].sig_bin;
                    const uint32_t page_bytes = p.S * D * 2;
                    const __half* kslice0 = p.k_pool + s * p.slice_kv;
                    const __half* vslice0 = p.v_pool + s * p.slice_kv;
                    // Each CTA prefetches the proven pages of its own estimate range (and the last
                    // CTA the newest page), skipping the pages its warps already prefetched
                    // speculatively: fewer bulk prefetches serialised in the copy engine ahead
                    // of the post-selection barrier.
                    const uint32_t lo = min(r_begin, n_cand), hi = min(r_end, n_cand);
                    const bool last = rank == C - 1;
                    for (uint32_t i = lo + uint32_t(tid - NTS); i < hi + (last ? 1u : 0u);
                         i += uint32_t(kThreads - NTS)) {
                        bool take;
                        uint32_t pg = i;
                        if (i >= hi) {
                            take = p.force != 0 && p.prefetch;  // the newest page
                            pg = P - 1;
                        } else {
                            const unsigned long long k = keys[key_slot(i)];
                            take = ok && unsigned(((k << shift) >> 32) >> 21) > bin;
                            const uint32_t blk = (i - r_begin) >> 5;
                            if (take && blk < uint32_t(kWarps) && s_spec_pg[blk] == i) take = false;
                        }
                        if (!take) continue;
                        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(kslice0 + size_t(pg) * p.S * D),
                                     "r"(page_bytes) : "memory");
                        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(vslice0 + size_t(pg) * p.S * D),
                                     "r"(page_bytes) : "memory");
                    }
                }
                for (int g = grpi; g < G; g += NGRP) {
                    const unsigned long long* kg = keys + size_t(g) * p.key_cap;
                    unsigned long long k16[KP];
                    const ulonglong2* src = reinterpret_cast<const ulonglong2*>(kg + key_slot(uint32_t(gt) * KP));
                    const bool has = uint32_t(gt) * KP < n_cand;  // rows past the keys stay out
#pragma unroll
                    for (int j = 0; j < KP / 2; ++j) {
                        const ulonglong2 v = has ? src[j] : make_ulonglong2(0ull, 0ull);
                        k16[2 * j] = v.x;
                        k16[2 * j + 1] = v.y;
                    }
                    if (g == 0) stamp(p.probe, 10);
                    block_select_reg<NTS, KP>(k16, n_cand, target, kg[0], sel + g * kMaxFusedK,
                                                   gsc[grpi], gt, 1 + grpi,
                                                   g == 0 ? p.probe : nullptr, G == 1 ? 7 : -1,
                                                   kThreads);
                    group_sync<NTS>(1 + grpi);  // scratch reuse for the next head

                }
            };
            if (G == 1 && smem_keys && n_cand <= uint32_t(kSelThreads * kSelKpt)) {
                // MHA up to 2048 candidates: 256 threads x 8 keys (half the serial per-thread
                // work of 128 x 16; 8 warps still prefetch): 19.19 -> 19.08 and 19.31 -> 19.21
                // us/layer in two same-box A/Bs (tools/ab_bench.sh); 512 x 4 without the
                // prefetch warps 19.24, with per-thread prefetch of its own proven keys 19.36.
                group_select(std::integral_constant<int, 2 * kSelThreads>{},
                             std::integral_constant<int, kSelKpt / 2>{});
            } else if (smem_keys && n_cand <= uint32_t(kSelThreads * kSelKpt)) {
                group_select(std::integral_constant<int, kSelThreads>{}, std::integral_constant<int, kSelKpt>{});
            } else if (smem_keys && n_cand <= uint32_t(2 * kSelThreads * kSelKpt)) {
                group_select(std::integral_constant<int, 2 * kSelThreads>{}, std::integral_constant<int, kSelKpt>{});
            } else if (smem_keys && n_cand <= uint32_t(kThreads * kSelKpt)) {
                for (int g = 0; g < G; ++g) {
                    const unsigned long long* kg = keys + size_t(g) * p.key_cap;
                    unsigned long long k16[kSelKpt];
                    const ulonglong2* src = reinterpret_cast<const ulonglong2*>(kg + key_slot(uint32_t(tid) * kSelKpt));
                    const bool has = uint32_t(tid) * kSelKpt < n_cand;
#pragma unroll
                    for (int j = 0; j < kSelKpt / 2; ++j) {
                        const ulonglong2 v = has ? src[j] : make_ulonglong2(0ull, 0ull);
                        k16[2 * j] = v.x;
                        k16[2 * j + 1] = v.y;
                    }
                    block_select_reg<kThreads, kSelKpt>(k16, n_cand, target, kg[0],
                                                        sel + g * kMaxFusedK, *big_sc, tid, 0,
                                                        g == 0 ? p.probe : nullptr);
                    __syncthreads();
                }
            } else {
                // Scores through HBM/L2 (large page counts, large GQA groups).
                for (int g = 0; g < G; ++g) {
                    unsigned long long kmax, kmin;
                    const double* src = p.ws_scores + (size_t(b) * Hq + size_t(kvh) * G + g) * p.Pmax;
                    const int kpt = load_keys<kThreads>(src, n_cand, pkeys, *big_sc, &kmax, &kmin);
                    block_select<kThreads>(pkeys, kpt, n_cand, target, kmax, kmin,
                                           sel + g * kMaxFusedK, *big_sc,
                                           g == 0 ? p.probe : nullptr);
                }
            }
        }
        if (tid < G && p.force) sel[tid * kMaxFusedK + target] = int32_t(P - 1);
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

    stamp(p.probe, 16);
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
        __syncwarp();  // reconverge the half-warp stores before the aligned barrier
        __syncthreads();
        if (g == 0) stamp(p.probe, 17);
        if (tid < D) {  // the CTA's partial of this head: channel tid
            __syncwarp();  // converged shuffles below (no divergent fallback path)
            // Lane w < kWarps of every warp computes warp w's weight once; the channel
            // sums then take the 16 weights by shuffle.
            const float mw = lane < kWarps ? s_m[lane] : -CUDART_INF_F;
            float M = mw;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
            const float myw = (mw == -CUDART_INF_F) ? 0.0f : exp2f(mw - M);
            const float myl = lane < kWarps ? s_l[lane] * myw : 0.0f;
            float L = 0.0f, acc = 0.0f;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) {
                L += __shfl_sync(0xffffffffu, myl, w);
                acc += s_o[w][tid] * __shfl_sync(0xffffffffu, myw, w);
            }
            // Partials layout [g][D+2][C] (element-major): rank 0 reads each element of the
            // C ranks as one vector.
            float* hbase = parts + size_t(g) * (D + 2) * C;
            if (C == 1 || rank == 0) {
                hbase[(2 + tid) * C + rank] = acc;
                if (tid == 0) {
                    hbase[rank] = M;
                    hbase[C + rank] = L;
                }
            } else {
                const uint32_t rb = map_rank(merge_bar, 0);
                st_async_f32(map_rank(hbase + (2 + tid) * C + rank, 0), acc, rb);
                if (tid == 0) {
                    st_async_f32(map_rank(hbase + rank, 0), M, rb);
                    st_async_f32(map_rank(hbase + C + rank, 0), L, rb);
                }
            }
        }
        __syncthreads();  // s_o / s_m reused by the next head; partials issued
    }
    stamp(p.probe, 18);
    if (C > 1 && rank != 0) return;  // the partials complete on rank 0's merge_bar
    if (C > 1) {
        if (tid == 0) mbar_wait_cluster(merge_bar, 0);  // every peer's partial has landed
        __syncthreads();
    }
    stamp(p.probe, 19);
    if (p.probe) {
        if (tid == 0) p.probe[blockIdx.x * kProbeSlots + 25] = clock64();
        __syncwarp();
    }

    // Rank 0: merge the C partials of every head in rank order: weights
    // w_r = exp2(m_r - M) / L (every thread computes its head's C weights itself), then
    // every channel is a C-term dot product.
    for (int i = tid; i < G * int(p.head_dim); i += kThreads) {
        const int g = i / int(p.head_dim), d = i % int(p.head_dim);
        const size_t bh = size_t(b) * Hq + size_t(kvh) * G + g;
        const float* hb = parts + size_t(g) * (D + 2) * C;  // [D+2][C]
        float Lg = 0.0f, acc = 0.0f;
        if (C == 4) {  // the common cluster: one vector per element
            const float4 m4 = reinterpret_cast<const float4*>(hb)[0];
            const float4 l4 = reinterpret_cast<const float4*>(hb)[1];
            const float4 o4 = reinterpret_cast<const float4*>(hb)[2 + d];
            const float mr[4] = {m4.x, m4.y, m4.z, m4.w}, lr[4] = {l4.x, l4.y, l4.z, l4.w},
                        orr[4] = {o4.x, o4.y, o4.z, o4.w};
            const float Mg = fmaxf(fmaxf(mr[0], mr[1]), fmaxf(mr[2], mr[3]));
#pragma unroll
            for (int r = 0; r < 4; ++r) {  // rank order, as the generic path
                const float w = (mr[r] == -CUDART_INF_F) ? 0.0f : exp2f(mr[r] - Mg);
                Lg = fmaf(lr[r], w, Lg);
                acc = fmaf(orr[r], w, acc);
            }
        } else {
            float Mg = -CUDART_INF_F;
            for (uint32_t r = 0; r < C; ++r) Mg = fmaxf(Mg, hb[r]);
            for (uint32_t r = 0; r < C; ++r) {
                const float mr = hb[r];
                const float w = (mr == -CUDART_INF_F) ? 0.0f : exp2f(mr - Mg);
                Lg = fmaf(hb[C + r], w, Lg);
                acc = fmaf(hb[(2 + d) * C + r], w, acc);
            }
        }
        acc = acc / Lg;
        if (p.out_dtype == QK_DTYPE_F32) static_cast<float*>(p.out)[bh * p.head_dim + d] = acc;
        else static_cast<__half*>(p.out)[bh * p.head_dim + d] = __float2half_rn(acc);
    }
    if (p.done_flag) {
        __syncthreads();  // this unit's outputs are written
        if (tid == 0) signal_done(p, gridDim.x / C);
    }
    stamp(p.probe, 20);
}

template <int D, int G>
int run_fused(qk_cache* c, FusedParams prm, uint32_t batch, uint32_t cluster,
              uint32_t max_pages, cudaStream_t st) {
    using LY = Layout<D, G>;
    // Selection keys of every head exchanged through the cluster's shared memory when they
    // fit.  The key array is sized for the cache's capacity (within the budget), not for
    // this launch's pages: a CUDA graph captured now replays on longer contexts, and a
    // launch whose candidates outgrow the array takes the HBM path inside the kernel.
    const uint32_t budget_slots = uint32_t(keys_budget(G) / (size_t(G) * 8)) & ~1u;
    const uint32_t full_slots = (key_slots(c->Pmax) + 1) & ~1u;  // even: 16-byte aligned rows
    const uint32_t cap = full_slots < budget_slots ? full_slots : budget_slots;
    prm.key_cap = key_slots(max_pages) <= cap ? cap : 0u;
    const size_t region_a = LY::region_a(c->Pmax);
    size_t smem = LY::bytes(c->Pmax, prm.key_cap, cluster);
    while (smem > kMaxSmem && cluster > 1) {  // large GQA groups: fewer partial slots
        cluster /= 2;
        smem = LY::bytes(c->Pmax, prm.key_cap, cluster);
    }
    if (smem > kMaxSmem && prm.key_cap) {
        prm.key_cap = 0;
        smem = LY::bytes(c->Pmax, 0, cluster);
    }
    if (smem > kMaxSmem) return set_error(QK_ERR_UNSUPPORTED, "qk_decode_step: shared memory");
    auto kern = decode_fused_kernel<D, G>;
    if (int rc = ensure_func_attrs(reinterpret_cast<const void*>(kern), smem, c->desc.device, true,
                                   "decode_fused_kernel attributes"))
        return rc;
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
    static const int pdl = getenv("QK_NO_PDL") ? 0 : 1;  // read once (per-launch cost)
    attrs[1].val.programmaticStreamSerializationAllowed = pdl;
    cfg.attrs = attrs;
    cfg.numAttrs = 2;
    c->launches++;
    if (c->host_graph_mode && prm.probe == nullptr && prm.layer < c->host_graphs.size()) {
        // Host step: replay this layer's captured launch while it is unchanged.
        auto& hg = c->host_graphs[prm.layer];
        std::vector<unsigned char> key(sizeof(prm) + 4 * sizeof(uint32_t));
        const uint32_t shape[4] = {cfg.gridDim.x, cluster, uint32_t(smem), uint32_t(region_a)};
        std::memcpy(key.data(), &prm, sizeof(prm));
        std::memcpy(key.data() + sizeof(prm), shape, sizeof(shape));
        if (hg.exec == nullptr || hg.key != key) {
            if (hg.exec) cudaGraphExecDestroy(hg.exec);
            hg.exec = nullptr;
            if (!c->capture_stream)
                if (int rc = cuda_check(cudaStreamCreateWithFlags(&c->capture_stream, cudaStreamNonBlocking),
                                        "capture stream"))
                    return rc;
            cudaGraph_t g = nullptr;
            cfg.stream = c->capture_stream;
            if (int rc = cuda_check(cudaStreamBeginCapture(c->capture_stream, cudaStreamCaptureModeThreadLocal),
                                    "host-step capture"))
                return rc;
            const cudaError_t le = cudaLaunchKernelEx(&cfg, kern, prm, uint32_t(region_a));
            const cudaError_t ee = cudaStreamEndCapture(c->capture_stream, &g);
            if (int rc = cuda_check(le != cudaSuccess ? le : ee, "host-step capture")) return rc;
            const cudaError_t ie = cudaGraphInstantiate(&hg.exec, g, 0);
            cudaGraphDestroy(g);
            if (int rc = cuda_check(ie, "host-step graph instantiate")) return rc;
            hg.key = std::move(key);
        }
        return cuda_check(cudaGraphLaunch(hg.exec, st), "decode_fused_kernel (graph)");
    }
    return cuda_check(cudaLaunchKernelEx(&cfg, kern, prm, uint32_t(region_a)), "decode_fused_kernel");
}

template <int D>
int dispatch_g(qk_cache* c, const FusedParams& prm, uint32_t batch, uint32_t cluster,
               uint32_t max_pages, cudaStream_t st) {
    switch (c->G) {
        case 1: return run_fused<D, 1>(c, prm, batch, cluster, max_pages, st);
        case 2: return run_fused<D, 2>(c, prm, batch, cluster, max_pages, st);
        case 4: return run_fused<D, 4>(c, prm, batch, cluster, max_pages, st);
        case 8: return run_fused<D, 8>(c, prm, batch, cluster, max_pages, st);
        default: return set_error(QK_ERR_UNSUPPORTED, "qk_decode_step: GQA group");
    }
}

// Unfused sequence of the same step (used when the fused kernel's limits -- kMaxFusedK
// selected pages per head, head_dim 64/128 -- are exceeded).
int decode_unfused(qk_cache* c, uint32_t layer, const __half* q, const __half* k,
                   const __half* v, uint32_t batch, const qk_selection_cfg& cfg,
                   uint32_t max_pages, void* out, int out_dtype, int32_t* pages,
                   uint32_t pstride, int32_t* counts, cudaStream_t st) {
    int rc = QK_OK;
    if (k) rc = launch_append(c, layer, k, v, batch, st);
    if (rc) return rc;
    // Grids and shared memory sized for the capacity, not this launch's pages: a CUDA graph
    // captured now must stay correct when its replays grow the context.
    rc = launch_estimate(c, layer, q, batch, c->ws_scores, c->Pmax, c->Pmax, st);
    if (rc) return rc;
    qk_selection_cfg eff = cfg;
    if (!cfg.per_layer_enabled) eff.token_budget = UINT32_MAX;
    int32_t* sel = pages ? pages : c->ws_pages;
    const uint32_t sstride = pages ? pstride : c->Pmax;
    int32_t* cnt = counts ? counts : c->ws_counts;
    rc = launch_topk(c, layer, c->ws_scores, c->Pmax, batch, eff, sel, sstride, cnt, c->Pmax, st);
    if (rc) return rc;
    const uint32_t kk = eff.token_budget / c->S;
    const uint32_t max_list = kk < c->Pmax ? kk : c->Pmax;
    return launch_attend(c, layer, q, batch, sel, sstride, cnt, kModePages, max_list, out, out_dtype,
                         nullptr, nullptr, st);
}

}  // namespace

// Cluster size: the largest power of two (<= 16) that keeps one wave of one CTA per SM
// (units * C <= 148) and leaves every CTA at least 64 pages to estimate.
uint32_t fused_cluster_size(const qk_cache* c, uint32_t batch, uint32_t pages) {
    const uint32_t units = batch * c->Hkv;
    uint32_t cl = 1;
    while (cl * 2 <= kMaxCluster && units * cl * 2 <= 148 && pages >= cl * 2 * 64) cl *= 2;
    return cl;
}

int launch_decode(qk_cache* c, uint32_t layer, const __half* q, const __half* k,
                  const __half* v, uint32_t batch, const qk_selection_cfg& cfg,
                  uint32_t max_pages, void* out, int out_dtype, int32_t* pages,
                  uint32_t pstride, int32_t* counts, cudaStream_t st) {
    const uint32_t kk = cfg.per_layer_enabled ? cfg.token_budget / c->S : UINT32_MAX;
    const bool fits = (kk >= c->Pmax || kk <= kMaxFusedK) && (c->D == 64 || c->D == 128);
    static const int force_path = [] {  // QK_DECODE_PATH=fused|unfused (experiments; read once)
        const char* e = getenv("QK_DECODE_PATH");
        return (e == nullptr || e[0] == 0) ? 0 : (e[0] == 'u' ? 2 : 1);
    }();
    // GQA with more (sequence, KV head) units than SMs: the fused kernel's one-CTA-per-unit
    // waves serialise the G heads' estimate chains and attention inside each CTA; the
    // separate kernels spread estimate, top-K and attention over the whole GPU (measured at
    // cfg4, 32 x 8 units: 557 -> 415 us/layer).
    const bool wide_gqa = c->G > 1 && batch * c->Hkv > 148u;
    if (!fits || force_path == 2 || (wide_gqa && force_path != 1))
        return decode_unfused(c, layer, q, k, v, batch, cfg, max_pages, out, out_dtype, pages,
                              pstride, counts, st);
    FusedParams prm;
    std::memset(&prm, 0, sizeof(prm));  // padding too: the host step keys its graphs on the bytes
    prm.k_pool = c->k_pool;
    prm.v_pool = c->v_pool;
    prm.meta = c->meta;
    prm.prange = c->prange;
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
    prm.mrow = c->Mrow;
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
    prm.keep_scores = c->keep_scores ? 1 : 0;
    static const int prefetch = getenv("QK_NO_PREFETCH") ? 0 : 1;  // read once
    prm.prefetch = prefetch;
    prm.scale_log2 = float(1.4426950408889634 / sqrt(double(c->desc.head_dim)));
    prm.probe = c->probe ? c->probe + size_t(layer) * c->B * c->Hkv * kMaxClusterCtas * kProbeSlots : nullptr;
    if (c->pending_done_flag) {  // the host step asked for a completion word (consumed here)
        prm.done_flag = c->pending_done_flag;
        prm.done_counter = c->done_counter;
        c->pending_done_flag = nullptr;
    }
    const uint32_t cluster = fused_cluster_size(c, batch, max_pages);
    switch (c->D) {
        case 64: return dispatch_g<64>(c, prm, batch, cluster, max_pages, st);
        case 128: return dispatch_g<128>(c, prm, batch, cluster, max_pages, st);
        default: return set_error(QK_ERR_UNSUPPORTED, "qk_decode_step: head_dim");
    }
}

}  // namespace qk

// select.cuh -- block-wide exact top-K page selection, shared by the standalone top-K
// kernel (topk.cu) and the fused decode kernel (decode.cu).
//
// Semantics: select_top_k, /root/reference/proj/core/src/criticality.cpp:36-81, for the
// `target` best of `n` candidate pages under the order (score desc, page asc).  The
// caller handles the early exits and force_include_recent (see topk.cu).
//
// Method (exact, no sort):
//   * scores -> order-preserving u64 keys; thread t owns pages [t*KPT, (t+1)*KPT), kept
//     in shared memory with one u64 of padding per thread (conflict-free row reads);
//   * the bits shared by every key (block min/max) are skipped, then 11-bit digits are
//     histogrammed (2048 bins) until the bin holding the target-th key either
//       - holds exactly the keys still needed  -> take the whole bin, or
//       - holds <= 32 keys -> one warp ranks them by (key desc, page asc) and yields the
//         exact threshold pair (T_key, T_page), or
//       - is a single 64-bit value shared by > 32 pages -> take the lowest pages;
//     random scores resolve in one pass, heavy ties in at most six;
//   * the selected pages are written in ascending order with one block-wide scan.
#pragma once

#include "qk_internal.cuh"

namespace qk {

// Optional phase stamps (QK_PROBE): slots 11..15 of the per-CTA record (decode.cu).
// QK_SEL_CYCLES (microbenchmarks only) records clock64 instead and enables fine stamps.
__device__ __forceinline__ void sel_stamp(unsigned long long* probe, int slot) {
    if (probe != nullptr) {  // (callers are warp-uniform)
        if (threadIdx.x == 0) {
            unsigned long long t;
#ifdef QK_SEL_CYCLES
            t = clock64();
#else
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
#endif
            probe[blockIdx.x * kProbeSlots + slot] = t;
        }
        __syncwarp();  // reconverge: a diverged warp would take the collectives' slow path
    }
}
#ifdef QK_SEL_CYCLES
#define QK_SEL_FINE(probe, slot) sel_stamp(probe, slot)
#else
#define QK_SEL_FINE(probe, slot) ((void)0)
#endif

template <int NT>
struct SelectScratch {
    alignas(16) unsigned int hist[2048 + 4];  // + a trash bin for branch-free increments
    alignas(16) unsigned int warp_sum[NT / 32 < 4 ? 4 : NT / 32];
    alignas(16) unsigned long long red_max[NT / 32 < 4 ? 4 : NT / 32];
    unsigned long long red_min[NT / 32 < 4 ? 4 : NT / 32];
    unsigned long long cand_key[32];
    unsigned int cand_idx[32];
    alignas(16) unsigned long long cand2[66];  // (key, index) pairs of the threshold bin + trash
    unsigned int cand_take[33];
    unsigned int selbits[NT / 2];  // block_select_reg: boundary-bin verdicts, 1 bit per key (KPT <= 16)
    int trash_out;
    // Early-signal of block_select_reg: after the first radix pass every key whose top
    // 11 bits (after the common prefix `sig_shift`) exceed `sig_bin` is selected.
    int sig_shift;
    unsigned int sig_bin;
    int sig_valid;
    unsigned int n_cand;
    unsigned int digit, above, count;
    unsigned long long t_key;
    unsigned int t_idx;
};

// Block-wide exclusive scan of one unsigned value per thread; returns (exclusive, total).
template <int NT>
__device__ __forceinline__ unsigned int block_excl_scan(unsigned int v, unsigned int* warp_sum,
                                                        unsigned int* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned int x = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += x;
    }
    if (lane == 31) warp_sum[warp] = incl;
    __syncthreads();
    unsigned int before = 0, all = 0;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) {
        const unsigned int s = warp_sum[w];
        before += (w < warp) ? s : 0u;
        all += s;
    }
    __syncthreads();  // warp_sum reusable
    *total = all;
    return before + incl - v;
}

__device__ __forceinline__ unsigned long long keyat(const unsigned long long* keys, int kpt,
                                                    uint32_t i) {
    return keys[(i / kpt) * (kpt + 1) + (i % kpt)];
}

// Loads score(0..n) -- `score(i)` returns candidate i's double (global data written
// earlier in the same kernel or by a prior one) -- as keys into `keys` (padded layout,
// capacity NT*(kpt+1)).  Returns kpt.
template <int NT, typename ScoreFn>
__device__ __forceinline__ int load_keys_fn(ScoreFn score, uint32_t n, unsigned long long* keys,
                                            SelectScratch<NT>& sc, unsigned long long* kmax_out,
                                            unsigned long long* kmin_out) {
    const int kpt = int((n + NT - 1) / NT);
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    unsigned long long kmax = 0, kmin = ~0ull;
    // Batches of 8 independent loads in flight before the first use (in-order issue
    // would otherwise pay one L2 round trip per score).
    for (int j0 = 0; j0 < kpt; j0 += 8) {
        double v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint32_t i = uint32_t(t) * kpt + j0 + j;
            v[j] = (j0 + j < kpt && i < n) ? score(i) : 0.0;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint32_t i = uint32_t(t) * kpt + j0 + j;
            if (j0 + j < kpt && i < n) {
                // -0 and +0 compare equal in the reference's sort (criticality.cpp:64-67: ties
                // go to the lower page): canonicalise before keying (user-supplied scores;
                // estimate sums start at +0 and are never -0).
                const unsigned long long u = order_key(__dadd_rn(v[j], 0.0));
                keys[t * (kpt + 1) + j0 + j] = u;
                kmax = u > kmax ? u : kmax;
                kmin = u < kmin ? u : kmin;
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long a = __shfl_xor_sync(0xffffffffu, kmax, o);
        const unsigned long long b = __shfl_xor_sync(0xffffffffu, kmin, o);
        kmax = a > kmax ? a : kmax;
        kmin = b < kmin ? b : kmin;
    }
    if (lane == 0) {
        sc.red_max[warp] = kmax;
        sc.red_min[warp] = kmin;
    }
    __syncthreads();
    kmax = sc.red_max[0];
    kmin = sc.red_min[0];
#pragma unroll
    for (int w = 1; w < NT / 32; ++w) {
        kmax = sc.red_max[w] > kmax ? sc.red_max[w] : kmax;
        kmin = sc.red_min[w] < kmin ? sc.red_min[w] : kmin;
    }
    *kmax_out = kmax;
    *kmin_out = kmin;
    return kpt;
}

// load_keys_fn over one score row: scores[0..n).
template <int NT>
__device__ __forceinline__ int load_keys(const double* __restrict__ scores, uint32_t n,
                                         unsigned long long* keys, SelectScratch<NT>& sc,
                                         unsigned long long* kmax_out,
                                         unsigned long long* kmin_out) {
    return load_keys_fn<NT>([scores](uint32_t i) { return __ldcg(scores + i); }, n, keys, sc,
                            kmax_out, kmin_out);
}

// Selects the `target` (1 <= target < n) best keys and writes their page indices,
// ascending, to out[0..target) (out may be global or shared).  All NT threads call.
template <int NT, typename OutT>
__device__ void block_select(const unsigned long long* keys, int kpt, uint32_t n,
                             uint32_t target, unsigned long long kmax, unsigned long long kmin,
                             OutT* out, SelectScratch<NT>& sc,
                             unsigned long long* probe = nullptr) {
    enum { TAKE_BIN = 0, PAIR = 1, EQUAL = 2 };
    const int t = threadIdx.x;
    const unsigned long long diff = kmax ^ kmin;
    int hb = diff ? 63 - __clzll(static_cast<long long>(diff)) : -1;
    unsigned long long mask = (hb >= 63) ? 0ull : (~0ull << (hb + 1));
    unsigned long long prefix = kmax & mask;
    uint32_t krem = target;
    uint32_t bin_count = n;
    int mode = EQUAL;
    bool resolved = false;
    if (hb < 0) {
        mode = (n <= 32) ? PAIR : EQUAL;  // every key equal
    }
    int pass = 0;
    while (hb >= 0) {
        const int lo = hb >= 10 ? hb - 10 : 0;
        const unsigned int dmask = (1u << (hb - lo + 1)) - 1u;
        for (int i = t; i < 2048; i += NT) sc.hist[i] = 0;
        __syncthreads();
        for (int j = 0; j < kpt; ++j) {
            const uint32_t i = uint32_t(t) * kpt + j;
            if (i < n) {
                const unsigned long long u = keys[t * (kpt + 1) + j];
                if ((u & mask) == prefix) atomicAdd(&sc.hist[(u >> lo) & dmask], 1u);
            }
        }
        __syncthreads();
        // Thread t sums bins [2047-8t-7, 2047-8t] (top bins first).
        unsigned int c[2048 / NT], s = 0;
#pragma unroll
        for (int j = 0; j < 2048 / NT; ++j) {
            c[j] = sc.hist[2047 - (2048 / NT) * t - j];
            s += c[j];
        }
        unsigned int total;
        const unsigned int excl = block_excl_scan<NT>(s, sc.warp_sum, &total);
        if (excl < krem && krem <= excl + s) {
            unsigned int above = excl;
#pragma unroll
            for (int j = 0; j < 2048 / NT; ++j) {
                if (above < krem && krem <= above + c[j]) {
                    sc.digit = 2047 - (2048 / NT) * t - j;
                    sc.above = above;
                    sc.count = c[j];
                }
                above += c[j];
            }
        }
        __syncthreads();
        krem -= sc.above;
        bin_count = sc.count;
        prefix |= static_cast<unsigned long long>(sc.digit) << lo;
        mask |= static_cast<unsigned long long>(dmask) << lo;
        __syncthreads();
        sel_stamp(probe, 11 + (pass < 2 ? pass : 2));
        ++pass;
        if (bin_count == krem) {
            mode = TAKE_BIN;
            resolved = true;
            break;
        }
        if (bin_count <= 32) {
            mode = PAIR;
            break;
        }
        hb = lo - 1;
        if (hb < 0) mode = EQUAL;  // > 32 pages share one 64-bit key
    }

    if (!resolved && mode == PAIR) {
        // Gather the <= 32 keys of the threshold bin and rank them in one warp.
        if (t == 0) sc.n_cand = 0;
        __syncthreads();
        for (int j = 0; j < kpt; ++j) {
            const uint32_t i = uint32_t(t) * kpt + j;
            if (i < n) {
                const unsigned long long u = keys[t * (kpt + 1) + j];
                if ((u & mask) == prefix) {
                    const unsigned int slot = atomicAdd(&sc.n_cand, 1u);
                    sc.cand_key[slot] = u;
                    sc.cand_idx[slot] = i;
                }
            }
        }
        __syncthreads();
        if (t < 32) {
            const unsigned int nc = sc.n_cand;
            if (uint32_t(t) < nc) {
                const unsigned long long mk = sc.cand_key[t];
                const unsigned int mi = sc.cand_idx[t];
                unsigned int rank = 0;
                for (unsigned int j = 0; j < nc; ++j) {
                    const unsigned long long ok = sc.cand_key[j];
                    rank += (ok > mk) || (ok == mk && sc.cand_idx[j] < mi);
                }
                if (rank == krem - 1) {
                    sc.t_key = mk;
                    sc.t_idx = mi;
                }
            }
        }
        __syncthreads();
    }
    sel_stamp(probe, 14);
    const unsigned long long t_key = sc.t_key;
    const unsigned int t_idx = sc.t_idx;

    // EQUAL mode needs, per key of the bin, the number of equal keys at lower pages.
    unsigned int eq_before = 0;
    if (!resolved && mode == EQUAL) {
        unsigned int e = 0;
        for (int j = 0; j < kpt; ++j) {
            const uint32_t i = uint32_t(t) * kpt + j;
            if (i < n) e += (keys[t * (kpt + 1) + j] & mask) == prefix;
        }
        unsigned int tot;
        eq_before = block_excl_scan<NT>(e, sc.warp_sum, &tot);
    }

    // Ascending compaction.
    unsigned int mine = 0;
    {
        unsigned int eq = eq_before;
        for (int j = 0; j < kpt; ++j) {
            const uint32_t i = uint32_t(t) * kpt + j;
            if (i >= n) break;
            const unsigned long long u = keys[t * (kpt + 1) + j];
            const unsigned long long um = u & mask;
            bool sel = um > prefix;
            if (um == prefix) {
                if (mode == TAKE_BIN) sel = true;
                else if (mode == PAIR) sel = (u > t_key) || (u == t_key && i <= t_idx);
                else sel = eq < krem;
                eq++;
            }
            mine += sel;
        }
    }
    unsigned int tot;
    unsigned int pos = block_excl_scan<NT>(mine, sc.warp_sum, &tot);
    {
        unsigned int eq = eq_before;
        for (int j = 0; j < kpt; ++j) {
            const uint32_t i = uint32_t(t) * kpt + j;
            if (i >= n) break;
            const unsigned long long u = keys[t * (kpt + 1) + j];
            const unsigned long long um = u & mask;
            bool sel = um > prefix;
            if (um == prefix) {
                if (mode == TAKE_BIN) sel = true;
                else if (mode == PAIR) sel = (u > t_key) || (u == t_key && i <= t_idx);
                else sel = eq < krem;
                eq++;
            }
            if (sel) out[pos++] = static_cast<OutT>(i);
        }
    }
    __syncthreads();
    sel_stamp(probe, 15);
}

// Inclusive warp scan of v; lane 31's value is the warp total.
__device__ __forceinline__ unsigned int warp_incl_scan(unsigned int v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned int x = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += x;
    }
    return v;
}

// Sum of v[w] over w < upto for the NW (multiple of 4) per-warp values in smem, read as
// 16-byte broadcast vectors.
template <int NW>
__device__ __forceinline__ unsigned int sum_below(const unsigned int* v, int upto) {
    unsigned int s = 0;
#pragma unroll
    for (int w4 = 0; w4 < NW / 4; ++w4) {
        const uint4 q = reinterpret_cast<const uint4*>(v)[w4];
        s += (4 * w4 + 0 < upto ? q.x : 0u) + (4 * w4 + 1 < upto ? q.y : 0u) +
             (4 * w4 + 2 < upto ? q.z : 0u) + (4 * w4 + 3 < upto ? q.w : 0u);
    }
    return s;
}

// Barrier over the NT threads of one selection group (named barrier `id`; id 0 with NT ==
// blockDim.x is __syncthreads).
template <int NT>
__device__ __forceinline__ void group_sync(int id) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(NT) : "memory");
}

// Padded position of key i in a key array read 16 keys per thread: 2 spare u64 after every
// 16 keys, so the 16-byte reads of 32 lanes spread over all banks.
__host__ __device__ __forceinline__ uint32_t key_slot(uint32_t i) { return i + 2u * (i >> 4); }
__host__ __device__ __forceinline__ uint32_t key_slots(uint32_t n) { return key_slot(n + 15u); }

// Exact top-`target` selection by a group of NT threads (NT/32 warps, gt = thread index in
// the group, barrier `bar`) over n <= NT*KPT keys held in registers: thread gt owns the keys
// of indices [gt*KPT, gt*KPT+KPT) (entries >= n are ignored); `ref` is any one of the n
// keys.  Same result as block_select -- the `target` best by (key desc, index asc), written
// ascending to out[0..target) -- built for latency: a phase costs one barrier plus the
// phase's instructions on every warp of the group, so the group is small (128 threads, one
// warp per scheduler; several groups can select different heads at once) and every step is
// shuffle-light:
//   * common key prefix: OR of key ^ ref (redux.sync per warp);
//   * 11-bit digit histogram (shared atomics); lane l of warp w sums bins of rank
//     [BPL*(32w + l), +BPL) from the top; the lane holding the krem-th key finds the bin;
//   * a threshold bin of <= 32 keys is gathered and each of its keys ranks itself;
//   * ascending compaction from per-thread counts (warp scan + per-warp totals).
// 1 <= target < n.  out is complete after the group's next barrier.
template <int NT, int KPT, typename OutT>
__device__ void block_select_reg_wide(const unsigned long long (&key)[KPT], uint32_t n,
                                      uint32_t target, unsigned long long ref, OutT* out,
                                      SelectScratch<NT>& sc, int gt, int bar,
                                      unsigned long long* probe = nullptr,
                                      long long* trace = nullptr) {
#define QK_TRACE(k) \
    if (trace != nullptr && gt == 0) trace[k] = clock64();
    constexpr int NW = NT / 32;
    constexpr int BPL = 2048 / NT;  // histogram bins per lane in the bin search
    static_assert(NW % 4 == 0 && NW <= 32 && BPL % 4 == 0, "geometry");
    enum { TAKE_BIN = 0, PAIR = 1, EQUAL = 2 };
    const int lane = gt & 31, warp = gt >> 5;
    const uint32_t i0 = uint32_t(gt) * KPT;
    uint4* hist4 = reinterpret_cast<uint4*>(sc.hist);

    // Zero the histogram; per-warp OR of key ^ ref = the bits where keys differ.
#pragma unroll
    for (int j = 0; j < BPL / 4; ++j) hist4[gt * (BPL / 4) + j] = make_uint4(0, 0, 0, 0);
    if (gt == 0) sc.n_cand = 0;
    unsigned long long dx = 0;
#pragma unroll
    for (int j = 0; j < KPT; ++j)
        if (i0 + j < n) dx |= key[j] ^ ref;
    {
        const unsigned int dhi = __reduce_or_sync(0xffffffffu, unsigned(dx >> 32));
        const unsigned int dlo = __reduce_or_sync(0xffffffffu, unsigned(dx));
        if (lane == 0) sc.red_max[warp] = (static_cast<unsigned long long>(dhi) << 32) | dlo;
    }
    group_sync<NT>(bar);
    unsigned long long diff = 0;
#pragma unroll
    for (int w2 = 0; w2 < NW / 2; ++w2) {
        const ulonglong2 q = reinterpret_cast<const ulonglong2*>(sc.red_max)[w2];
        diff |= q.x | q.y;
    }
    int hb = diff ? 63 - __clzll(static_cast<long long>(diff)) : -1;
    QK_TRACE(0);
    unsigned long long mask = (hb >= 63) ? 0ull : (~0ull << (hb + 1));
    unsigned long long prefix = ref & mask;
    uint32_t krem = target;
    int mode = (hb < 0 && n <= 32) ? PAIR : EQUAL;
    bool resolved = false;
    int pass = 0;
    while (hb >= 0) {
        const int lo = hb >= 10 ? hb - 10 : 0;
        const unsigned int dmask = (1u << (hb - lo + 1)) - 1u;
#pragma unroll
        for (int j = 0; j < KPT; ++j)
            if (i0 + j < n && (key[j] & mask) == prefix)
                atomicAdd(&sc.hist[(key[j] >> lo) & dmask], 1u);
        group_sync<NT>(bar);
        // This lane's bins, highest first: 2047 - BPL*gt - [0, BPL).
        unsigned int c[BPL], sl = 0;
#pragma unroll
        for (int j4 = 0; j4 < BPL / 4; ++j4) {
            const uint4 q = hist4[(2047 - BPL * gt) / 4 - j4];
            c[4 * j4 + 0] = q.w;
            c[4 * j4 + 1] = q.z;
            c[4 * j4 + 2] = q.y;
            c[4 * j4 + 3] = q.x;
        }
#pragma unroll
        for (int j = 0; j < BPL; ++j) sl += c[j];
        QK_TRACE(1);
        const unsigned int incl = warp_incl_scan(sl);
        if (lane == 31) sc.warp_sum[warp] = incl;
        QK_TRACE(2);
        group_sync<NT>(bar);
        unsigned int above = sum_below<NW>(sc.warp_sum, warp) + incl - sl;
        QK_TRACE(3);
        if (above < krem && krem <= above + sl) {  // exactly one lane of the group
#pragma unroll
            for (int j = 0; j < BPL; ++j) {
                if (above < krem && krem <= above + c[j]) {
                    sc.count = c[j];
                    sc.digit = 2047 - (BPL * gt + j);
                    sc.above = above;
                }
                above += c[j];
            }
        }
        group_sync<NT>(bar);
        krem -= sc.above;
        const uint32_t bin_count = sc.count;
        prefix |= static_cast<unsigned long long>(sc.digit) << lo;
        mask |= static_cast<unsigned long long>(dmask) << lo;
        QK_TRACE(4);
        sel_stamp(probe, 11 + (pass < 2 ? pass : 2));
        ++pass;
        if (bin_count == krem) {
            mode = TAKE_BIN;
            resolved = true;
            break;
        }
        if (bin_count <= 32) {
            mode = PAIR;
            break;
        }
        hb = lo - 1;
        if (hb < 0) {
            mode = EQUAL;  // > 32 keys share one 64-bit value
            break;
        }
        // Next pass: re-zero the histogram once everyone has read it and sc.*.
        group_sync<NT>(bar);
#pragma unroll
        for (int j = 0; j < BPL / 4; ++j) hist4[gt * (BPL / 4) + j] = make_uint4(0, 0, 0, 0);
        group_sync<NT>(bar);
    }

    // Per key: selected?  Keys above the threshold bin always; keys of the bin by mode.
    bool take[KPT];
#pragma unroll
    for (int j = 0; j < KPT; ++j) take[j] = (i0 + j < n) && (key[j] & mask) > prefix;
    if (resolved) {
#pragma unroll
        for (int j = 0; j < KPT; ++j) take[j] = take[j] || ((i0 + j < n) && (key[j] & mask) == prefix);
    } else if (mode == PAIR) {
        // Gather the <= 32 keys of the bin (sc.n_cand was zeroed before the first barrier
        // and is untouched since); thread m ranks candidate m; owners read the verdicts.
        int slot[KPT];
#pragma unroll
        for (int j = 0; j < KPT; ++j) {
            slot[j] = -1;
            if (i0 + j < n && (key[j] & mask) == prefix) {
                slot[j] = int(atomicAdd(&sc.n_cand, 1u));
                reinterpret_cast<ulonglong2*>(sc.cand2)[slot[j]] = make_ulonglong2(key[j], i0 + j);
            }
        }
        group_sync<NT>(bar);
        const unsigned int nc = sc.n_cand;
        QK_TRACE(5);
        if (uint32_t(gt) < nc) {
            const ulonglong2 me = reinterpret_cast<const ulonglong2*>(sc.cand2)[gt];
            unsigned int rank = 0;
#pragma unroll
            for (int m = 0; m < 32; ++m) {
                if (uint32_t(m) < nc) {
                    const ulonglong2 o = reinterpret_cast<const ulonglong2*>(sc.cand2)[m];
                    rank += (o.x > me.x) || (o.x == me.x && o.y < me.y);
                }
            }
            sc.cand_take[gt] = rank < krem;
        }
        group_sync<NT>(bar);
#pragma unroll
        for (int j = 0; j < KPT; ++j)
            if (slot[j] >= 0) take[j] = sc.cand_take[slot[j]] != 0;
    } else {
        // EQUAL: the krem lowest indices of the bin.
        unsigned int e = 0;
#pragma unroll
        for (int j = 0; j < KPT; ++j) e += (i0 + j < n) && (key[j] & mask) == prefix;
        const unsigned int incl = warp_incl_scan(e);
        if (lane == 31) sc.warp_sum[warp] = incl;
        group_sync<NT>(bar);
        unsigned int eq = sum_below<NW>(sc.warp_sum, warp) + incl - e;
#pragma unroll
        for (int j = 0; j < KPT; ++j)
            if (i0 + j < n && (key[j] & mask) == prefix) take[j] = eq++ < krem;
        group_sync<NT>(bar);  // warp_sum is rewritten below
    }
    QK_TRACE(6);
    sel_stamp(probe, 14);

    // Ascending compaction.
    unsigned int mine = 0;
#pragma unroll
    for (int j = 0; j < KPT; ++j) mine += take[j];
    const unsigned int incl = warp_incl_scan(mine);
    if (lane == 31) sc.warp_sum[warp] = incl;
    QK_TRACE(7);
    group_sync<NT>(bar);
    unsigned int pos = sum_below<NW>(sc.warp_sum, warp) + incl - mine;
    QK_TRACE(8);
#pragma unroll
    for (int j = 0; j < KPT; ++j)
        if (take[j]) out[pos++] = static_cast<OutT>(i0 + j);
    sel_stamp(probe, 15);
#undef QK_TRACE
}

// block_select_reg: the same selection with a 32-bit fast path.  Keys are shifted left
// past their common prefix once; the first 11-bit radix pass, the bin search and the
// verdicts then work on the high 32-bit word (one instruction per comparison instead of a
// 64-bit mask-and-compare).  A pass that leaves more than 32 keys of the threshold bin
// undecided (heavy ties) restarts in block_select_reg_wide.  Same contract.
// `signal_bar` >= 0: after the first pass (or on the way to the wide path) thread 0 of the
// group publishes (sig_shift, sig_bin, sig_valid) and the group arrives once on named
// barrier `signal_bar` with `signal_count` threads, so other warps can start work on the
// certainly-selected keys (the fused kernel prefetches their K/V pages).
template <int NT, int KPT, typename OutT>
__device__ void block_select_reg(const unsigned long long (&key)[KPT], uint32_t n, uint32_t target,
                                 unsigned long long ref, OutT* out, SelectScratch<NT>& sc, int gt,
                                 int bar, unsigned long long* probe = nullptr,
                                 int signal_bar = -1, int signal_count = 0) {
    auto signal = [&](int valid, int shift, unsigned int bin) {
        if (signal_bar < 0) return;
        if (gt == 0) {
            sc.sig_shift = shift;
            sc.sig_bin = bin;
            sc.sig_valid = valid;
        }
        asm volatile("bar.arrive %0, %1;" ::"r"(signal_bar), "r"(signal_count) : "memory");
    };
    constexpr int NW = NT / 32;
    constexpr int BPL = 2048 / NT;
    static_assert(NW % 4 == 0 && NW <= 32 && BPL % 4 == 0, "geometry");
    const int lane = gt & 31, warp = gt >> 5;
    const uint32_t i0 = uint32_t(gt) * KPT;
    const int nv = n > i0 ? int(min(uint32_t(KPT), n - i0)) : 0;  // valid keys of this thread
    uint4* hist4 = reinterpret_cast<uint4*>(sc.hist);

    static_assert(KPT <= 16 && 32 % KPT == 0,
                  "selbits: a thread's keys lie in one 32-bit verdict word (KPT divides 32)");
#pragma unroll
    for (int j = 0; j < BPL / 4; ++j) hist4[gt * (BPL / 4) + j] = make_uint4(0, 0, 0, 0);
    if (gt == 0) sc.n_cand = 0;
    if (gt < NT / 2) sc.selbits[gt] = 0u;
    unsigned long long dx = 0;
#pragma unroll
    for (int j = 0; j < KPT; ++j)
        if (j < nv) dx |= key[j] ^ ref;
    {
        const unsigned int dhi = __reduce_or_sync(0xffffffffu, unsigned(dx >> 32));
        const unsigned int dlo = __reduce_or_sync(0xffffffffu, unsigned(dx));
        if (lane == 0) sc.red_max[warp] = (static_cast<unsigned long long>(dhi) << 32) | dlo;
    }
    group_sync<NT>(bar);
    QK_SEL_FINE(probe, 20);
    unsigned long long diff = 0;
#pragma unroll
    for (int w2 = 0; w2 < NW / 2; ++w2) {
        const ulonglong2 q = reinterpret_cast<const ulonglong2*>(sc.red_max)[w2];
        diff |= q.x | q.y;
    }
    if (diff == 0) {  // every key equal: the lowest indices
        group_sync<NT>(bar);  // red_max read by all before the wide path reuses sc
        signal(0, 0, 0);
        block_select_reg_wide<NT, KPT>(key, n, target, ref, out, sc, gt, bar, probe);
        return;
    }
    const int shift = __clzll(static_cast<long long>(diff));  // common prefix length
    unsigned int h[KPT];  // top 32 bits after the common prefix; first digit = h >> 21
#pragma unroll
    for (int j = 0; j < KPT; ++j) {
        h[j] = unsigned((key[j] << shift) >> 32);
        // Branch-free: invalid entries count into the trash bin 2048.
        atomicAdd(&sc.hist[j < nv ? (h[j] >> 21) : 2048u], 1u);
    }
    QK_SEL_FINE(probe, 21);
    group_sync<NT>(bar);
    QK_SEL_FINE(probe, 22);
    unsigned int c[BPL], sl = 0;
#pragma unroll
    for (int j4 = 0; j4 < BPL / 4; ++j4) {
        const uint4 q = hist4[(2047 - BPL * gt) / 4 - j4];
        c[4 * j4 + 0] = q.w;
        c[4 * j4 + 1] = q.z;
        c[4 * j4 + 2] = q.y;
        c[4 * j4 + 3] = q.x;
    }
#pragma unroll
    for (int j = 0; j < BPL; ++j) sl += c[j];
    const unsigned int incl = warp_incl_scan(sl);
    if (lane == 31) sc.warp_sum[warp] = incl;
    QK_SEL_FINE(probe, 23);
    group_sync<NT>(bar);
    {
        unsigned int above = sum_below<NW>(sc.warp_sum, warp) + incl - sl;
        if (above < target && target <= above + sl) {  // exactly one lane of the group
#pragma unroll
            for (int j = 0; j < BPL; ++j) {
                if (above < target && target <= above + c[j]) {
                    sc.count = c[j];
                    sc.digit = 2047 - (BPL * gt + j);
                    sc.above = above;
                }
                above += c[j];
            }
        }
    }
    group_sync<NT>(bar);
    const unsigned int bin = sc.digit, bin_count = sc.count;
    const unsigned int krem = target - sc.above;
    sel_stamp(probe, 11);
    signal(1, shift, bin);  // keys of digit > bin are selected whatever happens next
    if (bin_count != krem && bin_count > 32) {  // needs more digits: the 64-bit path
        group_sync<NT>(bar);
        block_select_reg_wide<NT, KPT>(key, n, target, ref, out, sc, gt, bar, probe);
        return;
    }
    // Keys above the bin are in; keys of the bin by TAKE_BIN or by rank (<= 32 keys).
    // Per-thread 16-bit masks keep the register footprint small (the per-key arrays of an
    // earlier form serialised warp 0's ranking loads).
    unsigned int takem = 0, candm = 0;
#pragma unroll
    for (int j = 0; j < KPT; ++j) {
        const unsigned int d = h[j] >> 21;
        takem |= (j < nv && d > bin) ? 1u << j : 0u;
        candm |= (j < nv && d == bin) ? 1u << j : 0u;
    }
    if (bin_count == krem) {
        takem |= candm;
    } else {
        // Gather the bin's keys: warp-scanned slots, one shared atomic per warp.
        const unsigned int cnt = __popc(candm);
        const unsigned int incl_c = warp_incl_scan(cnt);
        unsigned int base = 0;
        if (lane == 31 && incl_c)  // plain atom (the intrinsic gets a warp-aggregation prologue)
            asm volatile("atom.shared.add.u32 %0, [%1], %2;"
                         : "=r"(base)
                         : "r"(static_cast<unsigned int>(__cvta_generic_to_shared(&sc.n_cand))), "r"(incl_c)
                         : "memory");
        base = __shfl_sync(0xffffffffu, base, 31) + incl_c - cnt;
#pragma unroll
        for (int j = 0; j < KPT; ++j) {  // static indices keep key[] in registers
            if ((candm >> j) & 1u) reinterpret_cast<ulonglong2*>(sc.cand2)[base++] = make_ulonglong2(key[j], i0 + j);
        }
        QK_SEL_FINE(probe, 24);
        group_sync<NT>(bar);
        QK_SEL_FINE(probe, 25);
        if (warp == 0) {  // lane m ranks candidate m; verdicts go to the key bitmap
            const unsigned int nc = sc.n_cand;
            const ulonglong2 me = reinterpret_cast<const ulonglong2*>(sc.cand2)[lane];
            unsigned int rank = 0;
            // Only the nc (<= 32, usually a few) gathered candidates: a warp-uniform trip
            // count (each iteration is a dependent compare chain of ~50 cycles).
            for (uint32_t m = 0; m < nc; ++m) {
                const ulonglong2 o = reinterpret_cast<const ulonglong2*>(sc.cand2)[m];
                rank += (o.x > me.x) | ((o.x == me.x) & (o.y < me.y));
            }
            if (uint32_t(lane) < nc && rank < krem) {
                const uint32_t idx = uint32_t(me.y);
                atomicOr(&sc.selbits[idx >> 5], 1u << (idx & 31));
            }
        }
        QK_SEL_FINE(probe, 26);
        group_sync<NT>(bar);
        takem |= candm & (sc.selbits[i0 >> 5] >> (i0 & 31));
    }
    sel_stamp(probe, 14);
    const unsigned int mine = __popc(takem);
    const unsigned int incl2 = warp_incl_scan(mine);
    if (lane == 31) sc.warp_sum[warp] = incl2;
    QK_SEL_FINE(probe, 27);
    group_sync<NT>(bar);
    unsigned int pos = sum_below<NW>(sc.warp_sum, warp) + incl2 - mine;
    for (unsigned int m = takem; m; m &= m - 1) out[pos++] = static_cast<OutT>(i0 + uint32_t(__ffs(m) - 1));
    sel_stamp(probe, 15);
}

}  // namespace qk

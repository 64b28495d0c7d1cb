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

// Optional phase stamps (QK_PROBE): slot 8.. of a 16-slot per-CTA record.
__device__ __forceinline__ void sel_stamp(unsigned long long* probe, int slot) {
    if (probe != nullptr && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        probe[blockIdx.x * 16 + slot] = t;
    }
}

template <int NT>
struct SelectScratch {
    unsigned int hist[2048];
    unsigned int warp_sum[NT / 32];
    unsigned long long red_max[NT / 32], red_min[NT / 32];
    unsigned long long cand_key[32];
    unsigned int cand_idx[32];
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

// Loads scores[0..n) (global, written earlier in the same kernel or by a prior one) as
// keys into `keys` (padded layout, capacity NT*(kpt+1)).  Returns kpt.
template <int NT>
__device__ __forceinline__ int load_keys(const double* __restrict__ scores, uint32_t n,
                                         unsigned long long* keys, SelectScratch<NT>& sc,
                                         unsigned long long* kmax_out,
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
            v[j] = (j0 + j < kpt && i < n) ? __ldcg(scores + i) : 0.0;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint32_t i = uint32_t(t) * kpt + j0 + j;
            if (j0 + j < kpt && i < n) {
                const unsigned long long u = order_key(v[j]);
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
        sel_stamp(probe, 9 + (pass < 2 ? pass : 2));
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
    sel_stamp(probe, 12);
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
    sel_stamp(probe, 13);
}

}  // namespace qk

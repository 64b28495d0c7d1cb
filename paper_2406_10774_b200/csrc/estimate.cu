// estimate.cu -- per-page criticality estimate (K2), bitwise equal to the reference.
//
// Reference: estimate_page_score / estimate_all,
// /root/reference/proj/core/src/criticality.cpp:9-34:
//     score = 0.0; for i ascending: score += std::max(q_i * max_i, q_i * min_i)   (double)
//
// Exactness argument (why this kernel reproduces the reference bit for bit):
//   * q_i, min_i, max_i are fp16 values, so q_i * x is a product of two 11-bit
//     significands: exact in double.  Hence fma(q_i, x, acc) == acc + (q_i * x) rounded
//     once, which is exactly the reference's `score += product`.
//   * max_i >= min_i always, so for q_i >= 0 the max is q_i*max_i and for q_i < 0 it is
//     q_i*min_i (equal products may differ only in the sign of zero, and adding +-0 to a
//     sum that starts at +0.0 never changes it).  The kernel therefore reads, per
//     channel, only the metadata row the query's sign selects: for MHA half of the
//     metadata bytes the reference's accounting charges (metrics.cpp:105).
//   * The fp64 chain per (query head, page) runs channel 0..D-1 in order in one thread.
//
// Work layout: one CTA per (PAGES pages, sequence, KV head); 128 threads.  The needed
// metadata rows (one contiguous run of PAGES*2 bytes per channel) are staged into shared
// memory with cp.async in four channel groups so the fp64 chains of group g overlap the
// loads of groups g+1.. .  MHA (G=1): each thread owns two adjacent pages (half2 reads,
// two independent chains).  GQA (G>1): each thread owns one page and G chains, the
// metadata is read once per KV head for all G query heads.
#include <cstdlib>

#include "qk_internal.cuh"

namespace qk {
namespace {

__device__ __forceinline__ double h2d(__half h) {
    double d;
    asm("cvt.f64.f16 %0, %1;" : "=d"(d) : "h"(__half_as_ushort(h)));
    return d;
}

// fp16 bits -> sel * 2^-1008 exactly (see decode.cu).
__device__ __forceinline__ double h2d_scaled(unsigned short h) {
    const uint32_t t = uint32_t(h) << 10;
    const uint32_t s = t & 0x02000000u;
    return __hiloint2double(int(t + s * 63u), 0);
}

// ---- MHA (G = 1): channel-split, certified -------------------------------------------------
//
// Thread (cg, pb) of a 256-thread CTA covers pages page0 + 8*pb .. +7 over the channel group
// cg (D/8 channels): one 16-byte load of the sign-selected row per channel (8 pages), all of
// them in flight at once, then 8 independent chains.  The 8 channel-group partials of a page
// meet in shared memory and are added pairwise; every partial is a sum of exact products,
// so the result is bitwise the reference's sequential sum whenever the page's magnitude
// record certifies that no partial sum can round (sum|q| * max|x| < 2^(53 + uq + ux), as
// the fused kernel, decode.cu); a failing page reruns the reference's chain.  Odd channels
// convert with the exact integer construction scaled by 2^-1008 (weights pre-scaled by
// 2^1008), even ones with F2F, so the XU and ALU pipes share the conversions.
constexpr int kMhaThreads = 256;
constexpr int kMhaPPC = 256;  // pages per CTA: 32 page blocks x 8 channel groups

template <int D>
__global__ void __launch_bounds__(kMhaThreads)
estimate_mha_kernel(const __half* __restrict__ meta, const uint32_t* __restrict__ prange,
                    const int32_t* __restrict__ len, const __half* __restrict__ q,
                    double* __restrict__ scores, uint32_t layer, uint32_t B, uint32_t Hkv,
                    uint32_t S, uint32_t head_dim, size_t slice_meta, uint32_t mrow,
                    uint32_t sstride) {
    constexpr int CPG = D / 8;                     // channels per group
    constexpr int ROUND = CPG < 16 ? CPG : 16;     // loads in flight per round
    __shared__ double dq[D], dw[D];
    __shared__ unsigned char need[D];
    __shared__ double part[8][kMhaPPC];
    __shared__ double s_qpart[D / 32];
    __shared__ unsigned int s_qcodep[D / 32];

    const uint32_t bh = blockIdx.y;
    const uint32_t b = bh / Hkv, kvh = bh % Hkv;
    const uint32_t n_tok = static_cast<uint32_t>(len[layer * B + b]);
    const uint32_t P = (n_tok + S - 1) / S;
    const uint32_t page0 = blockIdx.x * kMhaPPC;
    if (page0 >= P) return;
    const int tid = threadIdx.x, lane = tid & 31;
    if (tid < D) {
        const __half h = tid < int(head_dim) ? q[(size_t(b) * Hkv + kvh) * head_dim + tid]
                                             : __float2half(0.0f);
        const double x = double(__half2float(h));
        dq[tid] = x;
        dw[tid] = (tid & 1) ? x * 0x1p1008 : x;
        need[tid] = (x < 0.0) ? 0 : 1;  // the row index: min (0) or max (1)
        double a = fabs(x);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        const unsigned int code = __reduce_min_sync(0xffffffffu, ulp_code(__half_as_ushort(h)));
        if (lane == 0) {
            s_qpart[tid >> 5] = a;
            s_qcodep[tid >> 5] = code;
        }
    }
    __syncthreads();

    const size_t s = (size_t(layer) * B + b) * Hkv + kvh;
    const __half* mslice = meta + s * slice_meta;  // [2][D][mrow]
    if (tid < D) {
        // One L2 bulk prefetch per channel of this CTA's sign-selected row segment ahead of
        // the register loads (tools/microbench_meta.cu pattern F): 7.35 -> 6.84 us per cfg2
        // layer, graph-timed.  (Inside the fused kernel the same prefetch loses.)
        const uint32_t npg = min(uint32_t(kMhaPPC), ((P - page0) + 7u) & ~7u);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(
                         mslice + (size_t(need[tid]) * D + tid) * mrow + page0),
                     "r"(npg * 2u) : "memory");
    }
    const int cg = tid >> 5, pb = lane;            // warp = channel group: 512-byte loads
    const uint32_t pbase = page0 + uint32_t(pb) * 8;
    const bool act = pbase < P;
    double acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = 0.0;
#pragma unroll
    for (int r0 = 0; r0 < CPG; r0 += ROUND) {
        int4 v[ROUND];
#pragma unroll
        for (int k = 0; k < ROUND; ++k) {
            const int c = cg * CPG + r0 + k;
            v[k] = act ? ld_nc_v4(mslice + (size_t(need[c]) * D + c) * mrow + pbase)
                       : make_int4(0, 0, 0, 0);
        }
#pragma unroll
        for (int k = 0; k < ROUND; ++k) {
            const int c = cg * CPG + r0 + k;
            const double w = dw[c];
            const unsigned short* h = reinterpret_cast<const unsigned short*>(&v[k]);
#pragma unroll
            for (int j = 0; j < 8; ++j)
                acc[j] = __fma_rn(w, (c & 1) ? h2d_scaled(h[j]) : h2d(__ushort_as_half(h[j])), acc[j]);
        }
    }
    double2* dst = reinterpret_cast<double2*>(&part[cg][pb * 8]);
#pragma unroll
    for (int j = 0; j < 4; ++j) dst[j] = make_double2(acc[2 * j], acc[2 * j + 1]);
    __syncthreads();

    const uint32_t p = page0 + uint32_t(tid);
    if (p >= P || p >= sstride) return;
    double sc = ((part[0][tid] + part[1][tid]) + (part[2][tid] + part[3][tid])) +
                ((part[4][tid] + part[5][tid]) + (part[6][tid] + part[7][tid]));
    double qabs = 0.0;
    unsigned int qcode = 31u;
#pragma unroll
    for (int w = 0; w < D / 32; ++w) {
        qabs += s_qpart[w];
        qcode = min(qcode, s_qcodep[w]);
    }
    const uint32_t rec = __ldg(prange + s * mrow + p);
    const uint32_t xcode = rec >> 16;
    bool exact = xcode >= 31u || qcode >= 31u;  // all-zero operands
    if (!exact) {
        const double bound =
            __dmul_ru(qabs, double(__half2float(__ushort_as_half(uint16_t(rec & 0x7fffu)))));
        const int e = 5 + int(qcode) + int(xcode);
        exact = bound < __longlong_as_double(static_cast<long long>(e + 1023) << 52);
    }
    if (!exact) {  // the reference's sequential chain (criticality.cpp:16-21)
        double a = 0.0;
        for (int c = 0; c < D; ++c)
            a = __fma_rn(dq[c], h2d(mslice[(size_t(need[c]) * D + c) * mrow + p]), a);
        sc = a;
    }
    scores[(size_t(b) * Hkv + kvh) * sstride + p] = sc;
}

// ---- GQA (G > 1): sequential chains, the reference's order exactly ------------------------
//
// Thread = PB consecutive pages x all G query heads of one (sequence, KV head): per channel
// one 16-byte (8-page) load of each row some head needs, every value converted once (min
// row with F2F, max row with the scaled integer construction) and folded into the
// PB * G independent chains (enough to cover the DFMA latency; no certificate needed).
// The next channel group's loads are in flight while the current one is folded.
constexpr int kThreads = 128;

template <int G>
struct GqaGeom {
    static constexpr int PB = (G >= 8) ? 4 : 8;   // pages per thread (one 8/16-byte load)
    static constexpr int PPC = kThreads * PB;      // pages per CTA
    static constexpr int UNROLL = 4;               // channels per pipeline stage
};

template <int PB>
struct Piece;
template <>
struct Piece<8> {
    int4 v;
    __device__ __forceinline__ void load(const __half* p) { v = ld_nc_v4(p); }
    __device__ __forceinline__ void zero() { v = make_int4(0, 0, 0, 0); }
    __device__ __forceinline__ unsigned short at(int j) const {
        return reinterpret_cast<const unsigned short*>(&v)[j];
    }
};
template <>
struct Piece<4> {
    int2 v;
    __device__ __forceinline__ void load(const __half* p) {
        asm volatile("ld.global.nc.L1::no_allocate.v2.s32 {%0,%1}, [%2];"
                     : "=r"(v.x), "=r"(v.y) : "l"(p));
    }
    __device__ __forceinline__ void zero() { v = make_int2(0, 0); }
    __device__ __forceinline__ unsigned short at(int j) const {
        return reinterpret_cast<const unsigned short*>(&v)[j];
    }
};

template <int D, int G>
__global__ void __launch_bounds__(kThreads)
estimate_gqa_kernel(const __half* __restrict__ meta, const int32_t* __restrict__ len,
                    const __half* __restrict__ q, double* __restrict__ scores, uint32_t layer,
                    uint32_t B, uint32_t Hkv, uint32_t S, uint32_t head_dim, size_t slice_meta,
                    uint32_t mrow, uint32_t sstride) {
    using GM = GqaGeom<G>;
    constexpr int PB = GM::PB, PPC = GM::PPC, U = GM::UNROLL;
    __shared__ double dw[G * D];  // weights of the conversion path (max row scaled 2^1008)
    __shared__ unsigned char need[D];  // bit0: max row needed, bit1: min row needed

    const uint32_t bh = blockIdx.y;
    const uint32_t b = bh / Hkv, kvh = bh % Hkv;
    const uint32_t n_tok = static_cast<uint32_t>(len[layer * B + b]);
    const uint32_t P = (n_tok + S - 1) / S;
    const uint32_t page0 = blockIdx.x * PPC;
    if (page0 >= P) return;
    const int tid = threadIdx.x;
    for (int i = tid; i < G * D; i += kThreads) {
        const int g = i / D, c = i % D;
        const double x = c < int(head_dim)
                             ? double(__half2float(q[(size_t(b) * Hkv * G + size_t(kvh) * G + g) * head_dim + c]))
                             : 0.0;
        dw[i] = (x < 0.0) ? x : x * 0x1p1008;
    }
    __syncthreads();
    for (int c = tid; c < D; c += kThreads) {
        unsigned char m = 0;
#pragma unroll
        for (int g = 0; g < G; ++g) m |= (dw[g * D + c] < 0.0) ? 2 : 1;
        need[c] = m;
    }
    __syncthreads();

    const uint32_t pbase = page0 + uint32_t(tid) * PB;
    if (pbase >= P) return;
    const size_t s = (size_t(layer) * B + b) * Hkv + kvh;
    const __half* mslice = meta + s * slice_meta;  // [2][D][mrow]
    double acc[G][PB];
#pragma unroll
    for (int g = 0; g < G; ++g)
#pragma unroll
        for (int j = 0; j < PB; ++j) acc[g][j] = 0.0;

    Piece<PB> lo[2][U], hi[2][U];
    auto load = [&](int buf, int c0) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int c = c0 + u;
            const unsigned char m = need[c];
            if (m & 2) lo[buf][u].load(mslice + size_t(c) * mrow + pbase);
            else lo[buf][u].zero();
            if (m & 1) hi[buf][u].load(mslice + size_t(D + c) * mrow + pbase);
            else hi[buf][u].zero();
        }
    };
    auto fold = [&](int buf, int c0) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int c = c0 + u;
            double xl[PB], xh[PB];
#pragma unroll
            for (int j = 0; j < PB; ++j) {
                xl[j] = h2d(__ushort_as_half(lo[buf][u].at(j)));
                xh[j] = h2d_scaled(hi[buf][u].at(j));
            }
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const double w = dw[g * D + c];
                if (w < 0.0) {  // uniform over the CTA: a branch, not selects
#pragma unroll
                    for (int j = 0; j < PB; ++j) acc[g][j] = __fma_rn(w, xl[j], acc[g][j]);
                } else {
#pragma unroll
                    for (int j = 0; j < PB; ++j) acc[g][j] = __fma_rn(w, xh[j], acc[g][j]);
                }
            }
        }
    };
    load(0, 0);
#pragma unroll 1
    for (int c0 = 0; c0 < D; c0 += 2 * U) {
        if (c0 + U < D) load(1, c0 + U);
        fold(0, c0);
        if (c0 + U >= D) break;
        if (c0 + 2 * U < D) load(0, c0 + 2 * U);
        fold(1, c0 + U);
    }
#pragma unroll
    for (int j = 0; j < PB; ++j) {
        const uint32_t p = pbase + j;
        if (p >= P || p >= sstride) break;
#pragma unroll
        for (int g = 0; g < G; ++g)
            scores[(size_t(b) * Hkv * G + size_t(kvh) * G + g) * sstride + p] = acc[g][j];
    }
}

// Staged variant (PB = 8): the metadata pieces go through a kStages-deep cp.async pipeline
// in shared memory instead of register double buffers, so a thread keeps ~kStages x 128 B in
// flight without holding them in registers (more bytes in flight per SM, more CTAs per SM).
// Each thread copies and later reads only its own pieces: no CTA barrier in the loop.
constexpr int kStages = 4;

template <int D, int G>
__global__ void __launch_bounds__(kThreads)
estimate_gqa_staged_kernel(const __half* __restrict__ meta, const int32_t* __restrict__ len,
                           const __half* __restrict__ q, double* __restrict__ scores,
                           uint32_t layer, uint32_t B, uint32_t Hkv, uint32_t S,
                           uint32_t head_dim, size_t slice_meta, uint32_t mrow,
                           uint32_t sstride) {
    using GM = GqaGeom<G>;
    constexpr int PB = GM::PB, PPC = GM::PPC, U = GM::UNROLL;
    static_assert(PB == 8, "16-byte pieces");
    extern __shared__ __align__(16) int4 stage[];  // [kStages][2][U][kThreads]
    __shared__ double dw[G * D];
    __shared__ unsigned char need[D];

    const uint32_t bh = blockIdx.y;
    const uint32_t b = bh / Hkv, kvh = bh % Hkv;
    const uint32_t n_tok = static_cast<uint32_t>(len[layer * B + b]);
    const uint32_t P = (n_tok + S - 1) / S;
    const uint32_t page0 = blockIdx.x * PPC;
    if (page0 >= P) return;
    const int tid = threadIdx.x;
    for (int i = tid; i < G * D; i += kThreads) {
        const int g = i / D, c = i % D;
        const double x = c < int(head_dim)
                             ? double(__half2float(q[(size_t(b) * Hkv * G + size_t(kvh) * G + g) * head_dim + c]))
                             : 0.0;
        dw[i] = (x < 0.0) ? x : x * 0x1p1008;
    }
    __syncthreads();
    for (int c = tid; c < D; c += kThreads) {
        unsigned char m = 0;
#pragma unroll
        for (int g = 0; g < G; ++g) m |= (dw[g * D + c] < 0.0) ? 2 : 1;
        need[c] = m;
    }
    __syncthreads();

    const uint32_t pbase = page0 + uint32_t(tid) * PB;
    if (pbase >= P) return;
    const size_t s = (size_t(layer) * B + b) * Hkv + kvh;
    const __half* mslice = meta + s * slice_meta;  // [2][D][mrow]
    double acc[G][PB];
#pragma unroll
    for (int g = 0; g < G; ++g)
#pragma unroll
        for (int j = 0; j < PB; ++j) acc[g][j] = 0.0;

    constexpr int NB = D / U;  // channel blocks
    auto slot = [&](int st, int row, int u) -> int4* {
        return stage + ((st * 2 + row) * U + u) * kThreads + tid;
    };
    auto issue = [&](int cb) {
        if (cb < NB) {
            const int st = cb % kStages;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int c = cb * U + u;
                const unsigned char m = need[c];
                if (m & 2) cp_async16(slot(st, 0, u), mslice + size_t(c) * mrow + pbase);
                if (m & 1) cp_async16(slot(st, 1, u), mslice + size_t(D + c) * mrow + pbase);
            }
        }
        cp_async_commit();  // (empty groups keep the wait count uniform)
    };
#pragma unroll
    for (int cb = 0; cb < kStages - 1; ++cb) issue(cb);
#pragma unroll 1
    for (int cb = 0; cb < NB; ++cb) {
        cp_async_wait<kStages - 2>();
        const int st = cb % kStages;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int c = cb * U + u;
            const unsigned char m = need[c];
            const int4 lo = (m & 2) ? *slot(st, 0, u) : make_int4(0, 0, 0, 0);
            const int4 hi = (m & 1) ? *slot(st, 1, u) : make_int4(0, 0, 0, 0);
            const unsigned short* l16 = reinterpret_cast<const unsigned short*>(&lo);
            const unsigned short* h16 = reinterpret_cast<const unsigned short*>(&hi);
            double xl[PB], xh[PB];
#pragma unroll
            for (int j = 0; j < PB; ++j) {
                xl[j] = h2d(__ushort_as_half(l16[j]));
                xh[j] = h2d_scaled(h16[j]);
            }
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const double w = dw[g * D + c];
                if (w < 0.0) {
#pragma unroll
                    for (int j = 0; j < PB; ++j) acc[g][j] = __fma_rn(w, xl[j], acc[g][j]);
                } else {
#pragma unroll
                    for (int j = 0; j < PB; ++j) acc[g][j] = __fma_rn(w, xh[j], acc[g][j]);
                }
            }
        }
        issue(cb + kStages - 1);  // into the slot read in the previous iteration
    }
#pragma unroll
    for (int j = 0; j < PB; ++j) {
        const uint32_t p = pbase + j;
        if (p >= P || p >= sstride) break;
#pragma unroll
        for (int g = 0; g < G; ++g)
            scores[(size_t(b) * Hkv * G + size_t(kvh) * G + g) * sstride + p] = acc[g][j];
    }
}

template <int D, int G>
int run(const qk_cache* c, uint32_t layer, const __half* q, uint32_t batch, double* scores,
        uint32_t stride, uint32_t max_pages, cudaStream_t st) {
    if constexpr (G == 1) {
        const dim3 grid((max_pages + kMhaPPC - 1) / kMhaPPC, batch * c->Hkv);
        estimate_mha_kernel<D><<<grid, kMhaThreads, 0, st>>>(
            c->meta, c->prange, c->d_len, q, scores, layer, c->B, c->Hkv, c->S, c->desc.head_dim,
            c->slice_meta, c->Mrow, stride);
    } else {
        using GM = GqaGeom<G>;
        const dim3 grid((max_pages + GM::PPC - 1) / GM::PPC, batch * c->Hkv);
        // G = 2, 4 (16-byte pieces): the cp.async-staged kernel (cfg4: 388 -> 374 us per
        // layer step, 2-round A/B; deeper or narrower pipelines and 4 CTAs per SM were slower).
        static const bool staged = getenv("QK_GQA_REGISTER_ESTIMATE") == nullptr;  // A/B switch
        if constexpr (GM::PB == 8) {
            if (staged) {
                const size_t smem = size_t(kStages) * 2 * GM::UNROLL * kThreads * 16;
                auto kern = estimate_gqa_staged_kernel<D, G>;
                if (int rc = ensure_func_attrs(reinterpret_cast<const void*>(kern), smem,
                                               c->desc.device, false, "estimate_gqa_staged"))
                    return rc;
                kern<<<grid, kThreads, smem, st>>>(c->meta, c->d_len, q, scores, layer, c->B,
                                                   c->Hkv, c->S, c->desc.head_dim, c->slice_meta,
                                                   c->Mrow, stride);
                const_cast<qk_cache*>(c)->launches++;
                return cuda_check(cudaGetLastError(), "estimate_kernel");
            }
        }
        estimate_gqa_kernel<D, G><<<grid, kThreads, 0, st>>>(
            c->meta, c->d_len, q, scores, layer, c->B, c->Hkv, c->S, c->desc.head_dim,
            c->slice_meta, c->Mrow, stride);
    }
    const_cast<qk_cache*>(c)->launches++;
    return cuda_check(cudaGetLastError(), "estimate_kernel");
}

template <int D>
int dispatch_g(const qk_cache* c, uint32_t layer, const __half* q, uint32_t batch,
               double* scores, uint32_t stride, uint32_t max_pages, cudaStream_t st) {
    switch (c->G) {
        case 1: return run<D, 1>(c, layer, q, batch, scores, stride, max_pages, st);
        case 2: return run<D, 2>(c, layer, q, batch, scores, stride, max_pages, st);
        case 4: return run<D, 4>(c, layer, q, batch, scores, stride, max_pages, st);
        case 8: return run<D, 8>(c, layer, q, batch, scores, stride, max_pages, st);
        default: return set_error(QK_ERR_UNSUPPORTED, "qk_estimate: GQA group size must be 1, 2, 4 or 8");
    }
}

}  // namespace

int launch_estimate(const qk_cache* c, uint32_t layer, const __half* q, uint32_t batch,
                    double* scores, uint32_t stride, uint32_t max_pages, cudaStream_t st) {
    switch (c->D) {
        case 64: return dispatch_g<64>(c, layer, q, batch, scores, stride, max_pages, st);
        case 128: return dispatch_g<128>(c, layer, q, batch, scores, stride, max_pages, st);
        case 256: return dispatch_g<256>(c, layer, q, batch, scores, stride, max_pages, st);
        default: return set_error(QK_ERR_UNSUPPORTED, "qk_estimate: unsupported head_dim");
    }
}

}  // namespace qk

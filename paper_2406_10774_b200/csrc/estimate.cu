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

constexpr int kThreads = 128;
constexpr int kGroups = 4;

template <int D, int G, int PAGES>
__global__ void __launch_bounds__(kThreads)
estimate_kernel(const __half* __restrict__ meta, const int32_t* __restrict__ len,
                const __half* __restrict__ q, double* __restrict__ scores, uint32_t layer,
                uint32_t B, uint32_t Hkv, uint32_t S, uint32_t head_dim, size_t slice_meta,
                uint32_t mrow, uint32_t sstride) {
    constexpr int NROW = (G == 1) ? 1 : 2;  // metadata rows staged per channel
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __half* rows = reinterpret_cast<__half*>(smem_raw);                 // [NROW][D][PAGES]
    double* dq = reinterpret_cast<double*>(rows + NROW * D * PAGES);    // [G][D]
    __shared__ unsigned char need[D];  // bit0: max row needed, bit1: min row needed

    const uint32_t bh = blockIdx.y;
    const uint32_t b = bh / Hkv, kvh = bh % Hkv;
    const uint32_t n_tok = static_cast<uint32_t>(len[layer * B + b]);
    const uint32_t P = (n_tok + S - 1) / S;
    const uint32_t page0 = blockIdx.x * PAGES;
    if (page0 >= P) return;
    const uint32_t npg = min(uint32_t(PAGES), P - page0);
    const int n8 = int((npg + 7) / 8);  // 16-byte pieces per channel row

    // Query of the G heads sharing this KV head, widened to double (exact).
    for (int i = threadIdx.x; i < G * D; i += kThreads) {
        const int g = i / D, c = i % D;
        const size_t qh = size_t(kvh) * G + g;
        const float x = c < int(head_dim)
                            ? __half2float(q[(size_t(b) * Hkv * G + qh) * head_dim + c])
                            : 0.0f;
        dq[g * D + c] = double(x);
        if (G == 1) dq[D + c] = double(x) * 0x1p1008;  // weight of the scaled path
    }
    __syncthreads();
    for (int c = threadIdx.x; c < D; c += kThreads) {
        unsigned char m = 0;
#pragma unroll
        for (int g = 0; g < G; ++g) m |= (dq[g * D + c] < 0.0) ? 2 : 1;
        need[c] = m;
    }
    __syncthreads();

    const size_t s = (size_t(layer) * B + b) * Hkv + kvh;
    const __half* mslice = meta + s * slice_meta;
    constexpr int CH_PER_GROUP = D / kGroups;
#pragma unroll
    for (int grp = 0; grp < kGroups; ++grp) {
        const int n_items = CH_PER_GROUP * NROW * n8;
        for (int i = threadIdx.x; i < n_items; i += kThreads) {
            const int piece = i % n8;
            const int rest = i / n8;
            const int r = rest % NROW;
            const int c = grp * CH_PER_GROUP + rest / NROW;
            // G == 1: the single staged row is the one the query's sign selects.
            const int minmax = (G == 1) ? ((need[c] & 2) ? 0 : 1) : r;
            if (G > 1 && !(need[c] & (minmax == 0 ? 2 : 1))) continue;
            const __half* src = mslice + (size_t(minmax) * D + c) * mrow + page0 + piece * 8;
            __half* dst = rows + (size_t(r) * D + c) * PAGES + piece * 8;
            cp_async16(dst, src);
        }
        cp_async_commit();
    }

    if constexpr (G == 1) {
        const int j = threadIdx.x * 2;  // two adjacent pages
        const bool active = uint32_t(j) < npg;
        double acc0 = 0.0, acc1 = 0.0;
#pragma unroll
        for (int grp = 0; grp < kGroups; ++grp) {
            if (grp == 0) cp_async_wait<kGroups - 1>();
            if (grp == 1) cp_async_wait<kGroups - 2>();
            if (grp == 2) cp_async_wait<kGroups - 3>();
            if (grp == 3) cp_async_wait<0>();
            __syncthreads();
            if (active) {
#pragma unroll 8
                for (int cc = 0; cc < CH_PER_GROUP; ++cc) {
                    const int c = grp * CH_PER_GROUP + cc;
                    const __half2 h2 = *reinterpret_cast<const __half2*>(rows + size_t(c) * PAGES + j);
                    // Page 2j converts on the XU pipe, page 2j+1 with integer ops
                    // (h2d_scaled, weight pre-scaled by 2^1008): both pipes share the work.
                    acc0 = __fma_rn(dq[c], h2d(__low2half(h2)), acc0);
                    acc1 = __fma_rn(dq[D + c], h2d_scaled(__half_as_ushort(__high2half(h2))), acc1);
                }
            }
        }
        const uint32_t p = page0 + j;
        double* out = scores + (size_t(b) * Hkv + kvh) * sstride;
        if (active && p < P && p < sstride) out[p] = acc0;
        if (active && p + 1 < P && p + 1 < sstride) out[p + 1] = acc1;
    } else {
        const int j = threadIdx.x;  // PAGES == kThreads pages per CTA
        const bool active = uint32_t(j) < npg;
        double acc[G];
#pragma unroll
        for (int g = 0; g < G; ++g) acc[g] = 0.0;
#pragma unroll
        for (int grp = 0; grp < kGroups; ++grp) {
            if (grp == 0) cp_async_wait<kGroups - 1>();
            if (grp == 1) cp_async_wait<kGroups - 2>();
            if (grp == 2) cp_async_wait<kGroups - 3>();
            if (grp == 3) cp_async_wait<0>();
            __syncthreads();
            if (active) {
#pragma unroll 4
                for (int cc = 0; cc < CH_PER_GROUP; ++cc) {
                    const int c = grp * CH_PER_GROUP + cc;
                    const double lo = h2d(rows[(size_t(0) * D + c) * PAGES + j]);
                    const double hi = h2d(rows[(size_t(1) * D + c) * PAGES + j]);
#pragma unroll
                    for (int g = 0; g < G; ++g) {
                        const double w = dq[g * D + c];
                        acc[g] = __fma_rn(w, (w < 0.0) ? lo : hi, acc[g]);
                    }
                }
            }
        }
        const uint32_t p = page0 + j;
        if (active && p < P && p < sstride) {
#pragma unroll
            for (int g = 0; g < G; ++g)
                scores[(size_t(b) * Hkv * G + size_t(kvh) * G + g) * sstride + p] = acc[g];
        }
    }
}

template <int D, int G, int PAGES>
int run(const qk_cache* c, uint32_t layer, const __half* q, uint32_t batch, double* scores,
        uint32_t stride, uint32_t max_pages, cudaStream_t st) {
    constexpr int NROW = (G == 1) ? 1 : 2;
    const size_t smem = size_t(NROW) * D * PAGES * sizeof(__half) +
                        size_t(G == 1 ? 2 : G) * D * sizeof(double);
    auto kern = estimate_kernel<D, G, PAGES>;
    if (int rc = ensure_func_attrs(reinterpret_cast<const void*>(kern), smem, c->desc.device, false,
                                   "estimate_kernel attributes"))
        return rc;
    const uint32_t pages_per_cta = PAGES;
    const dim3 grid((max_pages + pages_per_cta - 1) / pages_per_cta, batch * c->Hkv);
    kern<<<grid, kThreads, smem, st>>>(c->meta, c->d_len, q, scores, layer, c->B, c->Hkv, c->S,
                                       c->desc.head_dim, c->slice_meta, c->Mrow, stride);
    const_cast<qk_cache*>(c)->launches++;
    return cuda_check(cudaGetLastError(), "estimate_kernel");
}

template <int D>
int dispatch_g(const qk_cache* c, uint32_t layer, const __half* q, uint32_t batch,
               double* scores, uint32_t stride, uint32_t max_pages, cudaStream_t st) {
    switch (c->G) {
        case 1: return run<D, 1, 2 * kThreads>(c, layer, q, batch, scores, stride, max_pages, st);
        case 2: return run<D, 2, kThreads>(c, layer, q, batch, scores, stride, max_pages, st);
        case 4: return run<D, 4, kThreads>(c, layer, q, batch, scores, stride, max_pages, st);
        case 8: return run<D, 8, kThreads>(c, layer, q, batch, scores, stride, max_pages, st);
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

// attend_warp.cuh -- the page-streaming inner loop shared by the split-KV attention
// kernel (attend.cu) and the fused decode kernel (decode.cu).
//
// One warp folds whole pages into an online-softmax state (m, l, o) in the base-2 domain:
// a page is S rows x D fp16, one contiguous block; lane (rgrp, chunk) reads 16 bytes of
// rows rgrp, rgrp+RPI, ... (RPI = 32 / (D/8) rows per warp-wide load), K and V of up to
// kBatchIters row groups are issued together, logits are reduced across the D/8 lanes of
// a row with shuffles, rows past the page's length are masked (partial newest page,
// attention.cpp:108-114).
#pragma once

#include <math_constants.h>

#include "qk_internal.cuh"

namespace qk {

constexpr int kBatchIters = 8;

__device__ __forceinline__ int4 ld_v4_coherent(const void* p) {
    int4 r;
    asm volatile("ld.global.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ void unpack8(const int4& v, float (&f)[8]) {
    const __half2* h = reinterpret_cast<const __half2*>(&v);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float2 x = __half22float2(h[i]);
        f[2 * i] = x.x;
        f[2 * i + 1] = x.y;
    }
}

// Folds one page (plen valid rows) into (m, l, o).  COHERENT selects plain loads (data
// written earlier in the same kernel) instead of the read-only path.  With `rows` (token
// granularity, attend_tokens) row r of the chunk is token rows[r] of the slice, i.e. at
// kpage + rows[r]*D with kpage the slice base; without it, row r is at kpage + r*D.  A chunk
// of consecutive tokens starting at a page boundary therefore loads and folds exactly what
// the page form does (bitwise equal results).
template <int D, bool COHERENT>
__device__ __forceinline__ void warp_fold_page(const __half* __restrict__ kpage,
                                               const __half* __restrict__ vpage, uint32_t plen,
                                               const float (&qf)[8], float scale_log2, float& m,
                                               float& l, float (&o)[8],
                                               const int32_t* __restrict__ rows = nullptr) {
    constexpr int CPR = D / 8;
    constexpr int RPI = 32 / CPR;
    const int lane = threadIdx.x & 31;
    const int chunk = lane % CPR, rgrp = lane / CPR;
    for (uint32_t r0 = 0; r0 < plen; r0 += kBatchIters * RPI) {
        int4 kv[kBatchIters], vv[kBatchIters];
#pragma unroll
        for (int it = 0; it < kBatchIters; ++it) {
            const uint32_t r = r0 + it * RPI + rgrp;
            if (r < plen) {
                const size_t row = rows ? size_t(uint32_t(rows[r])) : size_t(r);
                if (COHERENT) {
                    kv[it] = ld_v4_coherent(kpage + row * D + chunk * 8);
                    vv[it] = ld_v4_coherent(vpage + row * D + chunk * 8);
                } else {
                    kv[it] = ld_nc_v4(kpage + row * D + chunk * 8);
                    vv[it] = ld_nc_v4(vpage + row * D + chunk * 8);
                }
            } else {
                kv[it] = make_int4(0, 0, 0, 0);
                vv[it] = make_int4(0, 0, 0, 0);
            }
        }
        float sc[kBatchIters];
        float bmax = -CUDART_INF_F;
#pragma unroll
        for (int it = 0; it < kBatchIters; ++it) {
            float kf[8];
            unpack8(kv[it], kf);
            float d = 0.0f;
#pragma unroll
            for (int j = 0; j < 8; ++j) d = fmaf(qf[j], kf[j], d);
#pragma unroll
            for (int off = 1; off < CPR; off <<= 1) d += __shfl_xor_sync(0xffffffffu, d, off);
            const uint32_t r = r0 + it * RPI + rgrp;
            sc[it] = (r < plen) ? d * scale_log2 : -CUDART_INF_F;
            bmax = fmaxf(bmax, sc[it]);
        }
#pragma unroll
        for (int off = CPR; off < 32; off <<= 1)
            bmax = fmaxf(bmax, __shfl_xor_sync(0xffffffffu, bmax, off));
        const float m_new = fmaxf(m, bmax);
        const float alpha = exp2f(m - m_new);  // m == -inf on the first page -> 0
        l *= alpha;
#pragma unroll
        for (int j = 0; j < 8; ++j) o[j] *= alpha;
#pragma unroll
        for (int it = 0; it < kBatchIters; ++it) {
            const float p = exp2f(sc[it] - m_new);
            l += p;
            float vf[8];
            unpack8(vv[it], vf);
#pragma unroll
            for (int j = 0; j < 8; ++j) o[j] = fmaf(p, vf[j], o[j]);
        }
        m = m_new;
    }
}

// Folds the row groups of a warp: afterwards every lane with the same chunk holds the
// warp's (l, o) for its 8 channels.
template <int D>
__device__ __forceinline__ void warp_fold_rows(float& l, float (&o)[8]) {
    constexpr int CPR = D / 8;
#pragma unroll
    for (int off = CPR; off < 32; off <<= 1) {
        l += __shfl_xor_sync(0xffffffffu, l, off);
#pragma unroll
        for (int j = 0; j < 8; ++j) o[j] += __shfl_xor_sync(0xffffffffu, o[j], off);
    }
}

template <int D>
__device__ __forceinline__ void load_q8(const __half* __restrict__ qrow, uint32_t head_dim,
                                        float (&qf)[8]) {
    const int chunk = (threadIdx.x & 31) % (D / 8);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int c = chunk * 8 + j;
        qf[j] = c < int(head_dim) ? __half2float(qrow[c]) : 0.0f;
    }
}

}  // namespace qk

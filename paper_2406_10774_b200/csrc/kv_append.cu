// kv_append.cu -- KvCache::append with the page-metadata update fused in (K1), the
// page-parallel bulk prefill, and the read-back gathers used by the parity tests.
//
// Reference: KvCache::append, /root/reference/proj/core/src/kv_store.cpp:19-47.
//   token t -> page t/S, row t%S (:24-33); row 0 seeds min=max=key (:35-38); later rows
//   update channel-wise with strict '<' and '>' (:40-43), so among equal values (e.g.
//   -0 and +0) the first-seen one is kept.  Comparisons here are fp32 compares of the
//   exact fp16 values, written as explicit compare-and-select (fminf/__hmin do not
//   promise the first-seen zero sign).
#include "qk_internal.cuh"

namespace qk {
namespace {

// Page magnitude record (qk_internal.cuh) of one page, written by thread 0; the block is
// the page's D channel threads (D = 64, 128 or 256).
__device__ __forceinline__ void write_record(uint32_t* dst, __half mn, __half mx, int D) {
    __shared__ uint32_t scratch[8];
    uint32_t r;
    if (D == 64) r = page_record<64>(mn, mx, scratch, 1);
    else if (D == 128) r = page_record<128>(mn, mx, scratch, 1);
    else r = page_record<256>(mn, mx, scratch, 1);
    if (threadIdx.x == 0) *dst = r;
}


// One CTA per (sequence, KV head), one thread per channel.  Every CTA of a sequence reads
// the same token count; the last one to finish (ticket) bumps it, so no CTA can observe
// the new count early.
__global__ void append_kernel(__half* __restrict__ kp, __half* __restrict__ vp,
                              __half* __restrict__ meta, uint32_t* __restrict__ prange,
                              int32_t* __restrict__ len,
                              int32_t* __restrict__ ticket, int32_t* __restrict__ status,
                              const __half* __restrict__ k, const __half* __restrict__ v,
                              uint32_t layer, uint32_t B, uint32_t Hkv, uint32_t S, int D,
                              uint32_t head_dim, size_t slice_kv, size_t slice_meta, uint32_t mrow,
                              uint32_t capacity) {
    __shared__ int last;
    const uint32_t b = blockIdx.x, h = blockIdx.y, c = threadIdx.x;
    const uint32_t t = static_cast<uint32_t>(len[layer * B + b]);
    if (t >= capacity) {
        if (c == 0) record_status(status, QK_DEV_CAPACITY);
        return;
    }
    const uint32_t page = t / S, row = t % S;
    const size_t in = (size_t(b) * Hkv + h) * head_dim + c;
    const __half x = c < head_dim ? k[in] : __float2half(0.0f);
    const __half y = c < head_dim ? v[in] : __float2half(0.0f);
    const size_t s = (size_t(layer) * B + b) * Hkv + h;
    const size_t kv = s * slice_kv + (size_t(page) * S + row) * D + c;
    kp[kv] = x;
    vp[kv] = y;
    __half* mn = meta + meta_offset(slice_meta, mrow, s, page, D, 0, c);
    __half* mx = meta + meta_offset(slice_meta, mrow, s, page, D, 1, c);
    __half nmn = x, nmx = x;
    if (row != 0) {
        nmn = *mn;
        nmx = *mx;
        const float xf = __half2float(x);
        if (xf < __half2float(nmn)) nmn = x;
        if (xf > __half2float(nmx)) nmx = x;
    }
    *mn = nmn;
    *mx = nmx;
    write_record(prange + s * mrow + page, nmn, nmx, D);
    __syncthreads();
    if (c == 0) last = (atomicAdd(ticket + layer * B + b, 1) == int(Hkv) - 1);
    __syncthreads();
    if (last && c == 0) {
        ticket[layer * B + b] = 0;
        len[layer * B + b] = int32_t(t + 1);
    }
}

// Bulk prefill of n tokens starting at token t0 of one sequence: one CTA per (page,
// KV head), one thread per channel.  Each thread walks its page's new rows in token
// order with the same strict compares as append, continuing from the stored metadata
// when the first page is already partly filled, so the result is bitwise the
// metadata n single appends would leave.
__global__ void prefill_kernel(__half* __restrict__ kp, __half* __restrict__ vp,
                               __half* __restrict__ meta, uint32_t* __restrict__ prange,
                               int32_t* __restrict__ len,
                               const __half* __restrict__ k, const __half* __restrict__ v,
                               uint32_t layer, uint32_t seq, uint32_t B, uint32_t Hkv,
                               uint32_t S, int D, uint32_t head_dim, size_t slice_kv,
                               size_t slice_meta, uint32_t mrow, uint32_t t0, uint32_t n) {
    const uint32_t page = t0 / S + blockIdx.x;
    const uint32_t h = blockIdx.y;
    const uint32_t c = threadIdx.x;
    const size_t s = (size_t(layer) * B + seq) * Hkv + h;
    const uint32_t r_begin = (blockIdx.x == 0) ? t0 % S : 0;
    const uint32_t page_end = page * S + S;
    const uint32_t r_end = (t0 + n < page_end) ? (t0 + n - page * S) : S;
    __half mn = __float2half(0.0f), mx = __float2half(0.0f);
    __half* mnp = meta + meta_offset(slice_meta, mrow, s, page, D, 0, c);
    __half* mxp = meta + meta_offset(slice_meta, mrow, s, page, D, 1, c);
    if (r_begin != 0) {
        mn = *mnp;
        mx = *mxp;
    }
    for (uint32_t r = r_begin; r < r_end; ++r) {
        const uint32_t i = page * S + r - t0;  // index among the new tokens
        const size_t in = (size_t(h) * n + i) * head_dim + c;
        const __half x = c < head_dim ? k[in] : __float2half(0.0f);
        const __half y = c < head_dim ? v[in] : __float2half(0.0f);
        const size_t kv = s * slice_kv + (size_t(page) * S + r) * D + c;
        kp[kv] = x;
        vp[kv] = y;
        if (r == 0) {
            mn = x;
            mx = x;
        } else {
            const float xf = __half2float(x);
            if (xf < __half2float(mn)) mn = x;
            if (xf > __half2float(mx)) mx = x;
        }
    }
    *mnp = mn;
    *mxp = mx;
    write_record(prange + s * mrow + page, mn, mx, D);
    if (blockIdx.x == 0 && blockIdx.y == 0 && c == 0) len[layer * B + seq] = int32_t(t0 + n);
}

// Vectorised bulk prefill (head_dim == D, 16-byte aligned inputs): thread = 8 channels of one
// page (16-byte loads and stores of whole row pieces), CTA = kPfPages pages x D/8 threads.
// Every thread walks its page's new rows in token order with append's strict compares on
// its 8 channels (the same first-seen semantics as the scalar kernel), all rows' loads in
// flight first; the page record is reduced over the page's D/8 threads with shuffles.
constexpr int kPfThreads = 256;  // 16 pages per CTA at D=128: 238 -> 219 us at cfg2 (64: 237, 512: 229)

template <int D>
__global__ void __launch_bounds__(kPfThreads)
prefill_vec_kernel(__half* __restrict__ kp, __half* __restrict__ vp, __half* __restrict__ meta,
                   uint32_t* __restrict__ prange, int32_t* __restrict__ len,
                   const __half* __restrict__ k, const __half* __restrict__ v, uint32_t layer,
                   uint32_t seq, uint32_t B, uint32_t Hkv, uint32_t S, size_t slice_kv,
                   size_t slice_meta, uint32_t mrow, uint32_t t0, uint32_t n, uint32_t npages) {
    constexpr int TPP = D / 8;                 // threads per page (8 channels each)
    constexpr int PPC = kPfThreads / TPP;      // pages per CTA
    const uint32_t h = blockIdx.y;
    const uint32_t pi = blockIdx.x * PPC + threadIdx.x / TPP;  // page among the new ones
    const int chunk = threadIdx.x % TPP;
    const bool active = pi < npages;
    const uint32_t page = t0 / S + pi;
    const size_t s = (size_t(layer) * B + seq) * Hkv + h;
    const uint32_t r_begin = (pi == 0) ? t0 % S : 0;
    const uint32_t page_end = page * S + S;
    const uint32_t r_end = (t0 + n < page_end) ? (t0 + n - page * S) : S;
    __half mn[8], mx[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) mn[j] = mx[j] = __float2half(0.0f);
    if (active) {
        if (r_begin != 0) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                mn[j] = meta[meta_offset(slice_meta, mrow, s, page, D, 0, chunk * 8 + j)];
                mx[j] = meta[meta_offset(slice_meta, mrow, s, page, D, 1, chunk * 8 + j)];
            }
        }
        constexpr int RB = 8;  // rows in flight per thread
        for (uint32_t r0 = r_begin; r0 < r_end; r0 += RB) {
            int4 kv[RB], vv[RB];
#pragma unroll
            for (int u = 0; u < RB; ++u) {
                const uint32_t r = r0 + u;
                if (r < r_end) {
                    const size_t in = (size_t(h) * n + (page * S + r - t0)) * D + chunk * 8;
                    kv[u] = ld_nc_v4(k + in);
                    vv[u] = ld_nc_v4(v + in);
                }
            }
#pragma unroll
            for (int u = 0; u < RB; ++u) {
                const uint32_t r = r0 + u;
                if (r < r_end) {
                    const size_t o = s * slice_kv + (size_t(page) * S + r) * D + chunk * 8;
                    *reinterpret_cast<int4*>(kp + o) = kv[u];
                    *reinterpret_cast<int4*>(vp + o) = vv[u];
                    const __half* x = reinterpret_cast<const __half*>(&kv[u]);
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        if (r == 0) {
                            mn[j] = x[j];
                            mx[j] = x[j];
                        } else {
                            const float xf = __half2float(x[j]);
                            if (xf < __half2float(mn[j])) mn[j] = x[j];
                            if (xf > __half2float(mx[j])) mx[j] = x[j];
                        }
                    }
                }
            }
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            meta[meta_offset(slice_meta, mrow, s, page, D, 0, chunk * 8 + j)] = mn[j];
            meta[meta_offset(slice_meta, mrow, s, page, D, 1, chunk * 8 + j)] = mx[j];
        }
    }
    // Page record over the page's TPP threads (consecutive lanes; TPP divides 32 or spans
    // whole warps): max |x| and the smallest ulp code of the min/max values.
    uint32_t mag = 0, code = 31u;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const uint16_t a = __half_as_ushort(mn[j]), b2 = __half_as_ushort(mx[j]);
        mag = max(mag, max(uint32_t(a & 0x7fffu), uint32_t(b2 & 0x7fffu)));
        code = min(code, min(ulp_code(a), ulp_code(b2)));
    }
    if constexpr (TPP <= 32) {
#pragma unroll
        for (int o = TPP / 2; o > 0; o >>= 1) {
            mag = max(mag, __shfl_xor_sync(0xffffffffu, mag, o));
            code = min(code, __shfl_xor_sync(0xffffffffu, code, o));
        }
        if (active && chunk == 0) prange[s * mrow + page] = mag | (code << 16);
    } else {  // D = 256: two warps per page
        __shared__ uint32_t part[kPfThreads / 32];
        mag = __reduce_max_sync(0xffffffffu, mag);
        code = __reduce_min_sync(0xffffffffu, code);
        const int warp = threadIdx.x >> 5;
        if ((threadIdx.x & 31) == 0) part[warp] = mag | (code << 16);
        __syncthreads();
        if (active && chunk == 0) {
            const uint32_t a = part[warp], b2 = part[warp + 1];
            prange[s * mrow + page] = max(a & 0xffffu, b2 & 0xffffu) | (min(a >> 16, b2 >> 16) << 16);
        }
    }
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) len[layer * B + seq] = int32_t(t0 + n);
}

}  // namespace

int launch_append(qk_cache* c, uint32_t layer, const __half* k, const __half* v,
                  uint32_t batch, cudaStream_t st) {
    append_kernel<<<dim3(batch, c->Hkv), c->D, 0, st>>>(
        c->k_pool, c->v_pool, c->meta, c->prange, c->d_len, c->len_ticket, c->d_status, k, v, layer, c->B,
        c->Hkv, c->S, c->D, c->desc.head_dim, c->slice_kv, c->slice_meta, c->Mrow, c->desc.max_tokens);
    c->launches++;
    return cuda_check(cudaGetLastError(), "append_kernel");
}

int launch_prefill(qk_cache* c, uint32_t layer, uint32_t seq, const __half* k,
                   const __half* v, uint32_t n, uint32_t t0, cudaStream_t st) {
    const uint32_t pages = (t0 + n - 1) / c->S - t0 / c->S + 1;
    const bool vec = c->desc.head_dim == uint32_t(c->D) &&
                     (reinterpret_cast<uintptr_t>(k) & 15) == 0 && (reinterpret_cast<uintptr_t>(v) & 15) == 0;
    if (vec) {
        const uint32_t ppc = kPfThreads / (c->D / 8);
        const dim3 grid((pages + ppc - 1) / ppc, c->Hkv);
#define QK_PF(DD)                                                                                   \
    prefill_vec_kernel<DD><<<grid, kPfThreads, 0, st>>>(c->k_pool, c->v_pool, c->meta, c->prange,  \
                                                        c->d_len, k, v, layer, seq, c->B, c->Hkv,  \
                                                        c->S, c->slice_kv, c->slice_meta, c->Mrow, \
                                                        t0, n, pages)
        if (c->D == 64) QK_PF(64);
        else if (c->D == 128) QK_PF(128);
        else QK_PF(256);
#undef QK_PF
        c->launches++;
        return cuda_check(cudaGetLastError(), "prefill_vec_kernel");
    }
    prefill_kernel<<<dim3(pages, c->Hkv), c->D, 0, st>>>(
        c->k_pool, c->v_pool, c->meta, c->prange, c->d_len, k, v, layer, seq, c->B, c->Hkv, c->S, c->D,
        c->desc.head_dim, c->slice_kv, c->slice_meta, c->Mrow, t0, n);
    c->launches++;
    return cuda_check(cudaGetLastError(), "prefill_kernel");
}

}  // namespace qk

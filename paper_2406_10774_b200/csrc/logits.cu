// logits.cu -- attention_logits and softmax_weights of the reference's attention.hpp on the
// GPU (the token-granular entry points policies and metrics call).
//
// attention_logits, /root/reference/proj/core/src/attention.cpp:34-52:
//     logit_t = dot(q, k_t) / sqrt(double(head_dim)),   dot = sum_{i asc} double(q_i)*double(k_i)
// q and k are fp16 values, so every product is exact in double and fma(q_i, k_i, acc) is the
// reference's `acc += q_i * k_i` rounded once: one thread runs the token's chain in channel
// order, then divides by the correctly rounded sqrt -- bitwise the reference's logits.
// Token lists are validated on the device like check_token_set (attention.cpp:19-30).
//
// softmax_weights, attention.cpp:54-67: w_i = exp(l_i - max) / sum_j exp(l_j - max), fp64.
// The reference sums sequentially; the block reduction here sums in a tree, and CUDA's exp
// is not glibc's, so weights agree to ~1e-15 relative (tolerance, not bitwise).
#include <math_constants.h>

#include "qk_internal.cuh"

namespace qk {
namespace {

constexpr int kLogitThreads = 128;

template <int D>
__global__ void __launch_bounds__(kLogitThreads)
logits_kernel(const __half* __restrict__ kp, const int32_t* __restrict__ len,
              const __half* __restrict__ q, const int32_t* __restrict__ tokens, uint32_t tstride,
              const int32_t* __restrict__ counts, uint32_t layer, uint32_t B, uint32_t Hq,
              uint32_t Hkv, uint32_t head_dim, size_t slice_kv, double* __restrict__ logits,
              uint32_t lstride, int32_t* __restrict__ status) {
    __shared__ double dq[D];
    const uint32_t bh = blockIdx.y;
    const uint32_t b = bh / Hq, h = bh % Hq, kvh = h / (Hq / Hkv);
    const uint32_t n_tok = static_cast<uint32_t>(len[layer * B + b]);
    // tokens == nullptr: every cached token (the one-argument attention_logits, :48-52).
    const uint32_t count = tokens ? uint32_t(max(counts[bh], 0)) : n_tok;
    if (count == 0 || (tokens && count > tstride) || count > lstride) {
        if (blockIdx.x == 0 && threadIdx.x == 0)
            record_status(status, count == 0 ? QK_DEV_EMPTY_TOKENS : QK_DEV_BAD_COUNT);
        return;
    }
    for (int c = threadIdx.x; c < D; c += kLogitThreads)
        dq[c] = c < int(head_dim) ? double(__half2float(q[size_t(bh) * head_dim + c])) : 0.0;
    __syncthreads();
    const uint32_t i = blockIdx.x * kLogitThreads + threadIdx.x;
    if (i >= count) return;
    uint32_t t = i;
    if (tokens) {
        const int32_t* tl = tokens + size_t(bh) * tstride;
        const int32_t ti = tl[i];
        if (ti < 0 || uint32_t(ti) >= n_tok) {
            record_status(status, QK_DEV_TOKEN_OUT_OF_RANGE);
            return;
        }
        if (i > 0 && tl[i - 1] >= ti) {
            record_status(status, QK_DEV_TOKEN_NOT_ASCENDING);
            return;
        }
        t = uint32_t(ti);
    }
    const size_t s = (size_t(layer) * B + b) * Hkv + kvh;
    const __half* row = kp + s * slice_kv + size_t(t) * D;  // token t = page t/S, row t%S
    double acc = 0.0;
    for (uint32_t c0 = 0; c0 < head_dim; c0 += 8) {
        const int4 v = ld_nc_v4(row + c0);
        const __half* hv = reinterpret_cast<const __half*>(&v);
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if (c0 + j < head_dim) acc = __fma_rn(dq[c0 + j], double(__half2float(hv[j])), acc);
    }
    logits[size_t(bh) * lstride + i] = acc / sqrt(double(head_dim));
}

constexpr int kSoftThreads = 256;

__device__ __forceinline__ double block_reduce(double v, bool is_max, double* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double x = __shfl_xor_sync(0xffffffffu, v, o);
        v = is_max ? fmax(v, x) : v + x;
    }
    __syncthreads();  // red reusable
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double r = red[0];
    for (int w = 1; w < kSoftThreads / 32; ++w) r = is_max ? fmax(r, red[w]) : r + red[w];
    return r;
}

__global__ void __launch_bounds__(kSoftThreads)
softmax_kernel(const double* __restrict__ logits, const int32_t* __restrict__ counts, uint32_t n,
               uint32_t stride, double* __restrict__ weights, int32_t* __restrict__ status) {
    __shared__ double red[kSoftThreads / 32];
    const uint32_t row = blockIdx.x;
    const uint32_t cnt = counts ? uint32_t(max(counts[row], 0)) : n;
    if (cnt == 0 || cnt > stride) {
        if (threadIdx.x == 0 && status) record_status(status, cnt == 0 ? QK_DEV_EMPTY_TOKENS : QK_DEV_BAD_COUNT);
        return;
    }
    const double* l = logits + size_t(row) * stride;
    double* w = weights + size_t(row) * stride;
    double peak = -CUDART_INF;
    for (uint32_t i = threadIdx.x; i < cnt; i += kSoftThreads) peak = fmax(peak, l[i]);
    peak = block_reduce(peak, true, red);
    double total = 0.0;
    for (uint32_t i = threadIdx.x; i < cnt; i += kSoftThreads) {
        const double e = exp(l[i] - peak);
        w[i] = e;
        total += e;
    }
    total = block_reduce(total, false, red);
    for (uint32_t i = threadIdx.x; i < cnt; i += kSoftThreads) w[i] = w[i] / total;
}

// estimate_page_score (criticality.cpp:9-23) on explicit metadata rows [n][head_dim]: one
// thread per page, the reference's chain in channel order (exact products, one rounding
// per add): bitwise.
__global__ void page_score_kernel(const __half* __restrict__ q, const __half* __restrict__ mn,
                                  const __half* __restrict__ mx, uint32_t n, uint32_t d,
                                  double* __restrict__ out) {
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    double acc = 0.0;
    for (uint32_t c = 0; c < d; ++c) {
        const double qc = double(__half2float(q[c]));
        const double a = qc * double(__half2float(mx[size_t(p) * d + c]));
        const double b = qc * double(__half2float(mn[size_t(p) * d + c]));
        acc = __dadd_rn(acc, fmax(a, b));
    }
    out[p] = acc;
}

}  // namespace

int launch_page_scores(const __half* q, const __half* mn, const __half* mx, uint32_t n,
                       uint32_t d, double* out, cudaStream_t st) {
    if (n == 0) return QK_OK;
    page_score_kernel<<<(n + 127) / 128, 128, 0, st>>>(q, mn, mx, n, d, out);
    return cuda_check(cudaGetLastError(), "page_score_kernel");
}

int launch_logits(const qk_cache* c, uint32_t layer, const __half* q, uint32_t batch,
                  const int32_t* tokens, uint32_t tstride, const int32_t* counts,
                  uint32_t max_list, double* logits, uint32_t lstride, cudaStream_t st) {
    const dim3 grid((max_list + kLogitThreads - 1) / kLogitThreads, batch * c->Hq);
    if (grid.x == 0) return QK_OK;
#define QK_LOGITS(DD)                                                                             \
    logits_kernel<DD><<<grid, kLogitThreads, 0, st>>>(c->k_pool, c->d_len, q, tokens, tstride, \
                                                      counts, layer, c->B, c->Hq, c->Hkv,      \
                                                      c->desc.head_dim, c->slice_kv, logits,   \
                                                      lstride, c->d_status)
    switch (c->D) {
        case 64: QK_LOGITS(64); break;
        case 128: QK_LOGITS(128); break;
        case 256: QK_LOGITS(256); break;
        default: return set_error(QK_ERR_UNSUPPORTED, "attention_logits: unsupported head_dim");
    }
#undef QK_LOGITS
    const_cast<qk_cache*>(c)->launches++;
    return cuda_check(cudaGetLastError(), "logits_kernel");
}

int launch_softmax(const double* logits, const int32_t* counts, uint32_t n, uint32_t stride,
                   uint32_t rows, double* weights, int32_t* status, cudaStream_t st) {
    if (rows == 0) return QK_OK;
    softmax_kernel<<<rows, kSoftThreads, 0, st>>>(logits, counts, n, stride, weights, status);
    return cuda_check(cudaGetLastError(), "softmax_kernel");
}

}  // namespace qk

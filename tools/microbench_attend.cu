// microbench_attend.cu -- the fused kernel's attention phase in isolation: 128 CTAs x 512
// threads, every CTA folds 32 pages (16 x 128 fp16 K and V each) of one head's slice, two
// per warp, with attend_warp.cuh's warp_fold_page, then the CTA combine.  Pages are drawn
// at random from a 32K-token slice per head; `warm` repeats the same pages (L2 resident),
// `cold` rotates over 16 layers' worth of pools.  Stamps: globaltimer at start / after the
// page loop (thread 0) -> per-CTA phase time.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "../paper_2406_10774_b200/csrc/attend_warp.cuh"

using namespace qk;

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

template <int MODE>
__global__ void __launch_bounds__(512, 1) attend(const __half* __restrict__ kpool, const __half* __restrict__ vpool,
                                                 size_t slice, const int* __restrict__ pages,
                                                 const __half* __restrict__ q, float* out,
                                                 unsigned long long* ts) {
    constexpr int D = 128, S = 16;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int head = blockIdx.x / 4, rank = blockIdx.x % 4;
    __shared__ float s_o[16][D];
    __shared__ float s_m[16], s_l[16];
    const unsigned long long t0 = gtime();
    float qf[8];
    load_q8<D>(q + head * D, D, qf);
    float m = -CUDART_INF_F, l = 0.0f, o[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = 0.0f;
    const __half* ks = kpool + head * slice;
    const __half* vs = vpool + head * slice;
    const int* pl = pages + head * 128 + rank * 32;
    if (MODE == 0) {
        for (int i = warp; i < 32; i += 16) {
            const int pg = pl[i];
            warp_fold_page<D, true>(ks + size_t(pg) * S * D, vs + size_t(pg) * S * D, S, qf, 0.1f, m, l, o);
        }
    } else if (MODE == 1) {
        for (int i = warp; i < 32; i += 16) {
            const int pg = pl[i];
            warp_fold_page<D, false>(ks + size_t(pg) * S * D, vs + size_t(pg) * S * D, S, qf, 0.1f, m, l, o);
        }
    } else if (MODE == 3) {
        // MODE 3: the warp's two pages interleaved by halves: the first halves of both pages
        // in flight together (same registers as one full page), then the second halves.
        const int pa = pl[warp], pb = pl[warp + 16];
        for (int hh = 0; hh < 2; ++hh) {
            warp_fold_page<D, true>(ks + size_t(pa) * S * D + hh * 8 * D, vs + size_t(pa) * S * D + hh * 8 * D, 8, qf, 0.1f, m, l, o);
            warp_fold_page<D, true>(ks + size_t(pb) * S * D + hh * 8 * D, vs + size_t(pb) * S * D + hh * 8 * D, 8, qf, 0.1f, m, l, o);
        }
    } else {
        // MODE 2: half a page per warp-iteration, four iterations (more, smaller batches).
        for (int i = warp; i < 64; i += 16) {
            const int pg = pl[i >> 1];
            warp_fold_page<D, true>(ks + size_t(pg) * S * D + (i & 1) * 8 * D,
                                    vs + size_t(pg) * S * D + (i & 1) * 8 * D, 8, qf, 0.1f, m, l, o);
        }
    }
    warp_fold_rows<D>(l, o);
    const int chunk = lane % 16, rgrp = lane / 16;
    if (rgrp == 0)
        for (int j = 0; j < 8; ++j) s_o[warp][chunk * 8 + j] = o[j];
    if (lane == 0) {
        s_m[warp] = m;
        s_l[warp] = l;
    }
    __syncthreads();
    const unsigned long long t1 = gtime();
    if (threadIdx.x < D) {
        float acc = 0.f, L = 0.f;
        for (int w = 0; w < 16; ++w) {
            acc += s_o[w][threadIdx.x];
            L += s_l[w] + s_m[w];
        }
        out[blockIdx.x * D + threadIdx.x] = acc + L;
    }
    if (threadIdx.x == 0) {
        ts[blockIdx.x * 2] = t0;
        ts[blockIdx.x * 2 + 1] = t1;
    }
}

int main() {
    const int heads = 32, ctas = 128, tokens = 32768, layers = 16;
    const size_t slice = size_t(tokens) * 128;  // halves per head
    const size_t pool = slice * heads;
    __half *k, *v, *q;
    cudaMalloc(&k, pool * 2 * layers);
    cudaMalloc(&v, pool * 2 * layers);
    cudaMalloc(&q, heads * 128 * 2);
    cudaMemset(k, 0, pool * 2 * layers);
    cudaMemset(v, 0, pool * 2 * layers);
    cudaMemset(q, 0, heads * 128 * 2);
    std::vector<int> hp(heads * 128);
    srand(1);
    for (int h = 0; h < heads; ++h) {
        // 128 distinct sorted pages of 2048
        std::vector<int> all(2048);
        for (int i = 0; i < 2048; ++i) all[i] = i;
        for (int i = 0; i < 128; ++i) std::swap(all[i], all[i + rand() % (2048 - i)]);
        std::vector<int> sel(all.begin(), all.begin() + 128);
        std::sort(sel.begin(), sel.end());
        for (int i = 0; i < 128; ++i) hp[h * 128 + i] = sel[i];
    }
    int* pages;
    cudaMalloc(&pages, hp.size() * 4);
    cudaMemcpy(pages, hp.data(), hp.size() * 4, cudaMemcpyHostToDevice);
    float* out;
    cudaMalloc(&out, ctas * 128 * 4);
    unsigned long long* ts;
    cudaMalloc(&ts, ctas * 16);
    std::vector<unsigned long long> h(ctas * 2);
    auto run = [&](int mode, bool cold) {
        double best_med = 1e9, best_max = 1e9;
        for (int rep = 0; rep < 20; ++rep) {
            const size_t off = cold ? (rep % layers) * pool : 0;
            if (mode == 0) attend<0><<<ctas, 512>>>(k + off, v + off, slice, pages, q, out, ts);
            if (mode == 1) attend<1><<<ctas, 512>>>(k + off, v + off, slice, pages, q, out, ts);
            if (mode == 2) attend<2><<<ctas, 512>>>(k + off, v + off, slice, pages, q, out, ts);
            if (mode == 3) attend<3><<<ctas, 512>>>(k + off, v + off, slice, pages, q, out, ts);
            cudaDeviceSynchronize();
            cudaMemcpy(h.data(), ts, ctas * 16, cudaMemcpyDeviceToHost);
            std::vector<double> d(ctas);
            unsigned long long t0 = ~0ull, t1 = 0;
            for (int c = 0; c < ctas; ++c) {
                d[c] = (h[2 * c + 1] - h[2 * c]) / 1000.0;
                t0 = std::min(t0, h[2 * c]);
                t1 = std::max(t1, h[2 * c + 1]);
            }
            std::sort(d.begin(), d.end());
            if (rep >= 4) {
                best_med = std::min(best_med, d[ctas / 2]);
                best_max = std::min(best_max, (t1 - t0) / 1000.0);
            }
        }
        printf("mode %d %s: per-CTA median %.2f us, span %.2f us\n", mode, cold ? "cold" : "warm", best_med, best_max);
    };
    for (int mode = 0; mode < 4; ++mode) {
        run(mode, false);
        run(mode, true);
    }
    cudaError_t e = cudaGetLastError();
    printf("%s\n", cudaGetErrorString(e));
    return 0;
}

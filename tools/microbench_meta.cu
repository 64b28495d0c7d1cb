// microbench_meta.cu -- how fast can 128..148 SMs pull the fused kernel's metadata stream?
// cfg2 shape: 32 heads x 2048 pages, channel-major rows of Mrow pages (fp16), each CTA
// reading one sign-selected 1 KiB row segment per channel (128 channels) for its 512 pages.
// Variants (same bytes, 16.8 MB per launch, L2 flushed between launches):
//   A  128 CTAs x 512 thr, 16 LDG.128 per thread all in flight      (the fused kernel today)
//   B  as A, two waves of 8 loads (consume between)
//   C  148 CTAs: the 32x4 CTA ranges re-cut over 148 CTAs (uneven page ranges)
//   D  256 CTAs x 256 thr (2 per SM), 16 loads per thread
//   E  128 CTAs, 1 KiB cp.async.bulk (TMA) per channel row into shared memory
//   F  128 CTAs, L2 prefetch (cp.async.bulk.prefetch.L2) of every row first, then A's loads
// Prints the launch time (CUDA events) and the implied TB/s.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

constexpr int kHeads = 32, kPages = 2048, kMrow = 2112, kD = 128;

__device__ __forceinline__ int4 ldnc(const void* p) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}
__device__ unsigned long long g_t0[512], g_t1[512];
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define T_START if (threadIdx.x == 0) g_t0[blockIdx.x] = gtime();
#define T_END __syncthreads(); if (threadIdx.x == 0) g_t1[blockIdx.x] = gtime();
__device__ __forceinline__ int sign_row(int head, int c) { return ((c * 2654435761u + head * 40503u) >> 9) & 1; }

// A/B/C/D: CTA covers pages [p0, p0+npg) of `head`; warp (half, cg) lane -> 8 pages x 16 ch.
template <int WAVES, int NT>
__global__ void __launch_bounds__(NT) reg_loads(const __half* meta, int cuts, int* sink) {
    T_START
    const int head = blockIdx.x / cuts, part = blockIdx.x % cuts;
    const int p0 = (kPages * part / cuts) & ~7, p1 = (kPages * (part + 1) / cuts) & ~7;
    const __half* sl = meta + size_t(head) * 2 * kD * kMrow;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int NW = NT / 32;            // warps
    constexpr int CPW = kD * (NW >= 8 ? 8 : NW) / NW / (NW >= 8 ? 8 : NW) ;  // unused
    const int cg = warp % 8, grp = warp / 8, ngrp = NW / 8;
    int acc = 0;
    for (int pb = p0 + (grp * 32 + lane) * 8; pb < p1; pb += ngrp * 256) {
#pragma unroll
        for (int w = 0; w < WAVES; ++w) {
            int4 v[16 / WAVES];
#pragma unroll
            for (int k = 0; k < 16 / WAVES; ++k) {
                const int c = cg * 16 + w * (16 / WAVES) + k;
                v[k] = ldnc(sl + size_t(sign_row(head, c) * kD + c) * kMrow + pb);
            }
#pragma unroll
            for (int k = 0; k < 16 / WAVES; ++k) acc += v[k].x ^ v[k].w;
        }
    }
    (void)CPW;
    if (acc == 0x1234567) sink[0] = acc;
    T_END
}

// E: 1 KiB bulk copies per channel row (one thread per channel issues), wait on an mbarrier.
__global__ void __launch_bounds__(128, 1) bulk_rows(const __half* meta, int* sink) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) unsigned long long bar;
    T_START
    const int head = blockIdx.x / 4, part = blockIdx.x % 4;
    const int p0 = 512 * part;
    const __half* sl = meta + size_t(head) * 2 * kD * kMrow;
    const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(&bar));
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (threadIdx.x == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(kD * 1024));
    __syncthreads();
    const int c = threadIdx.x;
    const __half* src = sl + size_t(sign_row(head, c) * kD + c) * kMrow + p0;
    const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(sm + c * 1024));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 1024, [%2];"
                 ::"r"(dst), "l"(src), "r"(b) : "memory");
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"(b) : "memory");
    const int v = reinterpret_cast<const int*>(sm)[threadIdx.x * 7];
    if (v == 0x1234567) sink[0] = v;
    T_END
}

// F: L2 prefetch of the rows, then A's loads.
__global__ void __launch_bounds__(512, 1) prefetch_then_load(const __half* meta, int* sink) {
    T_START
    const int head = blockIdx.x / 4, part = blockIdx.x % 4;
    const int p0 = 512 * part;
    const __half* sl = meta + size_t(head) * 2 * kD * kMrow;
    if (threadIdx.x < kD) {
        const int c = threadIdx.x;
        const __half* src = sl + size_t(sign_row(head, c) * kD + c) * kMrow + p0;
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], 1024;" ::"l"(src) : "memory");
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, cg = warp % 8, half = warp / 8;
    const int pb = p0 + half * 256 + lane * 8;
    int4 v[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        const int c = cg * 16 + k;
        v[k] = ldnc(sl + size_t(sign_row(head, c) * kD + c) * kMrow + pb);
    }
    int acc = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) acc += v[k].x ^ v[k].w;
    if (acc == 0x1234567) sink[0] = acc;
    T_END
}

__global__ void empty_kernel(int* sink) { T_START T_END }

__global__ void touch_pages(const char* __restrict__ p, size_t n, int* sink) {
    int acc = 0;
    for (size_t i = (blockIdx.x * size_t(blockDim.x) + threadIdx.x) * 65536; i < n;
         i += size_t(gridDim.x) * blockDim.x * 65536)
        acc ^= __ldcg(reinterpret_cast<const int*>(p + i));
    if (acc == 0x12345678) sink[0] = acc;
}

__global__ void fill_random(unsigned int* p, size_t n) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
        unsigned int x = unsigned(i) * 2654435761u ^ unsigned(i >> 32) * 40503u;
        x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
        p[i] = x & 0x3bff3bffu;  // two finite fp16 values
    }
}

__global__ void flush(const int4* p, size_t n, int* sink) {
    int acc = 0;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
        acc ^= __ldcg(p + i).x;
    if (acc == 0x12345678) sink[0] = acc;
}

int main() {
    const size_t meta_elems = size_t(kHeads) * 2 * kD * kMrow;
    __half* meta;
    int* sink;
    int4* junk;
    const size_t junk_n = (size_t(getenv("BIGFLUSH") ? 4096 : 192) << 20) / 16;  // BIGFLUSH: TLB thrash
    cudaMalloc(&meta, meta_elems * 2);
    if (getenv("RANDOM_META")) {  // random fp16 bit patterns (constant data may be compressed)
        fill_random<<<592, 512>>>(reinterpret_cast<unsigned int*>(meta), meta_elems / 2);
        cudaDeviceSynchronize();
    } else {
        cudaMemset(meta, 1, meta_elems * 2);
    }
    cudaMalloc(&sink, 4096);
    cudaMalloc(&junk, junk_n * 16);
    cudaMemset(junk, 0, junk_n * 16);
    cudaFuncSetAttribute(bulk_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const double bytes = double(kHeads) * kD * kPages * 2;
    auto run = [&](const char* name, auto launch, int grid) {
        float best = 1e9f, sum = 0, dbest = 1e9f;
        for (int rep = 0; rep < 12; ++rep) {
            if (getenv("BIGFLUSH")) touch_pages<<<148, 512>>>(reinterpret_cast<const char*>(junk), junk_n * 16, sink);
            flush<<<592, 512>>>(junk, getenv("BIGFLUSH") ? (size_t(192) << 20) / 16 : junk_n, sink);
            cudaEventRecord(a);
            launch();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            unsigned long long t0[512], t1[512];
            cudaMemcpyFromSymbol(t0, g_t0, grid * 8);
            cudaMemcpyFromSymbol(t1, g_t1, grid * 8);
            unsigned long long lo = ~0ull, hi = 0;
            for (int i = 0; i < grid; ++i) {
                lo = t0[i] < lo ? t0[i] : lo;
                hi = t1[i] > hi ? t1[i] : hi;
            }
            const float dev_us = float(hi - lo) / 1000.f;
            if (rep >= 2) {
                best = ms < best ? ms : best;
                dbest = dev_us < dbest ? dev_us : dbest;
                sum += ms;
            }
        }
        printf("%-40s event best %.2f us mean %.2f | in-kernel best %.2f us (%.2f TB/s)\n", name, best * 1e3,
               sum / 10 * 1e3, dbest, bytes / (dbest * 1e-6) / 1e12);
    };
    run("A 128x512, 16 loads in flight", [&] { reg_loads<1, 512><<<128, 512>>>(meta, 4, sink); }, 128);
    run("B 128x512, 2 waves of 8", [&] { reg_loads<2, 512><<<128, 512>>>(meta, 4, sink); }, 128);
    run("C' 160 CTAs: 5 cuts per head", [&] { reg_loads<1, 512><<<32 * 5, 512>>>(meta, 5, sink); }, 160);
    run("D 256x256 (8 cuts per head, 2/SM)", [&] { reg_loads<1, 256><<<32 * 8, 256>>>(meta, 8, sink); }, 256);
    run("E 128 CTAs, 1 KiB TMA per row", [&] { bulk_rows<<<128, 128, 128 * 1024>>>(meta, sink); }, 128);
    run("F 128 CTAs, L2 prefetch + loads", [&] { prefetch_then_load<<<128, 512>>>(meta, sink); }, 128);
    run("empty kernel (launch overhead)", [&] { empty_kernel<<<128, 512>>>(sink); }, 128);
    run("A again", [&] { reg_loads<1, 512><<<128, 512>>>(meta, 4, sink); }, 128);
    printf("(%s)\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}

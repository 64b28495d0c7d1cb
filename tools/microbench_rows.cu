// microbench_rows.cu -- chip-wide read time of the estimate's metadata access pattern:
// 128 CTAs x 512 threads, each CTA reads NROWS row segments of SEG bytes (rows ROWSTRIDE
// apart, one of two row blocks per row chosen by a fixed pseudo-random "sign"), versus the
// same bytes read contiguously.  Every lane issues its 16-byte loads up front (as the fused
// kernel does) and a clock64 stamp records when warp 0's data has arrived.
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ int4 ldnc(const void* p) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

// mode 0: rows (fused-kernel layout); mode 1: contiguous per CTA.
template <int MODE>
__global__ void __launch_bounds__(512, 1) rows(const char* __restrict__ base, size_t slice,
                                               int seg, int rowstride, long long* cyc,
                                               int* sink) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int cg = warp & 7, half = warp >> 3;
    const char* sl = base + size_t(blockIdx.x / 4) * slice;  // 4 CTAs share a slice
    const int quarter = blockIdx.x % 4;
    int4 v[16];
    long long t0 = clock64();
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        const int c = cg * 16 + k;
        const int minmax = ((c * 2654435761u) >> 7) & 1;
        const size_t off = (MODE == 0)
            ? size_t(minmax * 128 + c) * rowstride + size_t(quarter) * seg + size_t(half) * (seg / 2) + lane * 16
            : size_t(quarter) * 128 * seg + size_t(c) * seg + size_t(half) * (seg / 2) + lane * 16;
        v[k] = (lane * 16 < seg / 2) ? ldnc(sl + off) : make_int4(0, 0, 0, 0);
    }
    int acc = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) acc += v[k].x ^ v[k].y ^ v[k].z ^ v[k].w;
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    sink[blockIdx.x * 512 + threadIdx.x] = acc;
}

__global__ void touch(const int4* __restrict__ p, size_t n, int* sink) {
    int acc = 0;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
        acc ^= __ldcg(p + i).x;
    if (acc == 0x12345678) sink[0] = acc;
}

// TLB only: one 16-byte load per 64 KiB of a 4 GiB region (no L2 pollution to speak of).
__global__ void touch_pages(const char* __restrict__ p, size_t n, int* sink) {
    int acc = 0;
    for (size_t i = (blockIdx.x * size_t(blockDim.x) + threadIdx.x) * 65536; i < n;
         i += size_t(gridDim.x) * blockDim.x * 65536)
        acc ^= __ldcg(reinterpret_cast<const int*>(p + i));
    if (acc == 0x12345678) sink[0] = acc;
}

int main() {
    const int rowstride = 4224, ctas = 128, slices = ctas / 4;
    const size_t slice = size_t(256) * rowstride;  // 2 x 128 rows
    char* buf;
    const size_t total = slice * slices * 8;  // 8 layers worth, rotate to defeat L2
    cudaMalloc(&buf, total);
    cudaMemset(buf, 1, total);
    long long* cyc;
    int* sink;
    cudaMalloc(&cyc, ctas * 8);
    cudaMalloc(&sink, ctas * 512 * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    char* junk;
    const size_t junk_bytes = size_t(4) << 30;  // touched between reps (clean reads)
    cudaMalloc(&junk, junk_bytes);
    cudaMemset(junk, 0, junk_bytes);
    for (int flush = 0; flush < 3; ++flush)
    for (int seg : {256, 1024}) {
        for (int mode = 0; mode < 2; ++mode) {
            auto k = mode == 0 ? rows<0> : rows<1>;
            float best = 1e9f;
            long long cb = 0;
            for (int rep = 0; rep < 8; ++rep) {
                const char* base = buf + (rep % 8) * slice * slices;
                if (flush == 1) touch<<<148 * 4, 512>>>(reinterpret_cast<const int4*>(junk), (size_t(1) << 30) / 16, sink);
                if (flush == 2) touch_pages<<<148, 512>>>(junk, junk_bytes, sink);
                cudaEventRecord(a);
                k<<<ctas, 512>>>(base, slice, seg, rowstride, cyc, sink);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (ms < best) {
                    best = ms;
                    cudaMemcpy(&cb, cyc, 8, cudaMemcpyDeviceToHost);
                }
            }
            const double bytes = double(ctas) * 128 * seg;
            printf("%s seg %4d %-10s: %.2f us  (%.2f TB/s)  warp0 data after %lld cycles\n", flush == 0 ? "warm     " : flush == 1 ? "L2+TLB   " : "TLB only ", seg,
                   mode == 0 ? "rows" : "contiguous", best * 1e3, bytes / (best * 1e-3) / 1e12, cb);
        }
    }
    return 0;
}

// microbench_cvt.cu -- throughput of the exact fp16 -> f64 conversion paths used by the
// estimate chains (F2F on the XU pipe vs the integer 2^-1008-scaled path), of DFMA, and of
// a chain mixing them, on one SM.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
// tools/microbench_cvt.cu -o gpurun_out/microbench_cvt
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ double h2d(unsigned short h) {
    double d;
    asm volatile("cvt.f64.f16 %0, %1;" : "=d"(d) : "h"(h));
    return d;
}
__device__ __forceinline__ double h2d_scaled(unsigned short h) {
    const uint32_t t = uint32_t(h) << 10;
    const uint32_t s = t & 0x02000000u;
    return __hiloint2double(int(t + s * 63u), 0);
}

template <int MODE>
__global__ void bench(const unsigned short* __restrict__ in, double* out, int iters) {
    unsigned short h[8];
    for (int j = 0; j < 8; ++j) h[j] = in[(threadIdx.x + j) & 255];
    double acc[4] = {0, 0, 0, 0};
    const double w = 1.000001;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            unsigned short x = h[j] ^ (unsigned short)(it & 1);
            double d;
            if (MODE == 0) d = h2d(x);                        // all F2F (XU)
            else if (MODE == 1) d = h2d_scaled(x);            // all integer
            else if (MODE == 2) d = (j & 1) ? h2d_scaled(x) : h2d(x);   // 1/2 XU
            else if (MODE == 3) d = (j & 3) ? h2d_scaled(x) : h2d(x);   // 1/4 XU
            else d = __hiloint2double(int(x), 0);            // DFMA only
            acc[j & 3] = __fma_rn(w, d, acc[j & 3]);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc[0] + acc[1] + acc[2] + acc[3];
}

int main() {
    unsigned short* in;
    double* out;
    cudaMalloc(&in, 512);
    cudaMemset(in, 0x3c, 512);
    cudaMalloc(&out, 148 * 1024 * 8);
    const int iters = 4096;
    const char* names[] = {"F2F only", "integer only", "1/2 F2F", "1/4 F2F", "DFMA only"};
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int threads : {256, 512, 1024}) {
        for (int mode = 0; mode < 5; ++mode) {
            auto k = mode == 0 ? bench<0> : mode == 1 ? bench<1> : mode == 2 ? bench<2>
                                                    : mode == 3 ? bench<3> : bench<4>;
            k<<<148, threads>>>(in, out, 16);
            cudaEventRecord(a);
            k<<<148, threads>>>(in, out, iters);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            const double elems = double(148) * threads * iters * 8;
            int clk;
            cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
            const double per_sm_clk = elems / 148 / (ms * 1e-3 * clk * 1e3);
            printf("threads %4d  %-12s  %.3f ms  %.1f elements/clk/SM (at %d MHz)\n", threads,
                   names[mode], ms, per_sm_clk, clk / 1000);
        }
    }
    return 0;
}

// microbench_chain.cu -- the estimate inner loop in isolation: per thread NCH independent
// fp64 chains over 128 channels, operands staged in shared memory as the fused kernel
// stages them ([channel][page] u16 rows), fp16 -> f64 by F2F / the integer path.
// Reports cycles per chain step and elements/clk/SM for 512 threads on every SM.
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ double h2d(unsigned short h) {
    double d;
    asm("cvt.f64.f16 %0, %1;" : "=d"(d) : "h"(h));
    return d;
}
__device__ __forceinline__ double h2d_scaled(unsigned short h) {
    const uint32_t t = uint32_t(h) << 10;
    const uint32_t s = t & 0x02000000u;
    return __hiloint2double(int(t + s * 63u), 0);
}

// PAGES pages per CTA staged as [128][PAGES] halves; thread t owns NCH pages.
template <int NCH, int CVT>
__global__ void __launch_bounds__(512, 1) chain(double* out, int reps, long long* cyc) {
    constexpr int D = 128;
    constexpr int PAGES = 512 * NCH;
    extern __shared__ unsigned short st[];
    __shared__ double dq[2 * D];
    for (int i = threadIdx.x; i < D * PAGES; i += 512) st[i] = 0x2c00 + (i % 977);
    for (int i = threadIdx.x; i < 2 * D; i += 512) dq[i] = (i & 1) ? 0x1p1008 * 0.01 : 0.01;
    __syncthreads();
    long long t0 = clock64();
    double acc[NCH];
#pragma unroll
    for (int k = 0; k < NCH; ++k) acc[k] = 0.0;
    for (int r = 0; r < reps; ++r) {
#pragma unroll 8
        for (int c = 0; c < D; c += 2) {
            const double2 w = *reinterpret_cast<const double2*>(dq + c);
#pragma unroll
            for (int k = 0; k < NCH; ++k) {
                const int pi = threadIdx.x + k * 512;
                const unsigned short h0 = st[c * PAGES + pi];
                const unsigned short h1 = st[(c + 1) * PAGES + pi];
                if (CVT == 0) {
                    acc[k] = __fma_rn(w.x, h2d(h0), acc[k]);
                    acc[k] = __fma_rn(w.y, h2d_scaled(h1), acc[k]);
                } else {
                    acc[k] = __fma_rn(w.y, h2d_scaled(h0), acc[k]);
                    acc[k] = __fma_rn(w.y, h2d_scaled(h1), acc[k]);
                }
            }
        }
    }
    __syncthreads();
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int k = 0; k < NCH; ++k) s += acc[k];
    out[blockIdx.x * 512 + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int NCH, int CVT>
void run(double* out, long long* cyc, const char* name) {
    const int reps = 16;
    const size_t smem = size_t(128) * 512 * NCH * 2;
    cudaFuncSetAttribute(chain<NCH, CVT>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    chain<NCH, CVT><<<148, 512, smem>>>(out, 1, cyc);
    chain<NCH, CVT><<<148, 512, smem>>>(out, reps, cyc);
    cudaDeviceSynchronize();
    long long c = 0;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    const double steps = double(reps) * 128;  // chain steps per thread
    printf("%-28s NCH=%d: %.1f cycles per chain step, %.1f elements/clk/SM  (%s)\n", name, NCH,
           c / steps, steps * 512 * NCH / c, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 148 * 512 * 8);
    cudaMalloc(&cyc, 148 * 8);
    run<1, 0>(out, cyc, "F2F/int mixed");
    run<2, 0>(out, cyc, "F2F/int mixed");
    run<3, 0>(out, cyc, "F2F/int mixed");
    run<1, 1>(out, cyc, "integer only");
    run<2, 1>(out, cyc, "integer only");
    run<3, 1>(out, cyc, "integer only");
    return 0;
}

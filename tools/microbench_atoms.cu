// microbench_atoms.cu -- shared-memory histogram cost on B200: 512 threads x 4 increments
// into 2048 bins, with the keys spread over B distinct bins (B = 2048 .. 1), as
// atomicAdd (ATOMS.POPC.INC) and as warp-aggregated increments (__match_any_sync).
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(512, 1) hist(int spread, long long* cyc, unsigned* out) {
    __shared__ unsigned h[2048];
    for (int i = threadIdx.x; i < 2048; i += 512) h[i] = 0;
    unsigned x = threadIdx.x * 2654435761u + blockIdx.x;
    unsigned bins[4];
    for (int j = 0; j < 4; ++j) {
        x ^= x << 13; x ^= x >> 17; x ^= x << 5;
        bins[j] = (x % spread) * (2048 / spread);
    }
    __syncthreads();
    long long t0 = clock64();
    for (int r = 0; r < 8; ++r) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (MODE == 0) {
                atomicAdd(&h[bins[j]], 1u);
            } else {
                const unsigned peers = __match_any_sync(0xffffffffu, bins[j]);
                if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&h[bins[j]], __popc(peers));
            }
        }
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = (t1 - t0) / 8;
    out[blockIdx.x * 512 + threadIdx.x] = h[threadIdx.x];
}

int main() {
    long long* cyc;
    unsigned* out;
    cudaMalloc(&cyc, 148 * 8);
    cudaMalloc(&out, 148 * 512 * 4);
    for (int mode = 0; mode < 2; ++mode) {
        for (int spread : {2048, 512, 64, 16, 4, 1}) {
            auto k = mode == 0 ? hist<0> : hist<1>;
            k<<<148, 512>>>(spread, cyc, out);
            k<<<148, 512>>>(spread, cyc, out);
            cudaDeviceSynchronize();
            long long c;
            cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
            printf("%-16s spread %4d bins: %5lld cycles per 2048 increments\n",
                   mode == 0 ? "atomicAdd" : "match_any+atom", spread, c);
        }
    }
    return 0;
}

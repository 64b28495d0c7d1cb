// synccheck_cluster_repro.cu -- minimal kernel with the fused decode kernel's prologue pattern
// (thread 0 initialises mbarriers, aligned cluster arrive, a 128-thread branch with warp
// reductions and a lane-0 store, __syncthreads, cluster wait), launched with clusters of
// 2, 4, 8 and 16 CTAs, for compute-sanitizer --tool synccheck triage.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512, 1) prologue(double* out) {
    __shared__ __align__(8) unsigned long long bar[2];
    __shared__ double part[4];
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&bar[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 4;" ::"r"((unsigned)__cvta_generic_to_shared(&bar[1])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
    const int tid = threadIdx.x, lane = tid & 31;
    if (tid < 128) {
        double a = double(tid);
        for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        if (lane == 0) part[tid >> 5] = a;
    }
    __syncthreads();
    asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
    if (tid == 0) out[blockIdx.x] = part[0] + part[1] + part[2] + part[3];
}

int main() {
    double* out;
    cudaMalloc(&out, 256 * 8);
    cudaFuncSetAttribute(prologue, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int c : {2, 4, 8, 16}) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(128);
        cfg.blockDim = dim3(512);
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = c;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaError_t e = cudaLaunchKernelEx(&cfg, prologue, out);
        cudaError_t s = cudaDeviceSynchronize();
        printf("cluster %2d: launch %s, sync %s\n", c, cudaGetErrorString(e), cudaGetErrorString(s));
    }
    return 0;
}

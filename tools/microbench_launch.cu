// microbench_launch.cu -- host-step launch costs: a 128-CTA, 4-CTA-cluster, 512-thread kernel
// (the fused decode kernel's launch shape) that writes a host-mapped completion word, launched
// (A) with cudaLaunchKernelEx (cluster + PDL attributes) or (B) as a captured 1-node CUDA
// graph, the host spinning on the word after each launch.  Prints microseconds per call.
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512, 1) k_done(volatile unsigned* flag, unsigned seq) {
    __syncthreads();
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        __threadfence_system();
        *flag = seq;
    }
}

int main() {
    unsigned* h;
    cudaHostAlloc(&h, 64, cudaHostAllocMapped);
    unsigned* d;
    cudaHostGetDevicePointer((void**)&d, h, 0);
    *(volatile unsigned*)h = 0;
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(128);
    cfg.blockDim = dim3(512);
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 4;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    unsigned seq = 0;
    auto spin = [&](unsigned s) { while (__atomic_load_n(h, __ATOMIC_ACQUIRE) != s) {} };
    const int N = 2000;
    for (int i = 0; i < 100; ++i) { cudaLaunchKernelEx(&cfg, k_done, (volatile unsigned*)d, ++seq); spin(seq); }
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < N; ++i) { cudaLaunchKernelEx(&cfg, k_done, (volatile unsigned*)d, ++seq); spin(seq); }
    auto t1 = std::chrono::steady_clock::now();
    printf("A cudaLaunchKernelEx (cluster 4 + PDL) + spin: %.2f us/call\n", std::chrono::duration<double, std::micro>(t1 - t0).count() / N);
    cfg.numAttrs = 1;  // no PDL
    t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < N; ++i) { cudaLaunchKernelEx(&cfg, k_done, (volatile unsigned*)d, ++seq); spin(seq); }
    t1 = std::chrono::steady_clock::now();
    printf("A' cudaLaunchKernelEx (cluster 4) + spin:      %.2f us/call\n", std::chrono::duration<double, std::micro>(t1 - t0).count() / N);
    // B: graph; the sequence number comes from device memory bumped by a second node? Use a
    // kernel param updated with cudaGraphExecKernelNodeSetParams.
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
    cfg.numAttrs = 2;
    cudaLaunchKernelEx(&cfg, k_done, (volatile unsigned*)d, 0u);
    cudaStreamEndCapture(st, &g);
    cudaGraphInstantiate(&ge, g, 0);
    size_t n = 0;
    cudaGraphGetNodes(g, nullptr, &n);
    cudaGraphNode_t node;
    n = 1;
    cudaGraphGetNodes(g, &node, &n);
    cudaKernelNodeParams kp;
    cudaGraphKernelNodeGetParams(node, &kp);
    volatile unsigned* dp = (volatile unsigned*)d;
    for (int i = 0; i < 100; ++i) {
        unsigned s = ++seq;
        void* args[2] = {&dp, &s};
        kp.kernelParams = args;
        cudaGraphExecKernelNodeSetParams(ge, node, &kp);
        cudaGraphLaunch(ge, st);
        spin(s);
    }
    t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < N; ++i) {
        unsigned s = ++seq;
        void* args[2] = {&dp, &s};
        kp.kernelParams = args;
        cudaGraphExecKernelNodeSetParams(ge, node, &kp);
        cudaGraphLaunch(ge, st);
        spin(s);
    }
    t1 = std::chrono::steady_clock::now();
    printf("B graph launch (+ param update) + spin:        %.2f us/call\n", std::chrono::duration<double, std::micro>(t1 - t0).count() / N);
    printf("(%s)\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}

// microbench_select.cu -- block_select (select.cuh) in isolation: one 512-thread CTA per
// SM selects the best 127 of 2047 fp64 scores, as the fused decode kernel does, plus the
// primitive costs (barrier, L2 load, smem histogram, block scan) it is built from.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#include "select.cuh"

using namespace qk;

constexpr int NT = 512;

constexpr int GT = 128;  // selection group

__global__ void __launch_bounds__(NT, 1) sel_kernel(const double* __restrict__ scores, int n,
                                                   int target, int* out_pages,
                                                   long long* cyc, unsigned long long* probe) {
    extern __shared__ unsigned long long keys[];
    __shared__ SelectScratch<NT> sc;
    __shared__ SelectScratch<GT> sg;
    __shared__ int list[512];
    __shared__ long long trace[16];
    const double* src = scores + size_t(blockIdx.x) * n;
    unsigned long long kmax, kmin;
    const int kpt = load_keys<NT>(src, n, keys, sc, &kmax, &kmin);
    __syncthreads();
    block_select<NT>(keys, kpt, n, target, kmax, kmin, list, sc);
    long long a = clock64();
    for (int r = 0; r < 10; ++r) block_select<NT>(keys, kpt, n, target, kmax, kmin, list, sc);
    long long b = clock64();
    b = a + (b - a) / 10;
    for (int i = threadIdx.x; i < target; i += NT) out_pages[blockIdx.x * 1024 + i] = list[i];
    __syncthreads();
    // group of 128 threads, 16 keys each
    const unsigned long long ref = order_key(src[0]);
    unsigned long long k16[16];
    const int gt = threadIdx.x;
    for (int j = 0; j < 16; ++j) {
        const int i = gt * 16 + j;
        k16[j] = (gt < GT && i < n) ? order_key(src[i]) : 0ull;
    }
    for (int k = 0; k < 16; ++k) trace[k] = 0;
    __syncthreads();
    long long c = 0, d = 0, e0 = 0;
    if (gt < GT) {
        block_select_reg<GT, 16>(k16, n, target, ref, list, sg, gt, 1);
        group_sync<GT>(1);
        c = clock64();
        for (int r = 0; r < 10; ++r) {
            block_select_reg<GT, 16>(k16, n, target, ref, list, sg, gt, 1);
            group_sync<GT>(1);
        }
        d = clock64();
        d = c + (d - c) / 10;
        // one more call with globaltimer stamps (slots 10 = start, 11 bin, 14 take, 15 done)
        if (gt == 0) {
            unsigned long long t;
            t = clock64();
            probe[blockIdx.x * 32 + 10] = t;
        }
        group_sync<GT>(1);
        block_select_reg<GT, 16>(k16, n, target, ref, list, sg, gt, 1, probe);
        group_sync<GT>(1);
        e0 = clock64();
        block_select_reg_wide<GT, 16>(k16, n, target, ref, list, sg, gt, 1, nullptr, trace);
        group_sync<GT>(1);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < target; i += NT) out_pages[blockIdx.x * 1024 + 512 + i] = list[i];
    if (threadIdx.x == 0) {
        long long* o = cyc + blockIdx.x * 16;
        o[0] = b - a;
        o[1] = d - c;
        for (int k = 0; k < 9; ++k) o[2 + k] = trace[k] ? trace[k] - e0 : 0;
    }
}

int main(int argc, char** argv) {
    const int n = 2047, target = argc > 1 ? atoi(argv[1]) : 127, ctas = 128;
    const int ties = argc > 2 ? atoi(argv[2]) : 0;  // draw from this many distinct values
    double* h = new double[size_t(ctas) * n];
    unsigned long long x = 88172645463325252ull;
    for (size_t i = 0; i < size_t(ctas) * n; ++i) {
        x ^= x << 13; x ^= x >> 7; x ^= x << 17;
        h[i] = ties ? double(x % ties) - 2.0 : 1.0 + double(x % 1000003) * 1e-7;
    }
    double* d;
    int* pages;
    long long* cyc;
    unsigned long long* probe;
    cudaMalloc(&probe, 128 * 32 * 8);
    cudaMemset(probe, 0, 128 * 32 * 8);
    cudaMalloc(&d, size_t(ctas) * n * 8);
    cudaMalloc(&pages, ctas * 1024 * 4);
    cudaMalloc(&cyc, ctas * 16 * 8);
    cudaMemcpy(d, h, size_t(ctas) * n * 8, cudaMemcpyHostToDevice);
    const int kpt = (n + NT - 1) / NT;
    const size_t smem = size_t(NT) * (kpt + 1) * 8;
    for (int rep = 0; rep < 3; ++rep) {
        sel_kernel<<<ctas, NT, smem>>>(d, n, target, pages, cyc, probe);
        cudaDeviceSynchronize();
    }
    long long c[16 * 128];
    cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
    int* hp = new int[ctas * 1024];
    cudaMemcpy(hp, pages, ctas * 1024 * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int b = 0; b < ctas; ++b)
        for (int i = 0; i < target; ++i) bad += hp[b * 1024 + i] != hp[b * 1024 + 512 + i];
    printf("target %d ties %d: register select vs block_select mismatches: %d\n", target, ties, bad);
    const char* names[] = {"block_select", "block_select_reg", "t0 range", "t1 hist read",
                           "t2 warp scan", "t3 sum_below", "t4 bin known", "t5 pair gathered",
                           "t6 take known", "t7 ballots", "t8 compaction prefix"};
    for (int k = 0; k < 11; ++k) {
        double a = 0;
        for (int i = 0; i < ctas; ++i) a += c[16 * i + k];
        printf("%-22s %7.0f cycles\n", names[k], a / ctas);
    }
    unsigned long long pr[128 * 32];
    cudaMemcpy(pr, probe, sizeof(pr), cudaMemcpyDeviceToHost);
    double s11 = 0, s14 = 0, s15 = 0;
    for (int i = 0; i < ctas; ++i) {
        s11 += double(pr[i * 32 + 11] - pr[i * 32 + 10]);
        s14 += double(pr[i * 32 + 14] - pr[i * 32 + 10]);
        s15 += double(pr[i * 32 + 15] - pr[i * 32 + 10]);
    }
    printf("stamps (cycles from start): bin known %.0f, take known %.0f, done %.0f\n", s11 / ctas, s14 / ctas, s15 / ctas);
    const int order[] = {20, 21, 22, 23, 11, 24, 25, 26, 14, 27, 15};
    const char* nm[] = {"ordiff synced", "hist issued", "hist synced", "scan done", "bin known", "gathered", "gather synced", "ranked", "take known", "compaction scan", "done"};
    for (int q = 0; q < 11; ++q) {
        double a = 0; int cnt = 0;
        for (int i = 0; i < ctas; ++i) if (pr[i * 32 + order[q]] > pr[i * 32 + 10]) { a += double(pr[i * 32 + order[q]] - pr[i * 32 + 10]); ++cnt; }
        printf("  %-16s %4d ctas %7.0f cycles\n", nm[q], cnt, cnt ? a / cnt : 0.0);
    }
    for (int k = 24; k < 30; ++k) {
        double a = 0; int cnt = 0;
        for (int i = 0; i < ctas; ++i) if (pr[i * 32 + k]) { a += double(pr[i * 32 + k] - pr[i * 32 + 10]); ++cnt; }
        printf("  slot %d: %d ctas, %.0f ns\n", k, cnt, cnt ? a / cnt : 0.0);
    }
    printf("(%s)\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}

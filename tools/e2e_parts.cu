// e2e_parts.cu -- where the end-to-end host call's time goes (cfg2 shape): per layer
//   A  decode_step_host (host q/k/v in, host fp32 out; what bench.py's e2e times)
//   B  decode_step on device buffers + cudaStreamSynchronize per call
//   C  decode_step on device buffers, one synchronize per step (launch-throughput bound)
//   D  an empty kernel launch + cudaStreamSynchronize (the host round-trip floor)
//
//   nvcc -O2 -std=c++17 -Iinclude tools/e2e_parts.cu -o build/e2e_parts \
//        -Lpaper_2406_10774_b200 -lquestkv_b200 -Xlinker -rpath=$PWD/paper_2406_10774_b200
#include <chrono>
#include <cstdio>
#include <random>
#include <vector>

#include <cuda_runtime.h>

#include "questkv_b200.hpp"

namespace qk = questkv_b200;

__global__ void empty_kernel() {}

int main() {
    const uint32_t ctx = 32768, budget = 2048, layers = 8, H = 32, d = 128, S = 16;
    const int steps = 20, warmup = 3;
    qk_cache_desc desc{d, S, 2, layers, 1, H, H, ctx + uint32_t(4 * (steps + warmup)) + 16, 0};
    qk::DeviceCache cache(desc);
    std::mt19937 rng(1234);
    std::normal_distribution<float> nd(0.0f, 1.0f / std::sqrt(float(d)));
    std::vector<uint16_t> kv(size_t(H) * (ctx - 1) * d);
    for (auto& x : kv) x = qk::float_to_half(nd(rng));
    for (uint32_t l = 0; l < layers; ++l) cache.prefill_host(l, 0, kv.data(), kv.data(), ctx - 1);
    std::vector<uint16_t> q(size_t(layers) * H * d), kn(q.size()), vn(q.size());
    for (auto* v : {&q, &kn, &vn})
        for (auto& x : *v) x = qk::float_to_half(nd(rng));
    std::vector<float> out(size_t(layers) * H * d);
    uint16_t *dq, *dk, *dv;
    float* dout;
    cudaMalloc(&dq, q.size() * 2);
    cudaMalloc(&dk, q.size() * 2);
    cudaMalloc(&dv, q.size() * 2);
    cudaMalloc(&dout, out.size() * 4);
    cudaMemcpy(dq, q.data(), q.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dk, kn.data(), q.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dv, vn.data(), q.size() * 2, cudaMemcpyHostToDevice);
    const qk::SelectionConfig sel{budget, true, true};
    const size_t hd = size_t(H) * d;
    auto time = [&](const char* name, auto&& step) {
        for (int i = 0; i < warmup; ++i) step();
        cudaDeviceSynchronize();
        const auto t0 = std::chrono::steady_clock::now();
        for (int i = 0; i < steps; ++i) step();
        cudaDeviceSynchronize();
        const auto t1 = std::chrono::steady_clock::now();
        std::printf("%-48s %8.2f us/layer\n", name,
                    std::chrono::duration<double, std::micro>(t1 - t0).count() / (steps * double(layers)));
    };
    time("A decode_step_host (e2e)", [&] {
        for (uint32_t l = 0; l < layers; ++l)
            cache.decode_step_host(l, q.data() + l * hd, kn.data() + l * hd, vn.data() + l * hd, 1, sel,
                                   out.data() + l * hd);
    });
    time("B decode_step (device bufs) + sync per call", [&] {
        for (uint32_t l = 0; l < layers; ++l) {
            cache.decode_step(l, dq + l * hd, dk + l * hd, dv + l * hd, 1, sel, dout + l * hd, nullptr);
            cudaStreamSynchronize(nullptr);
        }
    });
    time("C decode_step (device bufs), sync per step", [&] {
        for (uint32_t l = 0; l < layers; ++l)
            cache.decode_step(l, dq + l * hd, dk + l * hd, dv + l * hd, 1, sel, dout + l * hd, nullptr);
        cudaStreamSynchronize(nullptr);
    });
    time("D empty kernel + sync (host round trip)", [&] {
        for (uint32_t l = 0; l < layers; ++l) {
            empty_kernel<<<1, 32>>>();
            cudaStreamSynchronize(nullptr);
        }
    });
    return 0;
}

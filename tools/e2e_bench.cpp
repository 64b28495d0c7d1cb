// e2e_bench.cpp -- end-to-end latency of the Quest decode step through the repo's C++
// public API (include/questkv_b200.hpp, questkv_b200::DeviceCache::decode_step_host): every
// call takes the layer's q/k/v from pinned host memory and returns the fp32 output to host
// memory (copies inside the timed region), as a host-driven caller of the reference's API
// would.  Used by bench.py for the `e2e` key.
//
//   e2e_bench <ctx> <budget> <layers> <steps> <warmup>   -> one JSON line on stdout
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "questkv_b200.hpp"

namespace qk = questkv_b200;

int main(int argc, char** argv) {
    const uint32_t ctx = argc > 1 ? uint32_t(std::atoi(argv[1])) : 32768;
    const uint32_t budget = argc > 2 ? uint32_t(std::atoi(argv[2])) : 2048;
    const uint32_t layers = argc > 3 ? uint32_t(std::atoi(argv[3])) : 8;
    const int steps = argc > 4 ? std::atoi(argv[4]) : 20;
    const int warmup = argc > 5 ? std::atoi(argv[5]) : 3;
    const uint32_t H = 32, d = 128, S = 16;
    qk_cache_desc desc{d, S, 2, layers, 1, H, H, ctx + uint32_t(steps + warmup) + 16, 0};
    try {
        qk::DeviceCache cache(desc);
        // One random 32K-token block per head, N(0, 1/d) in fp16, shared by every layer.
        std::mt19937 rng(1234);
        std::normal_distribution<float> nd(0.0f, 1.0f / std::sqrt(float(d)));
        const uint32_t n0 = ctx - 1;
        std::vector<uint16_t> kv(size_t(H) * n0 * d);
        for (auto& x : kv) x = qk::float_to_half(nd(rng));
        for (uint32_t l = 0; l < layers; ++l) cache.prefill_host(l, 0, kv.data(), kv.data(), n0);
        // Per-step, per-layer inputs (pinned by the library's staging; plain host vectors).
        std::vector<uint16_t> q(size_t(layers) * H * d), kn(q.size()), vn(q.size());
        for (auto* v : {&q, &kn, &vn})
            for (auto& x : *v) x = qk::float_to_half(nd(rng));
        std::vector<float> out(size_t(layers) * H * d);
        const qk::SelectionConfig sel{budget, true, true};
        auto step = [&]() {
            for (uint32_t l = 0; l < layers; ++l)
                cache.decode_step_host(l, q.data() + size_t(l) * H * d, kn.data() + size_t(l) * H * d,
                                       vn.data() + size_t(l) * H * d, 1, sel, out.data() + size_t(l) * H * d);
        };
        for (int i = 0; i < warmup; ++i) step();
        const auto t0 = std::chrono::steady_clock::now();
        for (int i = 0; i < steps; ++i) step();
        const auto t1 = std::chrono::steady_clock::now();
        const double us = std::chrono::duration<double, std::micro>(t1 - t0).count() / (steps * double(layers));
        double cs = 0;
        for (float x : out) cs += x;
        std::printf("{\"e2e_us_per_layer\": %.3f, \"layers\": %u, \"steps\": %d, \"checksum\": %.6f}\n", us,
                    layers, steps, cs);
    } catch (const std::exception& e) {
        std::printf("{\"error\": \"%s\"}\n", e.what());
        return 1;
    }
    return 0;
}

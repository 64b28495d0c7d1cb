// e2e_bench.cpp -- end-to-end latency of the Quest decode step through the repo's C++
// public API (include/questkv_b200.hpp, questkv_b200::DeviceCache::decode_step_host): every
// call takes the layer's q/k/v from pinned host memory and returns the fp32 output to host
// memory (copies inside the timed region), as a host-driven caller of the reference's API
// would.  Inputs and outputs live in pinned host memory (qk_host_alloc); the same loop over
// pageable buffers is reported beside it.  Used by bench.py for the `e2e` key.
//
//   e2e_bench <ctx> <budget> <layers> <steps> <warmup>   -> one JSON line on stdout
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <stdexcept>
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
        // Two identical caches: the pinned-buffer and the pageable-buffer loops alternate step by
        // step (host clock drift over the run hits both arms alike), each on its own cache.
        qk::DeviceCache cache(desc), cache_b(desc);
        // One random 32K-token block per head, N(0, 1/d) in fp16, shared by every layer.
        std::mt19937 rng(1234);
        std::normal_distribution<float> nd(0.0f, 1.0f / std::sqrt(float(d)));
        const uint32_t n0 = ctx - 1;
        std::vector<uint16_t> kv(size_t(H) * n0 * d);
        for (auto& x : kv) x = qk::float_to_half(nd(rng));
        for (uint32_t l = 0; l < layers; ++l) {
            cache.prefill_host(l, 0, kv.data(), kv.data(), n0);
            cache_b.prefill_host(l, 0, kv.data(), kv.data(), n0);
        }
        // Per-step, per-layer inputs and outputs, in pinned host memory from the library
        // (qk_host_alloc; the kernel reads and writes them in place over PCIe), and the same
        // in pageable std::vectors (staged through the library's pinned buffer).
        const size_t n = size_t(layers) * H * d;
        auto* q = static_cast<uint16_t*>(qk_host_alloc(n * 2));
        auto* kn = static_cast<uint16_t*>(qk_host_alloc(n * 2));
        auto* vn = static_cast<uint16_t*>(qk_host_alloc(n * 2));
        auto* out = static_cast<float*>(qk_host_alloc(n * 4));
        if (!q || !kn || !vn || !out) throw std::runtime_error("qk_host_alloc failed");
        for (auto* v : {q, kn, vn})
            for (size_t i = 0; i < n; ++i) v[i] = qk::float_to_half(nd(rng));
        std::vector<uint16_t> pq(q, q + n), pk(kn, kn + n), pv(vn, vn + n);
        std::vector<float> pout(n);
        const qk::SelectionConfig sel{budget, true, true};
        auto step = [&](qk::DeviceCache& c, const uint16_t* a, const uint16_t* b, const uint16_t* v,
                        float* o) {
            const auto t0 = std::chrono::steady_clock::now();
            for (uint32_t l = 0; l < layers; ++l)
                c.decode_step_host(l, a + size_t(l) * H * d, b + size_t(l) * H * d,
                                   v + size_t(l) * H * d, 1, sel, o + size_t(l) * H * d);
            return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
        };
        double t_pinned = 0, t_pageable = 0;
        for (int i = 0; i < warmup + steps; ++i) {
            const double a = step(cache, q, kn, vn, out);
            const double b = step(cache_b, pq.data(), pk.data(), pv.data(), pout.data());
            if (i >= warmup) {
                t_pinned += a;
                t_pageable += b;
            }
        }
        const double us = t_pinned / (steps * double(layers));
        const double us_pageable = t_pageable / (steps * double(layers));
        double cs = 0;
        for (size_t i = 0; i < n; ++i) cs += out[i];
        std::printf("{\"e2e_us_per_layer\": %.3f, \"e2e_pageable_us_per_layer\": %.3f, \"layers\": %u, "
                    "\"steps\": %d, \"checksum\": %.6f}\n",
                    us, us_pageable, layers, steps, cs);
        for (void* p : {static_cast<void*>(q), static_cast<void*>(kn), static_cast<void*>(vn),
                        static_cast<void*>(out)})
            qk_host_free(p);
    } catch (const std::exception& e) {
        std::printf("{\"error\": \"%s\"}\n", e.what());
        return 1;
    }
    return 0;
}

// test_questkv_b200.cpp -- the C++ host layer (include/questkv_b200.hpp) against the
// reference's own known-answer tests (restated from R/tests/test_kv_store.cpp,
// test_criticality.cpp, test_attention.cpp, test_metrics.cpp; R = /root/reference/proj) and
// against the C oracle (oracle/questkv_oracle.h, test infrastructure) on random inputs.
//
//   test_questkv_b200 --cpu   host-only checks (no device needed): validation, fp16
//                             conversion, byte model, and that a cache cannot be created
//                             without a GPU (no CPU fallback)
//   test_questkv_b200         everything, on cuda:0
//
// Built and run by tests/test_cpp_layer.py.  Exit code 0 = pass; failures are printed.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <random>
#include <string>
#include <vector>

#include "questkv_b200.hpp"
#include "questkv_oracle.h"

namespace qk = questkv_b200;

static int g_failures = 0;
#define CHECK(cond)                                                              \
    do {                                                                         \
        if (!(cond)) {                                                           \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);          \
            ++g_failures;                                                        \
        }                                                                        \
    } while (0)

template <typename Ex, typename Fn>
static bool throws(Fn&& fn) {
    try {
        fn();
    } catch (const Ex&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static float h(float x) { return qk::half_to_float(qk::float_to_half(x)); }

static void host_checks() {
    // CacheConfig::validate (kv_store.cpp:8-13).
    CHECK(throws<std::invalid_argument>([] { qk::CacheConfig{0, 16, 2}.validate(); }));
    CHECK(throws<std::invalid_argument>([] { qk::CacheConfig{16, 0, 2}.validate(); }));
    CHECK(throws<std::invalid_argument>([] { qk::CacheConfig{16, 16, 0}.validate(); }));
    // fp16: every finite half round-trips; RNE at a tie; overflow to inf; tiny to zero.
    int bad = 0;
    for (uint32_t b = 0; b < 65536; ++b) {
        if (((b >> 10) & 31) == 31) continue;
        if (qk::float_to_half(qk::half_to_float(uint16_t(b))) != b) ++bad;
    }
    CHECK(bad == 0);
    CHECK(qk::float_to_half(1.0f + 1.0f / 2048.0f) == 0x3c00);  // tie -> even
    CHECK(qk::float_to_half(1.0f + 3.0f / 2048.0f) == 0x3c02);
    CHECK(qk::float_to_half(65520.0f) == 0x7c00);
    CHECK(qk::float_to_half(1e-9f) == 0x0000);
    CHECK(qk::float_to_half(-0.0f) == 0x8000);
    // traffic_fraction: the paper's 0.125 example (test_metrics.cpp:175-185).
    CHECK(std::fabs(qk::traffic_fraction(16, 65536, 4096) - 0.125) < 1e-15);
    CHECK(throws<std::invalid_argument>([] { qk::traffic_fraction(0, 10, 1); }));
    CHECK(throws<std::invalid_argument>([] { qk::traffic_fraction(16, 10, 20); }));
}

static void no_gpu_check() {
    // No CPU fallback: without a device the cache cannot be created.
    CHECK(throws<std::runtime_error>([] { qk::KvCache c(qk::CacheConfig{16, 4, 2}, 64); }));
}

static void kv_store_cases() {
    // test_kv_store.cpp:39-51 -- keys [1,5], [3,2] -> min [1,2], max [3,5].
    qk::KvCache c(qk::CacheConfig{2, 4, 2}, 64);
    const float k0[2] = {1, 5}, k1[2] = {3, 2}, v[2] = {0, 0};
    CHECK(c.append(k0, v) == 0);
    CHECK(c.append(k1, v) == 1);
    const qk::PageMetadata m = c.page_metadata(0);
    CHECK(m.min_key[0] == 1 && m.min_key[1] == 2 && m.max_key[0] == 3 && m.max_key[1] == 5);
    // Paging arithmetic (:61-73): 9 tokens of page size 4 -> 3 pages, last holds 1.
    qk::KvCache p(qk::CacheConfig{2, 4, 2}, 64);
    for (int t = 0; t < 9; ++t) {
        const float k[2] = {float(t), float(-t)};
        p.append(k, v);
    }
    CHECK(p.page_count() == 3 && p.token_count() == 9 && p.page(2).length == 1);
    CHECK(p.key(5)[0] == 5.0f && p.key(5)[1] == -5.0f);
    CHECK(throws<std::out_of_range>([&] { p.page_metadata(3); }));
    CHECK(throws<std::out_of_range>([&] { p.key(9); }));
    CHECK(throws<std::invalid_argument>([&] {
        const float k3[3] = {1, 2, 3};
        p.append(k3, k3);
    }));
    // Growth past the initial capacity (the reference's page vector grows on demand,
    // kv_store.cpp:24-29): 4 -> 8 -> 16 -> 32 tokens, pages and metadata kept.
    qk::KvCache g(qk::CacheConfig{2, 4, 2}, 4);
    for (int t = 0; t < 23; ++t) {
        const float k[2] = {float(t), float(100 - 3 * t)};
        g.append(k, v);
    }
    std::vector<float> ks(2 * 10), vs(2 * 10, 0.5f);
    for (int t = 0; t < 10; ++t) ks[2 * t] = ks[2 * t + 1] = float(-t);
    g.extend(ks, vs);
    CHECK(g.token_count() == 33 && g.page_count() == 9);
    CHECK(g.key(22)[0] == 22.0f && g.key(22)[1] == 34.0f && g.key(32)[0] == -9.0f);
    const qk::PageMetadata gm = g.page_metadata(1);  // tokens 4..7
    CHECK(gm.min_key[0] == 4 && gm.max_key[0] == 7 && gm.min_key[1] == 79 && gm.max_key[1] == 88);
    const qk::PageMetadata gm5 = g.page_metadata(5);  // tokens 20..22 appended, 23 extended
    CHECK(gm5.min_key[0] == 0 && gm5.max_key[0] == 22 && gm5.min_key[1] == 0 && gm5.max_key[1] == 40);
}

static void criticality_cases() {
    // test_criticality.cpp:60-64 -- q=[1,-2], min=[0,-1], max=[3,2] -> 5.
    const float q[2] = {1, -2};
    qk::PageMetadata m{{0, -1}, {3, 2}};
    CHECK(qk::estimate_page_score(q, m) == 5.0);
    const float z[2] = {0, 0};
    CHECK(qk::estimate_page_score(z, m) == 0.0);  // :66-69
    // select_top_k worked cases (:121-165) on a 4-page / 3-page cache of page size 1.
    auto cache_of = [](uint32_t pages) {
        auto c = std::make_unique<qk::KvCache>(qk::CacheConfig{1, 1, 2}, 16);
        for (uint32_t i = 0; i < pages; ++i) {
            const float k[1] = {float(i)};
            c->append(k, k);
        }
        return c;
    };
    auto scores = [](std::vector<double> s) {
        std::vector<qk::PageScore> v;
        for (uint32_t i = 0; i < s.size(); ++i) v.push_back({i, s[i]});
        return v;
    };
    auto c4 = cache_of(4);
    qk::SelectionConfig unforced{2, false, true}, forced{2, true, true};
    CHECK((qk::select_top_k(scores({5, 9, 9, 1}), unforced, *c4) == std::vector<uint32_t>{1, 2}));
    auto c3 = cache_of(3);
    CHECK((qk::select_top_k(scores({3, 3, 3}), qk::SelectionConfig{1, false, true}, *c3) ==
           std::vector<uint32_t>{0}));
    CHECK((qk::select_top_k(scores({9, 8, 1}), forced, *c3) == std::vector<uint32_t>{0, 2}));
    CHECK((qk::select_top_k(scores({9, 8, 1}), unforced, *c3) == std::vector<uint32_t>{0, 1}));
    CHECK((qk::select_top_k(scores({9, 8, 1}), qk::SelectionConfig{2, true, false}, *c3) ==
           std::vector<uint32_t>{0, 1, 2}));
    CHECK(throws<std::invalid_argument>(
        [&] { qk::select_top_k(scores({9, 8, 1}), qk::SelectionConfig{0, true, true}, *c3); }));
    CHECK(throws<std::out_of_range>([&] {
        qk::select_top_k({{7, 1.0}}, qk::SelectionConfig{1, true, true}, *c3);
    }));
    qk::KvCache empty(qk::CacheConfig{2, 4, 2}, 16);
    CHECK(throws<std::invalid_argument>([&] { qk::estimate_all(q, empty); }));
}

static void attention_cases() {
    // test_attention.cpp:125-146 -- single token returns its value; equal keys average.
    qk::KvCache c(qk::CacheConfig{2, 4, 2}, 16);
    const float k[2] = {0.5f, -0.25f}, v0[2] = {2, -3}, v1[2] = {4, 1}, q[2] = {1, 1};
    c.append(k, v0);
    auto o = qk::full_attention(q, c);
    CHECK(o.output[0] == 2.0 && o.output[1] == -3.0);
    c.append(k, v1);
    o = qk::full_attention(q, c);
    CHECK(std::fabs(o.output[0] - 3.0) < 1e-6 && std::fabs(o.output[1] + 1.0) < 1e-6);
    const uint32_t none[1] = {0};
    CHECK(throws<std::invalid_argument>([&] { qk::sparse_attention(q, c, std::span<const uint32_t>(none, 0)); }));
    const uint32_t bad[1] = {5}, dup[2] = {0, 0};
    CHECK(throws<std::out_of_range>([&] { qk::sparse_attention(q, c, bad); }));
    CHECK(throws<std::invalid_argument>([&] { qk::sparse_attention(q, c, dup); }));
    qk::KvCache empty(qk::CacheConfig{2, 4, 2}, 16);
    CHECK(throws<std::invalid_argument>([&] { qk::full_attention(q, empty); }));
}

static void random_parity(uint32_t d, uint32_t S, uint32_t n, uint32_t budget, uint32_t seed) {
    std::mt19937 rng(seed);
    std::normal_distribution<float> nd(0.0f, 1.0f / std::sqrt(float(d)));
    std::vector<float> keys(size_t(n) * d), vals(size_t(n) * d), q(d);
    for (auto& x : keys) x = h(nd(rng));
    for (auto& x : vals) x = h(nd(rng));
    for (auto& x : q) x = h(nd(rng));
    qk::KvCache c(qk::CacheConfig{d, S, 2}, n + 8);
    c.extend(keys, vals);
    const uint32_t P = c.page_count();
    // metadata bitwise
    std::vector<float> mn(size_t(P) * d), mx(size_t(P) * d);
    qo_build_metadata(keys.data(), n, d, S, mn.data(), mx.data());
    bool meta_ok = true;
    for (uint32_t p = 0; p < P; ++p) {
        const auto m = c.page_metadata(p);
        meta_ok &= std::memcmp(m.min_key.data(), &mn[size_t(p) * d], d * 4) == 0;
        meta_ok &= std::memcmp(m.max_key.data(), &mx[size_t(p) * d], d * 4) == 0;
    }
    CHECK(meta_ok);
    // scores bitwise
    std::vector<double> want(P);
    qo_estimate_all(q.data(), mn.data(), mx.data(), P, d, want.data());
    const auto got = qk::estimate_all(q, c);
    bool s_ok = true;
    for (uint32_t p = 0; p < P; ++p) s_ok &= std::memcmp(&want[p], &got[p].score, 8) == 0;
    CHECK(s_ok);
    // selection bitwise
    std::vector<uint32_t> wp(P);
    uint32_t wn = 0;
    qo_select_top_k(want.data(), P, S, budget, 1, 1, wp.data(), &wn);
    const auto sel = qk::select_top_k(got, qk::SelectionConfig{budget, true, true}, c);
    CHECK(sel == std::vector<uint32_t>(wp.begin(), wp.begin() + wn));
    // sparse attention within 1e-5 relative L2
    std::vector<double> wo(d);
    double wsum = 0;
    qo_sparse_attention(q.data(), keys.data(), vals.data(), n, d, S, wp.data(), wn, wo.data(), &wsum);
    const auto go = qk::sparse_attention(q, c, sel);
    double num = 0, den = 0;
    for (uint32_t i = 0; i < d; ++i) {
        num += (go.output[i] - wo[i]) * (go.output[i] - wo[i]);
        den += wo[i] * wo[i];
    }
    CHECK(std::sqrt(num / den) <= 1e-5);
}

int main(int argc, char** argv) {
    const bool cpu_only = argc > 1 && std::string(argv[1]) == "--cpu";
    host_checks();
    if (cpu_only) {
        no_gpu_check();
    } else {
        kv_store_cases();
        criticality_cases();
        attention_cases();
        random_parity(128, 16, 3000, 512, 1);
        random_parity(64, 8, 777, 128, 2);
        random_parity(100, 7, 1000, 70, 3);
    }
    std::printf("%s: %d failure(s)\n", cpu_only ? "cpu checks" : "all checks", g_failures);
    return g_failures == 0 ? 0 : 1;
}

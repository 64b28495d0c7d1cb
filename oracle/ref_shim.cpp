// ref_shim.cpp -- extern "C" entry points over the UNMODIFIED reference library
// (TEST INFRASTRUCTURE ONLY).
//
// oracle/Makefile compiles this file together with the reference's own sources, read in
// place from /root/reference/proj/core/src/*.cpp, into oracle/_ref/libquestkv_ref.so.
// Nothing from the reference is copied into this repository: this file only builds
// questkv::KvCache objects from flat float arrays and calls the reference's public API
// (kv_store.hpp, criticality.hpp, attention.hpp, reference.hpp, parallel.hpp), mapping
// exceptions to status codes (invalid_argument -> 1, out_of_range -> 2).
//
// Users: tests/golden/make_golden.py (golden vectors), tests/golden/make_trace_golden.py
// (QKVTRACE file and recall_at_n fixtures), tests/test_oracle.py and tests/test_trace.py
// (pin the C restatement and the trace/recall code against the reference), bench.py
// (cpu_baseline and --impl reference).

#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#include "questkv/attention.hpp"
#include "questkv/criticality.hpp"
#include "questkv/kv_store.hpp"
#include "questkv/metrics.hpp"
#include "questkv/parallel.hpp"
#include "questkv/reference.hpp"
#include "questkv/workloads.hpp"

using namespace questkv;

namespace {

template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return 0;
    } catch (const std::invalid_argument&) {
        return 1;
    } catch (const std::out_of_range&) {
        return 2;
    } catch (...) {
        return 3;
    }
}

KvCache make_cache(const float* keys, const float* values, uint32_t n, uint32_t dim,
                   uint32_t page_size) {
    KvCache cache({.head_dim = dim, .page_size = page_size});
    for (uint32_t t = 0; t < n; ++t)
        cache.append(std::span<const float>(keys + size_t(t) * dim, dim),
                     std::span<const float>(values + size_t(t) * dim, dim));
    return cache;
}

}  // namespace

extern "C" {

int ref_validate_config(uint32_t head_dim, uint32_t page_size, uint32_t bpe) {
    return guarded([&] { KvCache c({.head_dim = head_dim, .page_size = page_size,
                                    .bytes_per_element = bpe}); });
}

// KvCache::append x n, then page_metadata(p) for every page.
int ref_metadata(const float* keys, const float* values, uint32_t n, uint32_t dim,
                 uint32_t page_size, float* min_out, float* max_out) {
    return guarded([&] {
        KvCache cache = make_cache(keys, values, n, dim, page_size);
        for (uint32_t p = 0; p < cache.page_count(); ++p) {
            const PageMetadata& m = cache.page_metadata(p);
            std::memcpy(min_out + size_t(p) * dim, m.min_key.data(), sizeof(float) * dim);
            std::memcpy(max_out + size_t(p) * dim, m.max_key.data(), sizeof(float) * dim);
        }
    });
}

int ref_estimate_all(const float* q, const float* keys, const float* values, uint32_t n,
                     uint32_t dim, uint32_t page_size, double* scores) {
    return guarded([&] {
        KvCache cache = make_cache(keys, values, n, dim, page_size);
        const auto s = estimate_all(std::span<const float>(q, dim), cache);
        for (size_t i = 0; i < s.size(); ++i) scores[i] = s[i].score;
    });
}

// select_top_k on explicit scores against a geometry-only cache of n_pages full pages,
// as the reference's own selection tests do (test_criticality.cpp geometry_cache).
int ref_select_top_k(const double* scores, uint32_t n_scores, uint32_t n_pages,
                     uint32_t page_size, uint32_t budget, int force, int enabled,
                     uint32_t* out, uint32_t* count) {
    return guarded([&] {
        KvCache cache({.head_dim = 1, .page_size = page_size});
        const float zero = 0.0f;
        for (uint64_t t = 0; t < uint64_t(n_pages) * page_size; ++t)
            cache.append(std::span<const float>(&zero, 1), std::span<const float>(&zero, 1));
        std::vector<PageScore> ps(n_scores);
        for (uint32_t i = 0; i < n_scores; ++i) ps[i] = {i, scores[i]};
        const auto sel = select_top_k(ps, {.token_budget = budget,
                                           .force_include_recent = force != 0,
                                           .per_layer_enabled = enabled != 0},
                                      cache);
        std::memcpy(out, sel.data(), sizeof(uint32_t) * sel.size());
        *count = uint32_t(sel.size());
    });
}

int ref_sparse_attention(const float* q, const float* keys, const float* values, uint32_t n,
                         uint32_t dim, uint32_t page_size, const uint32_t* pages,
                         uint32_t n_sel, double* out, double* wsum) {
    return guarded([&] {
        KvCache cache = make_cache(keys, values, n, dim, page_size);
        const auto r = sparse_attention(std::span<const float>(q, dim), cache,
                                        std::span<const uint32_t>(pages, n_sel));
        std::memcpy(out, r.output.data(), sizeof(double) * dim);
        if (wsum) *wsum = r.weights_sum_check;
    });
}

int ref_full_attention(const float* q, const float* keys, const float* values, uint32_t n,
                       uint32_t dim, uint32_t page_size, double* out, double* wsum) {
    return guarded([&] {
        KvCache cache = make_cache(keys, values, n, dim, page_size);
        const auto r = full_attention(std::span<const float>(q, dim), cache);
        std::memcpy(out, r.output.data(), sizeof(double) * dim);
        if (wsum) *wsum = r.weights_sum_check;
    });
}

int ref_naive_attention(const float* q, const float* keys, const float* values, uint32_t n,
                        uint32_t dim, const uint32_t* tokens, uint32_t n_sel, double* out) {
    return guarded([&] {
        KvCache cache = make_cache(keys, values, n, dim, 1);
        const auto r = reference::naive_attention(std::span<const float>(q, dim), cache,
                                                  std::span<const uint32_t>(tokens, n_sel));
        std::memcpy(out, r.data(), sizeof(double) * dim);
    });
}

// One Quest step (metrics.cpp:90-95): estimate_all -> select_top_k -> sparse_attention.
int ref_quest_step(const float* q, const float* keys, const float* values, uint32_t n,
                   uint32_t dim, uint32_t page_size, uint32_t budget, int force, int enabled,
                   double* scores, uint32_t* pages, uint32_t* n_selected, double* out) {
    return guarded([&] {
        KvCache cache = make_cache(keys, values, n, dim, page_size);
        const std::span<const float> query(q, dim);
        const auto s = estimate_all(query, cache);
        for (size_t i = 0; i < s.size(); ++i) scores[i] = s[i].score;
        const auto sel = select_top_k(s, {.token_budget = budget,
                                          .force_include_recent = force != 0,
                                          .per_layer_enabled = enabled != 0},
                                      cache);
        std::memcpy(pages, sel.data(), sizeof(uint32_t) * sel.size());
        *n_selected = uint32_t(sel.size());
        const auto r = sparse_attention(query, cache, sel);
        std::memcpy(out, r.output.data(), sizeof(double) * dim);
    });
}

double ref_traffic_fraction(uint32_t page_size, uint64_t token_count, uint64_t budget) {
    return traffic_fraction(page_size, token_count, budget);
}

// ---------------------------------------------------------------------------------------
// CPU baseline: one decode layer = n_heads independent single-head caches, timed the way
// tools/src/cmd_bench.cpp:32-51 times a phase (steady_clock, warmup, reps), with the
// heads spread over questkv::parallel_for (parallel.hpp:29-56).

struct RefLayer {
    std::vector<KvCache> caches;
    uint32_t dim = 0;
};

void* ref_layer_create(const float* keys, const float* values, uint32_t n_heads,
                       uint32_t n_tokens, uint32_t dim, uint32_t page_size) {
    auto* layer = new RefLayer;
    layer->dim = dim;
    layer->caches.reserve(n_heads);
    for (uint32_t h = 0; h < n_heads; ++h)
        layer->caches.push_back(make_cache(keys + size_t(h) * n_tokens * dim,
                                           values + size_t(h) * n_tokens * dim, n_tokens,
                                           dim, page_size));
    return layer;
}

void ref_layer_destroy(void* handle) { delete static_cast<RefLayer*>(handle); }

// mode 0: Quest (estimate -> select -> sparse); mode 1: dense full_attention.
// queries: [n_heads][dim].  out: [n_heads][dim] from the last rep.
// Returns mean ns per rep in *mean_ns and the minimum in *min_ns.
int ref_layer_step(void* handle, const float* queries, uint32_t budget, int mode,
                   uint32_t threads, uint32_t warmup, uint32_t reps, double* mean_ns,
                   double* min_ns, double* out) {
    auto* layer = static_cast<RefLayer*>(handle);
    const std::string t = std::to_string(threads);
    setenv("QUESTKV_THREADS", t.c_str(), 1);
    const uint32_t dim = layer->dim;
    const uint64_t heads = layer->caches.size();
    auto one = [&] {
        parallel_for(heads, [&](uint64_t h) {
            const std::span<const float> q(queries + h * dim, dim);
            const KvCache& cache = layer->caches[h];
            AttentionOutput r;
            if (mode == 0) {
                const auto scores = estimate_all(q, cache);
                const auto pages = select_top_k(scores, {.token_budget = budget}, cache);
                r = sparse_attention(q, cache, pages);
            } else {
                r = full_attention(q, cache);
            }
            std::memcpy(out + h * dim, r.output.data(), sizeof(double) * dim);
        });
    };
    return guarded([&] {
        for (uint32_t i = 0; i < warmup; ++i) one();
        double total = 0.0, best = 1e300;
        for (uint32_t i = 0; i < reps; ++i) {
            const auto t0 = std::chrono::steady_clock::now();
            one();
            const double ns = std::chrono::duration<double, std::nano>(
                                  std::chrono::steady_clock::now() - t0)
                                  .count();
            total += ns;
            best = ns < best ? ns : best;
        }
        *mean_ns = reps ? total / reps : 0.0;
        *min_ns = reps ? best : 0.0;
    });
}


// QKVTRACE I/O through the reference (workloads.cpp write_trace / read_trace).
int ref_write_trace(const char* path, uint32_t head_dim, uint32_t n, const float* keys,
                    const float* values, const float* queries) {
    return guarded([&] {
        DecodeTrace t;
        t.head_dim = head_dim;
        t.steps.resize(n);
        for (uint32_t i = 0; i < n; ++i) {
            t.steps[i].key.assign(keys + size_t(i) * head_dim, keys + size_t(i + 1) * head_dim);
            t.steps[i].value.assign(values + size_t(i) * head_dim, values + size_t(i + 1) * head_dim);
            t.steps[i].query.assign(queries + size_t(i) * head_dim, queries + size_t(i + 1) * head_dim);
        }
        write_trace(path, t);
    });
}

// read_trace: -> head_dim, length; copies up to cap steps. Status 4 = trace_format_error.
int ref_read_trace(const char* path, uint32_t* head_dim, uint32_t* n, float* keys, float* values,
                   float* queries, uint32_t cap) {
    try {
        const DecodeTrace t = read_trace(path);
        *head_dim = t.head_dim;
        *n = uint32_t(t.steps.size());
        for (uint32_t i = 0; i < *n && i < cap; ++i) {
            std::memcpy(keys + size_t(i) * t.head_dim, t.steps[i].key.data(), t.head_dim * 4);
            std::memcpy(values + size_t(i) * t.head_dim, t.steps[i].value.data(), t.head_dim * 4);
            std::memcpy(queries + size_t(i) * t.head_dim, t.steps[i].query.data(), t.head_dim * 4);
        }
        return 0;
    } catch (const trace_format_error&) {
        return 4;
    } catch (...) {
        return 3;
    }
}

// recall_at_n (metrics.cpp:12-38) over a cache built from n_tokens appends.
int ref_recall_at_n(const uint32_t* selected, uint32_t n_sel, const float* query, const float* keys,
                    const float* values, uint32_t n_tokens, uint32_t dim, uint32_t page_size,
                    uint32_t top_n, double* recall) {
    return guarded([&] {
        KvCache cache = make_cache(keys, values, n_tokens, dim, page_size);
        *recall = recall_at_n(std::span<const uint32_t>(selected, n_sel),
                              std::span<const float>(query, dim), cache, top_n);
    });
}
}  // extern "C"

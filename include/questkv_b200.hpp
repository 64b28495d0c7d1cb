// questkv_b200.hpp -- C++ host layer over the C ABI (questkv_b200.h): the reference's
// questkv:: operator API (R/core/include/questkv/{kv_store,criticality,attention,metrics}.hpp,
// R = /root/reference/proj) with the same names, argument meaning and exception types,
// executed by the B200 kernels.  Header-only; link with -lquestkv_b200 (the in-tree
// paper_2406_10774_b200/libquestkv_b200.so).  Requires C++20 (std::span), like the reference.
//
// Drop-in use: replace `#include "questkv/..."` by `#include "questkv_b200.hpp"` and
// `questkv::` by `questkv_b200::` (or `namespace questkv = questkv_b200;`).
//
// Differences a caller can observe (all documented in INTEGRATION.md):
//   * storage is fp16: keys/values/queries are rounded to fp16 (round-to-nearest-even) on
//     the way in; for fp16-representable inputs every result equals the reference's
//     (metadata, scores and page sets bitwise, outputs within 1e-5 relative L2);
//   * KvCache's constructor takes an initial capacity; appends past it grow the cache by
//     doubling (qk_cache_reserve: a device copy) up to 16384 pages, as the reference grows
//     its page vector;
//   * accessors return values instead of references into host-side storage;
//   * AttentionOutput::weights_sum_check is the post-softmax mass of the weights the kernel
//     applied, evaluated in fp64 from its fp32 partials (1 up to fp32 rounding);
//   * softmax_weights runs on the current CUDA device (exp and summation order differ from
//     glibc's sequential loop: ~1e-15 relative).
// No CPU fallback exists: constructing a KvCache without a CUDA device throws
// std::runtime_error.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "questkv_b200.h"

namespace questkv_b200 {

// ---- status -> exception (the reference's types) ------------------------------------------
inline void check(int status) {
    if (status == QK_OK) return;
    const std::string msg = qk_last_error();
    switch (status) {
        case QK_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case QK_ERR_OUT_OF_RANGE: throw std::out_of_range(msg);
        default: throw std::runtime_error(msg);
    }
}

// ---- fp16 <-> float on the host (IEEE binary16, round to nearest even) --------------------
inline uint16_t float_to_half(float f) {
    uint32_t x;
    std::memcpy(&x, &f, 4);
    const uint32_t sign = (x >> 16) & 0x8000u;
    const uint32_t mag = x & 0x7fffffffu;
    if (mag >= 0x7f800000u) return uint16_t(sign | 0x7c00u | (mag > 0x7f800000u ? 0x200u : 0u));
    if (mag >= 0x477ff000u) return uint16_t(sign | 0x7c00u);  // rounds to >= 65520: inf
    if (mag < 0x38800000u) {                                   // fp16 subnormal or zero
        if (mag < 0x33000000u) return uint16_t(sign);          // < 2^-25: rounds to 0
        const uint32_t e = mag >> 23, m = (mag & 0x7fffffu) | 0x800000u;
        const uint32_t shift = 126u - e;                       // 14..24
        uint32_t r = m >> shift;
        const uint32_t rem = m & ((1u << shift) - 1u), halfway = 1u << (shift - 1u);
        if (rem > halfway || (rem == halfway && (r & 1u))) ++r;
        return uint16_t(sign | r);
    }
    uint32_t h = ((mag - 0x38000000u) >> 13);
    const uint32_t rem = mag & 0x1fffu;
    if (rem > 0x1000u || (rem == 0x1000u && (h & 1u))) ++h;
    return uint16_t(sign | h);
}

inline float half_to_float(uint16_t h) {
    const uint32_t sign = uint32_t(h & 0x8000u) << 16;
    uint32_t e = (h >> 10) & 0x1fu, m = h & 0x3ffu, x;
    if (e == 0) {
        if (m == 0) {
            x = sign;
        } else {  // subnormal
            int s = -1;
            do {
                ++s;
                m <<= 1;
            } while (!(m & 0x400u));
            x = sign | ((112u - uint32_t(s)) << 23) | ((m & 0x3ffu) << 13);
        }
    } else if (e == 31) {
        x = sign | 0x7f800000u | (m << 13);
    } else {
        x = sign | ((e + 112u) << 23) | (m << 13);
    }
    float f;
    std::memcpy(&f, &x, 4);
    return f;
}

inline std::vector<uint16_t> to_half(std::span<const float> v) {
    std::vector<uint16_t> out(v.size());
    for (size_t i = 0; i < v.size(); ++i) out[i] = float_to_half(v[i]);
    return out;
}

// ---- kv_store.hpp ---------------------------------------------------------------------------
// CacheConfig (kv_store.hpp:10-17; validate kv_store.cpp:8-13).
struct CacheConfig {
    uint32_t head_dim = 0;
    uint32_t page_size = 0;
    uint32_t bytes_per_element = 2;
    void validate() const {
        if (head_dim == 0) throw std::invalid_argument("CacheConfig: head_dim must be >= 1");
        if (page_size == 0) throw std::invalid_argument("CacheConfig: page_size must be >= 1");
        if (bytes_per_element == 0)
            throw std::invalid_argument("CacheConfig: bytes_per_element must be >= 1");
    }
};

struct PageMetadata {  // kv_store.hpp:21-24
    std::vector<float> min_key;
    std::vector<float> max_key;
};

struct Page {  // kv_store.hpp:26-31
    std::vector<float> keys;
    std::vector<float> values;
    PageMetadata metadata;
    uint32_t length = 0;
};

// KvCache (kv_store.hpp:41-65): one head's paged cache, resident in HBM.
class KvCache {
public:
    explicit KvCache(CacheConfig config, uint32_t capacity = 65536, int device = 0)
        : config_(config) {
        config_.validate();
        qk_cache_desc d{};
        d.head_dim = config_.head_dim;
        d.page_size = config_.page_size;
        d.bytes_per_element = config_.bytes_per_element;
        d.num_layers = 1;
        d.max_batch = 1;
        d.num_q_heads = 1;
        d.num_kv_heads = 1;
        d.max_tokens = capacity;
        d.device = device;
        check(qk_cache_create(&d, &cache_));
    }
    ~KvCache() {
        if (cache_) qk_cache_destroy(cache_);
    }
    KvCache(const KvCache&) = delete;
    KvCache& operator=(const KvCache&) = delete;
    KvCache(KvCache&& o) noexcept : config_(o.config_), cache_(o.cache_) { o.cache_ = nullptr; }

    // kv_store.cpp:19-47; returns the token index.
    uint32_t append(std::span<const float> key, std::span<const float> value) {
        if (key.size() != config_.head_dim || value.size() != config_.head_dim)
            throw std::invalid_argument("KvCache::append: vector dimension mismatch");
        const uint32_t t = token_count();
        ensure(uint64_t(t) + 1);
        const auto k = to_half(key), v = to_half(value);
        check(qk_append_host(cache_, 0, k.data(), v.data(), 1, nullptr));
        return t;
    }
    // n successive appends from [n][head_dim] rows (bulk prefill, same result).
    void extend(std::span<const float> keys, std::span<const float> values) {
        if (keys.size() != values.size() || keys.size() % config_.head_dim != 0)
            throw std::invalid_argument("KvCache::extend: shape mismatch");
        ensure(uint64_t(token_count()) + keys.size() / config_.head_dim);
        const auto k = to_half(keys), v = to_half(values);
        check(qk_prefill_host(cache_, 0, 0, k.data(), v.data(),
                              uint32_t(keys.size() / config_.head_dim), nullptr));
    }
    // kv_store.cpp:49-54 (out_of_range on a bad index).
    PageMetadata page_metadata(uint32_t page_index) const {
        if (page_index >= page_count())
            throw std::out_of_range("KvCache::page_metadata: page index out of range");
        std::vector<uint16_t> mn(config_.head_dim), mx(config_.head_dim);
        check(qk_read_metadata(cache_, 0, 0, 0, page_index, 1, mn.data(), mx.data(), nullptr));
        PageMetadata m;
        for (uint32_t c = 0; c < config_.head_dim; ++c) {
            m.min_key.push_back(half_to_float(mn[c]));
            m.max_key.push_back(half_to_float(mx[c]));
        }
        return m;
    }
    Page page(uint32_t page_index) const {
        if (page_index >= page_count()) throw std::out_of_range("KvCache::page: page index out of range");
        Page p;
        const uint32_t t0 = page_index * config_.page_size;
        p.length = std::min(config_.page_size, token_count() - t0);
        std::vector<uint16_t> k(size_t(p.length) * config_.head_dim), v(k.size());
        check(qk_read_kv(cache_, 0, 0, 0, t0, p.length, k.data(), v.data(), nullptr));
        for (size_t i = 0; i < k.size(); ++i) {
            p.keys.push_back(half_to_float(k[i]));
            p.values.push_back(half_to_float(v[i]));
        }
        p.metadata = page_metadata(page_index);
        return p;
    }
    std::vector<float> key(uint32_t token) const { return row(token, true); }
    std::vector<float> value(uint32_t token) const { return row(token, false); }

    const CacheConfig& config() const noexcept { return config_; }
    uint32_t token_count() const noexcept {
        uint32_t n = 0;
        qk_token_count(cache_, 0, 0, &n);
        return n;
    }
    uint32_t page_count() const noexcept {
        uint32_t n = 0;
        qk_page_count(cache_, 0, 0, &n);
        return n;
    }
    qk_cache* handle() const noexcept { return cache_; }

private:
    // Grows the slice (doubling) so that `tokens` fit: the reference's page vector growth.
    void ensure(uint64_t tokens) {
        qk_cache_desc d{};
        check(qk_cache_describe(cache_, &d));
        if (tokens <= d.max_tokens) return;
        const uint64_t cap = uint64_t(16384) * d.page_size;  // the ABI's page limit per slice
        const uint64_t want = std::max<uint64_t>(tokens, std::min<uint64_t>(2 * uint64_t(d.max_tokens), cap));
        check(qk_cache_reserve(cache_, uint32_t(std::min<uint64_t>(want, UINT32_MAX))));
    }
    std::vector<float> row(uint32_t token, bool want_key) const {
        if (token >= token_count()) throw std::out_of_range("KvCache::key: token out of range");
        std::vector<uint16_t> k(config_.head_dim), v(config_.head_dim);
        check(qk_read_kv(cache_, 0, 0, 0, token, 1, k.data(), v.data(), nullptr));
        std::vector<float> out;
        for (uint32_t c = 0; c < config_.head_dim; ++c) out.push_back(half_to_float(want_key ? k[c] : v[c]));
        return out;
    }
    CacheConfig config_;
    qk_cache* cache_ = nullptr;
};

// ---- criticality.hpp ------------------------------------------------------------------------
struct PageScore {  // criticality.hpp:13-16
    uint32_t page_index = 0;
    double score = 0.0;
};

struct SelectionConfig {  // criticality.hpp:18-22
    uint32_t token_budget = 0;
    bool force_include_recent = true;
    bool per_layer_enabled = true;
};

// estimate_all (criticality.cpp:25-34): bitwise the reference's doubles.
inline std::vector<PageScore> estimate_all(std::span<const float> query, const KvCache& cache) {
    if (cache.page_count() == 0) throw std::invalid_argument("estimate_all: empty cache");
    if (query.size() != cache.config().head_dim)
        throw std::invalid_argument("estimate_page_score: dimension mismatch");
    const auto q = to_half(query);
    const uint32_t P = cache.page_count();
    std::vector<double> s(P);
    check(qk_estimate_host(cache.handle(), 0, q.data(), 1, s.data(), P, nullptr));
    std::vector<PageScore> out(P);
    for (uint32_t p = 0; p < P; ++p) out[p] = {p, s[p]};
    return out;
}

// estimate_page_score (criticality.cpp:9-23) on explicit metadata, on the GPU (no cache).
inline double estimate_page_score(std::span<const float> query, const PageMetadata& metadata) {
    const uint32_t d = uint32_t(metadata.min_key.size());
    if (d == 0 || query.size() != d || metadata.max_key.size() != d)
        throw std::invalid_argument("estimate_page_score: dimension mismatch");
    const auto q = to_half(query), mn = to_half(metadata.min_key), mx = to_half(metadata.max_key);
    int dev = 0;
    double score = 0.0;
    check(qk_estimate_metadata_host(q.data(), mn.data(), mx.data(), 1, d, &score, dev));
    return score;
}

// select_top_k (criticality.cpp:36-81), same early-exit order and errors.  estimate_all's
// form (one score per page, in page order) takes the radix top-K kernel; any other vector
// (any order, repeated pages) the pair-sorting kernel -- both on the GPU.
inline std::vector<uint32_t> select_top_k(const std::vector<PageScore>& scores,
                                          const SelectionConfig& config, const KvCache& cache) {
    const uint32_t P = cache.page_count();
    std::vector<uint32_t> all(P);
    for (uint32_t p = 0; p < P; ++p) all[p] = p;
    if (!config.per_layer_enabled) return all;
    if (config.token_budget < cache.config().page_size)
        throw std::invalid_argument("select_top_k: token_budget below page_size");
    if (scores.empty()) throw std::invalid_argument("select_top_k: no scores");
    for (const PageScore& s : scores)
        if (s.page_index >= P) throw std::out_of_range("select_top_k: score for nonexistent page");
    qk_selection_cfg cfg{config.token_budget, config.force_include_recent ? 1 : 0, 1};
    bool page_order = scores.size() == P;
    for (uint32_t p = 0; page_order && p < P; ++p) page_order = scores[p].page_index == p;
    if (page_order) {
        std::vector<double> s(P);
        for (uint32_t p = 0; p < P; ++p) s[p] = scores[p].score;
        std::vector<int32_t> pages(P);
        int32_t count = 0;
        check(qk_select_topk_host(cache.handle(), 0, s.data(), P, 1, &cfg, pages.data(), P, &count,
                                  nullptr));
        return std::vector<uint32_t>(pages.begin(), pages.begin() + count);
    }
    std::vector<uint32_t> idx(scores.size());
    std::vector<double> s(scores.size());
    for (size_t i = 0; i < scores.size(); ++i) {
        idx[i] = scores[i].page_index;
        s[i] = scores[i].score;
    }
    const uint32_t cap = std::max<uint32_t>({P, config.token_budget / cache.config().page_size, 1u});
    std::vector<int32_t> pages(cap);
    int32_t count = 0;
    check(qk_select_topk_pairs_host(cache.handle(), 0, 0, idx.data(), s.data(), uint32_t(s.size()),
                                    &cfg, pages.data(), cap, &count, nullptr));
    return std::vector<uint32_t>(pages.begin(), pages.begin() + count);
}

// ---- attention.hpp --------------------------------------------------------------------------
using LogitVector = std::vector<double>;  // attention.hpp:13

struct AttentionOutput {  // attention.hpp:15-18
    std::vector<double> output;
    double weights_sum_check = 0.0;
};

namespace detail {
// check_token_set (attention.cpp:19-30), same messages and exception types.
inline void check_token_set(const KvCache& cache, std::span<const uint32_t> tokens) {
    if (tokens.empty()) throw std::invalid_argument("attention: empty token set");
    const uint32_t n = cache.token_count();
    for (size_t i = 0; i < tokens.size(); ++i) {
        if (tokens[i] >= n) throw std::out_of_range("attention: token index out of range");
        if (i > 0 && tokens[i] <= tokens[i - 1])
            throw std::invalid_argument("attention: token set must be strictly ascending");
    }
}
}  // namespace detail

// attention_logits (attention.cpp:34-46): q.k_t / sqrt(d) over token_subset, bitwise.
inline LogitVector attention_logits(std::span<const float> query, const KvCache& cache,
                                    std::span<const uint32_t> token_subset) {
    detail::check_token_set(cache, token_subset);
    if (query.size() != cache.config().head_dim)
        throw std::invalid_argument("attention_logits: query dimension mismatch");
    const auto q = to_half(query);
    const std::vector<int32_t> toks(token_subset.begin(), token_subset.end());
    const int32_t count = int32_t(toks.size());
    LogitVector logits(toks.size());
    check(qk_attention_logits_host(cache.handle(), 0, q.data(), 1, toks.data(), uint32_t(toks.size()),
                                   &count, logits.data(), uint32_t(toks.size()), nullptr));
    return logits;
}

// attention_logits over every cached token (attention.cpp:48-52).
inline LogitVector attention_logits(std::span<const float> query, const KvCache& cache) {
    const uint32_t n = cache.token_count();
    if (n == 0) throw std::invalid_argument("attention: empty token set");
    if (query.size() != cache.config().head_dim)
        throw std::invalid_argument("attention_logits: query dimension mismatch");
    const auto q = to_half(query);
    LogitVector logits(n);
    check(qk_attention_logits_host(cache.handle(), 0, q.data(), 1, nullptr, 0, nullptr,
                                   logits.data(), n, nullptr));
    return logits;
}

// softmax_weights (attention.cpp:54-67), on the current CUDA device.
inline std::vector<double> softmax_weights(const LogitVector& logits) {
    if (logits.empty()) throw std::invalid_argument("softmax_weights: empty logits");
    std::vector<double> w(logits.size());
    int dev = 0;
    check(qk_softmax_weights_host(logits.data(), uint32_t(logits.size()), w.data(), dev));
    return w;
}

// attend_tokens (attention.cpp:69-84): attention over an explicit strictly ascending token set.
inline AttentionOutput attend_tokens(std::span<const float> query, const KvCache& cache,
                                     std::span<const uint32_t> tokens) {
    detail::check_token_set(cache, tokens);
    if (query.size() != cache.config().head_dim)
        throw std::invalid_argument("attention_logits: query dimension mismatch");
    const auto q = to_half(query);
    const std::vector<int32_t> toks(tokens.begin(), tokens.end());
    const int32_t count = int32_t(toks.size());
    std::vector<float> out(cache.config().head_dim);
    double wsum = 0.0;
    check(qk_attend_tokens_host(cache.handle(), 0, q.data(), 1, toks.data(), uint32_t(toks.size()),
                                &count, out.data(), nullptr, &wsum, nullptr));
    return {std::vector<double>(out.begin(), out.end()), wsum};
}

inline AttentionOutput full_attention(std::span<const float> query, const KvCache& cache) {
    if (cache.token_count() == 0) throw std::invalid_argument("full_attention: empty cache");
    if (query.size() != cache.config().head_dim)
        throw std::invalid_argument("attention: query dimension mismatch");
    const auto q = to_half(query);
    std::vector<float> out(cache.config().head_dim);
    double wsum = 0.0;
    check(qk_dense_attend_host(cache.handle(), 0, q.data(), 1, out.data(), nullptr, &wsum, nullptr));
    return {std::vector<double>(out.begin(), out.end()), wsum};
}

// sparse_attention (attention.cpp:94-116): any order accepted; empty -> invalid_argument,
// out of range -> out_of_range, duplicate -> invalid_argument.
inline AttentionOutput sparse_attention(std::span<const float> query, const KvCache& cache,
                                        std::span<const uint32_t> selected_pages) {
    if (selected_pages.empty()) throw std::invalid_argument("sparse_attention: empty page selection");
    if (query.size() != cache.config().head_dim)
        throw std::invalid_argument("attention: query dimension mismatch");
    std::vector<int32_t> pages(selected_pages.begin(), selected_pages.end());
    std::sort(pages.begin(), pages.end());
    for (size_t i = 0; i < pages.size(); ++i) {
        if (uint32_t(pages[i]) >= cache.page_count())
            throw std::out_of_range("sparse_attention: page index out of range");
        if (i > 0 && pages[i] == pages[i - 1])
            throw std::invalid_argument("sparse_attention: duplicate page index");
    }
    const auto q = to_half(query);
    const int32_t count = int32_t(pages.size());
    std::vector<float> out(cache.config().head_dim);
    double wsum = 0.0;
    check(qk_sparse_attend_host(cache.handle(), 0, q.data(), 1, pages.data(),
                                uint32_t(pages.size()), &count, out.data(), nullptr, &wsum,
                                nullptr));
    return {std::vector<double>(out.begin(), out.end()), wsum};
}

// ---- metrics.hpp (the byte model of the roofline) ------------------------------------------
inline double traffic_fraction(uint32_t page_size, uint64_t token_count, uint64_t token_budget) {
    if (page_size == 0) throw std::invalid_argument("traffic_fraction: zero page_size");
    if (token_count == 0 || token_budget == 0)
        throw std::invalid_argument("traffic_fraction: counts must be positive");
    if (token_budget > token_count)
        throw std::invalid_argument("traffic_fraction: budget exceeds token count");
    const uint64_t k = token_budget / page_size;
    return 1.0 / double(page_size) + double(k * page_size) / double(token_count);
}

// ---- the batched serving object -------------------------------------------------------------
// Every (layer, sequence, KV head) cache of a model in HBM; decode_step is the fused
// append -> estimate -> top-K -> attend launch (one kernel per layer step).
class DeviceCache {
public:
    explicit DeviceCache(const qk_cache_desc& desc) { check(qk_cache_create(&desc, &cache_)); }
    ~DeviceCache() {
        if (cache_) qk_cache_destroy(cache_);
    }
    DeviceCache(const DeviceCache&) = delete;
    DeviceCache& operator=(const DeviceCache&) = delete;
    qk_cache* handle() const noexcept { return cache_; }

    // Device pointers (fp16 bits), asynchronous on `stream`.
    void decode_step(uint32_t layer, const uint16_t* q, const uint16_t* k, const uint16_t* v,
                     uint32_t batch, const SelectionConfig& sel, float* out,
                     void* stream = nullptr) {
        qk_selection_cfg cfg{sel.token_budget, sel.force_include_recent ? 1 : 0,
                             sel.per_layer_enabled ? 1 : 0};
        check(qk_decode_step(cache_, layer, q, k, v, batch, &cfg, out, QK_DTYPE_F32, nullptr, 0,
                             nullptr, stream));
    }
    // Host buffers, synchronous.
    void decode_step_host(uint32_t layer, const uint16_t* q, const uint16_t* k,
                          const uint16_t* v, uint32_t batch, const SelectionConfig& sel,
                          float* out, void* stream = nullptr) {
        qk_selection_cfg cfg{sel.token_budget, sel.force_include_recent ? 1 : 0,
                             sel.per_layer_enabled ? 1 : 0};
        check(qk_decode_step_host(cache_, layer, q, k, v, batch, &cfg, out, stream));
    }
    void prefill_host(uint32_t layer, uint32_t seq, const uint16_t* k, const uint16_t* v,
                      uint32_t n_tokens, void* stream = nullptr) {
        check(qk_prefill_host(cache_, layer, seq, k, v, n_tokens, stream));
    }
    // Grow every slice to max_tokens (qk_cache_reserve; device copy, graphs re-captured).
    void reserve(uint32_t max_tokens) { check(qk_cache_reserve(cache_, max_tokens)); }

private:
    qk_cache* cache_ = nullptr;
};

}  // namespace questkv_b200

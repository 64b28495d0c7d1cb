// compat_check.cpp -- one driver, two builds (oracle/Makefile, target `compat`):
//   compat_check_ref : against the UNMODIFIED reference library (R/core/src/*.cpp);
//   compat_check_b200: the reference's own metrics.cpp and policies.cpp compiled UNCHANGED
//                      against include/questkv_compat (questkv:: -> questkv_b200::, the GPU
//                      library).
// It uses only the reference's questkv:: API (kv_store/criticality/attention/metrics/
// policies.hpp) on the same seeded fp16-representable inputs and prints one JSON object;
// tests/test_cpp_layer.py compares the two (pages, logits, scores, recall, byte counts and
// policy token sets exactly; outputs within 1e-5 relative L2; softmax weights 1e-12).
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <numeric>
#include <random>
#include <string>
#include <vector>

#include "questkv/attention.hpp"
#include "questkv/criticality.hpp"
#include "questkv/kv_store.hpp"
#include "questkv/metrics.hpp"
#include "questkv/policies.hpp"

namespace {

float f16(float x) { return static_cast<float>(static_cast<_Float16>(x)); }

std::vector<float> rand_vec(std::mt19937& rng, size_t n, float sd) {
    std::normal_distribution<float> nd(0.0f, sd);
    std::vector<float> v(n);
    for (auto& x : v) x = f16(nd(rng));
    return v;
}

void put(const char* key, const std::vector<double>& v, bool last = false) {
    std::printf("\"%s\": [", key);
    for (size_t i = 0; i < v.size(); ++i) std::printf("%s%.17g", i ? ", " : "", v[i]);
    std::printf("]%s\n", last ? "" : ",");
}
template <typename T>
void put_int(const char* key, const std::vector<T>& v) {
    std::printf("\"%s\": [", key);
    for (size_t i = 0; i < v.size(); ++i) std::printf("%s%lld", i ? ", " : "", (long long)v[i]);
    std::printf("],\n");
}

}  // namespace

int main() {
    using namespace questkv;
    const uint32_t d = 64, S = 16, L = 1500;
    const float sd = 1.0f / std::sqrt(float(d));
    std::mt19937 rng(2406);
    KvCache cache(CacheConfig{d, S, 2});
    for (uint32_t t = 0; t < L; ++t) {
        const auto k = rand_vec(rng, d, sd), v = rand_vec(rng, d, sd);
        cache.append(k, v);
    }
    const auto q = rand_vec(rng, d, sd);
    std::printf("{\n");

    // criticality: scores, page-order selection, arbitrary PageScore vectors.
    const auto scores = estimate_all(q, cache);
    std::vector<double> sv;
    for (const auto& s : scores) sv.push_back(s.score);
    put("scores", sv);
    const SelectionConfig sel{256, true, true};
    put_int("pages", select_top_k(scores, sel, cache));
    std::vector<PageScore> shuffled(scores.rbegin(), scores.rend());
    shuffled.push_back(scores[3]);  // a repeated page
    shuffled.push_back({7, 1e9});
    put_int("pages_shuffled", select_top_k(shuffled, sel, cache));
    put_int("pages_shuffled_noforce", select_top_k(shuffled, SelectionConfig{256, false, true}, cache));
    std::vector<PageScore> few = {{5, 0.0}, {2, -0.0}, {9, 0.0}, {2, 1.5}};
    put_int("pages_few", select_top_k(few, SelectionConfig{32, true, true}, cache));
    put_int("pages_few_all", select_top_k(few, SelectionConfig{4096, true, true}, cache));

    // attention.hpp
    const auto pages = select_top_k(scores, sel, cache);
    const auto sparse = sparse_attention(q, cache, pages);
    put("sparse", sparse.output);
    put("sparse_wsum", {sparse.weights_sum_check});
    const auto full = full_attention(q, cache);
    put("full", full.output);
    put("full_wsum", {full.weights_sum_check});
    std::vector<uint32_t> toks;
    for (uint32_t t = 3; t < L; t += 7) toks.push_back(t);
    const auto at = attend_tokens(q, cache, toks);
    put("tokens", at.output);
    put("tokens_wsum", {at.weights_sum_check});
    put("logits_all", attention_logits(q, cache));
    put("logits_sub", attention_logits(q, cache, toks));
    put("softmax_sub", softmax_weights(attention_logits(q, cache, toks)));

    // metrics.cpp (compiled unchanged in the b200 build)
    std::vector<uint32_t> sel_tokens;
    for (uint32_t p : pages)
        for (uint32_t r = 0; r < cache.page(p).length; ++r) sel_tokens.push_back(p * S + r);
    put("recall", {recall_at_n(sel_tokens, q, cache, 10), recall_at_n(sel_tokens, q, cache, 100)});
    const auto run = run_instrumented_quest_step(q, cache, sel);
    const auto rep = counted_bytes(run);
    put_int("bytes", std::vector<uint64_t>{run.metadata_bytes, run.kv_bytes, run.bytes_full,
                                           rep.bytes_loaded_counted});
    put("fraction_model", {rep.fraction_model});
    put_int("oracle_sparsity", std::vector<uint64_t>{oracle_sparsity(q, cache, 0.5),
                                                     oracle_sparsity(q, cache, 0.9)});
    put("output_error", {output_error(sparse.output, full.output)});

    // policies.cpp (compiled unchanged in the b200 build): a few decode steps per policy.
    std::vector<PolicyState> pols = {make_full_policy(), make_quest_policy(sel),
                                     make_h2o_policy(64, 8), make_tova_policy(64),
                                     make_streaming_policy(4, 60)};
    std::vector<std::vector<uint32_t>> sets(pols.size());
    for (int step = 0; step < 6; ++step) {
        const auto k = rand_vec(rng, d, sd), v = rand_vec(rng, d, sd), qq = rand_vec(rng, d, sd);
        const uint32_t t = cache.append(k, v);
        for (size_t i = 0; i < pols.size(); ++i) sets[i] = policy_step(pols[i], qq, cache, t);
    }
    for (size_t i = 0; i < pols.size(); ++i) {
        const std::string key = std::string("policy_") + policy_name(pols[i].kind);
        put_int(key.c_str(), sets[i]);
    }
    put("h2o_scores", pols[2].accumulated_scores, true);
    std::printf("}\n");
    return 0;
}

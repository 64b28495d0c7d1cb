/*
 * questkv_oracle.h -- CPU restatement of the Quest (arXiv 2406.10774) decode hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the parity checker for the CUDA path in
 * paper_2406_10774_b200/.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  The product path never links,
 * calls or falls back to anything under oracle/.
 *
 * Every function restates one reference function; the file:line it follows is given
 * beside it (paths relative to /root/reference/proj/).  Arithmetic is the reference's:
 * float storage, double accumulation in fixed ascending order, std::exp -> libm exp,
 * compiled without FMA contraction (-ffp-contract=off) so that it is bit-identical to
 * the reference built with g++ -O3 on x86-64 (no -mfma).
 *
 * Parity is pinned two ways (see tests/test_oracle.py):
 *   1. the reference's own known-answer tests (tests/test_*.cpp) restated as pytest cases;
 *   2. golden vectors produced by the real reference, compiled from /root/reference by
 *      oracle/Makefile into oracle/_ref/, committed under tests/golden/.
 */
#ifndef QUESTKV_ORACLE_H
#define QUESTKV_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    QO_OK = 0,
    QO_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
    QO_ERR_OUT_OF_RANGE = 2      /* std::out_of_range in the reference     */
};

/* CacheConfig::validate (core/src/kv_store.cpp:8-13). */
int qo_validate_config(uint32_t head_dim, uint32_t page_size, uint32_t bytes_per_element);

/* Page metadata after appending keys[0..n_tokens) one at a time through
 * KvCache::append (core/src/kv_store.cpp:19-47): page p covers tokens [p*S, p*S+S);
 * the first key seeds min=max (kv_store.cpp:35-38); later keys update with strict
 * '<' / '>' (kv_store.cpp:40-43).  keys: [n_tokens][dim] row-major.
 * min_out/max_out: [ceil(n/S)][dim]. */
void qo_build_metadata(const float *keys, uint32_t n_tokens, uint32_t dim,
                       uint32_t page_size, float *min_out, float *max_out);

/* estimate_page_score (core/src/criticality.cpp:9-23). */
double qo_estimate_page_score(const float *query, const float *min_key,
                              const float *max_key, uint32_t dim);

/* estimate_all (core/src/criticality.cpp:25-34); min/max: [n_pages][dim].
 * Returns QO_ERR_INVALID_ARGUMENT for an empty cache (n_pages == 0). */
int qo_estimate_all(const float *query, const float *min_keys, const float *max_keys,
                    uint32_t n_pages, uint32_t dim, double *scores_out);

/* select_top_k (core/src/criticality.cpp:36-81) for scores of pages 0..n_pages-1.
 * Writes the selected pages, ascending, to out (capacity n_pages) and the count to
 * *count.  Same early exits and errors as the reference, in the same order. */
int qo_select_top_k(const double *scores, uint32_t n_pages, uint32_t page_size,
                    uint32_t token_budget, int force_include_recent,
                    int per_layer_enabled, uint32_t *out, uint32_t *count);

/* attend_tokens (core/src/attention.cpp:69-84) over an explicit strictly ascending
 * token set; keys/values: [n_tokens][dim].  Errors as check_token_set (:19-30). */
int qo_attend_tokens(const float *query, const float *keys, const float *values,
                     uint32_t n_tokens, uint32_t dim, const uint32_t *tokens,
                     uint32_t n_sel, double *out, double *weights_sum_check);

/* sparse_attention (core/src/attention.cpp:94-116): pages in any order, validated
 * (empty -> invalid_argument, out of range -> out_of_range, duplicate ->
 * invalid_argument), expanded to tokens using each page's length. */
int qo_sparse_attention(const float *query, const float *keys, const float *values,
                        uint32_t n_tokens, uint32_t dim, uint32_t page_size,
                        const uint32_t *pages, uint32_t n_pages_sel, double *out,
                        double *weights_sum_check);

/* full_attention (core/src/attention.cpp:86-92). */
int qo_full_attention(const float *query, const float *keys, const float *values,
                      uint32_t n_tokens, uint32_t dim, double *out,
                      double *weights_sum_check);

/* reference::naive_attention (core/src/reference.cpp:9-41): long double, no max
 * subtraction. */
int qo_naive_attention(const float *query, const float *keys, const float *values,
                       uint32_t n_tokens, uint32_t dim, const uint32_t *tokens,
                       uint32_t n_sel, double *out);

/* One Quest step for one head (metrics.cpp:90-95: estimate_all -> select_top_k ->
 * sparse_attention) given the cache as flat arrays.  pages_out capacity: n_pages. */
int qo_quest_step(const float *query, const float *keys, const float *values,
                  uint32_t n_tokens, uint32_t dim, uint32_t page_size,
                  uint32_t token_budget, int force_include_recent, int per_layer_enabled,
                  double *scores_out, uint32_t *pages_out, uint32_t *n_selected,
                  double *out);

/* Byte accounting (core/src/metrics.cpp:54-66 and :90-108). */
double qo_traffic_fraction(uint32_t page_size, uint64_t token_count, uint64_t token_budget);
uint64_t qo_quest_step_bytes(uint32_t dim, uint32_t bytes_per_element, uint32_t n_pages,
                             uint64_t attended_tokens);

#ifdef __cplusplus
}
#endif
#endif /* QUESTKV_ORACLE_H */

/*
 * questkv_oracle.c -- CPU restatement of the Quest decode hot path (TEST INFRASTRUCTURE).
 * See questkv_oracle.h for the contract.  Citations are relative to
 * /root/reference/proj/.  Build: oracle/Makefile (gcc -O2 -ffp-contract=off).
 */
#include "questkv_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* kv_store.cpp:8-13 */
int qo_validate_config(uint32_t head_dim, uint32_t page_size, uint32_t bytes_per_element) {
    if (head_dim == 0 || page_size == 0 || bytes_per_element == 0)
        return QO_ERR_INVALID_ARGUMENT;
    return QO_OK;
}

/* kv_store.cpp:19-47 -- metadata as produced by successive appends. */
void qo_build_metadata(const float *keys, uint32_t n_tokens, uint32_t dim,
                       uint32_t page_size, float *min_out, float *max_out) {
    for (uint32_t t = 0; t < n_tokens; ++t) {
        const uint32_t page = t / page_size;
        const uint32_t row = t % page_size;
        const float *key = keys + (size_t)t * dim;
        float *mn = min_out + (size_t)page * dim;
        float *mx = max_out + (size_t)page * dim;
        if (row == 0) { /* first key of the page seeds the metadata (:35-38) */
            memcpy(mn, key, sizeof(float) * dim);
            memcpy(mx, key, sizeof(float) * dim);
        } else { /* strict compares keep the first-seen value on ties (:40-43) */
            for (uint32_t i = 0; i < dim; ++i) {
                if (key[i] < mn[i]) mn[i] = key[i];
                if (key[i] > mx[i]) mx[i] = key[i];
            }
        }
    }
}

/* criticality.cpp:9-23 -- std::max(a, b) is (a < b) ? b : a. */
double qo_estimate_page_score(const float *query, const float *min_key,
                              const float *max_key, uint32_t dim) {
    double score = 0.0;
    for (uint32_t i = 0; i < dim; ++i) {
        const double q = query[i];
        const double a = q * (double)max_key[i];
        const double b = q * (double)min_key[i];
        score += (a < b) ? b : a;
    }
    return score;
}

/* criticality.cpp:25-34 */
int qo_estimate_all(const float *query, const float *min_keys, const float *max_keys,
                    uint32_t n_pages, uint32_t dim, double *scores_out) {
    if (n_pages == 0) return QO_ERR_INVALID_ARGUMENT;
    for (uint32_t p = 0; p < n_pages; ++p)
        scores_out[p] = qo_estimate_page_score(query, min_keys + (size_t)p * dim,
                                               max_keys + (size_t)p * dim, dim);
    return QO_OK;
}

/* Ordering of criticality.cpp:62-67: score descending, lower page index first. */
static const double *g_sort_scores; /* qsort has no context argument */
static int by_score_desc_then_index(const void *pa, const void *pb) {
    const uint32_t a = *(const uint32_t *)pa, b = *(const uint32_t *)pb;
    const double sa = g_sort_scores[a], sb = g_sort_scores[b];
    if (sa != sb) return sa > sb ? -1 : 1;
    return a < b ? -1 : (a > b ? 1 : 0);
}
static int by_index(const void *pa, const void *pb) {
    const uint32_t a = *(const uint32_t *)pa, b = *(const uint32_t *)pb;
    return a < b ? -1 : (a > b ? 1 : 0);
}

/* criticality.cpp:36-81 */
int qo_select_top_k(const double *scores, uint32_t n_pages, uint32_t page_size,
                    uint32_t token_budget, int force_include_recent,
                    int per_layer_enabled, uint32_t *out, uint32_t *count) {
    *count = 0;
    if (!per_layer_enabled) { /* :47 */
        for (uint32_t p = 0; p < n_pages; ++p) out[p] = p;
        *count = n_pages;
        return QO_OK;
    }
    if (token_budget < page_size) return QO_ERR_INVALID_ARGUMENT; /* :50-51 */
    if (n_pages == 0) return QO_ERR_INVALID_ARGUMENT;            /* :52-53 */
    const uint32_t k = token_budget / page_size;                 /* :58 */
    if (k >= n_pages) {                                          /* :59 */
        for (uint32_t p = 0; p < n_pages; ++p) out[p] = p;
        *count = n_pages;
        return QO_OK;
    }
    uint32_t *order = (uint32_t *)malloc(sizeof(uint32_t) * n_pages);
    for (uint32_t p = 0; p < n_pages; ++p) order[p] = p;
    g_sort_scores = scores;
    qsort(order, n_pages, sizeof(uint32_t), by_score_desc_then_index); /* :62-67 */
    for (uint32_t i = 0; i < k; ++i) out[i] = order[i];                /* :69-71 */
    free(order);
    if (force_include_recent) { /* :73-77 */
        const uint32_t last = n_pages - 1;
        int found = 0;
        for (uint32_t i = 0; i < k; ++i) found |= (out[i] == last);
        if (!found) out[k - 1] = last; /* drop the weakest pick */
    }
    qsort(out, k, sizeof(uint32_t), by_index); /* :79 */
    *count = k;
    return QO_OK;
}

/* attention.cpp:19-30 */
static int check_token_set(uint32_t n_tokens, const uint32_t *tokens, uint32_t n_sel) {
    if (n_sel == 0) return QO_ERR_INVALID_ARGUMENT;
    for (uint32_t i = 0; i < n_sel; ++i) {
        if (tokens[i] >= n_tokens) return QO_ERR_OUT_OF_RANGE;
        if (i > 0 && tokens[i] <= tokens[i - 1]) return QO_ERR_INVALID_ARGUMENT;
    }
    return QO_OK;
}

/* attention.cpp:12-17 */
static double dot(const float *a, const float *b, uint32_t dim) {
    double acc = 0.0;
    for (uint32_t i = 0; i < dim; ++i) acc += (double)a[i] * (double)b[i];
    return acc;
}

/* attention.cpp:34-52 (logits), :54-67 (softmax), :69-84 (weighted sum). */
int qo_attend_tokens(const float *query, const float *keys, const float *values,
                     uint32_t n_tokens, uint32_t dim, const uint32_t *tokens,
                     uint32_t n_sel, double *out, double *weights_sum_check) {
    const int err = check_token_set(n_tokens, tokens, n_sel);
    if (err) return err;
    const double scale = sqrt((double)dim);
    double *w = (double *)malloc(sizeof(double) * n_sel);
    for (uint32_t i = 0; i < n_sel; ++i)
        w[i] = dot(query, keys + (size_t)tokens[i] * dim, dim) / scale;
    double peak = w[0]; /* std::max_element: first maximum */
    for (uint32_t i = 1; i < n_sel; ++i)
        if (peak < w[i]) peak = w[i];
    double total = 0.0;
    for (uint32_t i = 0; i < n_sel; ++i) {
        w[i] = exp(w[i] - peak);
        total += w[i];
    }
    for (uint32_t i = 0; i < n_sel; ++i) w[i] /= total;
    for (uint32_t c = 0; c < dim; ++c) out[c] = 0.0;
    double wsum = 0.0;
    for (uint32_t i = 0; i < n_sel; ++i) {
        const float *v = values + (size_t)tokens[i] * dim;
        for (uint32_t c = 0; c < dim; ++c) out[c] += w[i] * (double)v[c];
        wsum += w[i];
    }
    if (weights_sum_check) *weights_sum_check = wsum;
    free(w);
    return QO_OK;
}

static int by_u32(const void *pa, const void *pb) { return by_index(pa, pb); }

/* attention.cpp:94-116 */
int qo_sparse_attention(const float *query, const float *keys, const float *values,
                        uint32_t n_tokens, uint32_t dim, uint32_t page_size,
                        const uint32_t *pages, uint32_t n_pages_sel, double *out,
                        double *weights_sum_check) {
    if (n_pages_sel == 0) return QO_ERR_INVALID_ARGUMENT;
    const uint32_t n_pages = (n_tokens + page_size - 1) / page_size;
    uint32_t *sorted = (uint32_t *)malloc(sizeof(uint32_t) * n_pages_sel);
    memcpy(sorted, pages, sizeof(uint32_t) * n_pages_sel);
    qsort(sorted, n_pages_sel, sizeof(uint32_t), by_u32);
    for (uint32_t i = 0; i < n_pages_sel; ++i) {
        if (sorted[i] >= n_pages) { free(sorted); return QO_ERR_OUT_OF_RANGE; }
        if (i > 0 && sorted[i] == sorted[i - 1]) { free(sorted); return QO_ERR_INVALID_ARGUMENT; }
    }
    uint32_t *tokens = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)n_pages_sel * page_size);
    uint32_t n_sel = 0;
    for (uint32_t i = 0; i < n_pages_sel; ++i) {
        const uint32_t first = sorted[i] * page_size;
        const uint32_t length =
            (sorted[i] == n_pages - 1) ? n_tokens - (n_pages - 1) * page_size : page_size;
        for (uint32_t row = 0; row < length; ++row) tokens[n_sel++] = first + row;
    }
    const int err = qo_attend_tokens(query, keys, values, n_tokens, dim, tokens, n_sel, out,
                                     weights_sum_check);
    free(tokens);
    free(sorted);
    return err;
}

/* attention.cpp:86-92 */
int qo_full_attention(const float *query, const float *keys, const float *values,
                      uint32_t n_tokens, uint32_t dim, double *out,
                      double *weights_sum_check) {
    if (n_tokens == 0) return QO_ERR_INVALID_ARGUMENT;
    uint32_t *tokens = (uint32_t *)malloc(sizeof(uint32_t) * n_tokens);
    for (uint32_t t = 0; t < n_tokens; ++t) tokens[t] = t;
    const int err = qo_attend_tokens(query, keys, values, n_tokens, dim, tokens, n_tokens,
                                     out, weights_sum_check);
    free(tokens);
    return err;
}

/* reference.cpp:9-41 */
int qo_naive_attention(const float *query, const float *keys, const float *values,
                       uint32_t n_tokens, uint32_t dim, const uint32_t *tokens,
                       uint32_t n_sel, double *out) {
    if (n_sel == 0) return QO_ERR_INVALID_ARGUMENT;
    for (uint32_t i = 0; i < n_sel; ++i)
        if (tokens[i] >= n_tokens) return QO_ERR_OUT_OF_RANGE;
    const long double scale = sqrtl((long double)dim);
    long double *e = (long double *)malloc(sizeof(long double) * n_sel);
    long double normalizer = 0.0L;
    for (uint32_t i = 0; i < n_sel; ++i) {
        const float *k = keys + (size_t)tokens[i] * dim;
        long double logit = 0.0L;
        for (uint32_t c = 0; c < dim; ++c) logit += (long double)query[c] * (long double)k[c];
        e[i] = expl(logit / scale);
        normalizer += e[i];
    }
    long double *acc = (long double *)calloc(dim, sizeof(long double));
    for (uint32_t i = 0; i < n_sel; ++i) {
        const long double weight = e[i] / normalizer;
        const float *v = values + (size_t)tokens[i] * dim;
        for (uint32_t c = 0; c < dim; ++c) acc[c] += weight * (long double)v[c];
    }
    for (uint32_t c = 0; c < dim; ++c) out[c] = (double)acc[c];
    free(acc);
    free(e);
    return QO_OK;
}

/* metrics.cpp:90-95 */
int qo_quest_step(const float *query, const float *keys, const float *values,
                  uint32_t n_tokens, uint32_t dim, uint32_t page_size,
                  uint32_t token_budget, int force_include_recent, int per_layer_enabled,
                  double *scores_out, uint32_t *pages_out, uint32_t *n_selected,
                  double *out) {
    const uint32_t n_pages = (n_tokens + page_size - 1) / page_size;
    if (n_pages == 0) return QO_ERR_INVALID_ARGUMENT;
    float *mn = (float *)malloc(sizeof(float) * (size_t)n_pages * dim);
    float *mx = (float *)malloc(sizeof(float) * (size_t)n_pages * dim);
    qo_build_metadata(keys, n_tokens, dim, page_size, mn, mx);
    int err = qo_estimate_all(query, mn, mx, n_pages, dim, scores_out);
    free(mn);
    free(mx);
    if (err) return err;
    err = qo_select_top_k(scores_out, n_pages, page_size, token_budget, force_include_recent,
                          per_layer_enabled, pages_out, n_selected);
    if (err) return err;
    return qo_sparse_attention(query, keys, values, n_tokens, dim, page_size, pages_out,
                               *n_selected, out, 0);
}

/* metrics.cpp:54-66 */
double qo_traffic_fraction(uint32_t page_size, uint64_t token_count, uint64_t token_budget) {
    const uint64_t k = token_budget / page_size;
    return 1.0 / (double)page_size + (double)(k * page_size) / (double)token_count;
}

/* metrics.cpp:105-106: metadata 2*d*bpe per page, KV 2*d*bpe per attended token. */
uint64_t qo_quest_step_bytes(uint32_t dim, uint32_t bytes_per_element, uint32_t n_pages,
                             uint64_t attended_tokens) {
    const uint64_t vec = (uint64_t)dim * bytes_per_element;
    return 2 * vec * n_pages + 2 * vec * attended_tokens;
}

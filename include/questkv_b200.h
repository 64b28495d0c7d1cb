/*
 * questkv_b200.h -- C ABI of the B200-native Quest decode hot path.
 *
 * This is the drop-in boundary for the reference's C++ operator API (questkv::,
 * /root/reference/proj/core/include/questkv/).  Every entry point below names the
 * reference interface it replaces (file:line).  The reference works on ONE attention
 * head per KvCache with float vectors on the host; this ABI is batched and
 * device-resident: one qk_cache holds every (layer, sequence, KV head) cache of a model,
 * with fp16 pages and fp16 per-page min/max key metadata in HBM.  A (layer, sequence,
 * KV head) slice of a qk_cache behaves exactly like one questkv::KvCache fed the same
 * values widened to float.
 *
 * Conventions
 *   - Plain C: pointers, sizes, POD structs.  fp16 tensors are passed as uint16_t
 *     (IEEE binary16 bit patterns); device pointers unless the name says _host.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).  Every
 *     call is asynchronous and ordered on `stream` unless documented as synchronous;
 *     that ordering is the reference's single-writer rule (kv_store.hpp:39-40).
 *   - Every call returns an int status.  No C++ exception crosses this boundary:
 *       QK_OK                    success
 *       QK_ERR_INVALID_ARGUMENT  where the reference throws std::invalid_argument
 *       QK_ERR_OUT_OF_RANGE      where the reference throws std::out_of_range
 *       QK_ERR_CUDA              a CUDA runtime error (message in qk_last_error())
 *       QK_ERR_UNSUPPORTED       a geometry the kernels are not built for
 *     qk_last_error() returns the calling thread's last message.
 *   - No CPU fallback exists: every compute entry point launches sm_100a kernels.
 *
 * Tensor layouts (caller-owned, device):
 *   q      [batch][num_q_heads][head_dim]            fp16
 *   k, v   [batch][num_kv_heads][head_dim]            fp16 (one new token per sequence)
 *   scores [batch][num_q_heads][scores_stride]        f64, scores_stride >= max_pages
 *   pages  [batch][num_q_heads][pages_stride]         int32, ascending page indices
 *   counts [batch][num_q_heads]                       int32
 *   out    [batch][num_q_heads][head_dim]             f32 or fp16 (qk_dtype)
 *   lse    [batch][num_q_heads]                       f32 natural-log LSE of logits/sqrt(d)
 *   weights_sum [batch][num_q_heads]                  f64 AttentionOutput::weights_sum_check
 *   tokens [batch][num_q_heads][tokens_stride]        int32, strictly ascending token indices
 *   logits [batch][num_q_heads][logits_stride]        f64
 * Query head h reads KV head h / (num_q_heads / num_kv_heads) (GQA); every query head
 * selects its own pages (the reference's single-head semantics applied per query head).
 */
#ifndef QUESTKV_B200_H
#define QUESTKV_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QK_ABI_VERSION 2

#if defined(__GNUC__)
#define QK_API __attribute__((visibility("default")))
#else
#define QK_API
#endif

enum qk_status {
    QK_OK = 0,
    QK_ERR_INVALID_ARGUMENT = 1,
    QK_ERR_OUT_OF_RANGE = 2,
    QK_ERR_CUDA = 3,
    QK_ERR_UNSUPPORTED = 4
};

enum qk_dtype { QK_DTYPE_F32 = 0, QK_DTYPE_F16 = 1 };

typedef struct qk_cache qk_cache;

/* CacheConfig (kv_store.hpp:10-17) plus the batching the reference leaves to callers. */
typedef struct qk_cache_desc {
    uint32_t head_dim;          /* CacheConfig::head_dim, 1..256                       */
    uint32_t page_size;         /* CacheConfig::page_size, 1..64                       */
    uint32_t bytes_per_element; /* CacheConfig::bytes_per_element; 2 (fp16 pools)      */
    uint32_t num_layers;        /* independent caches per (sequence, KV head)          */
    uint32_t max_batch;         /* sequences                                           */
    uint32_t num_q_heads;       /* multiple of num_kv_heads                            */
    uint32_t num_kv_heads;
    uint32_t max_tokens;        /* capacity of each (layer, sequence, KV head) cache   */
    int32_t device;             /* CUDA device ordinal                                 */
} qk_cache_desc;

/* SelectionConfig (criticality.hpp:18-22). */
typedef struct qk_selection_cfg {
    uint32_t token_budget;
    int32_t force_include_recent; /* default 1 in the reference */
    int32_t per_layer_enabled;    /* default 1 in the reference */
} qk_selection_cfg;

/* Message of the calling thread's last failed call ("" if none). */
QK_API const char *qk_last_error(void);
QK_API int qk_abi_version(void);

/* KvCache::KvCache (kv_store.cpp:15-17; validation kv_store.cpp:8-13).  Allocates every
 * pool, zero-fills it, sets all lengths to 0.  Zero head_dim/page_size/bpe ->
 * QK_ERR_INVALID_ARGUMENT (the reference's messages); bpe != 2, head_dim > 256 or
 * page_size > 64 -> QK_ERR_UNSUPPORTED. */
QK_API int qk_cache_create(const qk_cache_desc *desc, qk_cache **out);
QK_API int qk_cache_destroy(qk_cache *cache);
QK_API int qk_cache_describe(const qk_cache *cache, qk_cache_desc *out);
/* Bytes of HBM the cache holds (pools + metadata + workspaces). */
QK_API uint64_t qk_cache_device_bytes(const qk_cache *cache);
/* Logical pages per cache slice the pools are sized for (ceil(max_tokens/page_size)). */
QK_API uint32_t qk_cache_max_pages(const qk_cache *cache);
/* Grow every slice to hold max_tokens tokens (the reference's KvCache grows page by page,
 * kv_store.cpp:24-29): reallocates the pools, metadata and page-sized workspaces and copies
 * the cached pages, metadata and lengths into them.  Device-synchronising; a smaller or equal
 * max_tokens is a no-op.  Pointers captured before the call (CUDA graphs recorded by the
 * caller) refer to the old pools and must be re-captured.  More than 16384 pages per slice
 * -> QK_ERR_UNSUPPORTED; out of memory -> QK_ERR_CUDA with the cache unchanged. */
QK_API int qk_cache_reserve(qk_cache *cache, uint32_t max_tokens);

/* KvCache::token_count / page_count (kv_store.hpp:57-58) of one slice (all KV heads of a
 * sequence share it).  Host-side, never blocks. */
QK_API int qk_token_count(const qk_cache *cache, uint32_t layer, uint32_t seq, uint32_t *count);
QK_API int qk_page_count(const qk_cache *cache, uint32_t layer, uint32_t seq, uint32_t *count);

/* Drop every token of `layer` (all layers if layer == UINT32_MAX). */
QK_API int qk_reset(qk_cache *cache, uint32_t layer, void *stream);

/* KvCache::append (kv_store.cpp:19-47) for sequences 0..batch-1 of `layer`, every KV
 * head: token t = token_count lands in page t/S row t%S; row 0 seeds min=max=key, later
 * rows update with strict '<' / '>' (first-seen value kept on ties, so -0/+0 behave as
 * in the reference).  Metadata update is fused into the same kernel.  A full slice ->
 * QK_ERR_OUT_OF_RANGE; batch > max_batch -> QK_ERR_INVALID_ARGUMENT.  The previous
 * token counts are the appended tokens' indices (KvCache::append's return value). */
QK_API int qk_append(qk_cache *cache, uint32_t layer, const uint16_t *k, const uint16_t *v,
              uint32_t batch, void *stream);

/* n_tokens successive KvCache::append calls for one sequence (bulk prefill), every KV
 * head.  k, v: [num_kv_heads][n_tokens][head_dim] fp16.  Bitwise the same pages and
 * metadata as n_tokens single appends, built page-parallel. */
QK_API int qk_prefill(qk_cache *cache, uint32_t layer, uint32_t seq, const uint16_t *k,
               const uint16_t *v, uint32_t n_tokens, void *stream);

/* KvCache::page_metadata (kv_store.cpp:49-54): copies min_key/max_key of pages
 * [page0, page0+n) of one slice to host arrays [n][head_dim] (fp16 bits).  Synchronous
 * on `stream`.  A page past page_count -> QK_ERR_OUT_OF_RANGE. */
QK_API int qk_read_metadata(const qk_cache *cache, uint32_t layer, uint32_t seq, uint32_t kv_head,
                     uint32_t page0, uint32_t n_pages, uint16_t *min_host,
                     uint16_t *max_host, void *stream);

/* KvCache::key / value (kv_store.cpp:63-79): rows of tokens [token0, token0+n) to host
 * arrays [n][head_dim].  Synchronous.  A token past token_count -> QK_ERR_OUT_OF_RANGE. */
QK_API int qk_read_kv(const qk_cache *cache, uint32_t layer, uint32_t seq, uint32_t kv_head,
               uint32_t token0, uint32_t n_tokens, uint16_t *k_host, uint16_t *v_host,
               void *stream);

/* estimate_all (criticality.cpp:25-34) for every (sequence, query head) of a layer:
 * scores[b][h][p] = sum_{i ascending} max(q_i*max_i, q_i*min_i), p < page_count, in
 * fp64, bitwise equal to the reference (exact fp16 products, sequential fp64 adds).
 * Entries p >= page_count are left untouched.  An empty sequence ->
 * QK_ERR_INVALID_ARGUMENT. */
QK_API int qk_estimate(const qk_cache *cache, uint32_t layer, const uint16_t *q, uint32_t batch,
                double *scores, uint32_t scores_stride, void *stream);

/* select_top_k (criticality.cpp:36-81) per (sequence, query head): !per_layer_enabled ->
 * every page; token_budget < page_size -> QK_ERR_INVALID_ARGUMENT; K = budget/page_size
 * >= page_count -> every page; else the K best pages by (score desc, page asc), with
 * force_include_recent replacing the weakest pick by the newest page.  Output ascending;
 * counts[b][h] = pages written.  pages_stride >= min(K, max_pages) (>= max_pages when
 * selection can return every page). */
QK_API int qk_select_topk(const qk_cache *cache, uint32_t layer, const double *scores,
                   uint32_t scores_stride, uint32_t batch, const qk_selection_cfg *cfg,
                   int32_t *pages, uint32_t pages_stride, int32_t *counts, void *stream);

/* select_top_k (criticality.cpp:36-81) on an ARBITRARY PageScore vector of one
 * (layer, seq) cache: n (page_index, score) pairs in any order, repeated page indices
 * allowed, exactly the reference's rule -- disabled -> every page; budget < page_size ->
 * INVALID_ARGUMENT; n == 0 -> INVALID_ARGUMENT; a page_index >= page_count -> OUT_OF_RANGE
 * (device status, qk_check_status); K >= n -> every page; else the first K by (score desc,
 * page asc; -0 == +0), the K-th replaced by the newest page under force_include_recent,
 * ascending (duplicates kept, as the reference).  pages holds pages_capacity entries
 * (>= K, or >= page_count when every page is returned); *count = entries written.
 * n <= 16384.  The fast form for estimate_all's output is qk_select_topk. */
QK_API int qk_select_topk_pairs(qk_cache *cache, uint32_t layer, uint32_t seq,
                         const uint32_t *page_index, const double *scores, uint32_t n,
                         const qk_selection_cfg *cfg, int32_t *pages, uint32_t pages_capacity,
                         int32_t *count, void *stream);

/* sparse_attention (attention.cpp:94-116) over the listed pages, split-KV with an
 * fp32 log-sum-exp merge: logits q.k/sqrt(d), softmax renormalised over the selected
 * tokens, partial last page masked to its length.  Page lists must be strictly
 * ascending and in range (the form qk_select_topk writes); violations are recorded on
 * the device and reported by qk_check_status (the reference's out_of_range /
 * invalid_argument).  Every page count must be >= 1.  weights_sum (optional) receives
 * AttentionOutput::weights_sum_check (attention.cpp:81): the post-softmax mass of the
 * weights applied, evaluated in fp64 from the fp32 partials. */
QK_API int qk_sparse_attend(const qk_cache *cache, uint32_t layer, const uint16_t *q,
                     uint32_t batch, const int32_t *pages, uint32_t pages_stride,
                     const int32_t *counts, void *out, int32_t out_dtype, float *lse,
                     double *weights_sum, void *stream);

/* full_attention (attention.cpp:86-92): the same kernel over every page in order, so it
 * is bitwise equal to qk_sparse_attend given every page (the reference's full-budget
 * degeneracy, attention.hpp:34-36).  Empty sequence -> QK_ERR_INVALID_ARGUMENT. */
QK_API int qk_dense_attend(const qk_cache *cache, uint32_t layer, const uint16_t *q,
                    uint32_t batch, void *out, int32_t out_dtype, float *lse,
                    double *weights_sum, void *stream);

/* attend_tokens (attention.hpp:41-46, attention.cpp:69-84): attention over an explicit
 * token set per (sequence, query head), the token-granular form policies use.  Lists are
 * checked on the device like check_token_set (attention.cpp:19-30): an index >=
 * token_count -> OUT_OF_RANGE, not strictly ascending -> INVALID_ARGUMENT, empty ->
 * INVALID_ARGUMENT (reported by qk_check_status).  Chunks of page_size list entries are
 * folded like pages, so every token in order is bitwise qk_dense_attend. */
QK_API int qk_attend_tokens(const qk_cache *cache, uint32_t layer, const uint16_t *q,
                     uint32_t batch, const int32_t *tokens, uint32_t tokens_stride,
                     const int32_t *counts, void *out, int32_t out_dtype, float *lse,
                     double *weights_sum, void *stream);

/* attention_logits (attention.hpp:24-29, attention.cpp:34-52): logit_t = q.k_t / sqrt(d) in
 * fp64, bitwise the reference's (exact fp16 products, sequential fp64 sum, correctly
 * rounded sqrt and division).  tokens == NULL: every cached token of the sequence (the
 * one-argument overload; logits_stride >= token_count); else the listed tokens, validated
 * as qk_attend_tokens. */
QK_API int qk_attention_logits(const qk_cache *cache, uint32_t layer, const uint16_t *q,
                        uint32_t batch, const int32_t *tokens, uint32_t tokens_stride,
                        const int32_t *counts, double *logits, uint32_t logits_stride,
                        void *stream);

/* softmax_weights (attention.hpp:31, attention.cpp:54-67) over rows of device logits:
 * w = exp(l - max) / sum, fp64 (sum order and libm differ from the reference: ~1e-15
 * relative).  counts == NULL: every row holds n logits.  An empty row -> status
 * INVALID_ARGUMENT via qk_check_status(cache) (cache supplies the device and status). */
QK_API int qk_softmax_weights(qk_cache *cache, const double *logits, const int32_t *counts,
                       uint32_t n, uint32_t stride, uint32_t rows, double *weights,
                       void *stream);

/* One fused Quest decode step for a layer (the README's estimate -> select -> attend
 * loop, R/README.md:151-158, preceded by KvCache::append): appends k/v (if non-NULL),
 * then estimates, selects and attends in one kernel per step.  Results equal
 * qk_append + qk_estimate + qk_select_topk + qk_sparse_attend (same pages bitwise, same
 * outputs within fp32 rounding).  pages_out/counts_out (optional) receive the
 * selection.  Capturable in a CUDA graph. */
QK_API int qk_decode_step(qk_cache *cache, uint32_t layer, const uint16_t *q, const uint16_t *k,
                   const uint16_t *v, uint32_t batch, const qk_selection_cfg *cfg,
                   void *out, int32_t out_dtype, int32_t *pages_out, uint32_t pages_stride,
                   int32_t *counts_out, void *stream);

/* Same step from HOST buffers (pinned or pageable), synchronous, one launch and one
 * synchronisation per call.  The kernel reads q/k/v and writes the fp32 output over PCIe
 * (zero-copy): in place when a buffer is pinned and device-mapped (qk_host_alloc,
 * cudaHostAlloc, cudaHostRegister), else through the cache's pinned staging buffer (a host
 * memcpy each way).  The reference-facing call for callers that keep activations on the
 * host. */
QK_API int qk_decode_step_host(qk_cache *cache, uint32_t layer, const uint16_t *q_host,
                        const uint16_t *k_host, const uint16_t *v_host, uint32_t batch,
                        const qk_selection_cfg *cfg, float *out_host, void *stream);

/* Pinned, device-mapped host memory for the host-buffer entry points' inputs and outputs
 * (read and written by the kernels in place); nullptr on failure.  Free with qk_host_free. */
QK_API void *qk_host_alloc(size_t bytes);
QK_API void qk_host_free(void *ptr);

/* Host-buffer forms of the entry points above, for callers that keep activations on the
 * host (the questkv:: C++ layer in questkv_b200.hpp binds these).  Each stages its
 * inputs through the cache's device workspaces, runs the device entry point on `stream`
 * and copies the result back; all are synchronous and return the same statuses.
 * Arrays have the device forms' layouts; outputs are f32 (out) / f64 (scores). */
QK_API int qk_append_host(qk_cache *cache, uint32_t layer, const uint16_t *k_host,
                          const uint16_t *v_host, uint32_t batch, void *stream);
QK_API int qk_prefill_host(qk_cache *cache, uint32_t layer, uint32_t seq, const uint16_t *k_host,
                           const uint16_t *v_host, uint32_t n_tokens, void *stream);
QK_API int qk_estimate_host(const qk_cache *cache, uint32_t layer, const uint16_t *q_host,
                            uint32_t batch, double *scores_host, uint32_t scores_stride,
                            void *stream);
QK_API int qk_select_topk_host(const qk_cache *cache, uint32_t layer, const double *scores_host,
                               uint32_t scores_stride, uint32_t batch,
                               const qk_selection_cfg *cfg, int32_t *pages_host,
                               uint32_t pages_stride, int32_t *counts_host, void *stream);
/* Page lists are validated on the host first, with sparse_attention's errors
 * (attention.cpp:99-106): empty -> INVALID_ARGUMENT, out of range -> OUT_OF_RANGE,
 * duplicate / not ascending -> INVALID_ARGUMENT. */
QK_API int qk_sparse_attend_host(const qk_cache *cache, uint32_t layer, const uint16_t *q_host,
                                 uint32_t batch, const int32_t *pages_host,
                                 uint32_t pages_stride, const int32_t *counts_host,
                                 float *out_host, float *lse_host, double *wsum_host,
                                 void *stream);
QK_API int qk_dense_attend_host(const qk_cache *cache, uint32_t layer, const uint16_t *q_host,
                                uint32_t batch, float *out_host, float *lse_host,
                                double *wsum_host, void *stream);
/* Host arrays; the page range is checked on the host first (the reference's order). */
QK_API int qk_select_topk_pairs_host(qk_cache *cache, uint32_t layer, uint32_t seq,
                                     const uint32_t *page_index_host, const double *scores_host,
                                     uint32_t n, const qk_selection_cfg *cfg, int32_t *pages_host,
                                     uint32_t pages_capacity, int32_t *count_host, void *stream);
/* Token lists validated on the host first with check_token_set's errors and messages. */
QK_API int qk_attend_tokens_host(const qk_cache *cache, uint32_t layer, const uint16_t *q_host,
                                 uint32_t batch, const int32_t *tokens_host,
                                 uint32_t tokens_stride, const int32_t *counts_host,
                                 float *out_host, float *lse_host, double *wsum_host,
                                 void *stream);
QK_API int qk_attention_logits_host(const qk_cache *cache, uint32_t layer,
                                    const uint16_t *q_host, uint32_t batch,
                                    const int32_t *tokens_host, uint32_t tokens_stride,
                                    const int32_t *counts_host, double *logits_host,
                                    uint32_t logits_stride, void *stream);
/* estimate_page_score (criticality.cpp:9-23) on explicit metadata, host arrays:
 * q [head_dim], min/max [n_pages][head_dim] (fp16 bits) -> scores [n_pages], bitwise the
 * reference's doubles; computed on `device` (per-device scratch, no cache needed). */
QK_API int qk_estimate_metadata_host(const uint16_t *q_host, const uint16_t *min_host,
                                     const uint16_t *max_host, uint32_t n_pages,
                                     uint32_t head_dim, double *scores_host, int32_t device);
/* softmax_weights on one host vector, computed on `device` (empty -> INVALID_ARGUMENT
 * "softmax_weights: empty logits", as the reference). */
QK_API int qk_softmax_weights_host(const double *logits_host, uint32_t n, double *weights_host,
                                   int32_t device);

/* ---- GQA group-shared selection -------------------------------
 * An OPT-IN variant, NOT the reference's semantics (the reference selects per query head,
 * criticality.cpp:36-81): ONE page set per (sequence, KV head), chosen by select_top_k's
 * rule (early exits, (score desc, page asc), force_include_recent) from a group score
 * that combines the G exact per-query-head estimates of a page:
 *   QK_GROUP_MAX  max over the group's query heads (exact, order-free)
 *   QK_GROUP_SUM  fp64 sum in query-head order ((s_0 + s_1) + s_2) + ...
 * Every query head of the group then attends over the shared pages (sparse_attention,
 * attention.cpp:94-116, fp32 accumulate); K/V pages are read once per group and the
 * Q.K^T / P.V contractions run on the tensor cores (mma.sync m16n8k16, G <= 8 heads,
 * head_dim <= 128).  Group page lists / counts are [batch][num_kv_heads][stride] /
 * [batch][num_kv_heads]; everything else as the per-head entry points. */
enum qk_group_reduce { QK_GROUP_MAX = 1, QK_GROUP_SUM = 2 };

/* select_top_k over the group scores of estimate_all's per-head scores (layout of
 * qk_estimate's output). */
QK_API int qk_select_topk_grouped(const qk_cache *cache, uint32_t layer, const double *scores,
                                  uint32_t scores_stride, uint32_t batch,
                                  const qk_selection_cfg *cfg, int32_t group_reduce,
                                  int32_t *pages, uint32_t pages_stride, int32_t *counts,
                                  void *stream);
/* Every query head of a group attends over its group's page list (strictly ascending, in
 * range; violations reported by qk_check_status as for qk_sparse_attend). */
QK_API int qk_sparse_attend_grouped(const qk_cache *cache, uint32_t layer, const uint16_t *q,
                                    uint32_t batch, const int32_t *pages, uint32_t pages_stride,
                                    const int32_t *counts, void *out, int32_t out_dtype,
                                    void *stream);
/* append (optional) -> qk_estimate -> qk_select_topk_grouped -> qk_sparse_attend_grouped on
 * `stream` (capturable in a CUDA graph). */
QK_API int qk_decode_step_grouped(qk_cache *cache, uint32_t layer, const uint16_t *q,
                                  const uint16_t *k, const uint16_t *v, uint32_t batch,
                                  const qk_selection_cfg *cfg, int32_t group_reduce, void *out,
                                  int32_t out_dtype, int32_t *pages_out, uint32_t pages_stride,
                                  int32_t *counts_out, void *stream);

/* Diagnostics / parity: with `on`, qk_decode_step estimates every page (also the forced
 * newest page, and when the budget covers the cache) and keeps the scores for
 * qk_debug_step_scores.  Off by default: the fused step then skips scores selection
 * cannot use. */
QK_API int qk_debug_keep_scores(qk_cache *cache, int32_t on);

/* Re-reads the device token counts into the host-side shadow (synchronous).  Needed
 * after replaying a captured CUDA graph of qk_decode_step, whose appends advance only the
 * device counts. */
QK_API int qk_sync_lengths(qk_cache *cache, void *stream);

/* Synchronises `stream` and returns (and clears) the first error a kernel recorded on
 * the device since the last check (invalid page list, capacity overflow). */
QK_API int qk_check_status(qk_cache *cache, void *stream);

/* Diagnostics: with QK_PROBE=1 in the environment at qk_cache_create, the fused decode
 * kernel records up to 32 %globaltimer stamps per CTA at its phase boundaries, one record per
 * layer ([layer][max_batch*num_kv_heads*16][32] u64; see
 * decode.cu; tools/probe_fused.py prints the timeline).  Copies the first n and clears
 * the record (synchronous). */
QK_API int qk_debug_probe(qk_cache *cache, uint64_t *host, uint32_t n, void *stream);

/* Diagnostics: the page scores the last qk_decode_step computed for (seq, q_head), pages
 * [0, n) -- the fused kernel keeps them in an internal workspace (synchronous). */
QK_API int qk_debug_step_scores(qk_cache *cache, uint32_t seq, uint32_t q_head, double *host,
                                uint32_t n, void *stream);

/* Launches of this library's kernels since the cache was created (all entry points). */
QK_API uint64_t qk_kernel_launches(const qk_cache *cache);

#ifdef __cplusplus
}
#endif
#endif /* QUESTKV_B200_H */

/* TEST INFRASTRUCTURE ONLY — the checker, never the product.
 *
 * absp_oracle: a plain-C restatement of the reference's decode-time block-sparse
 * attention path (/root/reference/proj/src, C++20), one sequence at a time, over
 * the SAME paged bf16 layout the CUDA library uses:
 *
 *   k_pool / v_pool : uint16 bf16 bit patterns, [H][pool_pages][P][d]
 *   page_table      : uint32 [ceil(n / P)] page ids, shared by all heads
 *                     (the reference hands out identical ids per head,
 *                      kv_cache.cpp:53-60)
 *
 * Every function cites the reference code it restates. Parity is pinned by
 * tests/test_oracle_*.py against (a) the reference's own known-answer tests
 * (proj/tests/*\.cpp), re-expressed, and (b) the unmodified reference core
 * compiled into oracle/_ref/ (see oracle/Makefile) on the same inputs, plus the
 * committed fixtures in tests/golden/.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline/reference legs
 * may load this library.
 */
#ifndef ABSP_ORACLE_H
#define ABSP_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* 0 ok; 1 invalid argument; 2 out of range (mirrors the reference exception classes) */

/* build_offsets, centroids.cpp:78-84. offsets: H+1 entries. */
void absp_oracle_offsets(size_t n, const uint32_t* block_sizes, size_t H, uint64_t* offsets);

/* compute_block_centroids + compute_one_centroid, centroids.cpp:18-43, 86-120.
 * method 0 = mean (fp64 accumulate, *(1/cnt), cast), 1 = maxmin.
 * values, values_min: [total][d] fp32 (values_min only for maxmin). */
int absp_oracle_centroids(const uint16_t* k_pool, size_t pool_pages, const uint32_t* page_table,
                          size_t n, size_t H, size_t d, size_t P, const uint32_t* block_sizes,
                          int method, float* values, float* values_min);

/* quantize_store / quantize_one_head / quantize_segment, quantizer.cpp:16-73, 84-111.
 * One array (the mean store, or one maxmin array). bits in {2,4,8}; mode 0 sym, 1 asym.
 * codes: [total][d] one per byte; scales, zps: [H][d]. */
int absp_oracle_quantize(const float* values, const uint64_t* offsets, size_t H, size_t d,
                         int bits, int mode, uint8_t* codes, float* scales, float* zps);

/* estimate_scores(q, QuantizedCentroidStore) = estimate_batched + centroid_score,
 * engine.cpp:34-67, 79-97. q: [H][d]; scores: [total]. codes_min etc. only for maxmin. */
void absp_oracle_scores_quant(const float* q, const uint8_t* codes, const uint8_t* codes_min,
                              const float* scales, const float* zps, const float* scales_min,
                              const float* zps_min, const uint64_t* offsets, size_t H, size_t d,
                              int bits, int mode, int method, float* scores);

/* estimate_scores(q, CentroidStore), engine.cpp:21-32. */
void absp_oracle_scores_f32(const float* q, const float* values, const float* values_min,
                            const uint64_t* offsets, size_t H, size_t d, int method,
                            float* scores);

/* select_topk -> select_impl -> select_head, engine.cpp:119-178.
 * blocks: [H][max_k] (score-descending, ties to lower index), counts: [H],
 * budgets (may be NULL): [H] = ceil(T / B_h). */
int absp_oracle_select(const float* scores, const uint64_t* offsets, const uint32_t* block_sizes,
                       size_t H, size_t n, size_t token_budget, uint32_t* blocks, size_t max_k,
                       uint32_t* counts, uint32_t* budgets);

/* sparse_attention + attend_rows + dot_f32, engine.cpp:180-210, 285-327, reading rows
 * through block_to_pages (kv_cache.cpp:118-138). q, out: [H][d] fp32. */
int absp_oracle_attend(const float* q, const uint16_t* k_pool, const uint16_t* v_pool,
                       size_t pool_pages, const uint32_t* page_table, size_t n, size_t H, size_t d,
                       size_t P, const uint32_t* block_sizes, const uint32_t* blocks, size_t max_k,
                       const uint32_t* counts, float* out);

/* full_attention_oracle, engine.cpp:357-403 (fp64). q, out: [H][d]. */
int absp_oracle_full_attention(const float* q, const uint16_t* k_pool, const uint16_t* v_pool,
                               size_t pool_pages, const uint32_t* page_table, size_t n, size_t H,
                               size_t d, size_t P, float* out);

#ifdef __cplusplus
}
#endif
#endif

/*
 * absp.h — C ABI of the B200-native AB-Sparse decode-attention path.
 *
 * This is the drop-in boundary for the reference's hot path
 * (/root/reference/proj, namespace absparse). The reference exposes free C++
 * functions over std::vector-backed stores; this ABI exposes the same
 * operations over device memory, batched over sequences and GQA groups:
 *
 *   absp_config_validate   <- EngineConfig::validate          config.cpp:48-78
 *   absp_set_assignment    <- BlockAssignment::validate       centroids.cpp:59-76
 *                             (block-size table per KV head)  centroids.hpp:12-23
 *   absp_kv_bind           <- PagedKVCache (page pools + page tables)
 *                                                             kv_cache.hpp:26-67
 *   absp_build_store       <- compute_block_centroids         centroids.hpp:56-57
 *                             + quantize_store                quantizer.hpp:43
 *   absp_append            <- PagedKVCache::append            kv_cache.cpp:44-70
 *                             + refresh_tail_centroids        centroids.cpp:158-163
 *                             + requantize_heads (all heads)  quantizer.cpp:113-150
 *   absp_select            <- estimate_scores(q, qstore)      engine.hpp:47-49
 *                             + select_topk                   engine.hpp:61-64
 *   absp_attend            <- populate_page_spans             engine.hpp:71
 *                             + sparse_attention              engine.hpp:79-80
 *   absp_decode_step       <- the estimate->select->attend part of
 *                             DecodeEngine::step              engine.cpp:450-461
 *   absp_download_*        <- read-back in the reference layouts
 *                             (CentroidStore / QuantizedCentroidStore /
 *                              estimate_scores output)        centroids.hpp:31-52,
 *                                                             quantizer.hpp:18-38
 *
 * Extensions the reference lacks: a batch of sequences
 * (per-sequence length), GQA (num_q_heads = G * num_kv_heads; selection is per
 * KV head on the fp32 left-to-right group sum of the G queries; attention runs
 * for every query head over its KV head's selection), bf16 KV/query storage.
 *
 * Conventions
 *  - Every entry point returns absp_status; on failure absp_last_error() holds a
 *    thread-local message. Status codes map 1:1 onto the reference's exception
 *    classes (std::invalid_argument, std::out_of_range, std::runtime_error,
 *    std::logic_error) plus CUDA / allocation failures.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    Calls are stream-ordered and asynchronous unless documented otherwise; no
 *    hidden device synchronisation on the decode path.
 *  - Device buffers passed in are borrowed (caller-owned); store, scores,
 *    selections and partials are context-owned.
 *  - bf16 tensors are raw 16-bit patterns (uint16_t / void*).
 *  - Layouts:
 *      k_pool, v_pool : bf16 [num_kv_heads][pool_pages][page_size][head_dim]
 *                       (per-head page pools, kv_cache.cpp:36-41)
 *      page_table     : uint32 [batch][max_pages_per_seq]; one table per
 *                       sequence shared by all KV heads (the reference hands
 *                       identical ids to every head, kv_cache.cpp:53-60)
 *      q              : bf16 [batch][num_q_heads][head_dim]; q head hq belongs
 *                       to KV head hq / G
 *      out            : fp32 [batch][num_q_heads][head_dim]
 *      blocks         : uint32 [batch][num_kv_heads][blocks_stride], block ids
 *                       in score-descending order (ties -> lower id), as
 *                       SelectionResult::blocks (engine.hpp:23)
 *      counts         : uint32 [batch][num_kv_heads]
 *
 * Thread safety: one context per device per host thread; stores are immutable
 * between absp_build_store calls.
 */
#ifndef ABSP_H
#define ABSP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ABSP_ABI_VERSION 1
#define ABSP_MAX_CANDIDATES 16

typedef enum absp_status {
    ABSP_OK = 0,
    ABSP_EINVAL = 1,    /* std::invalid_argument: shapes, config, preconditions */
    ABSP_ERANGE = 2,    /* std::out_of_range: indices                           */
    ABSP_ECAPACITY = 3, /* std::runtime_error: capacity                         */
    ABSP_ESTATE = 4,    /* std::logic_error: call order / engine state          */
    ABSP_ECUDA = 5,     /* CUDA runtime error (device, launch, copy)            */
    ABSP_ENOMEM = 6     /* device allocation failure                            */
} absp_status;

typedef enum absp_centroid_method {
    ABSP_CENTROID_MEAN = 0,  /* CentroidMethod::kMean   (config.hpp:11) */
    ABSP_CENTROID_MAXMIN = 1 /* CentroidMethod::kMaxMin                 */
} absp_centroid_method;

typedef enum absp_quant_mode {
    ABSP_QUANT_SYM = 0, /* QuantMode::kSymmetric  (config.hpp:13) */
    ABSP_QUANT_ASYM = 1 /* QuantMode::kAsymmetric                 */
} absp_quant_mode;

/* Mirrors EngineConfig (config.hpp:36-52) + batch/GQA/capacity fields. */
typedef struct absp_config {
    uint32_t num_kv_heads;   /* EngineConfig::num_heads                              */
    uint32_t num_q_heads;    /* GQA: G * num_kv_heads (G in 1..8)                    */
    uint32_t head_dim;       /* EngineConfig::head_dim; kernels: 64 or 128            */
    uint32_t page_size;      /* EngineConfig::page_size                              */
    uint32_t num_candidates; /* |candidate_block_sizes|                              */
    uint32_t candidate_block_sizes[ABSP_MAX_CANDIDATES];
    uint32_t token_budget;    /* EngineConfig::token_budget (T)                      */
    uint32_t centroid_method; /* absp_centroid_method                                */
    uint32_t quant_bits;      /* 0 = full-precision store (quant = nullopt); 2, 4, 8 */
    uint32_t quant_mode;      /* absp_quant_mode                                     */
    uint32_t max_batch;       /* sequences per layer                                 */
    uint32_t max_seq_len;     /* capacity in tokens (store segments are reserved)    */
    uint32_t num_layers;      /* independent layers (stores/bindings) per context    */
} absp_config;

typedef struct absp_ctx absp_ctx;

/* Per-layer shape information (host-side, valid after absp_kv_bind). */
typedef struct absp_layer_info {
    uint32_t batch;
    uint32_t max_select;      /* max over (b,h) of min(N_h, K_h): minimal blocks_stride */
    uint64_t total_centroids; /* sum over (b,h) of N_h                                   */
    uint64_t store_bytes;     /* device bytes of codes + params (+ fp32 centroids)       */
    uint64_t kv_bytes_selected; /* bf16 K+V bytes the attention reads for a full-budget step */
    uint64_t code_bytes;      /* bytes of packed codes read by one scoring pass          */
} absp_layer_info;

int absp_abi_version(void);
const char* absp_last_error(void);

/* EngineConfig::validate (config.cpp:48-78) plus the GPU build's own limits:
 * head_dim 64 or 128; GQA group size G <= 8; page_size a power of two <= 128; block
 * sizes any multiple of page_size up to 128 (the reference's rule, capped at the
 * 128-row attention chunk); token_budget / min block size <= 2048. */
absp_status absp_config_validate(const absp_config* cfg);

absp_status absp_ctx_create(int device, const absp_config* cfg, absp_ctx** out);
absp_status absp_ctx_destroy(absp_ctx* ctx);

/* Per-KV-head block sizes B_h for `layer` (BlockAssignment::validate,
 * centroids.cpp:59-76: each B_h a candidate and a multiple of page_size). */
absp_status absp_set_assignment(absp_ctx* ctx, uint32_t layer, const uint32_t* block_sizes);

/* Borrow the caller's paged KV cache for `layer`. seq_lens is a HOST array of
 * `batch` entries (each 1..max_seq_len); page_table is a DEVICE array
 * [batch][max_pages_per_seq]. Invalidates the layer's store. */
absp_status absp_kv_bind(absp_ctx* ctx, uint32_t layer, const void* k_pool, const void* v_pool,
                         uint64_t pool_pages, const uint32_t* page_table,
                         uint32_t max_pages_per_seq, const uint32_t* seq_lens, uint32_t batch);

/* Prefill-time centroid build + quantization (compute_block_centroids +
 * quantize_store) for every (sequence, KV head) of the layer. */
absp_status absp_build_store(absp_ctx* ctx, uint32_t layer, void* stream);

/* Decode-time append + store maintenance, the first half of DecodeEngine::step
 * (engine.cpp:443-449): appends one token per sequence — k_new / v_new bf16
 * [batch][num_kv_heads][head_dim] (device) are written to row n % P of page
 * page_table[b][n / P] (PagedKVCache::append, kv_cache.cpp:44-70; the caller's
 * page table must map position n) — then refresh_tail_centroids and
 * requantize_heads over every head (centroids.cpp:122-163, quantizer.cpp:113-150),
 * leaving the store equal to one built from scratch on the grown cache (done
 * incrementally: only code words whose channel parameters changed are re-encoded).
 * ECAPACITY when a sequence would exceed max_seq_len or its page table. Stream-
 * ordered: the grown unit layout is uploaded on `stream` (staged through a ring of
 * pinned buffers sized at bind), so a layer's appends and decode steps belong on
 * one stream; the host waits only if more than 4 appends of the layer are still
 * queued ahead of the GPU. No device buffer is reallocated (capacity-reserved at
 * bind); see absp_layout_version for captured graphs. */
absp_status absp_append(absp_ctx* ctx, uint32_t layer, const void* k_new, const void* v_new, void* stream);

/* estimate_scores on the group-summed query + select_topk for every
 * (sequence, KV head). Writes blocks/counts (device). blocks_stride >= info.max_select. */
absp_status absp_select(absp_ctx* ctx, uint32_t layer, const void* q, uint32_t* blocks,
                        uint32_t blocks_stride, uint32_t* counts, void* stream);

/* sparse_attention over an explicit selection (device blocks/counts; any block
 * list of valid, distinct ids per (b,h), count >= 1). out: fp32 device. */
absp_status absp_attend(absp_ctx* ctx, uint32_t layer, const void* q, const uint32_t* blocks,
                        uint32_t blocks_stride, const uint32_t* counts, float* out, void* stream);

/* Validation of the explicit selections given to absp_attend since the last call
 * (the reference's check_selection / block_to_pages, engine.cpp:212-232,
 * kv_cache.cpp:118-138): ABSP_EINVAL for an empty selection or a count above
 * blocks_stride, ABSP_ERANGE for a block id >= N_h or a page-table entry outside the
 * pools. absp_attend itself never reads out of bounds (offending entries are
 * dropped, an empty unit's output is zero); this call synchronises `stream` and
 * clears the flags. */
absp_status absp_attend_validate(absp_ctx* ctx, uint32_t layer, void* stream);

/* Version of the layer's decode-step layout: bumped by absp_kv_bind and by any
 * absp_append that changes a kernel argument of absp_decode_step (grid sizes, work
 * counts — while sequences are shorter than the token budget, or a unit crosses a
 * top-k size class). Device buffers are capacity-reserved at bind, so a CUDA graph
 * the caller captured over absp_decode_step / absp_attend_selected stays valid as
 * long as this value is unchanged. */
uint64_t absp_layout_version(absp_ctx* ctx, uint32_t layer);

/* sparse_attention over the layer's most recent selection (made by absp_select or
 * absp_decode_step): the attention half of a decode step, e.g. to run it on another
 * stream than the selection. */
absp_status absp_attend_selected(absp_ctx* ctx, uint32_t layer, const void* q, float* out,
                                 void* stream);

/* The selection half of absp_decode_step into the layer's own buffers (the fused
 * selection kernel; blocks / counts / page list), without the attention: pair with
 * absp_attend_selected, e.g. to time or stream the two halves separately. */
absp_status absp_select_step(absp_ctx* ctx, uint32_t layer, const void* q, void* stream);

/* select + attend using context-owned selection buffers (the per-step hot path). */
absp_status absp_decode_step(absp_ctx* ctx, uint32_t layer, const void* q, float* out,
                             void* stream);

/* End-to-end variant with HOST buffers: copies q_host (bf16 [batch][Hq][d]) to the
 * device, runs absp_decode_step, copies the fp32 output back to out_host and
 * synchronises the stream. Pinned host memory recommended. */
absp_status absp_decode_step_host(absp_ctx* ctx, uint32_t layer, const void* q_host,
                                  float* out_host, void* stream);

/* The last selection made by absp_decode_step for `layer` (device pointers,
 * context-owned, valid until the next step on that layer). */
absp_status absp_last_selection(absp_ctx* ctx, uint32_t layer, const uint32_t** blocks,
                                uint32_t* blocks_stride, const uint32_t** counts);

absp_status absp_get_layer_info(absp_ctx* ctx, uint32_t layer, absp_layer_info* info);

/* The last selection of `layer` (absp_decode_step's or absp_select's context-owned
 * buffers) copied to HOST memory in SelectionResult::blocks order (engine.hpp:19-26):
 * blocks uint32 [batch][num_kv_heads][blocks_stride] (blocks_stride from
 * absp_last_selection), counts uint32 [batch][num_kv_heads]. Synchronous. */
absp_status absp_download_selection(absp_ctx* ctx, uint32_t layer, uint32_t* blocks, uint32_t* counts);

/* Read back one sequence's store in the reference layouts (synchronous):
 *   offsets           : uint64 [H+1]       (CentroidStore::offsets)
 *   values/values_min : fp32 [total][d]    (CentroidStore::values / values_min;
 *                                           available when the store keeps fp32
 *                                           centroids, i.e. always in this build)
 *   codes/codes_min   : uint8 [total][d]   (one code per byte, unpacked)
 *   scales, zps (+_min): fp32 [H][d]
 * Any pointer may be NULL. */
absp_status absp_download_store(absp_ctx* ctx, uint32_t layer, uint32_t seq, uint64_t* offsets,
                                float* values, float* values_min, uint8_t* codes,
                                uint8_t* codes_min, float* scales, float* zps, float* scales_min,
                                float* zps_min);

/* Scores of the last absp_select/absp_decode_step for one sequence, flattened
 * like estimate_scores' output (fp32 [total]); synchronous. */
absp_status absp_download_scores(absp_ctx* ctx, uint32_t layer, uint32_t seq, float* scores);

/* Diagnostics of absp_decode_step's fused selection (INT4 mean stores, select.cu):
 * with diagnostics enabled for the layer, decode steps also store every centroid's
 * approximate score A_i (the linearised score up to a per-unit constant) and the
 * per-unit bound E with |S_i - C_u - A_i| <= E (S_i the exact score). Off by default. */
absp_status absp_set_filter_diagnostics(absp_ctx* ctx, uint32_t layer, int enable);
/* One sequence's approximate scores (fp32 [total], estimate_scores layout) and the
 * per-KV-head bounds E_h of the last diagnostic decode step; synchronous. */
absp_status absp_download_filter_scores(absp_ctx* ctx, uint32_t layer, uint32_t seq, float* approx,
                                        float* err);

/* full_attention_oracle (engine.cpp:357-403) on the GPU: exact dense decode
 * attention of every query head over its sequence's whole cached context (the
 * layer's bound KV; no store needed), in fp64 like the reference. out fp32
 * [batch][Hq][d]. weights (optional, device fp64 [batch][Hq][weights_stride],
 * weights_stride >= the longest sequence): AttentionOutput::weights, the softmax
 * probabilities of every cached token (t < seq_len of the row's sequence).
 * Logits are bit-exact (bf16 products are exact in fp64, serial channel order);
 * the softmax denominator and the output sums are formed per split and merged, so
 * weights and outputs agree with the reference to fp64 rounding. The dense side of
 * the sparse/full A/B and the weight source of calibration. */
absp_status absp_full_attention(absp_ctx* ctx, uint32_t layer, const void* q, float* out, double* weights,
                                uint64_t weights_stride, void* stream);

/* attention_recall (calibrator.cpp:48-71) per (sequence, q head): the fraction of
 * the oracle's attention mass (weights from absp_full_attention, same layout) on
 * tokens inside the selected blocks of the head's KV head (blocks / counts as
 * absp_select writes them). recall: device fp64 [batch][Hq]. The per-KV-head
 * recall of the reference (G = 1) is the q-head value; with GQA the calibrator
 * averages the G heads of a group. */
absp_status absp_attention_recall(absp_ctx* ctx, uint32_t layer, const double* weights, uint64_t weights_stride,
                                  const uint32_t* blocks, uint32_t blocks_stride, const uint32_t* counts,
                                  double* recall, void* stream);

/* One calibration sample (the per-trace body of profile_sensitivity and
 * transfer_check, calibrator.cpp:73-106 / :159-200) on the GPU, synchronous: the trace
 * (keys / values fp32 [num_kv_heads][seq_len][head_dim], queries fp32
 * [num_q_heads][head_dim], host memory, stored as bf16 like every input of this build)
 * becomes a paged cache with sequential pages (cache_from_trace, workload.cpp:311-330);
 * absp_full_attention gives the oracle weights; for every candidate block size a
 * uniform assignment is built, quantized (cfg's QuantSpec), estimated and selected at
 * cfg->token_budget, and its attention_recall written to recalls (fp64
 * [num_kv_heads][num_candidates], RecallTable::recalls layout, calibrator.hpp:15-28;
 * with GQA the mean over the G query heads of a KV head). With `assignment`
 * (block size per KV head) its recall per KV head goes to assigned_recall.
 * cfg->max_batch / max_seq_len / num_layers are ignored. The reference skips traces
 * with seq_len <= token_budget; so does the host side of this build. */
absp_status absp_profile_sample(int device, const absp_config* cfg, const float* keys, const float* values,
                                const float* queries, uint64_t seq_len, const uint32_t* assignment,
                                double* recalls, double* assigned_recall);

/* Deterministic counter-based N(0,1)-like bf16 generator used by the benchmark
 * and tests (same bytes as oracle/synth.py): element i of stream s gets
 * splitmix64(seed + golden * (s * 2^40 + i + 1)) -> Irwin-Hall(4 x u16) -> fp32
 * (one rounding) -> bf16 (RNE). */
absp_status absp_fill_synthetic_bf16(void* dst, uint64_t count, uint64_t seed,
                                     uint64_t stream_id, void* stream);

/* Number of kernel launches the library issued since context creation
 * (benchmark accounting). */
uint64_t absp_launch_count(absp_ctx* ctx);

/* ---------------------------------------------------------------------------
 * DecodeEngine (engine.hpp:90-129, engine.cpp:405-463) for one sequence, with no
 * caller-side device memory: the engine owns its paged bf16 KV cache (per-head pools,
 * sequential page ids as kv_cache.cpp:53-60 hands out), a one-layer context, a stream
 * and pinned staging buffers. Host fp32 in, host fp32 out; inputs are stored as bf16
 * (RNE), all arithmetic runs in the sm_100a kernels.
 * ------------------------------------------------------------------------- */
typedef struct absp_engine absp_engine;

/* DecodeEngine::DecodeEngine(config, assignment, capacity_tokens): validates the config
 * (EngineConfig::validate) and the per-KV-head block sizes (BlockAssignment::validate);
 * cfg->max_batch / max_seq_len / num_layers are replaced by 1 / capacity / 1. */
absp_status absp_engine_create(int device, const absp_config* cfg, const uint32_t* block_sizes,
                               uint64_t capacity_tokens, absp_engine** out);
absp_status absp_engine_destroy(absp_engine* engine);

/* DecodeEngine::prefill (engine.cpp:414-440): keys / values are host spans of
 * keys_len / values_len floats, head-major [H][tokens][d] with head h starting at
 * h * (len / H); the first num_tokens tokens of every head are cached, then the
 * centroid store is built and quantized. ESTATE if already prefilled, EINVAL if a
 * span is smaller than num_tokens, ECAPACITY above the capacity. Synchronous. */
absp_status absp_engine_prefill(absp_engine* engine, const float* keys, uint64_t keys_len, const float* values,
                                uint64_t values_len, uint64_t num_tokens);

/* DecodeEngine::step (engine.cpp:442-463): appends keys / values ([H][d] host fp32),
 * maintains the store (refresh_tail_centroids + requantize_heads), then estimate ->
 * select -> attend for `query` ([Hq][d] host fp32). Writes out [Hq][d] (host fp32),
 * the ordered selection per KV head (blocks [H][blocks_stride] and counts [H], host;
 * either may be NULL) and whether seq_len <= token_budget (the reference's full-
 * attention fallback: every block is then selected and attended). ESTATE before
 * prefill, EINVAL on a size mismatch, ECAPACITY at capacity. Synchronous. */
absp_status absp_engine_step(absp_engine* engine, const float* keys, uint64_t keys_len, const float* values,
                             uint64_t values_len, const float* query, uint64_t query_len, float* out,
                             uint32_t* blocks, uint32_t blocks_stride, uint32_t* counts,
                             int* full_attention_fallback);

/* Current sequence length, the minimal blocks_stride (ceil(T / min block size)) and the
 * engine's context (layer 0), e.g. for absp_download_store (DecodeEngine::centroids /
 * quantized). */
absp_status absp_engine_info(absp_engine* engine, uint64_t* seq_len, uint32_t* blocks_stride, absp_ctx** ctx);

#ifdef __cplusplus
}
#endif
#endif /* ABSP_H */

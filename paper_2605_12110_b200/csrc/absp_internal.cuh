// Internal declarations shared by the sm_100a kernels and the C-ABI host layer.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "absp.h"

namespace absp {

// The thread-local message absp_last_error() returns (api.cu).
void set_last_error(const std::string& msg);

// ---------------------------------------------------------------------------
// Per-(sequence, KV head) "unit" metadata, device-resident, one array per layer.
// A unit is the reference's per-head segment of one sequence
// (CentroidStore offsets[h]..offsets[h+1], centroids.hpp:31-40).
struct UnitDesc {
    uint32_t seq;        // b
    uint32_t head;       // h (KV head)
    uint32_t block;      // B_h
    uint32_t n_tokens;   // seq_len of b
    uint32_t n_blocks;   // N = ceil(n / B_h)
    uint32_t budget;     // K = ceil(T / B_h)
    uint32_t cap;        // capacity-reserved centroids = ceil(max_seq / B_h)
    uint32_t pad_;
    uint64_t seg;        // first centroid slot of this unit (prefix sum of cap)
};

// Work item of the scoring kernel: centroids [start, end) of one unit.
struct ScoreItem {
    uint32_t unit;
    uint32_t start;
    uint32_t end;
    uint32_t pad_;
};
// Scoring work split: CTA c scores items [item_begin[c], item_begin[c+1]), an
// equal share of the layer's flattened centroids cut at unit boundaries.
struct ScoreWork {
    const ScoreItem* items;
    const uint32_t* item_begin;  // [grid + 1]
    uint32_t grid;
    uint32_t* scored;            // [units] centroids scored this step (table scorer; null: none),
                                 // lets the top-k of a unit start before the whole grid ends
};

// Everything a kernel needs about one bound layer.
struct LayerView {
    // config
    uint32_t H, G, D, P;
    uint32_t bits, mode, method;
    uint32_t batch, units;
    uint32_t max_pages;      // page-table row length
    uint64_t pool_pages;     // pages per head in the pools
    // KV
    const uint16_t* k_pool;
    const uint16_t* v_pool;
    const uint32_t* page_table;
    // store
    const UnitDesc* desc;
    float* values;      // fp32 centroids [seg][d] (maxmin: max-array)
    float* values_min;  // maxmin min-array
    uint32_t* codes;    // packed rows [seg][W], word order per code_word_pos
    uint32_t* codes_min;
    float* scales;      // [units][d]
    float* zps;
    float* scales_min;
    float* zps_min;
    float* scores;      // [seg]
    // quantization statistics (build_store.cu)
    float* qstat;       // frozen per-channel statistics [arrays][units][2][d]
    float* qpart;       // build scratch: per-slice statistics [arrays][units][slices][2][d]
    uint32_t* wmask;    // decode-time maintenance: changed code words [arrays][units]
};

// Packed code rows: centroid i of a unit occupies W = D*bits/32 consecutive words
// (64 B at int4, d = 128; the reference's row [centroid][d] at bits/8 bytes per
// code). Inside a row the 16-byte groups are XOR-swizzled by the centroid index,
// so that a straight bulk copy of consecutive rows into shared memory can be read
// one row per lane with conflict-free 16-byte loads: 8 consecutive rows cover all
// 8 bank groups for every logical group g. Word w of row i sits at
//     ((w / 4) ^ key(i)) * 4 + w % 4,  key(i) = (i >> (3 - log2 U)) & (U - 1),
// U = W / 4 groups per row (W in {4, 8, 16, 32}).
__host__ __device__ constexpr uint32_t code_row_key(uint32_t i, uint32_t W) {
    return W <= 4 ? 0u : (i >> (W == 8 ? 2 : W == 16 ? 1 : 0)) & (W / 4 - 1);
}
__host__ __device__ constexpr uint32_t code_word_pos(uint32_t i, uint32_t w, uint32_t W) {
    return (((w >> 2) ^ code_row_key(i, W)) << 2) | (w & 3u);
}

// Launch with programmatic stream serialisation (PDL): the kernel may begin while
// the previous kernel of the stream finishes; it orders itself with griddep_wait()
// (ptx.cuh). Works inside CUDA-graph capture (programmatic edges).
template <typename... Exp, typename... Act>
cudaError_t launch_pdl(void (*kernel)(Exp...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Act&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<Act&&>(args)...);
}

// Launch wrappers (each returns cudaGetLastError after the launch).
cudaError_t launch_build_store(const LayerView& L, uint32_t max_cap, cudaStream_t s, int* launches);
cudaError_t launch_refresh_store(const LayerView& L, uint32_t max_cap, cudaStream_t s, int* launches);
cudaError_t launch_append_rows(const LayerView& L, const uint16_t* k_new, const uint16_t* v_new, cudaStream_t s,
                               int* launches);
cudaError_t launch_score(const LayerView& L, const uint16_t* q, const ScoreWork& work, cudaStream_t s,
                         int* launches);
cudaError_t init_score_attributes();  // per device, once
cudaError_t init_topk_attributes();   // per device, once
// Selected blocks resolved to pool pages, laid out by global attention chunk:
// unit u's slot s = entry * (B/P) + page lives at index chunk_base[u] * ns + s, so
// chunk w's slots are [w * ns, (w + 1) * ns). Written by the top-k kernel (decode
// step) or k_resolve_pages (explicit selections), read by the attention producer.
struct PageList {
    uint32_t* page;               // head * pool_pages + pool page id
    uint16_t* valid;              // valid rows of the page (0 = empty slot)
    const uint32_t* chunk_base;   // [units + 1] first chunk of each unit (work list)
    uint32_t ns;                  // page slots per chunk = kAttnChunkRows / P
};
// ready (decode step, else null): per-unit "selection published" flags, raised by the
// selection kernel after the unit's blocks and page list are written (release) and
// re-armed by the attention merge; the attention producer starts a unit on its flag.
// Top-k launch classes: units grouped by the register variant their block count
// needs (topk_items), so a layer with mixed block sizes does not run every unit with
// the keys-per-thread of its largest one. units = null: one launch.
constexpr int kTopkClasses = 8;
struct TopkClasses {
    const uint32_t* units;           // [units] grouped by class
    uint32_t begin[kTopkClasses + 1];
    uint32_t items[kTopkClasses];    // keys per thread of each class (0: L2-resident keys)
};
uint32_t topk_items(uint32_t n_blocks);
// scored (else null): the scorer's per-unit completion counters (ScoreWork::scored);
// a unit's top-k starts once its count reaches N and re-arms it.
cudaError_t launch_topk(const LayerView& L, uint32_t max_nblocks, uint32_t max_budget,
                        uint32_t* blocks, uint32_t stride, uint32_t* counts, const PageList& pages,
                        uint32_t* ready, uint32_t* scored, const TopkClasses& classes, cudaStream_t s,
                        int* launches);
// Explicit-selection validation bits (k_resolve_pages -> absp_attend_validate).
constexpr uint32_t kAttendErrEmpty = 1u;  // a unit with count 0        (invalid_argument)
constexpr uint32_t kAttendErrBlock = 2u;  // block id >= n_blocks        (out_of_range)
constexpr uint32_t kAttendErrCount = 4u;  // count > blocks_stride       (invalid_argument)
constexpr uint32_t kAttendErrPage = 8u;   // page-table entry >= pool_pages (out_of_range)
cudaError_t launch_resolve_pages(const LayerView& L, const uint32_t* blocks, uint32_t stride,
                                 const uint32_t* counts, const PageList& pages, uint32_t* err, cudaStream_t s,
                                 int* launches);
// Attention work list: all 128-row chunks of all units, unit-major.
struct AttendWork {
    const uint32_t* chunk_unit;  // [n_work] unit of each chunk
    const uint32_t* chunk_idx;   // [n_work] chunk index within its unit
    const uint32_t* chunk_base;  // [units + 1] first chunk of each unit
    const uint32_t* unit_run;    // [units] first CTA of the unit | number of CTA runs << 16
    uint32_t n_work;             // total chunks
    uint32_t max_runs;           // partial slots per unit (one per CTA run)
    uint32_t* unit_done;         // [units] completion counters (zero between launches)
    uint32_t grid;               // persistent CTAs: min(n_work, SMs); CTA c owns chunks
                                 // [c * n_work / grid, (c + 1) * n_work / grid)
};
cudaError_t launch_attend(const LayerView& L, const uint16_t* q, const PageList& pages, uint32_t* ready,
                          const AttendWork& work, float* part_o, float* part_ml, float* out, cudaStream_t s,
                          int* launches);
size_t attend_smem_bytes(uint32_t D, uint32_t P);
// Fused decode-step selection (select.cu): estimate + select + page resolution per
// (sequence, KV head) unit in one kernel over balanced slices of the units' centroids
// (the last slice of a unit to finish finalizes it); the same ordered selections as
// launch_score + launch_topk (INT4 mean stores).
bool select_fused_supported(const LayerView& L);
// One slice of the fused selection: rows [r nd / n, (r + 1) nd / n) of unit `unit`'s
// candidate domain (nd = N, or N - 1 when the trailing block is forced), one CTA each;
// `first` is the unit's first slice (its bounds are slot[first .. first + n)).
struct SliceDesc {
    uint32_t unit, r, n, first;
};
struct SelectPlan {
    uint32_t rows;       // slice size S (rows)
    uint32_t stages;     // code-ring stages (2..4)
    uint32_t cand_cap;   // candidates the finalize orders
    uint32_t pg_cap;     // candidate page ids the finalize prefetches
    uint32_t n_slices;   // grid
    bool ok;             // fits in shared memory
};
struct SelectWork {
    const SliceDesc* slices;  // [n_slices], unit order
    uint32_t* slot;           // [4 n_slices] per-slice key range (min, max), bound t_r
    uint32_t* arrive;         // [units] slices done this step (zero between steps)
    uint32_t* keys;           // [store segment] integer filter keys
};
SelectPlan plan_select(const std::vector<UnitDesc>& desc, uint32_t max_budget, uint32_t D, int num_sms,
                       std::vector<SliceDesc>* slices);
uint64_t select_slices_bound(const std::vector<UnitDesc>& desc);
size_t select_fused_smem(uint32_t D, uint32_t stages, uint32_t cand_cap, uint32_t pg_cap, uint32_t rows);
cudaError_t init_select_attributes();  // per device, once
cudaError_t launch_select_fused(const LayerView& L, const uint16_t* q, const SelectPlan& plan, const SelectWork& work,
                                uint32_t* blocks, uint32_t stride, uint32_t* counts, const PageList& pages,
                                uint32_t* ready, float* diag_approx, float* diag_err, uint16_t* q_copy, cudaStream_t s,
                                int* launches);
// q_copy (else null): q is read from (device-mapped pinned) host memory; each unit's
// finalizing CTA copies the unit's G query rows to q_copy (device) for the attention.
cudaError_t init_attend_attributes();  // per device, once
// Dense fp64 decode attention with weights (dense.cu; full_attention_oracle,
// engine.cpp:357-403) and attention_recall (calibrator.cpp:48-71).
uint32_t full_attention_splits(uint32_t units, uint32_t max_tokens, int num_sms);
cudaError_t launch_full_attention(const LayerView& L, const uint16_t* q, uint32_t splits, double* weights,
                                  uint64_t wstride, double* part_o, double* part_ml, double* stats, float* out,
                                  cudaStream_t s, int* launches);
cudaError_t launch_recall(const LayerView& L, uint32_t max_nblocks, const double* weights, uint64_t wstride,
                          const uint32_t* blocks, uint32_t stride, const uint32_t* counts, double* recall,
                          cudaStream_t s, int* launches);
cudaError_t launch_fill_synth(uint16_t* dst, uint64_t count, uint64_t seed, uint64_t stream_id,
                              cudaStream_t s);

// Per-unit ready flags sit one per 128-byte line (flag u at ready[u * kReadyStride]): the
// attention producers poll them while the selection publishes, spread over L2 slices.
constexpr uint32_t kReadyStride = 32;

// Rows per attention chunk (one pipeline stage), see attend.cu.
constexpr uint32_t kAttnChunkRows = 128;
// Consumer warps per attention CTA; each owns a 16-row split of every chunk with
// its own online-softmax state and partials (partial slots per chunk).
constexpr uint32_t kAttnSplits = 8;
// Resident scoring CTAs per SM (score.cu: 256 threads, <= 128 registers).
constexpr uint32_t kScoreCtasPerSm = 2;

}  // namespace absp

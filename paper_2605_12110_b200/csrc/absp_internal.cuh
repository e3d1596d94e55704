// Internal declarations shared by the sm_100a kernels and the C-ABI host layer.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "absp.h"

namespace absp {

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

// Work item of the scoring kernel: a run of centroids of one unit.
struct ScoreItem {
    uint32_t unit;
    uint32_t start;
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
    uint32_t* codes;    // packed, per unit [words][cap]
    uint32_t* codes_min;
    float* scales;      // [units][d]
    float* zps;
    float* scales_min;
    float* zps_min;
    float* scores;      // [seg]
};

// Launch wrappers (each returns cudaGetLastError after the launch).
cudaError_t launch_build_store(const LayerView& L, uint32_t max_cap, cudaStream_t s, int* launches);
cudaError_t launch_score(const LayerView& L, const uint16_t* q, const ScoreItem* items,
                         uint32_t n_items, cudaStream_t s, int* launches);
// Selected blocks resolved to pool pages, laid out by global attention chunk:
// unit u's slot s = entry * (B/P) + page lives at index chunk_base[u] * ns + s, so
// chunk w's slots are [w * ns, (w + 1) * ns).
struct PageList {
    uint32_t* page;               // head * pool_pages + pool page id
    uint16_t* valid;              // valid rows of the page (0 = empty slot)
    const uint32_t* chunk_base;   // [units + 1] first chunk of each unit (work list)
    uint32_t ns;                  // page slots per chunk = kAttnChunkRows / P
};
cudaError_t launch_topk(const LayerView& L, uint32_t max_nblocks, uint32_t max_budget,
                        uint32_t* blocks, uint32_t stride, uint32_t* counts, const PageList& pages,
                        cudaStream_t s, int* launches);
cudaError_t launch_resolve_pages(const LayerView& L, const uint32_t* blocks, uint32_t stride,
                                 const uint32_t* counts, const PageList& pages, cudaStream_t s,
                                 int* launches);
// Attention work list: all 128-row chunks of all units, unit-major.
struct AttendWork {
    const uint32_t* chunk_unit;  // [n_work] unit of each chunk
    const uint32_t* chunk_idx;   // [n_work] chunk index within its unit
    const uint32_t* chunk_base;  // [units + 1] first chunk of each unit
    uint32_t n_work;             // total chunks
    uint32_t slots_per_unit;     // partial slots reserved per unit (max chunks of a unit)
    uint32_t* unit_done;         // [units] completion counters (zero between launches)
    uint32_t grid;               // persistent CTAs (one per SM)
};
cudaError_t launch_attend(const LayerView& L, const uint16_t* q, const PageList& pages,
                          const uint32_t* counts, const AttendWork& work,
                          float* part_o, float* part_ml, float* out, cudaStream_t s,
                          int* launches);
size_t attend_smem_bytes(uint32_t D, uint32_t P);
cudaError_t init_attend_attributes();  // per device, once
cudaError_t launch_fill_synth(uint16_t* dst, uint64_t count, uint64_t seed, uint64_t stream_id,
                              cudaStream_t s);

// Rows per attention chunk (one pipeline stage), see attend.cu.
constexpr uint32_t kAttnChunkRows = 128;
// Consumer warps per attention CTA; each owns a 16-row split of every chunk with
// its own online-softmax state and partials (partial slots per chunk).
constexpr uint32_t kAttnSplits = 8;
// Centroids per scoring CTA, see score.cu.
constexpr uint32_t kScoreItemCentroids = 2048;

}  // namespace absp

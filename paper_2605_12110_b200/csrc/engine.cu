// DecodeEngine as a C-ABI object (include/absp.h, absp_engine_*): the reference's
// DecodeEngine (engine.hpp:90-129, engine.cpp:405-463) for one sequence, on the GPU,
// with no PyTorch. It owns the paged KV cache (bf16 per-head pools with the
// reference allocator's sequential page ids, kv_cache.cpp:53-60), a one-layer absp
// context (quantized centroid store), a stream and the staging buffers, and runs
//   prefill : fp32 [H][tokens][d] -> bf16 pages (k_stage_rows) -> absp_kv_bind +
//             absp_build_store             (engine.cpp:414-440)
//   step    : fp32 k, v, q -> bf16 (k_stage_rows) -> absp_append (append +
//             refresh_tail_centroids + requantize_heads) -> absp_decode_step
//             (estimate -> select -> attend) -> output + selection to the host
//                                          (engine.cpp:442-463)
// The fp32 -> bf16 rounding (RNE) of the inputs is the build's storage format (SURVEY.md
// Appendix A); every arithmetic result comes from the sm_100a kernels. While
// seq_len <= token_budget every block is selected, so the sparse kernel computes the
// full attention the reference falls back to (full_attention_fallback is reported).
#include <cuda_runtime.h>

#include <algorithm>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "absp_internal.cuh"

namespace absp {
namespace {

__device__ __forceinline__ uint16_t f32_to_bf16_rne(float f) {
    uint32_t u = __float_as_uint(f);
    if ((u & 0x7fffffffu) > 0x7f800000u) return uint16_t((u >> 16) | 0x40u);  // quiet NaN
    u += 0x7fffu + ((u >> 16) & 1u);
    return uint16_t(u >> 16);
}

// rows x d fp32 -> bf16: row r = (head h, token i) of src (head stride src_hs floats,
// tokens contiguous) lands at dst + (h * dst_hs + t0 + i) * d.
__global__ void k_stage_rows(const float* __restrict__ src, uint64_t src_hs, uint32_t tokens, uint32_t heads,
                             uint32_t d, uint16_t* __restrict__ dst, uint64_t dst_hs, uint64_t t0) {
    const uint64_t total = uint64_t(heads) * tokens * d;
    for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < total;
         e += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t row = e / d, c = e % d;
        const uint64_t h = row / tokens, i = row % tokens;
        dst[(h * dst_hs + t0 + i) * d + c] = f32_to_bf16_rne(src[h * src_hs + i * d + c]);
    }
}

cudaError_t stage_rows(const float* src, uint64_t src_hs, uint32_t tokens, uint32_t heads, uint32_t d,
                       uint16_t* dst, uint64_t dst_hs, uint64_t t0, cudaStream_t s) {
    const uint64_t total = uint64_t(heads) * tokens * d;
    if (total == 0) return cudaSuccess;
    const uint64_t blocks = std::min<uint64_t>((total + 255) / 256, 148 * 32);
    k_stage_rows<<<unsigned(blocks), 256, 0, s>>>(src, src_hs, tokens, heads, d, dst, dst_hs, t0);
    return cudaGetLastError();
}

}  // namespace
}  // namespace absp

using namespace absp;

struct absp_engine {
    int device = 0;
    absp_config cfg{};
    std::vector<uint32_t> block_sizes;
    uint64_t capacity = 0, pages = 0, seq_len = 0;
    bool prefilled = false;
    absp_ctx* ctx = nullptr;
    cudaStream_t stream = nullptr;
    uint16_t* k_pool = nullptr;  // bf16 [H][pages][P][d]
    uint16_t* v_pool = nullptr;
    uint32_t* page_table = nullptr;  // [1][pages], sequential ids
    float* stage_f32 = nullptr;      // step inputs k | v | q (fp32)
    uint16_t* stage_bf16 = nullptr;  // k_new | v_new | q (bf16)
    float* out_dev = nullptr;        // [Hq][d]
    float* host_in = nullptr;        // pinned: k | v | q
    float* host_out = nullptr;       // pinned: out
    uint32_t* host_sel = nullptr;    // pinned: blocks [H][stride] | counts [H]
    uint32_t sel_stride = 0;
};

namespace {

absp_status efail(absp_status st, const std::string& msg) {
    set_last_error(msg);  // absp_last_error()
    return st;
}

#define ENG_CUDA(call)                                                                        \
    do {                                                                                      \
        cudaError_t e__ = (call);                                                             \
        if (e__ != cudaSuccess) return efail(ABSP_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e__)); \
    } while (0)

// Propagates a C-ABI failure with its message.
#define ENG_ABI(call)                                                 \
    do {                                                              \
        absp_status s__ = (call);                                     \
        if (s__ != ABSP_OK) return s__; /* message already set */     \
    } while (0)

struct Dev {
    int prev = -1;
    explicit Dev(int d) {
        cudaGetDevice(&prev);
        cudaSetDevice(d);
    }
    ~Dev() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

void release(absp_engine* e) {
    if (!e) return;
    Dev dg(e->device);
    if (e->ctx) absp_ctx_destroy(e->ctx);
    if (e->stream) cudaStreamSynchronize(e->stream);
    cudaFree(e->k_pool);
    cudaFree(e->v_pool);
    cudaFree(e->page_table);
    cudaFree(e->stage_f32);
    cudaFree(e->stage_bf16);
    cudaFree(e->out_dev);
    cudaFreeHost(e->host_in);
    cudaFreeHost(e->host_out);
    cudaFreeHost(e->host_sel);
    if (e->stream) cudaStreamDestroy(e->stream);
    delete e;
}

}  // namespace

extern "C" {

absp_status absp_engine_create(int device, const absp_config* config, const uint32_t* block_sizes,
                               uint64_t capacity_tokens, absp_engine** out) {
    if (!out || !config || !block_sizes) return efail(ABSP_EINVAL, "engine_create: null pointer");
    *out = nullptr;
    if (capacity_tokens == 0) return efail(ABSP_EINVAL, "init_cache: capacity must be positive");  // kv_cache.cpp:163-165
    if (capacity_tokens > 0xffffffffull) return efail(ABSP_EINVAL, "engine_create: capacity above 2^32 tokens");
    absp_config c = *config;
    c.max_batch = 1;
    c.num_layers = 1;
    c.max_seq_len = uint32_t(capacity_tokens);
    auto* e = new absp_engine;
    e->device = device;
    e->cfg = c;
    e->capacity = capacity_tokens;
    e->block_sizes.assign(block_sizes, block_sizes + c.num_kv_heads);
    absp_status st = absp_ctx_create(device, &c, &e->ctx);  // EngineConfig::validate + device checks
    if (st != ABSP_OK) {
        delete e;
        return st;
    }
    st = absp_set_assignment(e->ctx, 0, block_sizes);  // BlockAssignment::validate (engine.cpp:410)
    if (st != ABSP_OK) {
        release(e);
        return st;
    }
    Dev dg(device);
    const uint64_t H = c.num_kv_heads, D = c.head_dim, P = c.page_size, Hq = c.num_q_heads;
    e->pages = (capacity_tokens + P - 1) / P;
    e->sel_stride = (c.token_budget + c.candidate_block_sizes[0] - 1) / c.candidate_block_sizes[0];
    const size_t pool = H * e->pages * P * D;
    cudaError_t ce = cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking);
    if (ce == cudaSuccess) ce = cudaMalloc(&e->k_pool, pool * 2);
    if (ce == cudaSuccess) ce = cudaMalloc(&e->v_pool, pool * 2);
    if (ce == cudaSuccess) ce = cudaMemset(e->k_pool, 0, pool * 2);
    if (ce == cudaSuccess) ce = cudaMemset(e->v_pool, 0, pool * 2);
    if (ce == cudaSuccess) ce = cudaMalloc(&e->page_table, e->pages * 4);
    if (ce == cudaSuccess) ce = cudaMalloc(&e->stage_f32, (2 * H + Hq) * D * 4);
    if (ce == cudaSuccess) ce = cudaMalloc(&e->stage_bf16, (2 * H + Hq) * D * 2);
    if (ce == cudaSuccess) ce = cudaMalloc(&e->out_dev, Hq * D * 4);
    if (ce == cudaSuccess) ce = cudaMallocHost(&e->host_in, (2 * H + Hq) * D * 4);
    if (ce == cudaSuccess) ce = cudaMallocHost(&e->host_out, Hq * D * 4);
    if (ce == cudaSuccess) ce = cudaMallocHost(&e->host_sel, (H * e->sel_stride + H) * 4);
    if (ce == cudaSuccess) {  // the reference allocator: token t of every head on page t / P
        std::vector<uint32_t> ids(e->pages);
        for (uint64_t p = 0; p < e->pages; ++p) ids[p] = uint32_t(p);
        ce = cudaMemcpy(e->page_table, ids.data(), e->pages * 4, cudaMemcpyHostToDevice);
    }
    if (ce != cudaSuccess) {
        set_last_error(std::string("engine_create: ") + cudaGetErrorString(ce));
        release(e);
        return ce == cudaErrorMemoryAllocation ? ABSP_ENOMEM : ABSP_ECUDA;
    }
    *out = e;
    return ABSP_OK;
}

absp_status absp_engine_destroy(absp_engine* e) {
    release(e);
    return ABSP_OK;
}

absp_status absp_engine_prefill(absp_engine* e, const float* keys, uint64_t keys_len, const float* values,
                                uint64_t values_len, uint64_t num_tokens) {
    nvtxRangePushA("absp_engine_prefill");
    struct Pop { ~Pop() { nvtxRangePop(); } } nvtx_pop_;
    if (!e) return efail(ABSP_EINVAL, "null engine");
    if (e->prefilled) return efail(ABSP_ESTATE, "prefill: engine already prefilled");  // engine.cpp:416
    const uint64_t H = e->cfg.num_kv_heads, D = e->cfg.head_dim, P = e->cfg.page_size;
    if (num_tokens == 0 || !keys || !values || keys_len < H * num_tokens * D || values_len < H * num_tokens * D)
        return efail(ABSP_EINVAL, "prefill: tensor smaller than num_tokens");  // engine.cpp:420-423
    if (num_tokens > e->capacity)  // PagedKVCache::append (kv_cache.cpp:48-50)
        return efail(ABSP_ECAPACITY, "append: kv cache at capacity (" + std::to_string(e->capacity) + " tokens)");
    Dev dg(e->device);
    // head h's tokens start at h * (keys_len / H) floats (engine.cpp:424-431); staged in
    // chunks of whole tokens through one device buffer
    const uint64_t k_hs = keys_len / H, v_hs = values_len / H;
    const uint64_t chunk = std::max<uint64_t>(1, std::min<uint64_t>(num_tokens, (64ull << 20) / (H * D * 4)));
    float* dbuf = nullptr;
    ENG_CUDA(cudaMalloc(&dbuf, H * chunk * D * 4));
    cudaError_t ce = cudaSuccess;
    for (int kv = 0; kv < 2 && ce == cudaSuccess; ++kv) {
        const float* src = kv ? values : keys;
        const uint64_t hs = kv ? v_hs : k_hs;
        uint16_t* pool = kv ? e->v_pool : e->k_pool;
        for (uint64_t t0 = 0; t0 < num_tokens && ce == cudaSuccess; t0 += chunk) {
            const uint64_t cnt = std::min(chunk, num_tokens - t0);
            ce = cudaMemcpy2DAsync(dbuf, cnt * D * 4, src + t0 * D, hs * 4, cnt * D * 4, H, cudaMemcpyHostToDevice,
                                   e->stream);
            if (ce == cudaSuccess)
                ce = stage_rows(dbuf, cnt * D, uint32_t(cnt), uint32_t(H), uint32_t(D), pool, e->pages * P, t0, e->stream);
            if (ce == cudaSuccess) ce = cudaStreamSynchronize(e->stream);  // dbuf is reused
        }
    }
    cudaFree(dbuf);
    if (ce != cudaSuccess) return efail(ABSP_ECUDA, std::string("prefill staging: ") + cudaGetErrorString(ce));
    const uint32_t n = uint32_t(num_tokens);
    ENG_ABI(absp_kv_bind(e->ctx, 0, e->k_pool, e->v_pool, e->pages, e->page_table, uint32_t(e->pages), &n, 1));
    ENG_ABI(absp_build_store(e->ctx, 0, e->stream));  // compute_block_centroids + quantize_store
    ENG_CUDA(cudaStreamSynchronize(e->stream));
    e->seq_len = num_tokens;
    e->prefilled = true;
    return ABSP_OK;
}

absp_status absp_engine_step(absp_engine* e, const float* keys, uint64_t keys_len, const float* values,
                             uint64_t values_len, const float* query, uint64_t query_len, float* out,
                             uint32_t* blocks, uint32_t blocks_stride, uint32_t* counts, int* full_attention_fallback) {
    nvtxRangePushA("absp_engine_step");
    struct Pop { ~Pop() { nvtxRangePop(); } } nvtx_pop_;
    if (!e) return efail(ABSP_EINVAL, "null engine");
    if (!e->prefilled) return efail(ABSP_ESTATE, "step: call prefill first");  // engine.cpp:444
    const uint64_t H = e->cfg.num_kv_heads, D = e->cfg.head_dim, Hq = e->cfg.num_q_heads;
    if (!keys || !values || keys_len != H * D || values_len != H * D)  // kv_cache.cpp:45-47
        return efail(ABSP_EINVAL, "append: expected num_heads * head_dim floats per tensor");
    if (!query || query_len != Hq * D)  // engine.cpp:74-76
        return efail(ABSP_EINVAL, "estimate_scores: query dimension mismatch");
    if (!out) return efail(ABSP_EINVAL, "step: null output");
    if (blocks && blocks_stride < e->sel_stride)
        return efail(ABSP_EINVAL, "step: blocks_stride below ceil(token_budget / min block size)");
    if (e->seq_len >= e->capacity)  // kv_cache.cpp:48-50
        return efail(ABSP_ECAPACITY, "append: kv cache at capacity (" + std::to_string(e->capacity) + " tokens)");
    Dev dg(e->device);
    std::copy(keys, keys + H * D, e->host_in);
    std::copy(values, values + H * D, e->host_in + H * D);
    std::copy(query, query + Hq * D, e->host_in + 2 * H * D);
    ENG_CUDA(cudaMemcpyAsync(e->stage_f32, e->host_in, (2 * H + Hq) * D * 4, cudaMemcpyHostToDevice, e->stream));
    ENG_CUDA(stage_rows(e->stage_f32, D, 1, uint32_t(2 * H + Hq), uint32_t(D), e->stage_bf16, 1, 0, e->stream));
    const uint16_t* k_new = e->stage_bf16;
    const uint16_t* v_new = e->stage_bf16 + H * D;
    const uint16_t* q = e->stage_bf16 + 2 * H * D;
    ENG_ABI(absp_append(e->ctx, 0, k_new, v_new, e->stream));  // append + refresh + requantize
    ENG_ABI(absp_decode_step(e->ctx, 0, q, e->out_dev, e->stream));  // estimate -> select -> attend
    ENG_CUDA(cudaMemcpyAsync(e->host_out, e->out_dev, Hq * D * 4, cudaMemcpyDeviceToHost, e->stream));
    const uint32_t* sb = nullptr;
    const uint32_t* sc = nullptr;
    uint32_t stride = 0;
    ENG_ABI(absp_last_selection(e->ctx, 0, &sb, &stride, &sc));
    ENG_CUDA(cudaMemcpyAsync(e->host_sel, sb, H * stride * 4, cudaMemcpyDeviceToHost, e->stream));
    ENG_CUDA(cudaMemcpyAsync(e->host_sel + H * stride, sc, H * 4, cudaMemcpyDeviceToHost, e->stream));
    ENG_CUDA(cudaStreamSynchronize(e->stream));
    ++e->seq_len;
    std::copy(e->host_out, e->host_out + Hq * D, out);
    for (uint64_t h = 0; h < H; ++h) {
        const uint32_t cnt = e->host_sel[H * stride + h];
        if (counts) counts[h] = cnt;
        if (blocks)
            for (uint32_t i = 0; i < cnt; ++i) blocks[h * blocks_stride + i] = e->host_sel[h * stride + i];
    }
    if (full_attention_fallback) *full_attention_fallback = e->seq_len <= e->cfg.token_budget ? 1 : 0;
    return ABSP_OK;
}

absp_status absp_engine_info(absp_engine* e, uint64_t* seq_len, uint32_t* blocks_stride, absp_ctx** ctx) {
    if (!e) return efail(ABSP_EINVAL, "null engine");
    if (seq_len) *seq_len = e->seq_len;
    if (blocks_stride) *blocks_stride = e->sel_stride;
    if (ctx) *ctx = e->ctx;
    return ABSP_OK;
}

}  // extern "C"

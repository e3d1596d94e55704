// One calibration sample on the GPU (include/absp.h, absp_profile_sample): the body of
// the reference's profile_sensitivity / transfer_check loops (calibrator.cpp:86-106,
// :172-196) for one trace:
//
//   cache_from_trace            -> bf16 per-head pools with sequential pages (one upload)
//   full_attention_oracle       -> absp_full_attention (fp64, weights)       dense.cu
//   for every candidate B:       uniform assignment, compute_block_centroids +
//                                quantize_store -> absp_build_store,
//                                estimate + select_topk -> absp_select,
//                                attention_recall -> absp_attention_recall   dense.cu
//   (+ the same for a given assignment: transfer_check's adaptive recall)
//
// One context holds a layer per assignment, all bound to the same pools, so the trace
// crosses PCIe once. The host side (averaging over samples, assign_block_sizes,
// normalized_recall, the matched-uniform delta) stays in absp.hpp / absparse.py as the
// reference's host code is; every number here comes from the sm_100a kernels.
#include <cuda_runtime.h>

#include <algorithm>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "absp_internal.cuh"

namespace absp {
namespace {

__device__ __forceinline__ uint16_t bf16_rne(float f) {
    uint32_t u = __float_as_uint(f);
    if ((u & 0x7fffffffu) > 0x7f800000u) return uint16_t((u >> 16) | 0x40u);  // quiet NaN
    u += 0x7fffu + ((u >> 16) & 1u);
    return uint16_t(u >> 16);
}

// [H][n][d] fp32 -> [H][pages * P][d] bf16 (sequential pages: token t is row t of the
// head's pool; the rows past n of the last page stay zero)
__global__ void k_trace_to_pool(const float* __restrict__ src, uint32_t H, uint64_t n, uint32_t d,
                                uint64_t rows_per_head, uint16_t* __restrict__ dst) {
    const uint64_t total = uint64_t(H) * n * d;
    for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < total;
         e += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t h = e / (n * d), r = e % (n * d);
        dst[h * rows_per_head * d + r] = bf16_rne(src[e]);
    }
}

__global__ void k_to_bf16(const float* __restrict__ src, uint64_t count, uint16_t* __restrict__ dst) {
    for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < count; e += uint64_t(gridDim.x) * blockDim.x)
        dst[e] = bf16_rne(src[e]);
}

__global__ void k_iota(uint32_t* p, uint32_t n) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = i;
}

absp_status cfail(absp_status st, const std::string& msg) {
    set_last_error(msg);
    return st;
}

// Owns every device allocation of one sample.
struct Sample {
    int prev = -1;
    absp_ctx* ctx = nullptr;
    std::vector<void*> bufs;
    explicit Sample(int dev) {
        cudaGetDevice(&prev);
        cudaSetDevice(dev);
    }
    template <typename T>
    cudaError_t alloc(T** p, size_t count) {
        void* v = nullptr;
        const cudaError_t e = cudaMalloc(&v, std::max<size_t>(count, 1) * sizeof(T));
        if (e == cudaSuccess) {
            bufs.push_back(v);
            *p = static_cast<T*>(v);
        }
        return e;
    }
    ~Sample() {
        if (ctx) absp_ctx_destroy(ctx);
        for (void* v : bufs) cudaFree(v);
        if (prev >= 0) cudaSetDevice(prev);
    }
};

#define CAL_CUDA(call)                                                                                 \
    do {                                                                                               \
        cudaError_t e__ = (call);                                                                      \
        if (e__ != cudaSuccess) return cfail(ABSP_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e__)); \
    } while (0)
#define CAL_ABI(call)                                \
    do {                                                 \
        absp_status s__ = (call);                        \
        if (s__ != ABSP_OK) return s__;                  \
    } while (0)

}  // namespace
}  // namespace absp

using namespace absp;

extern "C" absp_status absp_profile_sample(int device, const absp_config* config, const float* keys,
                                           const float* values, const float* queries, uint64_t seq_len,
                                           const uint32_t* assignment, double* recalls, double* assigned_recall) {
    nvtxRangePushA("absp_profile_sample");
    struct Pop { ~Pop() { nvtxRangePop(); } } nvtx_pop_;
    if (!config || !keys || !values || !queries || !recalls)
        return cfail(ABSP_EINVAL, "profile_sample: null pointer");
    CAL_ABI(absp_config_validate(config));
    if (seq_len == 0) return cfail(ABSP_EINVAL, "profile_sample: empty trace");
    if (seq_len > 0xffffffffull) return cfail(ABSP_EINVAL, "profile_sample: trace longer than 2^32 tokens");
    if (assignment && !assigned_recall) return cfail(ABSP_EINVAL, "profile_sample: null assigned_recall");
    absp_config cfg = *config;
    const uint32_t H = cfg.num_kv_heads, Hq = cfg.num_q_heads, G = Hq / H, D = cfg.head_dim, P = cfg.page_size;
    const uint32_t nc = cfg.num_candidates;
    const uint32_t n = uint32_t(seq_len);
    const uint32_t layers = nc + (assignment ? 1u : 0u);
    cfg.max_batch = 1;
    cfg.max_seq_len = n;
    cfg.num_layers = layers;
    const uint64_t pages = (uint64_t(n) + P - 1) / P;

    Sample smp(device);
    float* f32 = nullptr;
    uint16_t *kp = nullptr, *vp = nullptr, *q = nullptr;
    uint32_t* pt = nullptr;
    float* out = nullptr;
    double *w = nullptr, *rec = nullptr;
    CAL_CUDA(smp.alloc(&f32, uint64_t(H) * n * D));
    CAL_CUDA(smp.alloc(&kp, uint64_t(H) * pages * P * D));
    CAL_CUDA(smp.alloc(&vp, uint64_t(H) * pages * P * D));
    CAL_CUDA(smp.alloc(&q, uint64_t(Hq) * D));
    CAL_CUDA(smp.alloc(&pt, pages));
    CAL_CUDA(smp.alloc(&out, uint64_t(Hq) * D));
    CAL_CUDA(smp.alloc(&w, uint64_t(Hq) * n));
    CAL_CUDA(smp.alloc(&rec, uint64_t(Hq) * layers));
    CAL_CUDA(cudaMemset(kp, 0, uint64_t(H) * pages * P * D * 2));
    CAL_CUDA(cudaMemset(vp, 0, uint64_t(H) * pages * P * D * 2));
    const unsigned grid = 148 * 8;
    // cache_from_trace (workload.cpp:311-330): the trace's rows in order, pages handed out
    // sequentially (kv_cache.cpp:53-60)
    CAL_CUDA(cudaMemcpy(f32, keys, uint64_t(H) * n * D * 4, cudaMemcpyHostToDevice));
    k_trace_to_pool<<<grid, 256>>>(f32, H, n, D, pages * P, kp);
    CAL_CUDA(cudaGetLastError());
    CAL_CUDA(cudaMemcpy(f32, values, uint64_t(H) * n * D * 4, cudaMemcpyHostToDevice));
    k_trace_to_pool<<<grid, 256>>>(f32, H, n, D, pages * P, vp);
    CAL_CUDA(cudaGetLastError());
    CAL_CUDA(cudaMemcpy(f32, queries, uint64_t(Hq) * D * 4, cudaMemcpyHostToDevice));
    k_to_bf16<<<4, 256>>>(f32, uint64_t(Hq) * D, q);
    k_iota<<<4, 256>>>(pt, uint32_t(pages));
    CAL_CUDA(cudaGetLastError());

    CAL_ABI(absp_ctx_create(device, &cfg, &smp.ctx));
    std::vector<uint32_t*> blk(layers), cnt(layers);
    std::vector<uint32_t> stride(layers);
    for (uint32_t l = 0; l < layers; ++l) {
        std::vector<uint32_t> bs(H);
        for (uint32_t h = 0; h < H; ++h) bs[h] = l < nc ? cfg.candidate_block_sizes[l] : assignment[h];
        CAL_ABI(absp_set_assignment(smp.ctx, l, bs.data()));
        CAL_ABI(absp_kv_bind(smp.ctx, l, kp, vp, pages, pt, uint32_t(pages), &n, 1));
        CAL_ABI(absp_build_store(smp.ctx, l, nullptr));
        absp_layer_info info{};
        CAL_ABI(absp_get_layer_info(smp.ctx, l, &info));
        stride[l] = std::max(info.max_select, 1u);
        CAL_CUDA(smp.alloc(&blk[l], uint64_t(H) * stride[l]));
        CAL_CUDA(smp.alloc(&cnt[l], H));
        CAL_ABI(absp_select(smp.ctx, l, q, blk[l], stride[l], cnt[l], nullptr));
    }
    CAL_ABI(absp_full_attention(smp.ctx, 0, q, out, w, n, nullptr));
    for (uint32_t l = 0; l < layers; ++l)
        CAL_ABI(absp_attention_recall(smp.ctx, l, w, n, blk[l], stride[l], cnt[l], rec + uint64_t(l) * Hq, nullptr));
    std::vector<double> h_rec(uint64_t(Hq) * layers);
    CAL_CUDA(cudaMemcpy(h_rec.data(), rec, h_rec.size() * 8, cudaMemcpyDeviceToHost));
    // per KV head: the mean over its G query heads (G = 1: the reference's per-head recall),
    // RecallTable layout recalls[h * nc + ci] (calibrator.hpp:15-28)
    for (uint32_t l = 0; l < layers; ++l)
        for (uint32_t h = 0; h < H; ++h) {
            double acc = 0.0;
            for (uint32_t g = 0; g < G; ++g) acc += h_rec[uint64_t(l) * Hq + h * G + g];
            const double r = G == 1 ? acc : acc / double(G);
            if (l < nc) recalls[uint64_t(h) * nc + l] = r;
            else assigned_recall[h] = r;
        }
    return ABSP_OK;
}

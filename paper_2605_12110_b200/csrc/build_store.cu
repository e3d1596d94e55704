// Prefill-time centroid build and quantization (sm_100a).
//
// Reference: compute_block_centroids / compute_one_centroid (centroids.cpp:18-43,
// 86-120) and quantize_store / quantize_segment (quantizer.cpp:16-111).
// Every arithmetic step uses the *_rn intrinsics so nvcc never contracts or
// reorders it: the stored centroids, scales, zero points and codes are
// bit-identical to the reference on the same (bf16-upcast) keys.
//
// HBM layout written here (per layer, capacity-reserved per unit u=(b,h)):
//   values   fp32 [seg_u + i][D]                 (CentroidStore::values)
//   scales   fp32 [u][D], zps fp32 [u][D]         (per (head, channel) params)
//   codes    u32  [(seg_u + i) * W + code_word_pos(i, w, W)]   W = D*bits/32
//            words per centroid row; word w holds channels w*(32/bits) ..
//            +32/bits-1, low bits first. Rows are contiguous per unit so the
//            scorer bulk-copies runs of rows into shared memory (score.cu).
#include "absp_internal.cuh"

#include <math.h>

namespace absp {
namespace {

__device__ __forceinline__ float bf16f(uint16_t x) { return __uint_as_float(uint32_t(x) << 16); }

// Mean / maxmin centroid of block i of unit u for channel c. One thread per
// (centroid, channel); rows are visited in token order exactly like the
// reference loop (centroids.cpp:25-31), so the fp64 sum is bit-identical even
// for inputs whose sum would be order-sensitive.
template <int D, int METHOD>
__global__ void __launch_bounds__(D * 8) k_centroids(LayerView L) {
    const uint32_t u = blockIdx.y;
    const UnitDesc du = L.desc[u];
    const uint32_t c = threadIdx.x % D;
    const uint32_t i = blockIdx.x * 8 + threadIdx.x / D;
    if (i >= du.n_blocks) return;
    const uint32_t begin = i * du.block;
    const uint32_t end = min(begin + du.block, du.n_tokens);
    const uint32_t* pt = L.page_table + size_t(du.seq) * L.max_pages;
    const size_t head_base = size_t(du.head) * L.pool_pages;
    const size_t out = (du.seg + i) * D + c;
    if (METHOD == ABSP_CENTROID_MEAN) {
        double acc = 0.0;
        for (uint32_t t = begin; t < end; ++t) {
            const size_t row = ((head_base + pt[t / L.P]) * L.P + t % L.P) * D;
            acc = __dadd_rn(acc, double(bf16f(L.k_pool[row + c])));
        }
        const double inv = __ddiv_rn(1.0, double(end - begin));
        L.values[out] = __double2float_rn(__dmul_rn(acc, inv));
    } else {
        float hi = -INFINITY, lo = INFINITY;
        for (uint32_t t = begin; t < end; ++t) {
            const size_t row = ((head_base + pt[t / L.P]) * L.P + t % L.P) * D;
            const float v = bf16f(L.k_pool[row + c]);
            hi = (hi < v) ? v : hi;  // std::max(hi, v)
            lo = (v < lo) ? v : lo;  // std::min(lo, v)
        }
        L.values[out] = hi;
        L.values_min[out] = lo;
    }
}

// Per-(unit, channel) quantization parameters (quantizer.cpp:24-43).
// min/max/absmax are order-independent, so the channel is reduced by
// 1024/D partitions in parallel.
template <int D>
__global__ void __launch_bounds__(1024) k_qparams(LayerView L, const float* values, float* scales,
                                                  float* zps) {
    constexpr int PARTS = 1024 / D;
    __shared__ float s_lo[PARTS][D];
    __shared__ float s_hi[PARTS][D];
    const uint32_t u = blockIdx.x;
    const UnitDesc du = L.desc[u];
    const uint32_t c = threadIdx.x % D;
    const uint32_t p = threadIdx.x / D;
    const bool asym = L.mode == ABSP_QUANT_ASYM;
    float lo = INFINITY, hi = -INFINITY, amax = 0.0f;
    for (uint32_t i = p; i < du.n_blocks; i += PARTS) {
        const float v = values[(du.seg + i) * D + c];
        lo = (v < lo) ? v : lo;
        hi = (hi < v) ? v : hi;
        const float a = fabsf(v);
        amax = (amax < a) ? a : amax;
    }
    s_lo[p][c] = asym ? lo : amax;
    s_hi[p][c] = hi;
    __syncthreads();
    if (p != 0) return;
    for (int q = 1; q < PARTS; ++q) {
        const float l2 = s_lo[q][c], h2 = s_hi[q][c];
        if (asym) {
            lo = (l2 < lo) ? l2 : lo;
            hi = (hi < h2) ? h2 : hi;
        } else {
            amax = (amax < l2) ? l2 : amax;
        }
    }
    const float floor_ = 1e-8f;  // kRangeFloor, quantizer.cpp:11
    float scale, zp;
    if (asym) {
        const float range = __fsub_rn(hi, lo);
        const float levels = float((1 << L.bits) - 1);
        scale = __fdiv_rn(range < floor_ ? floor_ : range, levels);
        zp = lo;
    } else {
        const float mid = float((1 << (L.bits - 1)) - 1);
        scale = __fdiv_rn(amax < floor_ ? floor_ : amax, mid);
        zp = 0.0f;
    }
    scales[size_t(u) * D + c] = scale;
    zps[size_t(u) * D + c] = zp;
}

// Encode + pack (quantizer.cpp:45-58): code = clamp(round((v - zp) / scale)) for
// asym, clamp(round(v / scale), -mid, mid) + mid for sym; std::round is
// half-away-from-zero, which is CUDA roundf.
template <int D, int BITS>
__global__ void __launch_bounds__(32 * (D * BITS / 32)) k_encode(LayerView L, const float* values,
                                                                 const float* scales,
                                                                 const float* zps,
                                                                 uint32_t* codes) {
    constexpr int W = D * BITS / 32;
    constexpr int CPW = 32 / BITS;
    const uint32_t u = blockIdx.y;
    const UnitDesc du = L.desc[u];
    const uint32_t i = blockIdx.x * 32 + threadIdx.x;
    const uint32_t w = threadIdx.y;
    if (i >= du.n_blocks) return;
    const bool asym = L.mode == ABSP_QUANT_ASYM;
    const int levels = (1 << BITS) - 1;
    const int mid = (1 << (BITS - 1)) - 1;
    uint32_t word = 0;
#pragma unroll
    for (int k = 0; k < CPW; ++k) {
        const uint32_t c = w * CPW + k;
        const float v = values[(du.seg + i) * D + c];
        const float sc = scales[size_t(u) * D + c];
        int q;
        if (asym) {
            const float zp = zps[size_t(u) * D + c];
            q = int(roundf(__fdiv_rn(__fsub_rn(v, zp), sc)));
            q = q < 0 ? 0 : (q > levels ? levels : q);
        } else {
            q = int(roundf(__fdiv_rn(v, sc)));
            q = (q < -mid ? -mid : (q > mid ? mid : q)) + mid;
        }
        word |= uint32_t(q) << (k * BITS);
    }
    codes[(du.seg + i) * W + code_word_pos(i, w, W)] = word;
}

// Decode-time append (PagedKVCache::append, kv_cache.cpp:44-70): token n of
// sequence b goes to row n % P of page page_table[b][n / P] of every KV head.
// One CTA per unit (b, h), one thread per channel; n is the unit's n_tokens
// before the append.
__global__ void k_append_rows(LayerView L, const uint16_t* __restrict__ k_new, const uint16_t* __restrict__ v_new,
                              uint16_t* k_pool, uint16_t* v_pool) {
    const uint32_t u = blockIdx.x;
    const UnitDesc du = L.desc[u];
    const uint32_t n = du.n_tokens;
    const uint32_t page = L.page_table[size_t(du.seq) * L.max_pages + n / L.P];
    const size_t row = ((size_t(du.head) * L.pool_pages + page) * L.P + n % L.P) * L.D;
    const size_t src = (size_t(du.seq) * L.H + du.head) * L.D;
    for (uint32_t c = threadIdx.x; c < L.D; c += blockDim.x) {
        k_pool[row + c] = k_new[src + c];
        v_pool[row + c] = v_new[src + c];
    }
}

// refresh_tail_centroid (centroids.cpp:122-156): after one appended token only the
// trailing block of a unit changed (the previous partial tail, or a block that just
// started); it is recomputed exactly like k_centroids. One CTA per unit.
template <int D, int METHOD>
__global__ void __launch_bounds__(D) k_tail_centroid(LayerView L) {
    const uint32_t u = blockIdx.x;
    const UnitDesc du = L.desc[u];
    const uint32_t c = threadIdx.x;
    const uint32_t i = du.n_blocks - 1;
    const uint32_t begin = i * du.block;
    const uint32_t end = min(begin + du.block, du.n_tokens);
    const uint32_t* pt = L.page_table + size_t(du.seq) * L.max_pages;
    const size_t head_base = size_t(du.head) * L.pool_pages;
    const size_t out = (du.seg + i) * D + c;
    if (METHOD == ABSP_CENTROID_MEAN) {
        double acc = 0.0;
        for (uint32_t t = begin; t < end; ++t) {
            const size_t row = ((head_base + pt[t / L.P]) * L.P + t % L.P) * D;
            acc = __dadd_rn(acc, double(bf16f(L.k_pool[row + c])));
        }
        const double inv = __ddiv_rn(1.0, double(end - begin));
        L.values[out] = __double2float_rn(__dmul_rn(acc, inv));
    } else {
        float hi = -INFINITY, lo = INFINITY;
        for (uint32_t t = begin; t < end; ++t) {
            const size_t row = ((head_base + pt[t / L.P]) * L.P + t % L.P) * D;
            const float v = bf16f(L.k_pool[row + c]);
            hi = (hi < v) ? v : hi;
            lo = (v < lo) ? v : lo;
        }
        L.values[out] = hi;
        L.values_min[out] = lo;
    }
}

template <int D>
cudaError_t build_d(const LayerView& L, uint32_t max_cap, bool tail_only, cudaStream_t s, int* launches) {
    if (tail_only) {  // decode-time maintenance: only each unit's trailing block changed
        if (L.method == ABSP_CENTROID_MEAN)
            k_tail_centroid<D, ABSP_CENTROID_MEAN><<<L.units, D, 0, s>>>(L);
        else
            k_tail_centroid<D, ABSP_CENTROID_MAXMIN><<<L.units, D, 0, s>>>(L);
    } else {
        const dim3 gc((max_cap + 7) / 8, L.units);
        if (L.method == ABSP_CENTROID_MEAN)
            k_centroids<D, ABSP_CENTROID_MEAN><<<gc, D * 8, 0, s>>>(L);
        else
            k_centroids<D, ABSP_CENTROID_MAXMIN><<<gc, D * 8, 0, s>>>(L);
    }
    ++*launches;
    if (L.bits == 0) return cudaGetLastError();
    const int arrays = L.method == ABSP_CENTROID_MAXMIN ? 2 : 1;
    for (int a = 0; a < arrays; ++a) {
        const float* vals = a ? L.values_min : L.values;
        float* sc = a ? L.scales_min : L.scales;
        float* zp = a ? L.zps_min : L.zps;
        uint32_t* cd = a ? L.codes_min : L.codes;
        k_qparams<D><<<L.units, 1024, 0, s>>>(L, vals, sc, zp);
        ++*launches;
        const dim3 ge((max_cap + 31) / 32, L.units);
        switch (L.bits) {
            case 2: k_encode<D, 2><<<ge, dim3(32, D * 2 / 32), 0, s>>>(L, vals, sc, zp, cd); break;
            case 4: k_encode<D, 4><<<ge, dim3(32, D * 4 / 32), 0, s>>>(L, vals, sc, zp, cd); break;
            default: k_encode<D, 8><<<ge, dim3(32, D * 8 / 32), 0, s>>>(L, vals, sc, zp, cd); break;
        }
        ++*launches;
    }
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_build_store(const LayerView& L, uint32_t max_cap, cudaStream_t s, int* launches) {
    if (L.D == 64) return build_d<64>(L, max_cap, false, s, launches);
    return build_d<128>(L, max_cap, false, s, launches);
}

// DecodeEngine::step's maintenance after an append (engine.cpp:445-449):
// refresh_tail_centroids, then requantize_heads over every head — per-(unit,
// channel) parameters from all centroids and every code re-encoded, which is
// exactly what quantizing the grown store from scratch gives.
cudaError_t launch_refresh_store(const LayerView& L, uint32_t max_cap, cudaStream_t s, int* launches) {
    if (L.D == 64) return build_d<64>(L, max_cap, true, s, launches);
    return build_d<128>(L, max_cap, true, s, launches);
}

cudaError_t launch_append_rows(const LayerView& L, const uint16_t* k_new, const uint16_t* v_new, cudaStream_t s,
                               int* launches) {
    k_append_rows<<<L.units, 128, 0, s>>>(L, k_new, v_new, const_cast<uint16_t*>(L.k_pool),
                                          const_cast<uint16_t*>(L.v_pool));
    ++*launches;
    return cudaGetLastError();
}

}  // namespace absp

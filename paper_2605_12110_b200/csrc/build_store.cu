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
#include "common.cuh"

#include <math.h>

#include <algorithm>

namespace absp {
namespace {

constexpr uint32_t kStatRows = 256;  // centroid rows per statistics slice (k_qstats)

__device__ __forceinline__ float ref_min(float a, float b) { return (b < a) ? b : a; }  // std::min(a, b)

// Centroid i of unit u over channels [c0, c0 + 8): the block's valid rows in token
// order, 16-byte loads of 8 bf16 keys, exactly the reference loop
// (compute_one_centroid, centroids.cpp:18-43): mean = fp64 sum * (1.0 / cnt) cast
// to float; maxmin = std::max / std::min from -inf / +inf.
template <int METHOD>
__device__ __forceinline__ void centroid8(const LayerView& L, const UnitDesc& du, uint32_t i, uint32_t c0,
                                          float hi_out[8], float lo_out[8]) {
    const uint32_t begin = i * du.block;
    const uint32_t end = min(begin + du.block, du.n_tokens);
    const uint32_t P = L.P;
    const uint32_t* pt = L.page_table + size_t(du.seq) * L.max_pages;
    const size_t head_base = size_t(du.head) * L.pool_pages;
    double acc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        acc[k] = 0.0;
        hi_out[k] = -INFINITY;
        lo_out[k] = INFINITY;
    }
    auto take = [&](const uint4 x) {
        const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const float v = bf16f(uint16_t(w[k / 2] >> (16 * (k & 1))));
            if (METHOD == ABSP_CENTROID_MEAN) {
                acc[k] = __dadd_rn(acc[k], double(v));
            } else {
                hi_out[k] = ref_max(hi_out[k], v);  // std::max(out, row)
                lo_out[k] = ref_min(lo_out[k], v);  // std::min(out, row)
            }
        }
    };
    // page by page (a block starts on a page boundary: B is a multiple of P); the next
    // page's id is loaded while this page's rows are, and up to 8 rows are in flight
    uint32_t t = begin;
    uint32_t page = pt[t / P];
    while (t < end) {
        const uint32_t r0 = t % P;
        const uint32_t n = min(P - r0, end - t);
        const uint32_t next = t + n < end ? pt[(t + n) / P] : 0u;
        const uint16_t* base = L.k_pool + ((head_base + page) * P + r0) * L.D + c0;
        uint32_t j = 0;
        for (; j + 8 <= n; j += 8) {
            uint4 x[8];
#pragma unroll
            for (int r = 0; r < 8; ++r) x[r] = __ldg(reinterpret_cast<const uint4*>(base + size_t(j + r) * L.D));
#pragma unroll
            for (int r = 0; r < 8; ++r) take(x[r]);
        }
        for (; j < n; ++j) take(__ldg(reinterpret_cast<const uint4*>(base + size_t(j) * L.D)));
        t += n;
        page = next;
    }
    if (METHOD == ABSP_CENTROID_MEAN) {
        const double inv = __ddiv_rn(1.0, double(end - begin));
#pragma unroll
        for (int k = 0; k < 8; ++k) hi_out[k] = __double2float_rn(__dmul_rn(acc[k], inv));
    }
}

__device__ __forceinline__ void store8(float* dst, const float v[8]) {
    reinterpret_cast<float4*>(dst)[0] = make_float4(v[0], v[1], v[2], v[3]);
    reinterpret_cast<float4*>(dst)[1] = make_float4(v[4], v[5], v[6], v[7]);
}

// compute_block_centroids (centroids.cpp:86-120): thread = (centroid, 8 channels);
// a warp reads whole 256 B key rows of two (D = 128) or four (D = 64) centroids.
template <int D, int METHOD>
__global__ void __launch_bounds__(256) k_centroids(LayerView L) {
    constexpr uint32_t TPC = D / 8, CPB = 256 / TPC;
    const uint32_t u = blockIdx.y;
    const UnitDesc du = L.desc[u];
    const uint32_t i = blockIdx.x * CPB + threadIdx.x / TPC;
    if (i >= du.n_blocks) return;
    const uint32_t c0 = (threadIdx.x % TPC) * 8;
    float hi[8], lo[8];
    centroid8<METHOD>(L, du, i, c0, hi, lo);
    store8(L.values + (du.seg + i) * D + c0, hi);
    if (METHOD == ABSP_CENTROID_MAXMIN) store8(L.values_min + (du.seg + i) * D + c0, lo);
}

// quantize_segment's parameters (quantizer.cpp:24-43) from the channel statistics.
__device__ __forceinline__ void qparams_of(float lo, float hi, float amax, bool asym, uint32_t bits, float& scale,
                                           float& zp) {
    const float floor_ = 1e-8f;  // kRangeFloor, quantizer.cpp:11
    if (asym) {
        const float range = __fsub_rn(hi, lo);
        scale = __fdiv_rn(range < floor_ ? floor_ : range, float((1u << bits) - 1u));
        zp = lo;
    } else {
        scale = __fdiv_rn(amax < floor_ ? floor_ : amax, float((1u << (bits - 1)) - 1u));
        zp = 0.0f;
    }
}

// Channel statistics, split so decode-time maintenance is incremental and exact:
// the "frozen" statistics cover every centroid but the trailing one (which is the
// only centroid an append changes); the full statistics are the frozen ones
// combined with the trailing centroid. std::min / std::max keep the earlier
// element on ties, so combining contiguous index ranges in index order reproduces
// the reference's sequential loop bit for bit (-0 vs +0 included); absmax is
// order-free. Per (array, unit, channel) two floats: a = lo (asym) or absmax (sym),
// b = hi.
//
// k_qstats: slice `blockIdx.x` of kStatRows frozen centroids, 1024/(D/4)
// contiguous partitions per slice (float4 loads, one warp per D = 128 row),
// partitions combined in order.
template <int D>
__global__ void __launch_bounds__(1024) k_qstats(LayerView L, float* __restrict__ part, uint32_t max_slices) {
    constexpr uint32_t TPR = D / 4, PARTS = 1024 / TPR, RPP = kStatRows / PARTS;
    __shared__ float s_a[PARTS][D];
    __shared__ float s_b[PARTS][D];
    const uint32_t u = blockIdx.y, arr = blockIdx.z, sl = blockIdx.x;
    const UnitDesc du = L.desc[u];
    const uint32_t nfrozen = du.n_blocks - 1;
    const uint32_t r0 = sl * kStatRows;
    if (r0 >= nfrozen) return;
    const bool asym = L.mode == ABSP_QUANT_ASYM;
    const float* vals = (arr ? L.values_min : L.values) + du.seg * D;
    const uint32_t p = threadIdx.x / TPR, c4 = (threadIdx.x % TPR) * 4;
    float a[4], b[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        a[k] = asym ? INFINITY : 0.0f;
        b[k] = -INFINITY;
    }
    const uint32_t rb = r0 + p * RPP, re = min(rb + RPP, nfrozen);
#pragma unroll 4
    for (uint32_t i = rb; i < re; ++i) {
        const float4 f = __ldcs(reinterpret_cast<const float4*>(vals + size_t(i) * D + c4));
        const float v[4] = {f.x, f.y, f.z, f.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            a[k] = asym ? ref_min(a[k], v[k]) : ref_max(a[k], fabsf(v[k]));
            b[k] = ref_max(b[k], v[k]);
        }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        s_a[p][c4 + k] = a[k];
        s_b[p][c4 + k] = b[k];
    }
    __syncthreads();
    if (threadIdx.x >= D) return;
    const uint32_t c = threadIdx.x;
    float A = s_a[0][c], B = s_b[0][c];
    for (uint32_t q = 1; q < PARTS; ++q) {
        A = asym ? ref_min(A, s_a[q][c]) : ref_max(A, s_a[q][c]);
        B = ref_max(B, s_b[q][c]);
    }
    float* dst = part + ((size_t(arr) * L.units + u) * max_slices + sl) * 2 * D;
    dst[c] = A;
    dst[D + c] = B;
}

// k_qfinal: slices in order -> frozen statistics; with the trailing centroid ->
// scale / zero point. One CTA per (unit, array), one thread per channel.
template <int D>
__global__ void __launch_bounds__(D) k_qfinal(LayerView L, const float* __restrict__ part, uint32_t max_slices) {
    const uint32_t u = blockIdx.x, arr = blockIdx.y, c = threadIdx.x;
    const UnitDesc du = L.desc[u];
    const bool asym = L.mode == ABSP_QUANT_ASYM;
    const uint32_t nfrozen = du.n_blocks - 1;
    const uint32_t nsl = (nfrozen + kStatRows - 1) / kStatRows;
    float A = asym ? INFINITY : 0.0f, B = -INFINITY;
    const float* src = part + (size_t(arr) * L.units + u) * max_slices * 2 * D;
    for (uint32_t sl = 0; sl < nsl; ++sl) {
        A = asym ? ref_min(A, src[sl * 2 * D + c]) : ref_max(A, src[sl * 2 * D + c]);
        B = ref_max(B, src[sl * 2 * D + D + c]);
    }
    float* fs = L.qstat + (size_t(arr) * L.units + u) * 2 * D;
    fs[c] = A;
    fs[D + c] = B;
    const float v = (arr ? L.values_min : L.values)[(du.seg + du.n_blocks - 1) * D + c];
    float scale, zp;
    qparams_of(ref_min(A, v), ref_max(B, v), ref_max(A, fabsf(v)), asym, L.bits, scale, zp);
    (arr ? L.scales_min : L.scales)[size_t(u) * D + c] = scale;
    (arr ? L.zps_min : L.zps)[size_t(u) * D + c] = zp;
}

// One code (quantizer.cpp:45-58): asym clamp(round((v - zp) / scale), 0, levels),
// sym clamp(round(v / scale), -mid, mid) + mid; std::round is half away from zero.
// The quotient is first formed with the rounded reciprocal (relative error
// <= 2^-23 against the IEEE quotient); only when that lies within 1e-4 of a
// rounding boundary k + 1/2 (or |q| >= 512) is the IEEE division done, so the
// rounded integer is always the one the reference gets.
__device__ __forceinline__ uint32_t encode_code(float v, float sc, float rc, float zp, bool asym, int levels,
                                                int mid) {
    const float num = asym ? __fsub_rn(v, zp) : v;
    float y = __fmul_rn(num, rc);
    const float fr = fabsf(__fsub_rn(y, truncf(y)));
    if (!(fabsf(y) < 512.0f) || fabsf(__fsub_rn(fr, 0.5f)) < 1e-4f) y = __fdiv_rn(num, sc);
    int q = int(roundf(y));
    if (asym) q = q < 0 ? 0 : (q > levels ? levels : q);
    else q = (q < -mid ? -mid : (q > mid ? mid : q)) + mid;
    return uint32_t(q);
}

// Encode + pack: thread = (centroid row, code word), float4 loads of the word's
// 32/BITS channels. wmask (decode-time maintenance) restricts the pass to the words
// whose channel parameters changed, plus the whole trailing row.
constexpr uint32_t kEncodeRows = 256;  // centroid rows per k_encode CTA

template <int D, int BITS>
__global__ void __launch_bounds__(256, BITS == 2 ? 2 : (BITS == 4 ? 3 : 4)) k_encode(LayerView L, const uint32_t* __restrict__ wmask) {
    constexpr uint32_t W = D * BITS / 32, CPW = 32 / BITS, RPI = 256 / W, F4 = CPW / 4;
    const uint32_t u = blockIdx.y;
    const UnitDesc du = L.desc[u];
    const uint32_t begin = blockIdx.x * kEncodeRows;
    if (begin >= du.n_blocks) return;
    const uint32_t end = min(begin + kEncodeRows, du.n_blocks);
    const uint32_t tail = du.n_blocks - 1;
    const bool has_tail = tail < end;
    const uint32_t arrays = L.method == ABSP_CENTROID_MAXMIN ? 2u : 1u;
    const bool asym = L.mode == ABSP_QUANT_ASYM;
    const int levels = (1 << BITS) - 1, mid = (1 << (BITS - 1)) - 1;
    const uint32_t w = threadIdx.x % W, r_in = threadIdx.x / W;
    for (uint32_t a = 0; a < arrays; ++a) {
        const bool word_changed = wmask ? ((wmask[a * L.units + u] >> w) & 1u) : true;
        if (!word_changed && !(has_tail && (tail - begin) % RPI == r_in)) continue;
        // this thread's CPW channels: parameters in registers for all its rows
        float sc[CPW], rc[CPW], zp[CPW];
        const float* gs = (a ? L.scales_min : L.scales) + size_t(u) * D + w * CPW;
        const float* gz = (a ? L.zps_min : L.zps) + size_t(u) * D + w * CPW;
#pragma unroll
        for (uint32_t k4 = 0; k4 < F4; ++k4) {
            const float4 s4 = *reinterpret_cast<const float4*>(gs + 4 * k4);
            const float4 z4 = *reinterpret_cast<const float4*>(gz + 4 * k4);
            sc[4 * k4] = s4.x; sc[4 * k4 + 1] = s4.y; sc[4 * k4 + 2] = s4.z; sc[4 * k4 + 3] = s4.w;
            zp[4 * k4] = z4.x; zp[4 * k4 + 1] = z4.y; zp[4 * k4 + 2] = z4.z; zp[4 * k4 + 3] = z4.w;
        }
#pragma unroll
        for (uint32_t k = 0; k < CPW; ++k) rc[k] = __frcp_rn(sc[k]);
        const float* vals = a ? L.values_min : L.values;
        uint32_t* codes = a ? L.codes_min : L.codes;
        auto encode_row = [&](uint32_t i, const float4* f) {
            uint32_t word = 0;
            bool exact = !asym;
            if (asym) {
                // y = (v - zp) * (1/scale) >= 0; floor(y + 1/2 -+ 2^-10) by a round-down add
                // of 2^23. Equal floors put no rounding boundary within 2^-10 of y + 1/2, and
                // |y - fl((v - zp) / scale)| <= 3 * 2^-24 * y, so the floor is the reference's
                // round-half-away code; otherwise the word is redone with the IEEE division.
                constexpr float kLo = 0.5f - 0.0009765625f, kHi = 0.5f + 0.0009765625f, kMagic = 8388608.0f;
                uint32_t diff = 0;
#pragma unroll
                for (uint32_t k4 = 0; k4 < F4; ++k4) {
                    const float v[4] = {f[k4].x, f[k4].y, f[k4].z, f[k4].w};
#pragma unroll
                    for (uint32_t k = 0; k < 4; ++k) {
                        const uint32_t c = k4 * 4 + k;
                        const float y = __fmul_rn(__fsub_rn(v[k], zp[c]), rc[c]);
                        const uint32_t qa = __float_as_uint(__fadd_rd(__fadd_rn(y, kLo), kMagic));
                        const uint32_t qb = __float_as_uint(__fadd_rd(__fadd_rn(y, kHi), kMagic));
                        diff |= qa ^ qb;
                        diff |= y < 4096.0f ? 0u : 1u;
                        const uint32_t q = min(qa - 0x4B000000u, uint32_t(levels));
                        word |= q << (c * BITS);
                    }
                }
                exact = diff != 0u;
            }
            if (exact) {
                word = 0;
#pragma unroll
                for (uint32_t k4 = 0; k4 < F4; ++k4) {
                    const float v[4] = {f[k4].x, f[k4].y, f[k4].z, f[k4].w};
#pragma unroll
                    for (uint32_t k = 0; k < 4; ++k) {
                        const uint32_t c = k4 * 4 + k;
                        word |= encode_code(v[k], sc[c], rc[c], zp[c], asym, levels, mid) << (c * BITS);
                    }
                }
            }
            codes[(du.seg + i) * W + code_word_pos(i, w, W)] = word;
        };
        auto src_of = [&](uint32_t i) {
            return reinterpret_cast<const float4*>(vals + (du.seg + i) * D + w * CPW);
        };
        if (!word_changed) {  // only the trailing row
            float4 f[F4];
#pragma unroll
            for (uint32_t k4 = 0; k4 < F4; ++k4) f[k4] = __ldcs(src_of(tail) + k4);
            encode_row(tail, f);
            continue;
        }
        for (uint32_t i0 = begin + r_in; i0 < end; i0 += 4 * RPI) {
            float4 f[4][F4];  // four rows loaded before any is encoded
#pragma unroll
            for (uint32_t j = 0; j < 4; ++j) {
                const uint32_t i = i0 + j * RPI;
#pragma unroll
                for (uint32_t k4 = 0; k4 < F4; ++k4)
                    f[j][k4] = i < end ? __ldcs(src_of(i) + k4) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (uint32_t j = 0; j < 4; ++j)
                if (i0 + j * RPI < end) encode_row(i0 + j * RPI, f[j]);
        }
    }
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

// DecodeEngine::step's maintenance after one appended token (engine.cpp:445-449):
// refresh_tail_centroids recomputes the trailing block (centroids.cpp:122-156), and
// requantize_heads re-derives every head's parameters and codes from scratch
// (quantizer.cpp:113-150). Only the trailing centroid changed, so the same result
// comes from the frozen statistics: when the token opened a new block, the previous
// trailing centroid (now final) is folded into them; the new parameters are the
// frozen statistics combined with the new trailing centroid. Channels whose scale
// or zero point changed bit-wise are flagged per code word (wmask) for k_encode;
// every other code is unchanged by construction. One CTA per unit, one thread per
// group of 8 channels.
template <int D, int METHOD>
__global__ void __launch_bounds__(D / 8) k_refresh(LayerView L) {
    const uint32_t u = blockIdx.x;
    const UnitDesc du = L.desc[u];
    const uint32_t c0 = threadIdx.x * 8;
    const uint32_t i = du.n_blocks - 1;
    float tv[2][8];
    centroid8<METHOD>(L, du, i, c0, tv[0], tv[1]);
    store8(L.values + (du.seg + i) * D + c0, tv[0]);
    if (METHOD == ABSP_CENTROID_MAXMIN) store8(L.values_min + (du.seg + i) * D + c0, tv[1]);
    if (L.bits == 0) return;
    const bool asym = L.mode == ABSP_QUANT_ASYM;
    const bool opened = du.n_blocks >= 2 && (du.n_tokens - 1) % du.block == 0;
    const uint32_t cpw = 32 / L.bits;
    constexpr uint32_t arrays = METHOD == ABSP_CENTROID_MAXMIN ? 2u : 1u;
#pragma unroll
    for (uint32_t a = 0; a < arrays; ++a) {
        const float* vals = a ? L.values_min : L.values;
        float* fs = L.qstat + (size_t(a) * L.units + u) * 2 * D;
        float* scales = (a ? L.scales_min : L.scales) + size_t(u) * D;
        float* zps = (a ? L.zps_min : L.zps) + size_t(u) * D;
        uint32_t changed = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint32_t c = c0 + k;
            float A = fs[c], B = fs[D + c];
            if (opened) {
                const float vo = vals[(du.seg + i - 1) * D + c];
                A = asym ? ref_min(A, vo) : ref_max(A, fabsf(vo));
                B = ref_max(B, vo);
                fs[c] = A;
                fs[D + c] = B;
            }
            const float v = tv[a][k];
            float scale, zp;
            qparams_of(ref_min(A, v), ref_max(B, v), ref_max(A, fabsf(v)), asym, L.bits, scale, zp);
            if (__float_as_uint(scale) != __float_as_uint(scales[c]) || __float_as_uint(zp) != __float_as_uint(zps[c])) {
                scales[c] = scale;
                zps[c] = zp;
                changed |= 1u << (c / cpw);
            }
        }
        // OR over the CTA's D/8 threads (lanes of one warp)
#pragma unroll
        for (int off = D / 16; off > 0; off >>= 1) changed |= __shfl_xor_sync((1u << (D / 8)) - 1u, changed, off);
        if (threadIdx.x == 0) L.wmask[a * L.units + u] = changed;
    }
}

template <int D>
cudaError_t build_d(const LayerView& L, uint32_t max_cap, bool tail_only, cudaStream_t s, int* launches) {
    const bool mm = L.method == ABSP_CENTROID_MAXMIN;
    if (tail_only) {  // decode-time maintenance: only each unit's trailing block changed
        if (mm) k_refresh<D, ABSP_CENTROID_MAXMIN><<<L.units, D / 8, 0, s>>>(L);
        else k_refresh<D, ABSP_CENTROID_MEAN><<<L.units, D / 8, 0, s>>>(L);
    } else {
        const dim3 gc((max_cap + 256 / (D / 8) - 1) / (256 / (D / 8)), L.units);
        if (mm) k_centroids<D, ABSP_CENTROID_MAXMIN><<<gc, 256, 0, s>>>(L);
        else k_centroids<D, ABSP_CENTROID_MEAN><<<gc, 256, 0, s>>>(L);
    }
    ++*launches;
    if (L.bits == 0) return cudaGetLastError();
    const uint32_t arrays = mm ? 2u : 1u;
    if (!tail_only) {
        const uint32_t slices = std::max<uint32_t>(1u, (max_cap + kStatRows - 1) / kStatRows);
        k_qstats<D><<<dim3(slices, L.units, arrays), 1024, 0, s>>>(L, L.qpart, slices);
        k_qfinal<D><<<dim3(L.units, arrays), D, 0, s>>>(L, L.qpart, slices);
        *launches += 2;
    }
    const uint32_t* mask = tail_only ? L.wmask : nullptr;
    const dim3 ge((max_cap + kEncodeRows - 1) / kEncodeRows, L.units);
    switch (L.bits) {
        case 2: k_encode<D, 2><<<ge, 256, 0, s>>>(L, mask); break;
        case 4: k_encode<D, 4><<<ge, 256, 0, s>>>(L, mask); break;
        default: k_encode<D, 8><<<ge, 256, 0, s>>>(L, mask); break;
    }
    ++*launches;
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_build_store(const LayerView& L, uint32_t max_cap, cudaStream_t s, int* launches) {
    if (L.D == 64) return build_d<64>(L, max_cap, false, s, launches);
    return build_d<128>(L, max_cap, false, s, launches);
}

// DecodeEngine::step's maintenance after an append (engine.cpp:445-449):
// refresh_tail_centroids + requantize_heads, incrementally (k_refresh): the result
// is what quantizing the grown store from scratch gives, bit for bit.
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

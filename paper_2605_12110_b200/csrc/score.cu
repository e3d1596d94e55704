// Kernel 1: quantized centroid scoring with dequantization fused into the load
// (sm_100a).
//
// Reference: estimate_batched / centroid_score (engine.cpp:34-67, 79-97):
//     acc = 0; for c in 0..d-1: acc += q[c] * (zp[c] + code[c] * scale[c])
// in fp32, serial in c, no FMA (the reference build emits none). Selection must
// be bit-exact, so the scores must be too: one thread owns one centroid and
// walks the channels in order with separately-rounded adds.
//
// The three roundings inside the sum term depend only on (c, code), so for
// bits <= 4 each CTA precomputes the exact product table
//     tbl[c][code] = fl(q[c] * fl(zp[c] + fl(code * scale[c])))
// in shared memory (16 x 128 x 4 B = 8 KB at int4): the inner loop is then one
// nibble extract, one conflict-free LDS (all lanes read the same 64 B row of
// the table, distinct codes land in distinct banks) and one FADD per element.
// GQA: q is the left-to-right fp32 sum of the group's G queries (SURVEY.md
// Appendix A).
#include "absp_internal.cuh"

namespace absp {
namespace {

constexpr int kThreads = 256;
constexpr int kPerThread = kScoreItemCentroids / kThreads;  // centroids per thread per item
constexpr int kBatch = 2;                                    // centroids per thread per batch

__device__ __forceinline__ float bf16f(uint16_t x) { return __uint_as_float(uint32_t(x) << 16); }

__device__ __forceinline__ float ref_max(float a, float b) { return (a < b) ? b : a; }

// Group-summed query for unit (b, h) into smem.
template <int D>
__device__ __forceinline__ void load_query(const LayerView& L, const UnitDesc& du,
                                           const uint16_t* q, float* qs) {
    for (uint32_t c = threadIdx.x; c < D; c += blockDim.x) {
        const uint16_t* qb = q + (size_t(du.seq) * L.H * L.G + size_t(du.head) * L.G) * D + c;
        float acc = bf16f(qb[0]);
        for (uint32_t g = 1; g < L.G; ++g) acc = __fadd_rn(acc, bf16f(qb[size_t(g) * D]));
        qs[c] = acc;
    }
}

// Byte offset (code * 4) of nibble/crumb k of a packed code word, for a 4-byte
// table entry. 4-bit: two masked copies hold the even / odd nibbles pre-scaled by 4
// in their bytes, and one PRMT per code extracts a byte (1.5 ALU ops per code).
template <int BITS>
struct CodeOffsets {
    uint32_t a, b, w;
    __device__ __forceinline__ explicit CodeOffsets(uint32_t word) : w(word) {
        if (BITS == 4) {
            a = (word << 2) & 0x3c3c3c3cu;  // nibbles 0,2,4,6 (x4) in bytes 0..3
            b = (word >> 2) & 0x3c3c3c3cu;  // nibbles 1,3,5,7 (x4)
        }
    }
    __device__ __forceinline__ uint32_t operator()(int k) const {
        if (BITS == 4) return __byte_perm((k & 1) ? b : a, 0u, 0x4440u | uint32_t(k >> 1));
        return ((w >> (k * BITS)) & ((1u << BITS) - 1u)) << 2;
    }
};

// Table path: bits in {2, 4}; MAXMIN doubles the tables and code streams. A CTA
// scores one item (up to kScoreItemCentroids centroids of one unit) in batches of
// kThreads * kBatch, with the next batch's code words loaded while the current
// batch is scored.
template <int D, int BITS, bool ASYM, bool MAXMIN>
__global__ void __launch_bounds__(kThreads, 2) k_score_tbl(LayerView L, const uint16_t* q,
                                                           const ScoreItem* items) {
    constexpr int LV = 1 << BITS;
    constexpr int W = D * BITS / 32;
    constexpr int CPW = 32 / BITS;
    constexpr int NT = MAXMIN ? 2 : 1;
    constexpr int NW = MAXMIN ? 2 * W : W;  // words per centroid incl. the min array
    __shared__ float qs[D];
    __shared__ float prm[NT][2][D];
    __shared__ __align__(16) float tbl[NT * D * LV];

    const ScoreItem it = items[blockIdx.x];
    const UnitDesc du = L.desc[it.unit];
    const uint32_t end = min(it.start + uint32_t(kScoreItemCentroids), du.n_blocks);
    const uint32_t* codes = L.codes + du.seg * W;
    const uint32_t* codes_lo = MAXMIN ? L.codes_min + du.seg * W : nullptr;
    float* out = L.scores + du.seg;

    auto load = [&](uint32_t base, uint32_t (&wd)[kBatch][NW]) {
#pragma unroll
        for (int j = 0; j < kBatch; ++j) {
            uint32_t i = base + j * kThreads + threadIdx.x;
            i = i < end ? i : it.start;  // clamp: a valid centroid, result discarded
#pragma unroll
            for (int w = 0; w < W; ++w) {
                wd[j][w] = __ldg(codes + size_t(w) * du.cap + i);
                if (MAXMIN) wd[j][W + w] = __ldg(codes_lo + size_t(w) * du.cap + i);
            }
        }
    };
    auto score = [&](uint32_t base, const uint32_t (&wd)[kBatch][NW]) {
        float acc[kBatch];
#pragma unroll
        for (int j = 0; j < kBatch; ++j) acc[j] = 0.0f;
        const char* tb = reinterpret_cast<const char*>(tbl);
#pragma unroll
        for (int w = 0; w < W; ++w) {
            CodeOffsets<BITS> hi0(wd[0][w]), hi1(wd[kBatch - 1][w]);
            CodeOffsets<BITS> lo0(MAXMIN ? wd[0][W + w] : 0u), lo1(MAXMIN ? wd[kBatch - 1][W + w] : 0u);
#pragma unroll
            for (int k = 0; k < CPW; ++k) {
                const char* row = tb + (w * CPW + k) * LV * 4;
#pragma unroll
                for (int j = 0; j < kBatch; ++j) {
                    const CodeOffsets<BITS>& h = j == 0 ? hi0 : hi1;
                    float p = *reinterpret_cast<const float*>(row + h(k));
                    if (MAXMIN) {
                        const CodeOffsets<BITS>& l = j == 0 ? lo0 : lo1;
                        p = ref_max(p, *reinterpret_cast<const float*>(row + D * LV * 4 + l(k)));
                    }
                    acc[j] = __fadd_rn(acc[j], p);
                }
            }
        }
#pragma unroll
        for (int j = 0; j < kBatch; ++j) {
            const uint32_t i = base + j * kThreads + threadIdx.x;
            if (i < end) out[i] = acc[j];
        }
    };

    // batch 0's code words are in flight while the query, parameters and table are built
    uint32_t wa[kBatch][NW], wb[kBatch][NW];
    load(it.start, wa);

    load_query<D>(L, du, q, qs);
    for (uint32_t e = threadIdx.x; e < NT * 2 * D; e += kThreads) {
        const uint32_t t = e / (2 * D), which = (e / D) & 1, c = e % D;
        const float* src = which == 0 ? (t ? L.scales_min : L.scales) : (t ? L.zps_min : L.zps);
        prm[t][which][c] = src[size_t(it.unit) * D + c];
    }
    __syncthreads();
    const int mid = (1 << (BITS - 1)) - 1;
    for (uint32_t e = threadIdx.x; e < NT * D * LV; e += kThreads) {
        const uint32_t t = e / (D * LV), c = (e / LV) % D, k = e % LV;
        const float sc = prm[t][0][c], zp = prm[t][1][c];
        const float deq = ASYM ? __fadd_rn(zp, __fmul_rn(float(k), sc)) : __fmul_rn(float(int(k) - mid), sc);
        tbl[e] = __fmul_rn(qs[c], deq);
    }
    __syncthreads();

    constexpr uint32_t kStep = kThreads * kBatch;
    for (uint32_t base = it.start; base < end; base += 2 * kStep) {
        if (base + kStep < end) load(base + kStep, wb);
        score(base, wa);
        if (base + kStep >= end) break;
        if (base + 2 * kStep < end) load(base + 2 * kStep, wa);
        score(base + kStep, wb);
    }
}

// Direct path for int8 codes (a 256-entry table per channel would not fit).
template <int D, bool ASYM, bool MAXMIN>
__global__ void __launch_bounds__(kThreads) k_score_int8(LayerView L, const uint16_t* q,
                                                         const ScoreItem* items) {
    constexpr int W = D / 4;
    __shared__ float qs[D];
    __shared__ float prm[4][D];
    const ScoreItem it = items[blockIdx.x];
    const UnitDesc du = L.desc[it.unit];
    load_query<D>(L, du, q, qs);
    for (uint32_t c = threadIdx.x; c < D; c += kThreads) {
        prm[0][c] = L.scales[size_t(it.unit) * D + c];
        prm[1][c] = L.zps[size_t(it.unit) * D + c];
        if (MAXMIN) {
            prm[2][c] = L.scales_min[size_t(it.unit) * D + c];
            prm[3][c] = L.zps_min[size_t(it.unit) * D + c];
        }
    }
    __syncthreads();
    const int mid = 127;
    const uint32_t* codes = L.codes + du.seg * W;
    const uint32_t* codes_lo = MAXMIN ? L.codes_min + du.seg * W : nullptr;
    for (int j = 0; j < kPerThread; ++j) {
        const uint32_t i = it.start + j * kThreads + threadIdx.x;
        if (i >= du.n_blocks) continue;
        float acc = 0.0f;
        for (int w = 0; w < W; ++w) {
            const uint32_t word = __ldg(codes + size_t(w) * du.cap + i);
            const uint32_t wlo = MAXMIN ? __ldg(codes_lo + size_t(w) * du.cap + i) : 0u;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int c = w * 4 + k;
                const uint32_t code = (word >> (8 * k)) & 255u;
                const float deq = ASYM ? __fadd_rn(prm[1][c], __fmul_rn(float(code), prm[0][c]))
                                       : __fmul_rn(float(int(code) - mid), prm[0][c]);
                float p = __fmul_rn(qs[c], deq);
                if (MAXMIN) {
                    const uint32_t cl = (wlo >> (8 * k)) & 255u;
                    const float dl = ASYM ? __fadd_rn(prm[3][c], __fmul_rn(float(cl), prm[2][c]))
                                          : __fmul_rn(float(int(cl) - mid), prm[2][c]);
                    p = ref_max(p, __fmul_rn(qs[c], dl));
                }
                acc = __fadd_rn(acc, p);
            }
        }
        L.scores[du.seg + i] = acc;
    }
}

// Full-precision store (EngineConfig::quant == nullopt): engine.cpp:21-32.
template <int D, bool MAXMIN>
__global__ void __launch_bounds__(kThreads) k_score_f32(LayerView L, const uint16_t* q,
                                                        const ScoreItem* items) {
    __shared__ float qs[D];
    const ScoreItem it = items[blockIdx.x];
    const UnitDesc du = L.desc[it.unit];
    load_query<D>(L, du, q, qs);
    __syncthreads();
    for (int j = 0; j < kPerThread; ++j) {
        const uint32_t i = it.start + j * kThreads + threadIdx.x;
        if (i >= du.n_blocks) continue;
        const float* v = L.values + (du.seg + i) * D;
        const float* vl = MAXMIN ? L.values_min + (du.seg + i) * D : nullptr;
        float acc = 0.0f;
        for (int c = 0; c < D; c += 4) {
            const float4 a = *reinterpret_cast<const float4*>(v + c);
            const float av[4] = {a.x, a.y, a.z, a.w};
            float bv[4] = {0, 0, 0, 0};
            if (MAXMIN) {
                const float4 b = *reinterpret_cast<const float4*>(vl + c);
                bv[0] = b.x; bv[1] = b.y; bv[2] = b.z; bv[3] = b.w;
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                float p = __fmul_rn(qs[c + k], av[k]);
                if (MAXMIN) p = ref_max(p, __fmul_rn(qs[c + k], bv[k]));
                acc = __fadd_rn(acc, p);
            }
        }
        L.scores[du.seg + i] = acc;
    }
}

template <int D>
cudaError_t score_d(const LayerView& L, const uint16_t* q, const ScoreItem* items, uint32_t n,
                    cudaStream_t s) {
    const bool asym = L.mode == ABSP_QUANT_ASYM;
    const bool mm = L.method == ABSP_CENTROID_MAXMIN;
#define ABSP_SCORE(KERNEL, ...) KERNEL<__VA_ARGS__><<<n, kThreads, 0, s>>>(L, q, items)
    if (L.bits == 0) {
        if (mm) ABSP_SCORE(k_score_f32, D, true);
        else ABSP_SCORE(k_score_f32, D, false);
    } else if (L.bits == 8) {
        if (asym) { if (mm) ABSP_SCORE(k_score_int8, D, true, true); else ABSP_SCORE(k_score_int8, D, true, false); }
        else      { if (mm) ABSP_SCORE(k_score_int8, D, false, true); else ABSP_SCORE(k_score_int8, D, false, false); }
    } else if (L.bits == 4) {
        if (asym) { if (mm) ABSP_SCORE(k_score_tbl, D, 4, true, true); else ABSP_SCORE(k_score_tbl, D, 4, true, false); }
        else      { if (mm) ABSP_SCORE(k_score_tbl, D, 4, false, true); else ABSP_SCORE(k_score_tbl, D, 4, false, false); }
    } else {
        if (asym) { if (mm) ABSP_SCORE(k_score_tbl, D, 2, true, true); else ABSP_SCORE(k_score_tbl, D, 2, true, false); }
        else      { if (mm) ABSP_SCORE(k_score_tbl, D, 2, false, true); else ABSP_SCORE(k_score_tbl, D, 2, false, false); }
    }
#undef ABSP_SCORE
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_score(const LayerView& L, const uint16_t* q, const ScoreItem* items,
                         uint32_t n_items, cudaStream_t s, int* launches) {
    ++*launches;
    if (L.D == 64) return score_d<64>(L, q, items, n_items, s);
    return score_d<128>(L, q, items, n_items, s);
}

}  // namespace absp

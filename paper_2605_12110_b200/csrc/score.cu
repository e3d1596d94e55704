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
constexpr int kPerThread = kScoreItemCentroids / kThreads;  // centroids per thread

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

// Table path: bits in {2, 4}; MAXMIN doubles the tables and code streams.
template <int D, int BITS, bool ASYM, bool MAXMIN>
__global__ void __launch_bounds__(kThreads) k_score_tbl(LayerView L, const uint16_t* q,
                                                        const ScoreItem* items) {
    constexpr int LV = 1 << BITS;
    constexpr int W = D * BITS / 32;
    constexpr int CPW = 32 / BITS;
    constexpr uint32_t MASK = LV - 1;
    __shared__ float qs[D];
    __shared__ float tbl[(MAXMIN ? 2 : 1) * D * LV];

    const ScoreItem it = items[blockIdx.x];
    const UnitDesc du = L.desc[it.unit];
    const uint32_t* codes = L.codes + du.seg * W;
    const uint32_t* codes_lo = MAXMIN ? L.codes_min + du.seg * W : nullptr;
    float* out = L.scores + du.seg;

    // Issue every code-word load of this thread first (coalesced: one 128 B line per
    // warp per word), so HBM latency overlaps the table construction below.
    uint32_t idx[kPerThread];
    bool ok[kPerThread];
#pragma unroll
    for (int j = 0; j < kPerThread; ++j) {
        const uint32_t i = it.start + j * kThreads + threadIdx.x;
        ok[j] = i < du.n_blocks;
        idx[j] = ok[j] ? i : 0;
    }
    uint32_t word[kPerThread][W], wlo[kPerThread][MAXMIN ? W : 1];
#pragma unroll
    for (int w = 0; w < W; ++w)
#pragma unroll
        for (int j = 0; j < kPerThread; ++j) {
            word[j][w] = __ldg(codes + size_t(w) * du.cap + idx[j]);
            if (MAXMIN) wlo[j][w] = __ldg(codes_lo + size_t(w) * du.cap + idx[j]);
        }

    load_query<D>(L, du, q, qs);
    __syncthreads();
    const int mid = (1 << (BITS - 1)) - 1;
    for (int t = 0; t < (MAXMIN ? 2 : 1); ++t) {
        const float* sc = (t ? L.scales_min : L.scales) + size_t(it.unit) * D;
        const float* zp = (t ? L.zps_min : L.zps) + size_t(it.unit) * D;
        for (uint32_t e = threadIdx.x; e < D * LV; e += kThreads) {
            const uint32_t c = e / LV, k = e % LV;
            const float deq = ASYM ? __fadd_rn(zp[c], __fmul_rn(float(k), sc[c]))
                                   : __fmul_rn(float(int(k) - mid), sc[c]);
            tbl[t * D * LV + e] = __fmul_rn(qs[c], deq);
        }
    }
    __syncthreads();

    float acc[kPerThread];
#pragma unroll
    for (int j = 0; j < kPerThread; ++j) acc[j] = 0.0f;
#pragma unroll
    for (int w = 0; w < W; ++w) {
#pragma unroll
        for (int k = 0; k < CPW; ++k) {
            const float* row = tbl + (w * CPW + k) * LV;
#pragma unroll
            for (int j = 0; j < kPerThread; ++j) {
                float p = row[(word[j][w] >> (k * BITS)) & MASK];
                if (MAXMIN) p = ref_max(p, row[D * LV + ((wlo[j][w] >> (k * BITS)) & MASK)]);
                acc[j] = __fadd_rn(acc[j], p);
            }
        }
    }
#pragma unroll
    for (int j = 0; j < kPerThread; ++j)
        if (ok[j]) out[idx[j]] = acc[j];
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

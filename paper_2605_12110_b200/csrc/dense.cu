// Dense decode attention with attention weights (the reference's
// full_attention_oracle, engine.cpp:357-403) and the calibrator's
// attention_recall (calibrator.cpp:48-71), on sm_100a.
//
// This is the exact, fp64 path: the source of calibration weights (SURVEY.md
// §8(f3)) and the "full attention" side of the A/B (§8(f4)). The production
// sparse path never calls it.
//
// Arithmetic follows the reference op for op where it is order-free:
//   z_t = (sum_c q_c k_tc) * (1/sqrt(d))   fp64, serial over c. q and k are bf16
//          values, so every product is exact in fp64 and the FMA chain rounds
//          exactly like the reference's `z += q*k` loop: logits are bit-exact.
//   w_t = exp(z_t - M) / L,  o_c = sum_t w_t v_tc      fp64
// M is the exact maximum; L = sum_t exp(z_t - M) and the output sums are formed
// per split and merged (the reference sums serially over t), so weights and
// outputs agree with the reference to fp64 rounding (~1e-15 relative), not bit
// for bit.
//
// Layout. One CTA per (unit, split): a contiguous token range of one (sequence,
// KV head), streamed in 64-token sub-chunks through a 2-stage cp.async ring
// (K and V rows padded by 16 B so a row per lane is conflict-free). Logits for the
// G query heads of the group, an fp64 online softmax per head, and an fp64 PV
// accumulation (thread = channel x token quarter) per sub-chunk; the split's
// (m, l, o) partial goes to HBM and k_full_merge combines the splits.
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>

#include "absp_internal.cuh"
#include "common.cuh"
#include "ptx.cuh"

namespace absp {
namespace {

constexpr int kThreads = 256;
constexpr int kTS = 64;       // tokens per sub-chunk
constexpr int kStages = 2;

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

__device__ __forceinline__ double bf16d(uint32_t bits16) { return double(__uint_as_float(bits16 << 16)); }

template <int D>
struct FullSmem {
    static constexpr int kRow = D * 2 + 16;  // padded row bytes
    unsigned char k[kStages][kTS * kRow];
    unsigned char v[kStages][kTS * kRow];
    double q[8][D];
    double z[8][kTS];     // logits, then probabilities
    double alpha[8];      // per-head rescale of this sub-chunk
    double red[kThreads / D - 1][8][D];  // PV partial sums of token parts 1..
};

// Partials: part[(u * S + s) * G + g] -> o [D] fp64; ml[...] -> (m, l).
template <int D, int NG>
__global__ void __launch_bounds__(kThreads) k_full_attn(LayerView L, const uint16_t* __restrict__ q,
                                                          uint32_t splits, double inv_sqrt_d,
                                                          double* __restrict__ weights, uint64_t wstride,
                                                          double* __restrict__ part_o,
                                                          double* __restrict__ part_ml) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    FullSmem<D>& sm = *reinterpret_cast<FullSmem<D>*>(smem_raw);
    constexpr int kRow = FullSmem<D>::kRow;
    constexpr int kPieces = D / 8;  // 16-byte pieces per row
    constexpr int kParts = kThreads / D;  // token parts of the PV phase
    const uint32_t u = blockIdx.x / splits, s = blockIdx.x % splits;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const UnitDesc du = L.desc[u];
    const uint32_t G = L.G, n = du.n_tokens;
    const uint32_t t_begin = uint32_t(uint64_t(s) * n / splits);
    const uint32_t t_end = uint32_t(uint64_t(s + 1) * n / splits);
    const uint32_t qh0 = du.head * G;
    const size_t qrow = size_t(du.seq) * L.H * G + qh0;  // first q row of the group

    griddep_wait();
    for (int i = tid; i < int(G * D); i += kThreads) {
        const uint32_t g = i / D, c = i % D;
        sm.q[g][c] = bf16d(q[(qrow + g) * D + c]);
    }
    const uint32_t* pt = L.page_table + size_t(du.seq) * L.max_pages;
    const size_t head_base = size_t(du.head) * L.pool_pages;
    auto issue = [&](uint32_t t0, int stage) {
        // 64 rows x kPieces pieces per tensor; rows past t_end are not loaded
        for (int i = tid; i < kTS * kPieces; i += kThreads) {
            const int r = i / kPieces, p = i % kPieces;
            const uint32_t t = t0 + r;
            if (t >= t_end) continue;
            const size_t row = (head_base + __ldg(pt + t / L.P)) * L.P + t % L.P;
            const uint32_t off = r * kRow + p * 16;
            cp_async16(smem_u32(sm.k[stage] + off), L.k_pool + row * D + p * 8);
            cp_async16(smem_u32(sm.v[stage] + off), L.v_pool + row * D + p * 8);
        }
        cp_async_commit();
    };

    double m_run = -INFINITY, l_run = 0.0;  // warp g's running max / denominator (g = warp < G)
    double acc[8];
#pragma unroll
    for (int g = 0; g < 8; ++g) acc[g] = 0.0;
    const int c_pv = tid % D, part = tid / D;

    const uint32_t n_sub = (t_end - t_begin + kTS - 1) / kTS;
    if (n_sub > 0) issue(t_begin, 0);
    for (uint32_t it = 0; it < n_sub; ++it) {
        const int stage = it % kStages;
        const uint32_t t0 = t_begin + it * kTS;
        if (it + 1 < n_sub) {
            issue(t0 + kTS, (it + 1) % kStages);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        // ---- logits: thread = (token, heads g0, g0 + 4 [, ...])
        {
            const int t = tid & (kTS - 1), g0 = tid / kTS;
            const bool live = t0 + t < t_end;
            double z[NG];
#pragma unroll
            for (int j = 0; j < NG; ++j) z[j] = 0.0;
            const unsigned char* krow = sm.k[stage] + t * kRow;
#pragma unroll 4
            for (int p = 0; p < kPieces; ++p) {
                const uint4 w = *reinterpret_cast<const uint4*>(krow + p * 16);
                const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const double kv = bf16d((ww[e >> 1] >> ((e & 1) * 16)) & 0xffffu);
#pragma unroll
                    for (int j = 0; j < NG; ++j) {
                        const int g = g0 + 4 * j;
                        if (g < int(G)) z[j] = fma(sm.q[g][p * 8 + e], kv, z[j]);
                    }
                }
            }
#pragma unroll
            for (int j = 0; j < NG; ++j) {
                const int g = g0 + 4 * j;
                if (g < int(G)) {
                    const double zz = live ? z[j] * inv_sqrt_d : -INFINITY;
                    sm.z[g][t] = zz;
                    if (live && weights)
                        weights[(size_t(du.seq) * L.H * G + qh0 + g) * wstride + t0 + t] = zz;
                }
            }
        }
        __syncthreads();
        // ---- online softmax: warp g owns head g (G <= 8)
        if (warp < int(G)) {
            const int g = warp;
            const double z0 = sm.z[g][lane], z1 = sm.z[g][lane + 32];
            double mx = fmax(z0, z1);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            const double m_new = fmax(m_run, mx);  // finite: the sub-chunk holds >= 1 live token
            const double a = exp(m_run - m_new);
            const double p0 = exp(z0 - m_new), p1 = exp(z1 - m_new);
            sm.z[g][lane] = p0;
            sm.z[g][lane + 32] = p1;
            double ps = p0 + p1;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, o);
            l_run = l_run * a + ps;
            m_run = m_new;
            if (lane == 0) sm.alpha[g] = a;
        }
        __syncthreads();
        // ---- PV: thread = (channel, token part)
        {
#pragma unroll
            for (int g = 0; g < 8; ++g)
                if (g < int(G)) acc[g] *= sm.alpha[g];
            const uint32_t live = min(uint32_t(kTS), t_end - t0);
            for (uint32_t t = part; t < live; t += kParts) {
                const double vv = bf16d(*reinterpret_cast<const uint16_t*>(sm.v[stage] + t * kRow + c_pv * 2));
#pragma unroll
                for (int g = 0; g < 8; ++g)
                    if (g < int(G)) acc[g] = fma(sm.z[g][t], vv, acc[g]);
            }
        }
        __syncthreads();  // the stage is re-filled next iteration
    }
    // ---- combine token parts, write the split's partial
    if (part > 0) {
#pragma unroll
        for (int g = 0; g < 8; ++g)
            if (g < int(G)) sm.red[part - 1][g][c_pv] = acc[g];
    }
    if (warp < int(G) && lane == 0) {
        const size_t pi = (size_t(u) * splits + s) * G + warp;
        part_ml[pi * 2] = m_run;
        part_ml[pi * 2 + 1] = l_run;
    }
    __syncthreads();
    if (part == 0) {
        for (int g = 0; g < int(G); ++g) {
            double o = acc[g];
#pragma unroll
            for (int p = 1; p < kParts; ++p) o += sm.red[p - 1][g][c_pv];
            part_o[((size_t(u) * splits + s) * G + g) * D + c_pv] = o;
        }
    }
    griddep_launch_dependents();
}

// One CTA per (unit, head of the group): M = max m_s, L = sum l_s e^(m_s - M),
// out_c = (sum o_sc e^(m_s - M)) / L; (M, L) kept for the weight normalisation.
template <int D>
__global__ void __launch_bounds__(D) k_full_merge(LayerView L, uint32_t splits, const double* __restrict__ part_o,
                                                  const double* __restrict__ part_ml, float* __restrict__ out,
                                                  double* __restrict__ stats) {
    griddep_wait();
    const uint32_t G = L.G;
    const uint32_t u = blockIdx.x / G, g = blockIdx.x % G;
    const UnitDesc du = L.desc[u];
    const int c = threadIdx.x;
    double M = -INFINITY;
    for (uint32_t s = 0; s < splits; ++s) {
        const double ls = part_ml[((size_t(u) * splits + s) * G + g) * 2 + 1];
        if (ls > 0.0) M = fmax(M, part_ml[((size_t(u) * splits + s) * G + g) * 2]);
    }
    double Lsum = 0.0, o = 0.0;
    for (uint32_t s = 0; s < splits; ++s) {
        const size_t pi = (size_t(u) * splits + s) * G + g;
        const double ls = part_ml[pi * 2 + 1];
        if (!(ls > 0.0)) continue;
        const double f = exp(part_ml[pi * 2] - M);
        Lsum += ls * f;
        o += part_o[pi * D + c] * f;
    }
    const size_t row = size_t(du.seq) * L.H * G + du.head * G + g;
    out[row * D + c] = float(o / Lsum);
    if (c == 0 && stats) {
        stats[row * 2] = M;
        stats[row * 2 + 1] = Lsum;
    }
    griddep_launch_dependents();
}

// weights[row][t] : z_t -> exp(z_t - M) / L (engine.cpp:388-395), t < n of the row's sequence.
__global__ void __launch_bounds__(256) k_full_weights(LayerView L, const double* __restrict__ stats,
                                                      double* __restrict__ weights, uint64_t wstride) {
    griddep_wait();
    const uint32_t row = blockIdx.y;  // sequence * Hq + q head
    const uint32_t Hq = L.H * L.G;
    const uint32_t b = row / Hq, h = (row % Hq) / L.G;
    const uint32_t n = L.desc[size_t(b) * L.H + h].n_tokens;
    const double M = stats[row * 2], Lsum = stats[row * 2 + 1];
    double* w = weights + size_t(row) * wstride;
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x)
        w[t] = exp(w[t] - M) / Lsum;
    griddep_launch_dependents();
}

// attention_recall (calibrator.cpp:48-71) per (sequence, q head): the weight mass
// on tokens whose block is selected. Block membership comes from a bitmap of the
// unit's selection in shared memory; the sum is a fixed-order tree (deterministic).
constexpr int kRecallThreads = 512;
__global__ void __launch_bounds__(kRecallThreads) k_recall(LayerView L, const double* __restrict__ weights,
                                                           uint64_t wstride, const uint32_t* __restrict__ blocks,
                                                           uint32_t stride, const uint32_t* __restrict__ counts,
                                                           double* __restrict__ recall) {
    extern __shared__ uint32_t bitmap[];  // ceil(n_blocks / 32) words
    __shared__ double red[kRecallThreads / 32];
    griddep_wait();
    const uint32_t row = blockIdx.x;
    const uint32_t Hq = L.H * L.G;
    const uint32_t b = row / Hq, h = (row % Hq) / L.G;
    const uint32_t u = b * L.H + h;
    const UnitDesc du = L.desc[u];
    const uint32_t words = (du.n_blocks + 31) / 32;
    for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) bitmap[i] = 0u;
    __syncthreads();
    const uint32_t cnt = min(counts[u], stride);
    for (uint32_t e = threadIdx.x; e < cnt; e += blockDim.x) {
        const uint32_t blk = blocks[size_t(u) * stride + e];
        if (blk < du.n_blocks) atomicOr(&bitmap[blk >> 5], 1u << (blk & 31));
    }
    __syncthreads();
    const double* w = weights + size_t(row) * wstride;
    double acc = 0.0;
    for (uint32_t t = threadIdx.x; t < du.n_tokens; t += blockDim.x) {
        const uint32_t blk = t / du.block;
        if ((bitmap[blk >> 5] >> (blk & 31)) & 1u) acc += w[t];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
        double v = threadIdx.x < kRecallThreads / 32 ? red[threadIdx.x] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (threadIdx.x == 0) recall[row] = v;
    }
    griddep_launch_dependents();
}

template <int D, int NG>
cudaError_t set_full_attr() {
    return cudaFuncSetAttribute(k_full_attn<D, NG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                int(sizeof(FullSmem<D>)));
}

template <int D>
cudaError_t launch_full_d(const LayerView& L, const uint16_t* q, uint32_t splits, double* weights,
                          uint64_t wstride, double* part_o, double* part_ml, double* stats, float* out,
                          cudaStream_t s, int* launches) {
    const double inv_sqrt_d = 1.0 / sqrt(double(D));  // engine.cpp:370
    const dim3 grid(L.units * splits);
    cudaError_t e;
    if (L.G > 4) {
        if ((e = set_full_attr<D, 2>()) != cudaSuccess) return e;
        e = launch_pdl(k_full_attn<D, 2>, grid, dim3(kThreads), sizeof(FullSmem<D>), s, L, q, splits, inv_sqrt_d,
                       weights, wstride, part_o, part_ml);
    } else {
        if ((e = set_full_attr<D, 1>()) != cudaSuccess) return e;
        e = launch_pdl(k_full_attn<D, 1>, grid, dim3(kThreads), sizeof(FullSmem<D>), s, L, q, splits, inv_sqrt_d,
                       weights, wstride, part_o, part_ml);
    }
    if (e != cudaSuccess) return e;
    ++*launches;
    e = launch_pdl(k_full_merge<D>, dim3(L.units * L.G), dim3(D), 0, s, L, splits,
                   static_cast<const double*>(part_o), static_cast<const double*>(part_ml), out, stats);
    if (e != cudaSuccess) return e;
    ++*launches;
    if (weights) {
        e = launch_pdl(k_full_weights, dim3(16, L.batch * L.H * L.G), dim3(256), 0, s, L,
                       static_cast<const double*>(stats), weights, wstride);
        if (e != cudaSuccess) return e;
        ++*launches;
    }
    return cudaGetLastError();
}

}  // namespace

uint32_t full_attention_splits(uint32_t units, uint32_t max_tokens, int num_sms) {
    // about four CTAs per SM over the layer, at least 256 tokens per split
    const uint32_t want = (uint32_t(4 * num_sms) + units - 1) / units;
    const uint32_t cap = (max_tokens + 255) / 256;
    return std::max(1u, std::min(want, cap));
}

cudaError_t launch_full_attention(const LayerView& L, const uint16_t* q, uint32_t splits, double* weights,
                                  uint64_t wstride, double* part_o, double* part_ml, double* stats, float* out,
                                  cudaStream_t s, int* launches) {
    if (L.D == 128) return launch_full_d<128>(L, q, splits, weights, wstride, part_o, part_ml, stats, out, s, launches);
    if (L.D == 64) return launch_full_d<64>(L, q, splits, weights, wstride, part_o, part_ml, stats, out, s, launches);
    return cudaErrorInvalidValue;
}

cudaError_t launch_recall(const LayerView& L, uint32_t max_nblocks, const double* weights, uint64_t wstride,
                          const uint32_t* blocks, uint32_t stride, const uint32_t* counts, double* recall,
                          cudaStream_t s, int* launches) {
    const size_t smem = size_t((max_nblocks + 31) / 32) * 4;
    cudaError_t e = cudaFuncSetAttribute(k_recall, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    e = launch_pdl(k_recall, dim3(L.batch * L.H * L.G), dim3(kRecallThreads), smem, s, L, weights, wstride, blocks,
                   stride, counts, recall);
    if (e != cudaSuccess) return e;
    ++*launches;
    return cudaSuccess;
}

}  // namespace absp

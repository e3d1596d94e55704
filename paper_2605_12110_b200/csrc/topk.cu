// Kernel 2: per-(sequence, KV head) budgeted Top-K block selection (sm_100a).
//
// Reference: select_topk -> select_impl -> select_head (engine.cpp:119-178).
//   K = ceil(T / B); if N <= K every block is selected; otherwise the top K by
//   (score desc, index asc) with the trailing block N-1 forced in, which is
//   exactly {N-1} U top-(K-1) of blocks [0, N-1). The
//   output is ordered by the same key. -0.0 and +0.0 tie (the reference
//   compares with !=).
//
// Algorithm (one CTA per unit, no atomics on the hot loop):
//   1. Order-preserving u32 keys (+-0 folded to +0).
//   2. Exact radix select of the (K-1)-th largest key over [0, N-1) with 5-bit
//      digits: 32 bins == 32 lanes. Per warp-step of 32 keys, 5 ballots give
//      each lane (= bin) its count through one LOP chain + POPC, so a pass costs
//      ~10 warp instructions per 32 keys and no shared-memory atomics.
//      7 passes (5,5,5,5,5,5,2 bits) pin the threshold key tau and the number of
//      tau-valued keys still needed; ties at tau go to the lowest indices.
//   3. The <= K winners are gathered to shared memory as 64-bit composite keys
//      (key << 32 | ~index), all distinct, and bitonic-sorted descending, which
//      yields the reference order.
#include "absp_internal.cuh"

namespace absp {
namespace {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxSort = 2048;      // max K (power of two bound)
constexpr int kMaxSteps = 4096;     // max (N-1)/32 warp-steps for tie ranking

__device__ __forceinline__ uint32_t order_key(float f) {
    uint32_t u = __float_as_uint(f);
    if ((u & 0x7fffffffu) == 0u) u = 0u;  // -0.0 == +0.0
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__global__ void __launch_bounds__(kThreads) k_topk(LayerView L, uint32_t* blocks, uint32_t stride,
                                                   uint32_t* counts) {
    __shared__ uint32_t s_hist[kWarps][32];
    __shared__ uint32_t s_state[4];  // prefix, pmask, remaining, eq_total
    __shared__ uint32_t s_nsel;
    __shared__ unsigned long long s_sel[kMaxSort];
    __shared__ uint32_t s_eq[kMaxSteps];

    const uint32_t u = blockIdx.x;
    const UnitDesc du = L.desc[u];
    const uint32_t N = du.n_blocks;
    const uint32_t K = du.budget;
    const float* sc = L.scores + du.seg;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t sel_total = N <= K ? N : K;

    if (threadIdx.x == 0) {
        s_state[0] = 0u;
        s_state[1] = 0u;
        s_state[2] = N > K ? K - 1 : 0u;
        s_state[3] = 0u;
        s_nsel = 0u;
    }
    __syncthreads();

    const uint32_t n_cand = N > K ? N - 1 : 0u;  // radix-select domain [0, N-1)
    if (N > K && K > 1) {
        for (int pass = 0; pass < 7; ++pass) {
            const int nbits = pass < 6 ? 5 : 2;
            const int shift = pass < 6 ? 27 - 5 * pass : 0;
            const uint32_t prefix = s_state[0], pmask = s_state[1];
            uint32_t xm[5];
#pragma unroll
            for (int j = 0; j < 5; ++j) xm[j] = ((lane >> j) & 1u) ? 0u : 0xffffffffu;
            uint32_t cnt = 0;
            for (uint32_t s = warp; s * 32 < n_cand; s += kWarps) {
                const uint32_t i = s * 32 + lane;
                const uint32_t key = i < n_cand ? order_key(__ldg(sc + i)) : 0u;
                const uint32_t m = __ballot_sync(0xffffffffu, i < n_cand && (key & pmask) == prefix);
                if (m == 0u) continue;
                uint32_t mm = m;
#pragma unroll
                for (int j = 0; j < 5; ++j) {
                    if (j < nbits) {
                        const uint32_t b = __ballot_sync(0xffffffffu, (key >> (shift + j)) & 1u);
                        mm &= b ^ xm[j];
                    }
                }
                cnt += __popc(mm);
            }
            if (lane >= (1u << nbits)) cnt = 0;
            s_hist[warp][lane] = cnt;
            __syncthreads();
            if (warp == 0) {
                uint32_t tot = 0;
#pragma unroll
                for (int w = 0; w < kWarps; ++w) tot += s_hist[w][lane];
                // suffix sum: number of keys in bins above `lane`
                uint32_t incl = tot;  // inclusive suffix (bins >= lane)
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t v = __shfl_down_sync(0xffffffffu, incl, o);
                    if (lane + o < 32) incl += v;
                }
                const uint32_t above = incl - tot;
                const uint32_t rem = s_state[2];
                if (tot > 0 && above < rem && rem <= above + tot) {
                    s_state[0] = prefix | (lane << shift);
                    s_state[1] = pmask | (((1u << nbits) - 1u) << shift);
                    s_state[2] = rem - above;
                    s_state[3] = tot;
                }
            }
            __syncthreads();
        }
    }

    // ---- gather the winners -------------------------------------------------
    if (N <= K) {
        for (uint32_t i = threadIdx.x; i < N; i += kThreads)
            s_sel[i] = (uint64_t(order_key(sc[i])) << 32) | uint32_t(~i);
    } else {
        const uint32_t tau = s_state[0];
        const uint32_t need_eq = s_state[2];
        const bool all_eq = (K > 1) && need_eq == s_state[3];
        const bool use_tau = K > 1;
        // Tie ranking by index is only needed when tau-valued keys exceed the slots.
        if (use_tau && !all_eq) {
            for (uint32_t s = warp; s * 32 < n_cand; s += kWarps) {
                const uint32_t i = s * 32 + lane;
                const bool eq = i < n_cand && order_key(__ldg(sc + i)) == tau;
                const uint32_t m = __ballot_sync(0xffffffffu, eq);
                if (lane == 0) s_eq[s] = __popc(m);
            }
            __syncthreads();
            if (warp == 0) {  // exclusive scan over steps
                const uint32_t nsteps = (n_cand + 31) / 32;
                uint32_t carry = 0;
                for (uint32_t base = 0; base < nsteps; base += 32) {
                    const uint32_t v = base + lane < nsteps ? s_eq[base + lane] : 0u;
                    uint32_t incl = v;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
                        if (lane >= uint32_t(o)) incl += t;
                    }
                    if (base + lane < nsteps) s_eq[base + lane] = carry + incl - v;
                    carry += __shfl_sync(0xffffffffu, incl, 31);
                }
            }
            __syncthreads();
        }
        for (uint32_t s = warp; s * 32 < n_cand; s += kWarps) {
            const uint32_t i = s * 32 + lane;
            const uint32_t key = i < n_cand ? order_key(__ldg(sc + i)) : 0u;
            bool take = false;
            if (use_tau) {
                if (all_eq) {
                    take = i < n_cand && key >= tau;
                } else {
                    const uint32_t eqm = __ballot_sync(0xffffffffu, i < n_cand && key == tau);
                    const uint32_t rank = s_eq[s] + __popc(eqm & ((1u << lane) - 1u));
                    take = i < n_cand && (key > tau || (key == tau && rank < need_eq));
                }
            }
            const uint32_t tm = __ballot_sync(0xffffffffu, take);
            if (tm) {
                uint32_t base = 0;
                if (lane == 0) base = atomicAdd(&s_nsel, __popc(tm));
                base = __shfl_sync(0xffffffffu, base, 0);
                if (take) s_sel[base + __popc(tm & ((1u << lane) - 1u))] = (uint64_t(key) << 32) | uint32_t(~i);
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            const uint32_t t = N - 1;
            s_sel[K - 1] = (uint64_t(order_key(sc[t])) << 32) | uint32_t(~t);
        }
    }
    // pad to a power of two with the minimum composite (sorts last)
    uint32_t sp = 1;
    while (sp < sel_total) sp <<= 1;
    for (uint32_t i = sel_total + threadIdx.x; i < sp; i += kThreads) s_sel[i] = 0ull;
    __syncthreads();

    // ---- bitonic sort, descending ------------------------------------------
    for (uint32_t k = 2; k <= sp; k <<= 1) {
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t i = threadIdx.x; i < sp; i += kThreads) {
                const uint32_t ixj = i ^ j;
                if (ixj > i) {
                    const unsigned long long a = s_sel[i], b = s_sel[ixj];
                    const bool desc = (i & k) == 0;
                    if (desc ? (a < b) : (a > b)) {
                        s_sel[i] = b;
                        s_sel[ixj] = a;
                    }
                }
            }
            __syncthreads();
        }
    }
    uint32_t* out = blocks + size_t(u) * stride;
    for (uint32_t i = threadIdx.x; i < sel_total; i += kThreads) out[i] = ~uint32_t(s_sel[i]);
    if (threadIdx.x == 0) counts[u] = sel_total;
}

}  // namespace

cudaError_t launch_topk(const LayerView& L, uint32_t max_nblocks, uint32_t max_budget,
                        uint32_t* blocks, uint32_t stride, uint32_t* counts, cudaStream_t s,
                        int* launches) {
    if (max_budget > uint32_t(kMaxSort) || max_nblocks > uint32_t(kMaxSteps) * 32u)
        return cudaErrorInvalidValue;
    k_topk<<<L.units, kThreads, 0, s>>>(L, blocks, stride, counts);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace absp

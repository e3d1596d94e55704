// Kernel 2: per-(sequence, KV head) budgeted Top-K block selection (sm_100a).
//
// Reference: select_topk -> select_impl -> select_head (engine.cpp:119-178).
//   K = ceil(T / B); if N <= K every block is selected; otherwise the top K by
//   (score desc, index asc) with the trailing block N-1 forced in, which is
//   exactly {N-1} U top-(K-1) of blocks [0, N-1). The
//   output is ordered by the same key. -0.0 and +0.0 tie (the reference
//   compares with !=).
//
// Algorithm (one 512-thread CTA per unit, no atomics on the hot loop):
//   1. Order-preserving u32 keys (+-0 folded to +0), loaded once into registers
//      (ITEMS keys per thread, warp-step s = j*16 + warp covers indices
//      [32s, 32s+32)). Units with more than 512*64 blocks use the same code with
//      keys re-read from L2 each pass.
//   2. The bits shared by every key (AND vs OR reduction) are skipped; the
//      remaining bits are resolved MSB-first by an exact radix select with 5-bit
//      digits: 32 bins == 32 lanes. Per warp-step, 5 ballots give each lane (=bin)
//      its count through a LOP chain + POPC — ~10 warp instructions per 32 keys,
//      no shared-memory atomics. This pins the (K-1)-th largest key tau and how
//      many tau-valued keys are still needed; ties at tau go to the lowest indices.
//   3. The <= K winners are gathered to shared memory as 64-bit composite keys
//      (key << 32 | ~index), all distinct, and bitonic-sorted descending, which
//      is exactly the reference order.
#include "absp_internal.cuh"

namespace absp {
namespace {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxSort = 2048;   // max K
constexpr int kMaxSteps = 4096;  // max (N-1)/32 warp-steps for tie ranking

__device__ __forceinline__ uint32_t order_key(float f) {
    uint32_t u = __float_as_uint(f);
    if ((u & 0x7fffffffu) == 0u) u = 0u;  // -0.0 == +0.0
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

struct TopkSmem {
    uint32_t hist[kWarps][32];
    uint32_t red[2][kWarps];
    uint32_t state[4];  // prefix, pmask, remaining, eq_total
    uint32_t nsel;
    unsigned long long sel[kMaxSort];
    uint32_t eq[kMaxSteps];
};

// Key of warp-step item j: from registers (REG) or re-read from L2.
template <bool REG, int ITEMS>
struct Keys {
    uint32_t r[REG ? ITEMS : 1];
    const float* sc;
    uint32_t n_cand;
    __device__ __forceinline__ uint32_t get(int j, uint32_t i) const {
        if (REG) return r[j];
        return i < n_cand ? order_key(__ldg(sc + i)) : 0u;
    }
};

template <bool REG, int ITEMS>
__global__ void __launch_bounds__(kThreads) k_topk(LayerView L, uint32_t* blocks, uint32_t stride,
                                                   uint32_t* counts) {
    __shared__ TopkSmem sm;
    const uint32_t u = blockIdx.x;
    const UnitDesc du = L.desc[u];
    const uint32_t N = du.n_blocks;
    const uint32_t K = du.budget;
    const float* sc = L.scores + du.seg;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t sel_total = N <= K ? N : K;
    const uint32_t n_cand = N > K ? N - 1 : 0u;  // radix-select domain [0, N-1)
    // number of warp-steps each warp walks
    const uint32_t nsteps = (n_cand + 31) / 32;
    const int my_items = REG ? ITEMS : int((nsteps + kWarps - 1 - warp) / kWarps);

    Keys<REG, ITEMS> keys;
    keys.sc = sc;
    keys.n_cand = n_cand;
    if (REG) {
#pragma unroll
        for (int j = 0; j < (REG ? ITEMS : 1); ++j) {
            const uint32_t i = (j * kWarps + warp) * 32 + lane;
            keys.r[j] = i < n_cand ? order_key(__ldg(sc + i)) : 0u;
        }
    }
    if (threadIdx.x == 0) {
        sm.state[0] = 0u;
        sm.state[1] = 0u;
        sm.state[2] = N > K ? K - 1 : 0u;
        sm.state[3] = 0u;
        sm.nsel = 0u;
    }

    if (N > K && K > 1) {
        // ---- common prefix of all candidate keys ---------------------------
        uint32_t kand = 0xffffffffu, kor = 0u;
#pragma unroll
        for (int j = 0; j < my_items; ++j) {
            const uint32_t i = (j * kWarps + warp) * 32 + lane;
            if (i < n_cand) {
                const uint32_t k = keys.get(j, i);
                kand &= k;
                kor |= k;
            }
        }
        kand = __reduce_and_sync(0xffffffffu, kand);
        kor = __reduce_or_sync(0xffffffffu, kor);
        if (lane == 0) {
            sm.red[0][warp] = kand;
            sm.red[1][warp] = kor;
        }
        __syncthreads();
        kand = 0xffffffffu;
        kor = 0u;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            kand &= sm.red[0][w];
            kor |= sm.red[1][w];
        }
        const uint32_t diff = kand ^ kor;
        int lo_bit;  // bits [lo_bit, 32) are already decided
        if (diff == 0u) {  // every candidate key is equal
            if (threadIdx.x == 0) {
                sm.state[0] = kand;
                sm.state[1] = 0xffffffffu;
                sm.state[3] = n_cand;
            }
            lo_bit = 0;
        } else {
            lo_bit = 32 - __clz(diff);  // highest differing bit is lo_bit-1
            if (threadIdx.x == 0) {
                const uint32_t m = lo_bit >= 32 ? 0u : (0xffffffffu << lo_bit);
                sm.state[0] = kand & m;
                sm.state[1] = m;
            }
        }
        __syncthreads();

        // ---- radix select, 5-bit digits, MSB first ------------------------
        uint32_t xm[5];
#pragma unroll
        for (int b = 0; b < 5; ++b) xm[b] = ((lane >> b) & 1u) ? 0u : 0xffffffffu;
        while (lo_bit > 0) {
            const int nbits = lo_bit >= 5 ? 5 : lo_bit;
            const int shift = lo_bit - nbits;
            const uint32_t prefix = sm.state[0], pmask = sm.state[1];
            uint32_t cnt = 0;
#pragma unroll
            for (int j = 0; j < my_items; ++j) {
                const uint32_t i = (j * kWarps + warp) * 32 + lane;
                const uint32_t key = keys.get(j, i);
                const uint32_t m = __ballot_sync(0xffffffffu, i < n_cand && (key & pmask) == prefix);
                if (m == 0u) continue;
                uint32_t mm = m;
#pragma unroll
                for (int b = 0; b < 5; ++b) {
                    if (b < nbits) mm &= __ballot_sync(0xffffffffu, (key >> (shift + b)) & 1u) ^ xm[b];
                }
                cnt += __popc(mm);
            }
            if (lane >= (1u << nbits)) cnt = 0;
            sm.hist[warp][lane] = cnt;
            __syncthreads();
            if (warp == 0) {
                uint32_t tot = 0;
#pragma unroll
                for (int w = 0; w < kWarps; ++w) tot += sm.hist[w][lane];
                uint32_t incl = tot;  // inclusive suffix sum over bins >= lane
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t v = __shfl_down_sync(0xffffffffu, incl, o);
                    if (lane + o < 32) incl += v;
                }
                const uint32_t above = incl - tot;
                const uint32_t rem = sm.state[2];
                if (tot > 0 && above < rem && rem <= above + tot) {
                    sm.state[0] = prefix | (lane << shift);
                    sm.state[1] = pmask | (((1u << nbits) - 1u) << shift);
                    sm.state[2] = rem - above;
                    sm.state[3] = tot;
                }
            }
            __syncthreads();
            lo_bit = shift;
        }
    }
    __syncthreads();

    // ---- gather the winners -------------------------------------------------
    if (N <= K) {
        for (uint32_t i = threadIdx.x; i < N; i += kThreads)
            sm.sel[i] = (uint64_t(order_key(sc[i])) << 32) | uint32_t(~i);
    } else {
        const uint32_t tau = sm.state[0];
        const uint32_t need_eq = sm.state[2];
        const bool use_tau = K > 1;
        const bool all_eq = use_tau && need_eq == sm.state[3];
        if (use_tau && !all_eq) {  // tie ranking by index among tau-valued keys
#pragma unroll
            for (int j = 0; j < my_items; ++j) {
                const uint32_t s = j * kWarps + warp;
                const uint32_t i = s * 32 + lane;
                const uint32_t m = __ballot_sync(0xffffffffu, i < n_cand && keys.get(j, i) == tau);
                if (lane == 0) sm.eq[s] = __popc(m);
            }
            __syncthreads();
            if (warp == 0) {  // exclusive scan over warp-steps (index order)
                uint32_t carry = 0;
                for (uint32_t base = 0; base < nsteps; base += 32) {
                    const uint32_t v = base + lane < nsteps ? sm.eq[base + lane] : 0u;
                    uint32_t incl = v;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
                        if (lane >= uint32_t(o)) incl += t;
                    }
                    if (base + lane < nsteps) sm.eq[base + lane] = carry + incl - v;
                    carry += __shfl_sync(0xffffffffu, incl, 31);
                }
            }
            __syncthreads();
        }
#pragma unroll
        for (int j = 0; j < my_items; ++j) {
            const uint32_t s = j * kWarps + warp;
            const uint32_t i = s * 32 + lane;
            const uint32_t key = keys.get(j, i);
            bool take = false;
            if (use_tau) {
                if (all_eq) {
                    take = i < n_cand && key >= tau;
                } else {
                    const uint32_t eqm = __ballot_sync(0xffffffffu, i < n_cand && key == tau);
                    const uint32_t rank = sm.eq[s] + __popc(eqm & ((1u << lane) - 1u));
                    take = i < n_cand && (key > tau || (key == tau && rank < need_eq));
                }
            }
            const uint32_t tm = __ballot_sync(0xffffffffu, take);
            if (tm) {
                uint32_t base = 0;
                if (lane == 0) base = atomicAdd(&sm.nsel, __popc(tm));
                base = __shfl_sync(0xffffffffu, base, 0);
                if (take) sm.sel[base + __popc(tm & ((1u << lane) - 1u))] = (uint64_t(key) << 32) | uint32_t(~i);
            }
        }
        if (threadIdx.x == 0) {
            const uint32_t t = N - 1;
            sm.sel[K - 1] = (uint64_t(order_key(sc[t])) << 32) | uint32_t(~t);
        }
    }
    uint32_t sp = 1;
    while (sp < sel_total) sp <<= 1;
    for (uint32_t i = sel_total + threadIdx.x; i < sp; i += kThreads) sm.sel[i] = 0ull;
    __syncthreads();

    // ---- bitonic sort, descending ------------------------------------------
    for (uint32_t k = 2; k <= sp; k <<= 1) {
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t i = threadIdx.x; i < sp; i += kThreads) {
                const uint32_t ixj = i ^ j;
                if (ixj > i) {
                    const unsigned long long a = sm.sel[i], b = sm.sel[ixj];
                    const bool desc = (i & k) == 0;
                    if (desc ? (a < b) : (a > b)) {
                        sm.sel[i] = b;
                        sm.sel[ixj] = a;
                    }
                }
            }
            __syncthreads();
        }
    }
    uint32_t* out = blocks + size_t(u) * stride;
    for (uint32_t i = threadIdx.x; i < sel_total; i += kThreads) out[i] = ~uint32_t(sm.sel[i]);
    if (threadIdx.x == 0) counts[u] = sel_total;
}

}  // namespace

cudaError_t launch_topk(const LayerView& L, uint32_t max_nblocks, uint32_t max_budget,
                        uint32_t* blocks, uint32_t stride, uint32_t* counts, cudaStream_t s,
                        int* launches) {
    if (max_budget > uint32_t(kMaxSort) || max_nblocks > uint32_t(kMaxSteps) * 32u)
        return cudaErrorInvalidValue;
    const uint32_t per_thread = (max_nblocks + kThreads - 1) / kThreads;
    const dim3 grid(L.units);
    if (per_thread <= 1) k_topk<true, 1><<<grid, kThreads, 0, s>>>(L, blocks, stride, counts);
    else if (per_thread <= 2) k_topk<true, 2><<<grid, kThreads, 0, s>>>(L, blocks, stride, counts);
    else if (per_thread <= 4) k_topk<true, 4><<<grid, kThreads, 0, s>>>(L, blocks, stride, counts);
    else if (per_thread <= 8) k_topk<true, 8><<<grid, kThreads, 0, s>>>(L, blocks, stride, counts);
    else if (per_thread <= 16) k_topk<true, 16><<<grid, kThreads, 0, s>>>(L, blocks, stride, counts);
    else if (per_thread <= 32) k_topk<true, 32><<<grid, kThreads, 0, s>>>(L, blocks, stride, counts);
    else if (per_thread <= 64) k_topk<true, 64><<<grid, kThreads, 0, s>>>(L, blocks, stride, counts);
    else k_topk<false, 1><<<grid, kThreads, 0, s>>>(L, blocks, stride, counts);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace absp

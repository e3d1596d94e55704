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
//      (ITEMS keys per thread; warp-step s = j*16 + warp covers [32s, 32s+32)).
//      Units with more than 512*64 blocks re-read the keys from L2 each pass.
//   2. Bits shared by every key (AND vs OR reduction) are skipped; the rest are
//      resolved MSB-first by an exact radix select with 5-bit digits: 32 bins ==
//      32 lanes; per warp-step, 5 ballots give each lane (= bin) its count through
//      a LOP chain + POPC. As soon as the keys still matching the running prefix
//      fit in shared memory they are compacted there, and the remaining passes
//      touch only them. This pins the (K-1)-th largest key tau and how many
//      tau-valued keys are still needed; ties at tau go to the lowest indices.
//   3. The <= K winners become 64-bit composite keys (key << 32 | ~index), all
//      distinct; their rank among each other is their output position (rank sort
//      for K <= 256, bitonic sort above), which is exactly the reference order.
//   4. The selection is published from shared memory with every selected block
//      resolved to its pool pages (the reference's populate_page_spans,
//      engine.cpp:271-283) for the attention producer; in the decode step the
//      unit's ready flag then lets the attention producer start on it.
#include "absp_internal.cuh"
#include "ptx.cuh"
#include "common.cuh"

namespace absp {
namespace {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxSort = 2048;   // max K
constexpr int kMaxSteps = 4096;  // max (N-1)/32 warp-steps for index tie ranking
constexpr int kCompact = 2048;   // compaction capacity (keys matching the prefix)

// Optional timeline instrumentation (debug builds with -DABSP_ATTN_TRACE).
#ifdef ABSP_ATTN_TRACE
constexpr int kTopkTraceSlots = 8;
__device__ unsigned long long g_topk_trace[1024 * kTopkTraceSlots];
__device__ __forceinline__ void topk_trace(int slot) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    if (blockIdx.x < 1024) g_topk_trace[blockIdx.x * kTopkTraceSlots + slot] = t;
}
#define TOPK_TRACE(slot) do { if (threadIdx.x == 0) topk_trace(slot); } while (0)
#else
#define TOPK_TRACE(slot) do {} while (0)
#endif


struct TopkSmem {
    uint32_t hist[kWarps][32];
    uint32_t red[2][kWarps];
    uint32_t state[6];  // prefix, pmask, remaining, eq_total, compacted count, compact flag
    uint32_t nsel;
    unsigned long long sel[kMaxSort];
    uint32_t outs[kMaxSort];  // the ordered selection, published from here
    union {
        uint32_t eq[kMaxSteps];
        struct {
            uint32_t key[kCompact];
            uint32_t idx[kCompact];
        } c;
    } u;
};

// Keys of a unit, thread (warp, lane) owning keys i = (j * kWarps + warp) * 32 + lane:
// in registers (REG), in dynamic shared memory (SMK: the largest units, whose
// register arrays would spill), or re-read from L2.
template <bool REG, int ITEMS, bool SMK>
struct Keys {
    uint32_t r[REG && !SMK ? ITEMS : 1];
    const uint32_t* sk;  // SMK: [n_cand] in shared memory
    const float* sc;
    uint32_t n_cand;
    __device__ __forceinline__ uint32_t get(int j, uint32_t i) const {
        if (SMK) return sk[i];
        if (REG) return r[j];
        return i < n_cand ? order_key(__ldcg(sc + i)) : 0u;
    }
    __device__ __forceinline__ uint32_t reg(int j, uint32_t warp, uint32_t lane) const {
        if (SMK) return sk[(j * kWarps + warp) * 32 + lane];
        return r[j];
    }
};

// One radix pass over a warp-step's 32 keys: adds this lane's bin count.
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ uint32_t bin_count(bool in, uint32_t key, uint32_t prefix, uint32_t pmask,
                                              int shift, int nbits, const uint32_t* xm) {
    const uint32_t m = __ballot_sync(0xffffffffu, in && (key & pmask) == prefix);
    if (m == 0u) return 0u;
    uint32_t mm = m;
#pragma unroll
    for (int b = 0; b < 5; ++b)
        if (b < nbits) mm &= __ballot_sync(0xffffffffu, (key >> (shift + b)) & 1u) ^ xm[b];
    return __popc(mm);
}

template <bool REG, int ITEMS, bool SMK>
__global__ void __launch_bounds__(kThreads, 1) k_topk(LayerView L, uint32_t* blocks, uint32_t stride,
                                                   uint32_t* counts, PageList pages, uint32_t* ready,
                                                   uint32_t* scored, const uint32_t* __restrict__ unit_list) {
    __shared__ TopkSmem sm;
    TOPK_TRACE(0);
    const uint32_t u = unit_list ? unit_list[blockIdx.x] : blockIdx.x;
    const UnitDesc du = L.desc[u];
    const uint32_t N = du.n_blocks;
    const uint32_t K = du.budget;
    const float* sc = L.scores + du.seg;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t sel_total = N <= K ? N : K;
    const uint32_t n_cand = N > K ? N - 1 : 0u;  // radix-select domain [0, N-1)
    const uint32_t nsteps = (n_cand + 31) / 32;
    const int my_items = REG ? ITEMS : int((nsteps + kWarps - 1 - warp) / kWarps);

    {   // the page resolution at the end reads the sequence's page-table row: the H units of
        // the sequence warm L2 with a slice each while the scores are being produced
        const uint32_t row_pages = (du.n_tokens + L.P - 1) / L.P;
        const uint32_t slice = (row_pages + L.H - 1) / L.H;
        const uint32_t* pt = L.page_table + size_t(du.seq) * L.max_pages;
        for (uint32_t p = du.head * slice + threadIdx.x * 32; p < min(row_pages, (du.head + 1) * slice);
             p += blockDim.x * 32)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(pt + p));
    }
    if (scored) {
        // the unit's scores are complete once the scorer's producers have published all
        // N of them (release); then re-arm the counter for the next step
        if (threadIdx.x == 0) {
            while (ld_acquire(scored + u) < N) __nanosleep(64);
            scored[u] = 0u;
        }
        __syncthreads();
    } else {
        griddep_wait();  // the scores are written by the scoring kernel of this step
    }
    // Only now may the attention kernel be scheduled. Its producers poll the per-unit
    // ready flags without a grid dependency wait; the flags of the previous step are
    // re-armed by that step's attention merges. Once every top-k CTA has seen its
    // unit's scores, the scorer of this step has run past its own griddep_wait, i.e.
    // the previous attention grid has completed and no stale flag is left to read.
    griddep_launch_dependents();
    const float tail_score = N > K ? __ldcg(sc + N - 1) : 0.0f;  // the trailing block, loaded early
    Keys<REG, ITEMS, SMK> keys;
    keys.sc = sc;
    keys.n_cand = n_cand;
    extern __shared__ uint32_t topk_keys[];  // SMK only: ITEMS * kThreads keys
    keys.sk = topk_keys;
    if (SMK) {
#pragma unroll 16
        for (int j = 0; j < ITEMS; ++j) {
            const uint32_t i = (j * kWarps + warp) * 32 + lane;
            topk_keys[i] = i < n_cand ? order_key(__ldcg(sc + i)) : 0u;
        }
    } else if (REG) {
#pragma unroll
        for (int j = 0; j < (REG ? ITEMS : 1); ++j) {
            const uint32_t i = (j * kWarps + warp) * 32 + lane;
            keys.r[j] = i < n_cand ? order_key(__ldcg(sc + i)) : 0u;
        }
    }
    if (threadIdx.x == 0) {
        sm.state[0] = 0u;
        sm.state[1] = 0u;
        sm.state[2] = N > K ? K - 1 : 0u;
        sm.state[3] = 0u;
        sm.state[4] = 0u;
        sm.state[5] = 0u;
        sm.nsel = 0u;
    }
    uint32_t xm[5];
#pragma unroll
    for (int b = 0; b < 5; ++b) xm[b] = ((lane >> b) & 1u) ? 0u : 0xffffffffu;
    __syncthreads();

    // ======== fast path: threshold from group maxima, exact order among few ========
    // x = lower edge of the (15-bit) bucket holding the (K-1)-th largest maximum of
    // groups of 4 keys. At least K-1 groups have a maximum >= x, so the candidates
    // {key >= x} contain the whole top-(K-1); typically only a little more than K-1
    // of them exist. They are compacted and ordered exactly among themselves.
    TOPK_TRACE(1);
    if (REG && N > K && K > 1) {
        constexpr int GS = ITEMS >= 4 ? 4 : 1;
        constexpr int NG = ITEMS / GS;
        const uint32_t K1 = K - 1;
        uint32_t gmax[NG];
#pragma unroll
        for (int gi = 0; gi < NG; ++gi) {
            uint32_t mx = 0;
#pragma unroll
            for (int j = gi * GS; j < gi * GS + GS; ++j) mx = max(mx, keys.reg(j, warp, lane));  // invalid keys are 0
            gmax[gi] = mx;
        }
        uint32_t kand = 0xffffffffu, kor = 0u;
#pragma unroll
        for (int gi = 0; gi < NG; ++gi)
            if (((gi * GS) * kWarps + warp) * 32 + lane < n_cand) {
                kand &= gmax[gi];
                kor |= gmax[gi];
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
        int lo_bit = (kand ^ kor) ? 32 - __clz(kand ^ kor) : 0;
        uint32_t prefix = lo_bit >= 32 ? 0u : (kand & (0xffffffffu << lo_bit));
        uint32_t pmask = lo_bit >= 32 ? 0u : (0xffffffffu << lo_bit);
        uint32_t rem = K1;
        for (int pass = 0; pass < 3 && lo_bit > 0; ++pass) {
            const int nbits = lo_bit >= 5 ? 5 : lo_bit;
            const int shift = lo_bit - nbits;
            uint32_t cnt = 0;
#pragma unroll
            for (int gi = 0; gi < NG; ++gi) {
                const bool in = ((gi * GS) * kWarps + warp) * 32 + lane < n_cand;
                cnt += bin_count(in, gmax[gi], prefix, pmask, shift, nbits, xm);
            }
            if (lane >= (1u << nbits)) cnt = 0;
            sm.hist[warp][lane] = cnt;
            __syncthreads();
            if (warp == 0) {
                uint32_t tot = 0;
#pragma unroll
                for (int w = 0; w < kWarps; ++w) tot += sm.hist[w][lane];
                uint32_t incl = tot;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t v = __shfl_down_sync(0xffffffffu, incl, o);
                    if (lane + o < 32) incl += v;
                }
                const uint32_t above = incl - tot;
                if (tot > 0 && above < rem && rem <= above + tot) {
                    sm.state[0] = prefix | (lane << shift);
                    sm.state[2] = rem - above;
                }
            }
            __syncthreads();
            prefix = sm.state[0];
            rem = sm.state[2];
            pmask |= ((1u << nbits) - 1u) << shift;
            lo_bit = shift;
        }
        TOPK_TRACE(2);
        const uint32_t x = prefix;  // bucket lower edge: low bits zero
        uint32_t c = 0;
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) c += keys.reg(j, warp, lane) >= x && (j * kWarps + warp) * 32 + lane < n_cand;
        c = __reduce_add_sync(0xffffffffu, c);
        __syncthreads();
        if (lane == 0) sm.red[0][warp] = c;
        __syncthreads();
        uint32_t C = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) C += sm.red[0][w];
        if (C >= K1 && C <= uint32_t(kMaxSort)) {
            // compact the candidates as composite keys (key << 32 | ~index): each warp
            // writes at its prefix of the per-warp counts, no atomics
            uint32_t pos = 0;
            for (uint32_t w = 0; w < warp; ++w) pos += sm.red[0][w];
#pragma unroll
            for (int j = 0; j < ITEMS; ++j) {
                const uint32_t i = (j * kWarps + warp) * 32 + lane;
                const uint32_t kj = keys.reg(j, warp, lane);
                const bool in = i < n_cand && kj >= x;
                const uint32_t m = __ballot_sync(0xffffffffu, in);
                if (in) sm.sel[pos + __popc(m & ((1u << lane) - 1u))] = (uint64_t(kj) << 32) | uint32_t(~i);
                pos += __popc(m);
            }
            __syncthreads();
            TOPK_TRACE(3);
            const unsigned long long ct = (uint64_t(order_key(tail_score)) << 32) | uint32_t(~(N - 1));
            uint32_t* out = sm.outs;
            if (C <= 256) {
                // rank among candidates = output position (composites are distinct);
                // tpc adjacent lanes share a candidate, each counting a strided share
                const uint32_t tpc = C <= 128 ? 4u : 2u;
                const uint32_t t = threadIdx.x, j = t / tpc, part = t % tpc;
                const bool valid = j < C;
                const unsigned long long me = valid ? sm.sel[j] : 0ull;
                uint32_t rank = 0;
                if (valid)
                    for (uint32_t o = part; o < C; o += tpc) rank += sm.sel[o] > me;
                for (uint32_t off = 1; off < tpc; off <<= 1) rank += __shfl_xor_sync(0xffffffffu, rank, off);
                bool above = false;  // a winner ranked before the trailing block
                if (valid && part == 0 && rank < K1) {
                    out[rank + (ct > me ? 1u : 0u)] = ~uint32_t(me);
                    above = me > ct;
                }
                const uint32_t n_above = __syncthreads_count(above);
                if (threadIdx.x == 0) sm.nsel = n_above;
            } else if (C <= 2u * kThreads) {
                // bitonic sort (descending) of 2 * kThreads composites, zero-padded: warp w
                // holds elements 64w + lane and 64w + 32 + lane in registers; distances
                // <= 32 are exchanged by shuffles / within the thread, larger ones through
                // shared memory (10 of the 55 stages), so most stages need no barrier
                for (uint32_t i = C + threadIdx.x; i < 2u * kThreads; i += kThreads) sm.sel[i] = 0ull;
                __syncthreads();
                const uint32_t p0 = warp * 64 + lane, p1 = p0 + 32;
                unsigned long long v0 = sm.sel[p0], v1 = sm.sel[p1];
                auto mx = [](unsigned long long a, unsigned long long b) { return a > b ? a : b; };
                auto mn = [](unsigned long long a, unsigned long long b) { return a > b ? b : a; };
                for (uint32_t k = 2; k <= 2u * kThreads; k <<= 1) {
                    uint32_t j = k >> 1;
                    if (j >= 64) {  // cross-warp stages through shared memory
                        sm.sel[p0] = v0;
                        sm.sel[p1] = v1;
                        __syncthreads();
                        for (; j >= 64; j >>= 1) {
                            for (uint32_t i = threadIdx.x; i < 2u * kThreads; i += kThreads) {
                                const uint32_t ixj = i ^ j;
                                if (ixj > i) {
                                    const unsigned long long a = sm.sel[i], b = sm.sel[ixj];
                                    if (((i & k) == 0) ? (a < b) : (a > b)) {
                                        sm.sel[i] = b;
                                        sm.sel[ixj] = a;
                                    }
                                }
                            }
                            __syncthreads();
                        }
                        v0 = sm.sel[p0];
                        v1 = sm.sel[p1];
                    }
                    if (j == 32) {  // the thread's own pair
                        const bool desc = (p0 & k) == 0;
                        const unsigned long long hi = mx(v0, v1), lo = mn(v0, v1);
                        v0 = desc ? hi : lo;
                        v1 = desc ? lo : hi;
                        j = 16;
                    }
                    for (; j > 0; j >>= 1) {  // partner lane ^ j, same register
                        const unsigned long long o0 = __shfl_xor_sync(0xffffffffu, v0, j);
                        const unsigned long long o1 = __shfl_xor_sync(0xffffffffu, v1, j);
                        const bool lower = (lane & j) == 0;
                        v0 = (lower == ((p0 & k) == 0)) ? mx(v0, o0) : mn(v0, o0);
                        v1 = (lower == ((p1 & k) == 0)) ? mx(v1, o1) : mn(v1, o1);
                    }
                }
                sm.sel[p0] = v0;
                sm.sel[p1] = v1;
                __syncthreads();
                for (uint32_t p = threadIdx.x; p < K1; p += kThreads) {
                    const unsigned long long me = sm.sel[p];
                    out[p + (ct > me ? 1u : 0u)] = ~uint32_t(me);
                    if (me > ct) atomicAdd(&sm.nsel, 1u);
                }
            } else {
                uint32_t sp = 1;
                while (sp < C) sp <<= 1;
                for (uint32_t i = C + threadIdx.x; i < sp; i += kThreads) sm.sel[i] = 0ull;
                __syncthreads();
                for (uint32_t k = 2; k <= sp; k <<= 1)
                    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
                        for (uint32_t i = threadIdx.x; i < sp; i += kThreads) {
                            const uint32_t ixj = i ^ j;
                            if (ixj > i) {
                                const unsigned long long a = sm.sel[i], b = sm.sel[ixj];
                                if (((i & k) == 0) ? (a < b) : (a > b)) {
                                    sm.sel[i] = b;
                                    sm.sel[ixj] = a;
                                }
                            }
                        }
                        __syncthreads();
                    }
                for (uint32_t p = threadIdx.x; p < K1; p += kThreads) {
                    const unsigned long long me = sm.sel[p];
                    out[p + (ct > me ? 1u : 0u)] = ~uint32_t(me);
                    if (me > ct) atomicAdd(&sm.nsel, 1u);
                }
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                out[sm.nsel] = N - 1;  // the trailing block sits after every larger winner
                TOPK_TRACE(4);
            }
            publish_selection(L, du, u, out, K, blocks, stride, counts, pages, ready);
            TOPK_TRACE(5);
            return;
        }
        // too many candidates (heavy ties near the threshold): exact path below
        if (threadIdx.x == 0) {
            sm.state[0] = 0u;
            sm.state[2] = K - 1;
            sm.state[4] = 0u;
        }
        __syncthreads();
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
        int lo_bit;  // bits [lo_bit, 32) are decided
        if (diff == 0u) {
            if (threadIdx.x == 0) {
                sm.state[0] = kand;
                sm.state[1] = 0xffffffffu;
                sm.state[3] = n_cand;
            }
            lo_bit = 0;
        } else {
            lo_bit = 32 - __clz(diff);
            if (threadIdx.x == 0) {
                const uint32_t m = lo_bit >= 32 ? 0u : (0xffffffffu << lo_bit);
                sm.state[0] = kand & m;
                sm.state[1] = m;
                sm.state[3] = n_cand;
            }
        }
        __syncthreads();

        // ---- radix select, 5-bit digits, MSB first ------------------------
        bool compact = false;
        while (lo_bit > 0) {
            const uint32_t prefix = sm.state[0], pmask = sm.state[1];
            // compact the keys still matching the prefix once they fit
            if (!compact && sm.state[3] <= uint32_t(kCompact)) {
#pragma unroll
                for (int j = 0; j < my_items; ++j) {
                    const uint32_t i = (j * kWarps + warp) * 32 + lane;
                    const uint32_t key = keys.get(j, i);
                    const bool in = i < n_cand && (key & pmask) == prefix;
                    const uint32_t m = __ballot_sync(0xffffffffu, in);
                    if (m) {
                        uint32_t base = 0;
                        if (lane == 0) base = atomicAdd(&sm.state[4], __popc(m));
                        base = __shfl_sync(0xffffffffu, base, 0);
                        if (in) {
                            const uint32_t p = base + __popc(m & ((1u << lane) - 1u));
                            sm.u.c.key[p] = key;
                            sm.u.c.idx[p] = i;
                        }
                    }
                }
                compact = true;
                __syncthreads();
            }
            const int nbits = lo_bit >= 5 ? 5 : lo_bit;
            const int shift = lo_bit - nbits;
            uint32_t cnt = 0;
            if (compact) {
                const uint32_t nc = sm.state[4];
                for (uint32_t s = warp; s * 32 < nc; s += kWarps) {
                    const uint32_t i = s * 32 + lane;
                    const uint32_t key = i < nc ? sm.u.c.key[i] : 0u;
                    cnt += bin_count(i < nc, key, prefix, pmask, shift, nbits, xm);
                }
            } else {
#pragma unroll
                for (int j = 0; j < my_items; ++j) {
                    const uint32_t i = (j * kWarps + warp) * 32 + lane;
                    cnt += bin_count(i < n_cand, keys.get(j, i), prefix, pmask, shift, nbits, xm);
                }
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
        if (threadIdx.x == 0) sm.state[5] = compact ? 1u : 0u;
    }
    __syncthreads();

    // ---- gather the winners -------------------------------------------------
    if (N <= K) {
        for (uint32_t i = threadIdx.x; i < N; i += kThreads)
            sm.sel[i] = (uint64_t(order_key(__ldcg(sc + i))) << 32) | uint32_t(~i);
    } else {
        const uint32_t tau = sm.state[0];
        const uint32_t need_eq = sm.state[2];
        const bool use_tau = K > 1;
        const bool all_eq = use_tau && need_eq == sm.state[3];
        const bool compacted = sm.state[5] != 0;
        // keys strictly above tau (and all tau-valued keys when every one is taken)
#pragma unroll
        for (int j = 0; j < my_items; ++j) {
            const uint32_t i = (j * kWarps + warp) * 32 + lane;
            const uint32_t key = keys.get(j, i);
            const bool take = use_tau && i < n_cand && (key > tau || (all_eq && key == tau));
            const uint32_t tm = __ballot_sync(0xffffffffu, take);
            if (tm) {
                uint32_t base = 0;
                if (lane == 0) base = atomicAdd(&sm.nsel, __popc(tm));
                base = __shfl_sync(0xffffffffu, base, 0);
                if (take) sm.sel[base + __popc(tm & ((1u << lane) - 1u))] = (uint64_t(key) << 32) | uint32_t(~i);
            }
        }
        if (use_tau && !all_eq) {
            // only `need_eq` of the tau-valued keys fit: the lowest indices win
            if (compacted) {
                const uint32_t nc = sm.state[4];
                for (uint32_t p = threadIdx.x; p < nc; p += kThreads) {
                    if (sm.u.c.key[p] != tau) continue;
                    const uint32_t my = sm.u.c.idx[p];
                    uint32_t rank = 0;
                    for (uint32_t o = 0; o < nc; ++o) rank += (sm.u.c.key[o] == tau && sm.u.c.idx[o] < my);
                    if (rank < need_eq) {
                        const uint32_t pos = atomicAdd(&sm.nsel, 1u);
                        sm.sel[pos] = (uint64_t(tau) << 32) | uint32_t(~my);
                    }
                }
            } else {
                __syncthreads();
#pragma unroll
                for (int j = 0; j < my_items; ++j) {
                    const uint32_t s = j * kWarps + warp;
                    const uint32_t i = s * 32 + lane;
                    const uint32_t m = __ballot_sync(0xffffffffu, i < n_cand && keys.get(j, i) == tau);
                    if (lane == 0) sm.u.eq[s] = __popc(m);
                }
                __syncthreads();
                if (warp == 0) {  // exclusive scan over warp-steps (index order)
                    uint32_t carry = 0;
                    for (uint32_t base = 0; base < nsteps; base += 32) {
                        const uint32_t v = base + lane < nsteps ? sm.u.eq[base + lane] : 0u;
                        uint32_t incl = v;
#pragma unroll
                        for (int o = 1; o < 32; o <<= 1) {
                            const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
                            if (lane >= uint32_t(o)) incl += t;
                        }
                        if (base + lane < nsteps) sm.u.eq[base + lane] = carry + incl - v;
                        carry += __shfl_sync(0xffffffffu, incl, 31);
                    }
                }
                __syncthreads();
#pragma unroll
                for (int j = 0; j < my_items; ++j) {
                    const uint32_t s = j * kWarps + warp;
                    const uint32_t i = s * 32 + lane;
                    const bool eq = i < n_cand && keys.get(j, i) == tau;
                    const uint32_t eqm = __ballot_sync(0xffffffffu, eq);
                    const bool take = eq && sm.u.eq[s] + __popc(eqm & ((1u << lane) - 1u)) < need_eq;
                    const uint32_t tm = __ballot_sync(0xffffffffu, take);
                    if (tm) {
                        uint32_t base = 0;
                        if (lane == 0) base = atomicAdd(&sm.nsel, __popc(tm));
                        base = __shfl_sync(0xffffffffu, base, 0);
                        if (take) sm.sel[base + __popc(tm & ((1u << lane) - 1u))] = (uint64_t(tau) << 32) | uint32_t(~i);
                    }
                }
            }
        }
        if (threadIdx.x == 0) {
            const uint32_t t = N - 1;
            sm.sel[K - 1] = (uint64_t(order_key(tail_score)) << 32) | uint32_t(~t);
        }
    }
    __syncthreads();

    // ---- order: (key desc, index asc) == composite desc -----------------------
    uint32_t* out = sm.outs;
    if (sel_total <= 256) {
        // rank sort: position = number of larger composites (all distinct)
        for (uint32_t i = threadIdx.x; i < sel_total; i += kThreads) {
            const unsigned long long me = sm.sel[i];
            uint32_t rank = 0;
            for (uint32_t o = 0; o < sel_total; ++o) rank += sm.sel[o] > me;
            out[rank] = ~uint32_t(me);
        }
    } else {
        uint32_t sp = 1;
        while (sp < sel_total) sp <<= 1;
        for (uint32_t i = sel_total + threadIdx.x; i < sp; i += kThreads) sm.sel[i] = 0ull;
        __syncthreads();
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
        for (uint32_t i = threadIdx.x; i < sel_total; i += kThreads) out[i] = ~uint32_t(sm.sel[i]);
    }
    publish_selection(L, du, u, out, sel_total, blocks, stride, counts, pages, ready);
}

}  // namespace

#ifdef ABSP_ATTN_TRACE
cudaError_t debug_topk_trace(void* dst, size_t bytes) {
    return cudaMemcpyFromSymbol(dst, g_topk_trace, bytes);
}
#endif

// Keys per thread of the register-resident variant for a unit of n blocks (0: too
// many for registers, keys re-read from L2).
uint32_t topk_items(uint32_t n_blocks) {
    const uint32_t per_thread = (n_blocks + kThreads - 1) / kThreads;
    for (uint32_t it = 1; it <= 64; it <<= 1)
        if (per_thread <= it) return it;
    return 0;
}

template <bool REG, int IT, bool SMK = false>
cudaError_t topk_launch(const LayerView& L, uint32_t grid, uint32_t* blocks, uint32_t stride, uint32_t* counts,
                        const PageList& pages, uint32_t* ready, uint32_t* scored, const uint32_t* unit_list,
                        cudaStream_t s) {
    return launch_pdl(k_topk<REG, IT, SMK>, dim3(grid), dim3(kThreads), SMK ? size_t(IT) * kThreads * 4 : 0, s, L,
                      blocks, stride, counts, pages, ready, scored, unit_list);
}

cudaError_t init_topk_attributes() {  // the shared-memory key variants: 32 / 64 / 128 KB of keys
    cudaError_t e = cudaFuncSetAttribute(k_topk<true, 16, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         16 * kThreads * 4);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_topk<true, 32, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             32 * kThreads * 4);
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(k_topk<true, 64, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                64 * kThreads * 4);
}

cudaError_t launch_topk_class(const LayerView& L, uint32_t items, uint32_t grid, uint32_t* blocks, uint32_t stride,
                              uint32_t* counts, const PageList& pages, uint32_t* ready, uint32_t* scored,
                              const uint32_t* unit_list, cudaStream_t s) {
    switch (items) {
        case 1: return topk_launch<true, 1>(L, grid, blocks, stride, counts, pages, ready, scored, unit_list, s);
        case 2: return topk_launch<true, 2>(L, grid, blocks, stride, counts, pages, ready, scored, unit_list, s);
        case 4: return topk_launch<true, 4>(L, grid, blocks, stride, counts, pages, ready, scored, unit_list, s);
        case 8: return topk_launch<true, 8>(L, grid, blocks, stride, counts, pages, ready, scored, unit_list, s);
        case 16: return topk_launch<true, 16, true>(L, grid, blocks, stride, counts, pages, ready, scored, unit_list, s);
        case 32: return topk_launch<true, 32, true>(L, grid, blocks, stride, counts, pages, ready, scored, unit_list, s);
        // 64 keys per thread would spill from registers: they live in shared memory
        case 64: return topk_launch<true, 64, true>(L, grid, blocks, stride, counts, pages, ready, scored, unit_list, s);
        default: return topk_launch<false, 1>(L, grid, blocks, stride, counts, pages, ready, scored, unit_list, s);
    }
}

cudaError_t launch_topk(const LayerView& L, uint32_t max_nblocks, uint32_t max_budget,
                        uint32_t* blocks, uint32_t stride, uint32_t* counts, const PageList& pages,
                        uint32_t* ready, uint32_t* scored, const TopkClasses& classes,
                        cudaStream_t s, int* launches) {
    if (max_budget > uint32_t(kMaxSort) || max_nblocks > uint32_t(kMaxSteps) * 32u)
        return cudaErrorInvalidValue;
    if (!classes.units) {  // one launch sized for the largest unit
        ++*launches;
        cudaError_t e = launch_topk_class(L, topk_items(max_nblocks), L.units, blocks, stride, counts, pages, ready,
                                          scored, nullptr, s);
        return e == cudaSuccess ? cudaGetLastError() : e;
    }
    // one launch per register class, units grouped by class (largest first)
    for (int c = 0; c < kTopkClasses; ++c) {
        const uint32_t n = classes.begin[c + 1] - classes.begin[c];
        if (n == 0) continue;
        ++*launches;
        cudaError_t e = launch_topk_class(L, classes.items[c], n, blocks, stride, counts, pages, ready, scored,
                                          classes.units + classes.begin[c], s);
        if (e != cudaSuccess) return e;
    }
    return cudaGetLastError();
}

// Page resolution for an explicit (caller-provided) selection: absp_attend. The
// selection is validated as the reference's check_selection / block_to_pages do
// (engine.cpp:212-232, kv_cache.cpp:118-138): an empty selection, a count above
// blocks_stride, a block id past the unit's blocks or a page-table entry outside the
// pools raises a bit of *err (read back by absp_attend_validate); offending entries
// are dropped, so no copy leaves the K/V pools.
__global__ void k_resolve_pages(LayerView L, const uint32_t* __restrict__ blocks, uint32_t stride,
                                const uint32_t* __restrict__ counts, PageList pages, uint32_t* err) {
    griddep_launch_dependents();
    griddep_wait();  // blocks / counts may come from the previous kernel
    const uint32_t u = blockIdx.x;
    const UnitDesc du = L.desc[u];
    const uint32_t ppb = du.block / L.P;
    const uint32_t E = kAttnChunkRows / du.block;
    const uint32_t cap = min(stride, du.n_blocks);  // entries the work list reserves
    const uint32_t raw = counts[u];
    const uint32_t cnt = min(raw, cap);
    uint32_t flags = 0;
    if (threadIdx.x == 0) {
        if (raw == 0) flags |= kAttendErrEmpty;
        if (raw > stride) flags |= kAttendErrCount;
    }
    const uint32_t slot_end = ((cap + E - 1) / E) * pages.ns;  // every slot of the unit's chunks (page_slot)
    const uint32_t* pt = L.page_table + size_t(du.seq) * L.max_pages;
    const uint32_t head_base = du.head * uint32_t(L.pool_pages);
    const size_t base = size_t(pages.chunk_base[u]) * pages.ns;
    for (uint32_t s = threadIdx.x; s < slot_end; s += blockDim.x) {
        const uint32_t w = s % pages.ns, ein = w / ppb, pp = w % ppb;
        const uint32_t e = (s / pages.ns) * E + ein;
        uint32_t v = 0, page = 0;
        if (ein < E && e < cnt) {
            const uint32_t blk = __ldg(blocks + size_t(u) * stride + e);
            if (blk >= du.n_blocks) {
                flags |= kAttendErrBlock;
            } else {
                const uint32_t t0 = blk * du.block + pp * L.P;
                if (t0 < du.n_tokens) {
                    const uint32_t pid = __ldg(pt + t0 / L.P);
                    if (pid >= L.pool_pages) {
                        flags |= kAttendErrPage;
                    } else {
                        v = min(L.P, du.n_tokens - t0);
                        page = head_base + pid;
                    }
                }
            }
        }
        pages.page[base + s] = page;
        pages.valid[base + s] = uint16_t(v);
    }
    if (flags && err) atomicOr(err, flags);
}
cudaError_t launch_resolve_pages(const LayerView& L, const uint32_t* blocks, uint32_t stride,
                                 const uint32_t* counts, const PageList& pages, uint32_t* err, cudaStream_t s,
                                 int* launches) {
    launch_pdl(k_resolve_pages, dim3(L.units), dim3(256), 0, s, L, blocks, stride, counts, pages, err);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace absp

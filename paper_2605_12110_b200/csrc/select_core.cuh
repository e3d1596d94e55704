// Core of the fused selection (select.cu): its constants and shared-memory header, the
// exact serial score, the filter's weight split and error bound, the sorts, and the
// finalize of one unit (threshold, candidates, exact scores, ranks, publication). See
// select.cu for the algorithm.
#pragma once

#include <math.h>

#include <algorithm>

#include "absp_internal.cuh"
#include "common.cuh"
#include "ptx.cuh"

namespace absp {
namespace selcore {
namespace {  // internal linkage (device helpers defined in a header)

constexpr int kSCons = 256;              // consumer threads (8 warps), one code row each per stage
constexpr int kSThreads = kSCons + 32;   // + producer warp
constexpr int kSWarps = kSThreads / 32;
constexpr int kSRows = kSCons;           // rows per stage
constexpr int kSStages = 4;
constexpr uint32_t kCandCapMax = 2048;   // candidate capacity bound (>= K, K <= T / min B <= 2048)
constexpr int kBins = 1024;
constexpr uint32_t kNoPrefetch = 0xfffffffeu;  // emit: resolve the block's pages from the page table
constexpr uint32_t kSliceMin = 256;      // slice rows: a multiple of kSliceMin ...
constexpr uint32_t kSliceMax = 4096;     // ... up to this
constexpr uint32_t kFinKeys = 8192;      // finalize: keys per TMA batch in shared memory
constexpr uint32_t kRefineMin = 48;      // finalize: keys in the threshold bin above which it is refined

// Optional timeline instrumentation (debug builds with -DABSP_ATTN_TRACE): per CTA,
// globaltimer stamps at the phase boundaries (tools/select_trace.py).
#ifdef ABSP_ATTN_TRACE
constexpr int kSelTraceSlots = 24;
__device__ unsigned long long g_sel_trace[4096 * kSelTraceSlots];
#define SEL_TRACE(slot)                                                                           \
    do {                                                                                          \
        if (threadIdx.x == 0 && blockIdx.x < 4096) {                                              \
            unsigned long long t_;                                                                \
            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_));                                 \
            g_sel_trace[blockIdx.x * kSelTraceSlots + (slot)] = t_;                               \
        }                                                                                         \
    } while (0)
#else
#define SEL_TRACE(slot) do {} while (0)
#endif

template <int D>
struct SelCfg {
    static constexpr int W = D / 8;        // int4 words per code row
    static constexpr int ROWB = W * 4;
    static constexpr int STAGEB = kSRows * ROWB;
    static constexpr int QB = 8 * D * 2;   // q rows (G <= 8)
    static constexpr int PB = 2 * D * 4;   // scales + zero points
    static constexpr int TBL = D * 16 * 4; // exact product table
};

// Fixed-size part of the shared memory (after the ring, keys, table and parameters).
struct SelHead {
    unsigned long long bars[2 * kSStages + 2];  // full[NS], empty[NS], params, finalize keys
    unsigned long long ct;               // finalize: the trailing block's composite
    int8_t hlw[kSCons / 32][2][128];     // per consumer warp: h and l per channel (D <= 128)
    float red[4][kSWarps];       // block reductions
    uint32_t tpg[kAttnChunkRows];  // finalize: the trailing block's pool pages
    uint32_t st[16];             // misc scalars
    alignas(16) uint32_t hist[kBins];
    uint32_t local_cnt;          // finalize: candidates found
    uint32_t cand_cnt;
    uint32_t overflow;
    uint32_t nsel;
    unsigned long long* cand;
    uint32_t* list;
    uint32_t* outs;
    uint32_t cap;
};

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

__device__ __forceinline__ void cons_sync() {  // named barrier 1: the consumer warps
    asm volatile("bar.sync 1, %0;\n" ::"n"(kSCons) : "memory");
}

// The reference's exact serial score of one packed code row (score.cu's op order:
// channel c = 8 w + k, acc = fl(acc + tbl[c][code])).
template <int W>
__device__ __forceinline__ float exact_row(const uint32_t* wd, const float* tbl) {
    float acc = 0.0f;
#pragma unroll
    for (int w = 0; w < W; ++w) {
#pragma unroll
        for (int k = 0; k < 8; ++k) acc = __fadd_rn(acc, tbl[(w * 8 + k) * 16 + ((wd[w] >> (4 * k)) & 15u)]);
    }
    return acc;
}

// Logical words of code row i (global memory, swizzled 16-byte groups).
template <int W>
__device__ __forceinline__ void load_row_global(const uint32_t* codes, uint64_t row, uint32_t i, uint32_t* wd) {
    constexpr int U = W / 4;
    const uint4* src = reinterpret_cast<const uint4*>(codes + row * W);
    const uint32_t key = code_row_key(i, W);
#pragma unroll
    for (int g = 0; g < U; ++g) {
        const uint4 v = __ldcg(src + (g ^ key));
        wd[4 * g] = v.x;
        wd[4 * g + 1] = v.y;
        wd[4 * g + 2] = v.z;
        wd[4 * g + 3] = v.w;
    }
}

// Bitonic sort of a[0, n) descending in shared memory (the power of two above n must
// fit the array; padded with 0, below every composite key).
__device__ void sort_desc(unsigned long long* a, uint32_t n) {
    uint32_t sp = 1;
    while (sp < n) sp <<= 1;
    for (uint32_t i = n + threadIdx.x; i < sp; i += blockDim.x) a[i] = 0ull;
    __syncthreads();
    for (uint32_t k = 2; k <= sp; k <<= 1)
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t i = threadIdx.x; i < sp; i += blockDim.x) {
                const uint32_t ixj = i ^ j;
                if (ixj > i) {
                    const unsigned long long x = a[i], y = a[ixj];
                    if (((i & k) == 0) ? (x < y) : (x > y)) {
                        a[i] = y;
                        a[ixj] = x;
                    }
                }
            }
            __syncthreads();
        }
}

// Leader: orders the n candidate composites and writes the unit's selection to
// sh.outs: all of them (N <= K), or the top K-1 with the trailing composite ct
// inserted at its rank. Returns the selection length.
__device__ uint32_t order_selection(SelHead& sh, uint32_t n, uint32_t K, bool trailing, unsigned long long ct,
                                    uint32_t N) {
    const uint32_t tid = threadIdx.x;
    const uint32_t K1 = trailing ? K - 1 : n;
    if (tid == 0) sh.nsel = 0u;
    if (n <= 256) {  // rank counting (composites are distinct)
        __syncthreads();
        for (uint32_t j = tid; j < n; j += blockDim.x) {
            const unsigned long long me = sh.cand[j];
            uint32_t rank = 0;
            for (uint32_t o = 0; o < n; ++o) rank += sh.cand[o] > me;
            if (rank < K1) {
                sh.outs[rank + (trailing && ct > me ? 1u : 0u)] = ~uint32_t(me);
                if (trailing && me > ct) atomicAdd(&sh.nsel, 1u);
            }
        }
    } else {
        sort_desc(sh.cand, n);
        for (uint32_t p = tid; p < K1; p += blockDim.x) {
            const unsigned long long me = sh.cand[p];
            sh.outs[p + (trailing && ct > me ? 1u : 0u)] = ~uint32_t(me);
            if (trailing && me > ct) atomicAdd(&sh.nsel, 1u);
        }
    }
    __syncthreads();
    if (trailing && tid == 0) sh.outs[sh.nsel] = N - 1;
    __syncthreads();
    return trailing ? K : n;
}

// Exact fallback of the leader (mass ties): every block of [0, n1) scored exactly
// into the scores buffer, the (K-1)-th largest by an 8-bit radix select over the
// keys re-read from L2, ties at the threshold taken by lowest index, then ordered.
template <int W>
__device__ void exact_fallback(const LayerView& L, const UnitDesc& du, SelHead& sh, const float* tbl, uint32_t K,
                               unsigned long long ct) {
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t N = du.n_blocks, n1 = N - 1, K1 = K - 1;
    float* sc = L.scores + du.seg;
    for (uint32_t i = tid; i < n1; i += blockDim.x) {
        uint32_t wd[W];
        load_row_global<W>(L.codes, du.seg + i, i, wd);
        sc[i] = exact_row<W>(wd, tbl);
    }
    __syncthreads();
    uint32_t prefix = 0, mask = 0, rem = K1, gt = 0;
    for (int shift = 24; shift >= 0; shift -= 8) {
        for (uint32_t i = tid; i < 256; i += blockDim.x) sh.hist[i] = 0u;
        __syncthreads();
        for (uint32_t i = tid; i < n1; i += blockDim.x) {
            const uint32_t key = order_key(__ldcg(sc + i));
            if ((key & mask) == prefix) atomicAdd(&sh.hist[(key >> shift) & 255u], 1u);
        }
        __syncthreads();
        if (tid == 0) {  // the digit holding the rem-th largest
            uint32_t cum = 0;
            for (int b = 255; b >= 0; --b) {
                if (cum + sh.hist[b] >= rem) {
                    sh.st[0] = uint32_t(b);
                    sh.st[1] = cum;
                    break;
                }
                cum += sh.hist[b];
            }
        }
        __syncthreads();
        prefix |= sh.st[0] << shift;
        mask |= 255u << shift;
        gt += sh.st[1];
        rem -= sh.st[1];
        __syncthreads();
    }
    const uint32_t tau = prefix, need_eq = rem;  // K1 = gt + need_eq
    if (tid == 0) sh.cand_cnt = 0u;
    __syncthreads();
    for (uint32_t i = tid; i < n1; i += blockDim.x) {
        const uint32_t key = order_key(__ldcg(sc + i));
        if (key > tau) sh.cand[atomicAdd(&sh.cand_cnt, 1u)] = (uint64_t(key) << 32) | uint32_t(~i);
    }
    // the first need_eq tau-valued keys in index order
    uint32_t taken = 0;
    for (uint32_t base = 0; base < n1 && taken < need_eq; base += blockDim.x) {
        const uint32_t i = base + tid;
        const bool eq = i < n1 && order_key(__ldcg(sc + i)) == tau;
        const uint32_t m = __ballot_sync(0xffffffffu, eq);
        if (lane == 0) sh.hist[warp] = __popc(m);
        __syncthreads();
        uint32_t before = taken;
        for (uint32_t w = 0; w < warp; ++w) before += sh.hist[w];
        before += __popc(m & ((1u << lane) - 1u));
        if (eq && before < need_eq) sh.cand[gt + before] = (uint64_t(tau) << 32) | uint32_t(~i);
        uint32_t tot = 0;
        for (uint32_t w = 0; w < blockDim.x / 32; ++w) tot += sh.hist[w];
        taken += tot;
        __syncthreads();
    }
    __syncthreads();
    order_selection(sh, K1, K, true, ct, N);
}


// Integer MMA: C[16x8] (s32) += A[16x32] (u8, row) * B[32x8] (s8, col), exact.
__device__ __forceinline__ void imma(int* c, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                     uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}

// Warp: the bin of hist[0, 1024) holding the kr-th largest element counted from the top
// bin (1 <= kr <= total). Lane l sums bins [32 l, 32 l + 32) (8 16-byte loads in a
// lane-rotated order: conflict-free), a suffix scan over the lanes finds the lane L
// holding it, and a second suffix scan over L's 32 bins (one per lane) the bin. Writes
// the bin and the number of elements in the bins above it.
__device__ __forceinline__ void find_bin_desc(const uint32_t* hist, uint32_t kr, uint32_t lane, uint32_t* bin,
                                              uint32_t* above) {
    uint32_t tot = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const uint4 x = *reinterpret_cast<const uint4*>(hist + lane * 32 + ((uint32_t(k) + lane) & 7u) * 4);
        tot += (x.x + x.y) + (x.z + x.w);
    }
    uint32_t incl = tot;  // elements in lanes >= this one (larger bins)
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t x = __shfl_down_sync(0xffffffffu, incl, o);
        if (lane + o < 32) incl += x;
    }
    const uint32_t hit = __ballot_sync(0xffffffffu, incl - tot < kr && kr <= incl);
    const uint32_t L = __ffs(hit) - 1;
    const uint32_t cumL = __shfl_sync(0xffffffffu, incl - tot, L);  // elements above lane L's bins
    const uint32_t c = hist[L * 32 + lane];
    uint32_t in2 = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t x = __shfl_down_sync(0xffffffffu, in2, o);
        if (lane + o < 32) in2 += x;
    }
    const uint32_t hit2 = __ballot_sync(0xffffffffu, cumL + in2 - c < kr && kr <= cumL + in2);
    const uint32_t i = __ffs(hit2) - 1;
    if (lane == i) {
        *bin = L * 32 + i;
        *above = cumL + in2 - c;
    }
}

// Bitonic sort (descending) of n <= 256 R composites a[0, 256 R), zero-padded, by the 8
// consumer warps (R elements per lane in registers: element warp*32R + 32 r + lane):
// distances 32 .. 16R inside a thread (register indices resolved at compile time, so v
// stays in registers), below 32 by shuffles, 32R and up through shared memory. The
// producer warp only joins the barriers.
template <int R>
__device__ void sortreg_desc(unsigned long long* a, uint32_t n) {
    constexpr uint32_t NE = 256u * R;
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (uint32_t i = n + tid; i < NE; i += blockDim.x) a[i] = 0ull;
    __syncthreads();
    SEL_TRACE(16);
    const bool act = warp < 8;
    const uint32_t base = warp * 32u * R + lane;
    unsigned long long v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = act ? a[base + 32 * r] : 0ull;
    for (uint32_t k = 2; k <= NE; k <<= 1) {
#ifdef SORT_PROBE
        if (threadIdx.x == 0) g_sort_clk[31 - __clz(k)] = clock64();
#endif
        if ((k >> 1) >= 32u * R) {  // cross-warp distances through shared memory
            if (k == 64u * R) SEL_TRACE(17);
            if (act) {
#pragma unroll
                for (int r = 0; r < R; ++r) a[base + 32 * r] = v[r];
            }
            __syncthreads();
            for (uint32_t j = k >> 1; j >= 32u * R; j >>= 1) {
                for (uint32_t i = tid; i < NE; i += blockDim.x) {
                    const uint32_t ixj = i ^ j;
                    if (ixj > i) {
                        const unsigned long long x = a[i], y = a[ixj];
                        if (((i & k) == 0) ? (x < y) : (x > y)) {
                            a[i] = y;
                            a[ixj] = x;
                        }
                    }
                }
                __syncthreads();
            }
            if (act) {
#pragma unroll
                for (int r = 0; r < R; ++r) v[r] = a[base + 32 * r];
            }
        }
        if (!act) continue;
        const uint32_t j0 = min(k >> 1, 16u * R);
#pragma unroll
        for (int jr = R / 2; jr >= 1; jr >>= 1) {  // distance 32 jr: registers r and r | jr
            if (uint32_t(32 * jr) > j0) continue;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                if (r & jr) continue;
                const bool desc = ((base + 32 * r) & k) == 0;
                const unsigned long long x = v[r], y = v[r | jr];
                const unsigned long long hi = x > y ? x : y, lo = x > y ? y : x;
                v[r] = desc ? hi : lo;
                v[r | jr] = desc ? lo : hi;
            }
        }
        for (uint32_t j = min(k >> 1, 16u); j > 0; j >>= 1) {  // lanes ^ j, same register
            const bool lower = (lane & j) == 0;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const unsigned long long o = __shfl_xor_sync(0xffffffffu, v[r], j);
                const bool desc = ((base + 32 * r) & k) == 0;
                v[r] = (lower == desc) ? (v[r] > o ? v[r] : o) : (v[r] > o ? o : v[r]);
            }
        }
    }
    SEL_TRACE(18);
    if (act) {
#pragma unroll
        for (int r = 0; r < R; ++r) a[base + 32 * r] = v[r];
    }
    __syncthreads();
}

// Shared-memory layout (host and device): ring [stages][rows][row bytes] (in the
// finalize: the candidate composites cand [cand_cap] u64, list / outs [cand_cap] u32, the
// candidates' prefetched pages cpg [pg_cap] u32 and a batch of the unit's keys) | the
// slice's keys [rows] (units of several key batches) | product table | q rows | scales,
// zps | SelHead.
template <int D>
struct SelLayout {
    size_t cand, list, cpg, fkeys, slk, tbl, prm, head, total;
    __host__ __device__ SelLayout(uint32_t stages, uint32_t cand_cap, uint32_t pg_cap, uint32_t rows) {
        cand = 0;
        list = size_t(cand_cap) * 8;
        cpg = list + size_t(cand_cap) * 4;
        fkeys = (cpg + size_t(pg_cap) * 4 + 15) & ~size_t(15);
        const size_t ring = size_t(stages) * SelCfg<D>::STAGEB, fin = fkeys + (kFinKeys + 8) * 4;
        slk = ((ring > fin ? ring : fin) + 15) & ~size_t(15);
        tbl = (slk + size_t(rows) * 4 + 15) & ~size_t(15);
        prm = tbl + SelCfg<D>::TBL;
        head = prm + SelCfg<D>::QB + SelCfg<D>::PB;
        total = (head + sizeof(SelHead) + 15) & ~size_t(15);
    }
};

// Everything the finalize of one unit needs (k_select's last-arriving slice, or the
// attention CTA that owns the unit's first chunk): the unit, its slices, the step's
// outputs and this CTA's shared-memory scratch (cand | list | cpg | key batch, the
// product table, the unit's q rows, scales and zero points).
template <int D>
struct FinIn {
    LayerView L;
    uint32_t u;
    UnitDesc du;
    uint32_t first, Cn;  // the unit's slices [first, first + Cn)
    SelectPlan plan;
    SelectWork sw;
    uint32_t* blocks;
    uint32_t stride;
    uint32_t* counts;
    PageList pages;
    uint32_t* ready;
    uint16_t* q_copy;
    unsigned long long* cand;
    uint32_t* list;
    uint32_t* cpg;
    uint32_t* skeys;
    float* tbl;
    const uint16_t* qrows;
    const float* scl;
    const float* zps;
};

// Finalize of unit a.u once every slice has arrived (their keys and key ranges in L2):
// threshold, candidates, exact scores, ranks, publication. sh.st[0] holds the unit's
// integer error bound E_int; sh.hist, local_cnt, nsel are zero and the keys mbarrier
// (bars[2 * kSStages + 1]) is initialised at phase 0. All kSThreads threads call it.
template <int D>
__device__ __forceinline__ void finalize_unit(const FinIn<D>& a, SelHead& sh) {
    using C = SelCfg<D>;
    constexpr int W = C::W;
    const LayerView& L = a.L;
    const uint32_t u = a.u;
    const UnitDesc du = a.du;
    const uint32_t N = du.n_blocks, K = du.budget;
    const bool all = N <= K;
    const uint32_t nd = all ? N : N - 1;
    const bool trailing = !all;
    const bool big = !all && K > 1 && a.Cn > 1 && nd > kFinKeys;
    uint32_t* gkeys = a.sw.keys + du.seg;
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t G = L.G;
    const bool asym = L.mode == ABSP_QUANT_ASYM;
    const uint16_t* qrows = a.qrows;
    const float* scl = a.scl;
    const float* zps = a.zps;
    float* tbl = a.tbl;
    unsigned long long* cand = a.cand;
    uint32_t* list = a.list;
    uint32_t* cpg = a.cpg;
    uint32_t* blocks = a.blocks;
    uint32_t* counts = a.counts;
    uint32_t* ready = a.ready;
    const uint32_t stride = a.stride;
    const PageList& pages = a.pages;
    auto qsum = [&](uint32_t c) {
        float qg[8];
#pragma unroll
        for (int g = 0; g < 8; ++g) qg[g] = uint32_t(g) < G ? bf16f(qrows[g * D + c]) : 0.0f;
        float qc = qg[0];
#pragma unroll
        for (int g = 1; g < 8; ++g)
            if (uint32_t(g) < G) qc = __fadd_rn(qc, qg[g]);
        return qc;
    };
    // ================================ finalize ==================================
    // Kept compact on purpose: the finalize runs once per unit on cold instruction caches
    // (a step streams more than L2 holds), so its time follows the instruction bytes it
    // traverses. Loops stay rolled; the unit's keys arrive by one TMA bulk copy per
    // batch of kFinKeys.
    const uint32_t ppb = du.block / L.P;
    const uint32_t* pt = L.page_table + size_t(du.seq) * L.max_pages;
    const uint32_t head_base = du.head * uint32_t(L.pool_pages);
    uint32_t* skeys = a.skeys;
    const uint32_t kbar = smem_u32(&sh.bars[2 * kSStages + 1]);
    uint32_t kphase = 0;
    // keys [k0, min(k0 + kFinKeys, nd)) -> skeys[off ..]; every thread waits for them
    auto fetch_keys = [&](uint32_t k0) -> uint32_t {
        const uint32_t k1 = min(nd, k0 + kFinKeys);
        const uintptr_t a = reinterpret_cast<uintptr_t>(gkeys + k0);
        const uint32_t off = uint32_t(a & 15u) / 4;
        if (tid == 0) {
            asm volatile("fence.proxy.async.global;\n" ::: "memory");  // generic-proxy keys -> TMA reads
            const uint32_t bytes = ((k1 - k0 + off) * 4 + 15) & ~15u;
            mbar_expect_tx(kbar, bytes);
            bulk_g2s(smem_u32(skeys), reinterpret_cast<const void*>(a & ~uintptr_t(15)), bytes, kbar);
        }
        return off;
    };
    auto wait_keys = [&]() {
        mbar_wait(kbar, kphase & 1u);
        ++kphase;
    };
    uint32_t koff = fetch_keys(0);
    if (a.q_copy)  // q read from host memory: the attention gets the unit's rows in device memory
        for (uint32_t i = tid; i < G * D / 8; i += kSThreads)
            reinterpret_cast<uint4*>(a.q_copy + size_t(u) * G * D)[i] = reinterpret_cast<const uint4*>(qrows)[i];
    if (warp == kSWarps - 1) {  // the unit's key range: min / max over its slices
        uint32_t mn = 0xffffffffu, mx = 0u, bnd = 0xffffffffu;
        for (uint32_t i = lane; i < a.Cn; i += 32) {
            mn = min(mn, __ldcg(a.sw.slot + 4 * (a.first + i)));
            mx = max(mx, __ldcg(a.sw.slot + 4 * (a.first + i) + 1));
            if (big) bnd = min(bnd, __ldcg(a.sw.slot + 4 * (a.first + i) + 2));  // written by big units' slices
        }
        mn = __reduce_min_sync(0xffffffffu, mn);
        mx = __reduce_max_sync(0xffffffffu, mx);
        bnd = __reduce_min_sync(0xffffffffu, bnd);
        if (lane == 0) {
            sh.st[7] = mn;
            sh.st[8] = mx;
            sh.st[14] = bnd;
        }
    } else {  // exact product table: warp w < 8 builds 16 channels x 16 codes
        constexpr uint32_t CPT = 16 * D / 8 / 32;  // codes per lane
        const uint32_t c = warp * (D / 8) + (lane % (D / 8)), code0 = (lane / (D / 8)) * CPT;
        const float qc = qsum(c), sc = scl[c], zp = zps[c], fc0 = float(code0);
#pragma unroll 1
        for (uint32_t k = 0; k < CPT; ++k) {
            const float fc = fc0 + float(k);  // exact small integers
            const float deq = asym ? __fadd_rn(zp, __fmul_rn(fc, sc)) : __fmul_rn(fc - 7.0f, sc);
            tbl[c * 16 + code0 + k] = __fmul_rn(qc, deq);
        }
    }
    wait_keys();
    __syncthreads();  // key range, table, first keys
    SEL_TRACE(2);
    const uint32_t e_int = sh.st[0];
    const bool one_batch = nd <= kFinKeys;
    uint32_t thr = 0u;
    if (big) {
        const uint32_t T = sh.st[14];  // min over the slices' bounds: >= K-1 keys are >= T
        thr = (e_int == 0xffffffffu || T < 2ull * e_int) ? 0u : T - 2u * e_int;
    } else if (!all && K > 1) {
        // T = lower edge of the histogram bin holding the (K-1)-th largest key, refined once
        // inside that bin: at least K-1 keys are >= T (a lower bound of the (K-1)-th largest;
        // exact when the second-level bins are one key value wide)
        const uint32_t kmin = sh.st[7], span = sh.st[8] - kmin;
        const uint32_t shift = span < uint32_t(kBins) ? 0u : 32u - __clz(span) - 10u;
        uint32_t lo = kmin, sh1 = shift, kr = K - 1, bin0 = 0xffffffffu;
        for (int level = 0; level < 2; ++level) {
            // level 0: every key; level 1: the keys of bin0, sub-bins of width 2^sh1
            for (uint32_t b0 = 0; b0 < nd; b0 += kFinKeys) {
                if (b0 > 0) {
                    __syncthreads();
                    koff = fetch_keys(b0);
                    wait_keys();
                }
                const uint32_t nb = min(kFinKeys, nd - b0);
#pragma unroll 4
                for (uint32_t i = tid; i < nb; i += kSThreads) {
                    const uint32_t k = skeys[koff + i];
                    if (level == 0) atomicAdd(&sh.hist[(k - kmin) >> shift], 1u);
                    else if (((k - kmin) >> shift) == bin0) atomicAdd(&sh.hist[(k - lo) >> sh1], 1u);
                }
            }
            if (!one_batch) {
                __syncthreads();
                koff = fetch_keys(0);
                wait_keys();
            }
            __syncthreads();
            if (level == 0) SEL_TRACE(11);
            if (warp == 0) find_bin_desc(sh.hist, kr, lane, &sh.st[1], &sh.st[9]);
            __syncthreads();
            const uint32_t bb = sh.st[1], above = sh.st[9];
            lo += bb << sh1;
            // a bin of few keys costs fewer extra candidates than a second pass costs time
            if (level == 1 || sh1 == 0 || sh.hist[bb] <= kRefineMin) break;
            bin0 = bb;
            kr -= above;
            sh1 = sh1 > 10 ? sh1 - 10 : 0;
            for (uint32_t i = tid; i < uint32_t(kBins); i += kSThreads) sh.hist[i] = 0u;
            __syncthreads();
        }
        SEL_TRACE(13);
        thr = (e_int == 0xffffffffu || lo < 2ull * e_int) ? 0u : lo - 2u * e_int;
    }
    if (all || K > 1) {  // candidates {I_i >= thr}: per-thread counts, per-warp slots
        for (uint32_t b0 = 0; b0 < nd; b0 += kFinKeys) {
            if (b0 > 0) {
                __syncthreads();
                koff = fetch_keys(b0);
                wait_keys();
            }
            const uint32_t nb = min(kFinKeys, nd - b0);
            uint32_t cnt = 0;
#pragma unroll 4
            for (uint32_t i = tid; i < nb; i += kSThreads) cnt += skeys[koff + i] >= thr ? 1u : 0u;
            uint32_t incl = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= uint32_t(o)) incl += v;
            }
            uint32_t base = 0;
            if (lane == 31 && incl) base = atomicAdd(&sh.local_cnt, incl);
            uint32_t pos = __shfl_sync(0xffffffffu, base, 31) + incl - cnt;
            if (cnt) {
#pragma unroll 1
                for (uint32_t i = tid; i < nb; i += kSThreads) {
                    if (skeys[koff + i] >= thr) {
                        if (pos < a.plan.cand_cap) list[pos] = b0 + i;
                        ++pos;
                    }
                }
            }
        }
    }
    __syncthreads();  // candidate list complete
    SEL_TRACE(8);
    const uint32_t n = sh.local_cnt;
#ifdef ABSP_ATTN_TRACE
    if (tid == 0 && blockIdx.x < 4096) g_sel_trace[blockIdx.x * kSelTraceSlots + 14] = n;
#endif
    // exact scores of the candidates and of the trailing block (entry n), their pages
    // prefetched into shared memory for the emit below
    const uint32_t n_sc = n <= a.plan.cand_cap ? n + (trailing ? 1u : 0u) : (trailing ? 1u : 0u);
    const bool pg_pre = pages.page && n <= a.plan.cand_cap && (n + 1) * ppb <= a.plan.pg_cap;
    // Rows in batches of the dead key buffer (512 rows at d = 128): every candidate row of
    // a batch is requested at once (16-byte cp.async pieces, as stored: swizzled), so a
    // batch costs one L2 round trip whatever the candidates per thread
    constexpr uint32_t kRowBatch = kFinKeys * 4 / C::ROWB;
    unsigned char* rowbuf = reinterpret_cast<unsigned char*>(skeys);
    for (uint32_t j0 = 0; j0 < n_sc; j0 += kRowBatch) {
        const uint32_t jn = min(n_sc, j0 + kRowBatch);
        __syncthreads();  // the key batch (or the previous row batch) is dead
        for (uint32_t e = tid; e < (jn - j0) * (W / 4); e += kSThreads) {
            const uint32_t jj = j0 + e / (W / 4), g = e % (W / 4);
            const uint32_t i = (n > a.plan.cand_cap || jj == n) ? N - 1 : list[jj];
            cp_async16(smem_u32(rowbuf + (jj - j0) * C::ROWB + g * 16), L.codes + (du.seg + i) * W + g * 4);
        }
        cp_async_commit();
        cp_async_wait0();
        __syncthreads();
        for (uint32_t j = j0 + tid; j < jn; j += kSThreads) {
            const bool tr = n > a.plan.cand_cap || j == n;  // the trailing block
            const uint32_t i = tr ? N - 1 : list[j];
            const uint32_t slot = tr ? n : j;
            if (pg_pre || (tr && pages.page)) {
#pragma unroll 1
                for (uint32_t pp = 0; pp < ppb; ++pp) {
                    const uint32_t t0 = i * du.block + pp * L.P;
                    const uint32_t pg = t0 < du.n_tokens ? head_base + __ldg(pt + t0 / L.P) : 0u;
                    if (tr) sh.tpg[pp] = pg;
                    else cpg[slot * ppb + pp] = pg;
                }
            }
            uint32_t wd[W];
            const unsigned char* src = rowbuf + (j - j0) * C::ROWB;
            const uint32_t key = code_row_key(i, W);
#pragma unroll
            for (int g = 0; g < W / 4; ++g) {
                const uint4 v = *reinterpret_cast<const uint4*>(src + ((g ^ key) << 4));
                wd[4 * g] = v.x;
                wd[4 * g + 1] = v.y;
                wd[4 * g + 2] = v.z;
                wd[4 * g + 3] = v.w;
            }
            const float x = exact_row<W>(wd, tbl);
            const unsigned long long comp = (uint64_t(order_key(x)) << 32) | uint32_t(~i);
            if (tr) sh.ct = comp;
            else cand[slot] = comp;
        }
    }
    __syncthreads();
    SEL_TRACE(9);
    const unsigned long long ct = trailing ? sh.ct : 0ull;
    const uint32_t K1 = trailing ? K - 1 : n;
    if (trailing && (K > 1) && (n > a.plan.cand_cap || n < K1)) {  // mass ties: exact fallback
        exact_fallback<W>(L, du, sh, tbl, K, ct);
        publish_selection(L, du, u, sh.outs, K, blocks, stride, counts, pages, ready);
        SEL_TRACE(12);
        return;
    }
    // Order and publish in one pass: the rank of a candidate among the candidates is its
    // output position (composites are distinct); the trailing block goes after every
    // winner above it. The thread that ranks a winner writes its block id and its pages
    // straight into the attention producer's page list.
    const uint32_t n_sel = trailing ? K : n;
    const size_t pbase = pages.page ? size_t(pages.chunk_base[u]) * pages.ns : 0;
    const uint32_t E = kAttnChunkRows / du.block;  // entries per attention chunk (page_slot)
    // j: candidate index (pages in cpg), kNoPrefetch (page table), ~0u: the trailing block
    auto emit = [&](uint32_t p, uint32_t blk, uint32_t j) {
        blocks[size_t(u) * stride + p] = blk;
        if (!pages.page) return;
#pragma unroll 1
        for (uint32_t pp = 0; pp < ppb; ++pp) {
            const uint32_t t0 = blk * du.block + pp * L.P;
            uint32_t v = 0, page = 0;
            if (t0 < du.n_tokens) {
                v = min(L.P, du.n_tokens - t0);
                page = j == ~0u ? sh.tpg[pp] : (pg_pre && j != kNoPrefetch) ? cpg[j * ppb + pp]
                                                                            : head_base + __ldg(pt + t0 / L.P);
            }
            const uint32_t slot = page_slot(p, pp, E, ppb, pages.ns);
            pages.page[pbase + slot] = page;
            pages.valid[pbase + slot] = uint16_t(v);
        }
    };
    bool above = false;  // a winner ranked before the trailing block
    if (trailing && K == 1) {
        // the trailing block only
    } else if (n <= uint32_t(kSThreads)) {
        const uint32_t tpc = n <= 36 ? 8u : n <= 72 ? 4u : n <= 144 ? 2u : 1u;  // threads per candidate
        const uint32_t j = tid / tpc, part = tid % tpc;
        const bool valid = j < n;
        const unsigned long long me = valid ? cand[j] : 0ull;
        uint32_t rank = 0;
        if (valid) {
#pragma unroll 4
            for (uint32_t o = part; o < n; o += tpc) rank += cand[o] > me;
        }
        for (uint32_t off = 1; off < tpc; off <<= 1) rank += __shfl_xor_sync(0xffffffffu, rank, off);
        if (valid && part == 0 && rank < K1) {
            above = trailing && me > ct;
            emit(rank + (trailing && ct > me ? 1u : 0u), ~uint32_t(me), j);
        }
    } else if (n <= 2048u && reinterpret_cast<unsigned char*>(a.skeys) - reinterpret_cast<unsigned char*>(cand) >=
                                 (n <= 1024u ? 8192 : 16384)) {
        // large sets (large budgets): sort (the 1024 / 2048 padded composites may overwrite
        // the dead candidate list / pages), emit by position
        if (n <= 1024u) sortreg_desc<4>(cand, n);
        else sortreg_desc<8>(cand, n);
        SEL_TRACE(15);
        for (uint32_t p = tid; p < K1; p += kSThreads) {
            const unsigned long long me = cand[p];
            if (trailing && me > ct) atomicAdd(&sh.nsel, 1u);
            emit(p + (trailing && ct > me ? 1u : 0u), ~uint32_t(me), kNoPrefetch);
        }
    } else {  // every thread ranks several candidates
        for (uint32_t j = tid; j < n; j += kSThreads) {
            const unsigned long long me = cand[j];
            uint32_t r0 = 0, r1 = 0, r2 = 0, r3 = 0;
            uint32_t o = 0;
            for (; o + 4 <= n; o += 4) {
                r0 += cand[o] > me;
                r1 += cand[o + 1] > me;
                r2 += cand[o + 2] > me;
                r3 += cand[o + 3] > me;
            }
            for (; o < n; ++o) r0 += cand[o] > me;
            const uint32_t rank = (r0 + r1) + (r2 + r3);
            if (rank < K1) {
                if (trailing && me > ct) atomicAdd(&sh.nsel, 1u);
                emit(rank + (trailing && ct > me ? 1u : 0u), ~uint32_t(me), j);
            }
        }
    }
    SEL_TRACE(10);
    uint32_t n_above = __syncthreads_count(above);
    if (n > uint32_t(kSThreads)) n_above = sh.nsel;  // (set before the barrier above)
    if (trailing && tid == 0) emit(n_above, N - 1, ~0u);
    if (pages.page) {  // the entries left in the unit's last attention chunk: empty slots
        const uint32_t e_end = (n_sel + E - 1) / E * E;
        for (uint32_t s = tid; s < (e_end - n_sel) * ppb; s += kSThreads) {
            const uint32_t slot = page_slot(n_sel + s / ppb, s % ppb, E, ppb, pages.ns);
            pages.page[pbase + slot] = 0u;
            pages.valid[pbase + slot] = 0u;
        }
    }
    if (tid == 0) counts[u] = n_sel;
    __syncthreads();
    if (ready && tid == 0)  // release: cumulative over the CTA's writes ordered by the barrier
        asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(ready + size_t(u) * kReadyStride), "r"(1u) : "memory");
    SEL_TRACE(12);
}

// The unit's weight split and the filter's error bound, by one warp (lane owns channels
// lane + 32 j; every warp computing it gets the same values): w_c = fl(q_c s_c) ~
// (sigma / 256)(256 h_c + l_c) with h, l int8 written to hl[0][c], hl[1][c]; returns
// E_int = ceil(E 256 / sigma) + 2 (0xffffffff when every weight is zero) with
// E = 2^-14 M + 15 sum_c |w_c - w^_c| (1.01) (see the header of select.cu).
template <int D>
__device__ __forceinline__ uint32_t unit_weights(const uint16_t* qrows, const float* scl, const float* zps, uint32_t G,
                                                 bool asym, uint32_t lane, int8_t (*hl)[128], float* E_out,
                                                 float* sigma_out) {
    auto qsum = [&](uint32_t c) {  // q_c = left-to-right fp32 group sum (score.cu)
        float qg[8];
#pragma unroll
        for (int g = 0; g < 8; ++g) qg[g] = uint32_t(g) < G ? bf16f(qrows[g * D + c]) : 0.0f;
        float qc = qg[0];
#pragma unroll
        for (int g = 1; g < 8; ++g)
            if (uint32_t(g) < G) qc = __fadd_rn(qc, qg[g]);
        return qc;
    };
    constexpr int CPL = D / 32;
    float wv[CPL];
    float wmax = 0.0f, M = 0.0f;
#pragma unroll
    for (int j = 0; j < CPL; ++j) {
        const uint32_t c = lane + 32 * j;
        const float qc = qsum(c), sc = scl[c], zp = zps[c];
        wv[j] = __fmul_rn(qc, sc);
        wmax = fmaxf(wmax, fabsf(wv[j]));
        // max_code |p_c(code)|: every rounding step is monotone in the code, so the
        // magnitude of the exact product peaks at code 0 or code 15
        const float d0 = asym ? zp : __fmul_rn(-7.0f, sc);
        const float d15 = asym ? __fadd_rn(zp, __fmul_rn(15.0f, sc)) : __fmul_rn(8.0f, sc);
        M += fmaxf(fabsf(__fmul_rn(qc, d0)), fabsf(__fmul_rn(qc, d15)));
    }
    wmax = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(wmax)));
    const float sigma = wmax / 127.0f, inv = wmax > 0.0f ? 127.0f / wmax : 0.0f;
    float resid = 0.0f;
#pragma unroll
    for (int j = 0; j < CPL; ++j) {
        const uint32_t c = lane + 32 * j;
        int h = 0, l = 0;
        if (sigma > 0.0f) {  // any h, l are valid: the bound uses the actual residual
            h = __float2int_rn(wv[j] * inv);
            h = h > 127 ? 127 : (h < -127 ? -127 : h);
            l = __float2int_rn((wv[j] - float(h) * sigma) * 256.0f * inv);
            l = l > 127 ? 127 : (l < -127 ? -127 : l);
        }
        hl[0][c] = int8_t(h);
        hl[1][c] = int8_t(l);
        resid += fabsf(wv[j] - sigma * (float(h) + float(l) * 0.00390625f)) + fabsf(wv[j]) * 0x1p-23f;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        resid += __shfl_xor_sync(0xffffffffu, resid, off);
        M += __shfl_xor_sync(0xffffffffu, M, off);
    }
    const float E = M * 0x1p-14f + 15.0f * resid * 1.01f;
    *E_out = E;
    *sigma_out = sigma;
    return sigma > 0.0f ? uint32_t(fminf(ceilf(E * 256.0f * inv), 1.0e9f)) + 2u : 0xffffffffu;
}

}  // namespace
}  // namespace selcore
}  // namespace absp

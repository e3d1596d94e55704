// Fused decode-step selection (sm_100a): estimate_scores + select_topk +
// populate_page_spans (engine.cpp:34-97, 119-178, 271-283) for INT4 mean stores in
// ONE kernel, one thread-block cluster of C CTAs per (sequence, KV head) unit, with
// the same ordered block lists the reference computes (bit-exact), but without the
// serial fp32 score of every centroid.
//
//   stream  : the producer warp bulk-copies (TMA) the CTA's slice of the unit's packed
//             code rows into a 4-stage ring, plus q and the unit's scale / zero point.
//   filter  : consumers compute, per centroid, the exact integer
//                 I_i = sum_c (256 h_c + l_c) code_ic   (codes 0..15, integer tensor cores:
//                 mma.sync m16n8k32 u8 x s8 -> s32 on code words fed by ldmatrix, even
//                 nibbles as bytes and odd nibbles x16 against separate B columns)
//             with w_c = fl(q_c s_c) ~ (sigma / 256)(256 h_c + l_c), h, l int8, so
//             A_i = (sigma / 256) I_i is the score up to the constant C = sum_c q_c zp_c
//             and a proven per-unit error bound
//                 |S_i - C - A_i| <= E = 2^-14 M + 15 sum_c |w_c - w^_c| (1.01)
//             (S_i the reference's serial fp32 score; M = sum_c max_code |p_c(code)|
//             bounds the products; the serial sum of 128 rounded products is within
//             ~131u M of the real sum, so 2^-14 keeps an 8x margin; the second term is
//             the weight quantisation exactly, codes <= 15). In integer units
//             E_int = ceil(E 256 / sigma) + 2.
//   bound   : every CTA finds a lower bound t_r of the ceil((K-1)/C)-th largest of its
//             slice's I (a 1024-bin histogram); T = min_r t_r (DSMEM exchange) is a lower
//             bound of the (K-1)-th largest I of the unit. Any block of the exact
//             top-(K-1) has I >= T - 2 E_int (else K-1 blocks score strictly higher), so
//             the candidates {I_i >= T - 2 E_int} (typically K-1 plus a few) contain it.
//   refine  : each CTA scores its candidates with the reference's exact serial fp32
//             arithmetic (product table, score.cu) and sends (key << 32 | ~index)
//             composites to the leader CTA's shared memory (DSMEM); the leader orders
//             them, keeps the top K-1, inserts the trailing block N-1 (forced, exactly
//             where its exact score ranks), and publishes blocks, counts, the page list
//             and the unit's ready flag for the attention producer (common.cuh).
//   fallback: more candidates than fit (mass ties) -> the leader scores every block
//             exactly into the scores buffer and runs an exact radix select (slow, rare,
//             identical result).
#include "absp_internal.cuh"
#include "common.cuh"
#include "ptx.cuh"

#include <math.h>

#include <algorithm>

namespace absp {
namespace {

constexpr int kSCons = 256;              // consumer threads (8 warps), one code row each per stage
constexpr int kSThreads = kSCons + 32;   // + producer warp
constexpr int kSWarps = kSThreads / 32;
constexpr int kSRows = kSCons;           // rows per stage
constexpr int kSStages = 4;
constexpr uint32_t kCandCapMax = 2048;   // candidate capacity bound (>= K, K <= T / min B <= 2048)
constexpr int kBins = 1024;

// Optional timeline instrumentation (debug builds with -DABSP_ATTN_TRACE): per CTA,
// globaltimer stamps at the phase boundaries (tools/select_trace.py).
#ifdef ABSP_ATTN_TRACE
constexpr int kSelTraceSlots = 16;
__device__ unsigned long long g_sel_trace[2048 * kSelTraceSlots];
#define SEL_TRACE(slot)                                                                           \
    do {                                                                                          \
        if (threadIdx.x == 0 && blockIdx.x < 2048) {                                              \
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

// Fixed-size part of the shared memory; the candidate arrays follow it:
//   cand [cand_cap] u64 (leader: composites), list / outs [cand_cap] u32 (this CTA's
//   candidate indices, then the leader's ordered selection).
struct SelHead {
    unsigned long long bars[2 * kSStages + 1];  // full[NS], empty[NS], params
    int8_t hlw[kSCons / 32][2][128];     // per consumer warp: h and l per channel (D <= 128)
    uint32_t tpg[kAttnChunkRows];        // leader: the trailing block's pool pages (prefetched)
    uint32_t tvl[kAttnChunkRows];        //         and their valid rows
    float red[4][kSWarps];       // block reductions
    uint32_t slot[8];            // per-rank local bounds t_r (written by every CTA of the cluster)
    uint32_t st[16];             // misc scalars
    uint32_t hist[kBins];
    uint32_t local_cnt;
    uint32_t cand_cnt;           // leader: composites received
    uint32_t overflow;           // leader: some CTA could not deliver all its candidates
    uint32_t nsel;
    unsigned long long* cand;
    uint32_t* list;
    uint32_t* outs;
    uint32_t cap;
};

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cluster_size() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;\n" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cluster_arrive() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// Address of `p` (this CTA's shared memory) in CTA `rank` of the cluster.
__device__ __forceinline__ uint32_t dsmem(const void* p, uint32_t rank) {
    uint32_t a;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(a) : "r"(smem_u32(p)), "r"(rank));
    return a;
}
__device__ __forceinline__ void st_cluster_u32(uint32_t addr, uint32_t v) {
    asm volatile("st.shared::cluster.u32 [%0], %1;\n" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void st_cluster_u64(uint32_t addr, unsigned long long v) {
    asm volatile("st.shared::cluster.u64 [%0], %1;\n" ::"r"(addr), "l"(v) : "memory");
}
__device__ __forceinline__ uint32_t atom_add_cluster(uint32_t addr, uint32_t v) {
    uint32_t old;
    asm volatile("atom.shared::cluster.add.u32 %0, [%1], %2;\n" : "=r"(old) : "r"(addr), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ void red_or_cluster(uint32_t addr, uint32_t v) {
    asm volatile("red.shared::cluster.or.b32 [%0], %1;\n" ::"r"(addr), "r"(v) : "memory");
}
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

// Shared-memory layout (host and device): ring [stages][rows][row bytes] | keys
// [slice_cap] | product table | q rows | scales, zps | SelHead | cand | list/outs.
template <int D>
struct SelLayout {
    size_t keys, tbl, prm, head, cand, list, total;
    __host__ __device__ SelLayout(uint32_t stages, uint32_t slice_cap, uint32_t cand_cap) {
        keys = size_t(stages) * SelCfg<D>::STAGEB;
        tbl = keys + ((size_t(slice_cap) * 4 + 15) & ~size_t(15));
        prm = tbl + SelCfg<D>::TBL;
        head = prm + SelCfg<D>::QB + SelCfg<D>::PB;
        cand = (head + sizeof(SelHead) + 15) & ~size_t(15);
        list = cand + size_t(cand_cap) * 8;
        total = list + size_t(cand_cap) * 4;
    }
};

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

template <int D>
__global__ void __launch_bounds__(kSThreads, 2) k_select(LayerView L, const uint16_t* __restrict__ q, uint32_t stages,
                                                       uint32_t slice_cap, uint32_t cand_cap, uint32_t* blocks,
                                                       uint32_t stride, uint32_t* counts, PageList pages,
                                                       uint32_t* ready, float* diag_approx, float* diag_err) {
    using C = SelCfg<D>;
    constexpr int W = C::W, NG = D / 32;  // code words per row, 16-byte groups (32 channels) per row
    extern __shared__ __align__(1024) unsigned char smem[];
    const SelLayout<D> lay(stages, slice_cap, cand_cap);
    unsigned char* ring = smem;
    uint32_t* keys = reinterpret_cast<uint32_t*>(smem + lay.keys);  // [slice_cap]
    float* tbl = reinterpret_cast<float*>(smem + lay.tbl);          // [D][16]
    unsigned char* prm_raw = smem + lay.prm;                         // q rows | scales | zps
    SelHead& sh = *reinterpret_cast<SelHead*>(smem + lay.head);
    const uint16_t* qrows = reinterpret_cast<const uint16_t*>(prm_raw);
    const float* scl = reinterpret_cast<const float*>(prm_raw + C::QB);
    const float* zps = scl + D;
    unsigned long long* cand = reinterpret_cast<unsigned long long*>(smem + lay.cand);
    uint32_t* list = reinterpret_cast<uint32_t*>(smem + lay.list);

    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t Cn = cluster_size(), r = cluster_rank();
    const uint32_t u = blockIdx.x / Cn;
    const UnitDesc du = L.desc[u];
    const uint32_t N = du.n_blocks, K = du.budget;
    const bool all = N <= K;               // every block selected (ordered)
    const uint32_t nd = all ? N : N - 1;   // candidate domain [0, nd)
    const uint32_t s0 = uint32_t((uint64_t(r) * nd) / Cn), s1 = uint32_t((uint64_t(r + 1) * nd) / Cn);
    const uint32_t ns = s1 - s0;
    const uint32_t n_chunks = (ns + kSRows - 1) / kSRows;
    const bool resident = n_chunks <= stages;  // the whole slice stays in the ring
    const bool trailing = !all;                // block N-1 is forced in (scored by the leader)

    SEL_TRACE(0);
    if (tid == 0) {
        sh.cand = cand;
        sh.list = list;
        sh.outs = list;  // the candidate list is dead once the composites are in
        sh.cap = cand_cap;
        for (int i = 0; i < kSStages; ++i) {
            mbar_init(smem_u32(&sh.bars[i]), 1);
            mbar_init(smem_u32(&sh.bars[kSStages + i]), kSCons / 32);
        }
        mbar_init(smem_u32(&sh.bars[2 * kSStages]), 1);
        mbar_fence_init();
        sh.local_cnt = 0u;
        sh.cand_cnt = 0u;
        sh.overflow = 0u;
        sh.nsel = 0u;
        sh.st[1] = 0u;
    }
    for (uint32_t i = tid; i < uint32_t(kBins); i += kSThreads) sh.hist[i] = 0u;
    {   // the page resolution at the end reads the sequence's page-table row: warm L2
        const uint32_t row_pages = (du.n_tokens + L.P - 1) / L.P;
        const uint32_t* pt = L.page_table + size_t(du.seq) * L.max_pages;
        const uint32_t a = uint32_t((uint64_t(r) * row_pages) / Cn), b = uint32_t((uint64_t(r + 1) * row_pages) / Cn);
        for (uint32_t p = a + tid * 32; p < b; p += kSThreads * 32) asm volatile("prefetch.global.L2 [%0];" ::"l"(pt + p));
    }
    __syncthreads();
    griddep_wait();  // codes / params (appends) and q are written by earlier kernels
    // The attention kernel may be scheduled now: every CTA of this grid is past its wait,
    // i.e. the previous step's attention has completed (its merges re-armed the ready flags).
    griddep_launch_dependents();
    // the leader's last thread fetches the trailing block's code row now; it is scored
    // exactly once the product table exists (after barrier #1)
    uint32_t trail[W];
    if (r == 0 && trailing && tid == kSThreads - 1) load_row_global<W>(L.codes, du.seg + N - 1, N - 1, trail);
    if (r == 0 && trailing && warp == kSWarps - 1 && pages.page) {  // and its pages
        const uint32_t ppb = du.block / L.P;
        const uint32_t* pt = L.page_table + size_t(du.seq) * L.max_pages;
        for (uint32_t pp = lane; pp < ppb; pp += 32) {
            const uint32_t t0 = (N - 1) * du.block + pp * L.P;
            sh.tvl[pp] = t0 < du.n_tokens ? min(L.P, du.n_tokens - t0) : 0u;
            sh.tpg[pp] = t0 < du.n_tokens ? du.head * uint32_t(L.pool_pages) + __ldg(pt + t0 / L.P) : 0u;
        }
    }
    SEL_TRACE(1);
    // this CTA's shared memory is initialised: no CTA of the cluster touches another's
    // before the matching wait (just before the first DSMEM access, after the filter)
    cluster_arrive();
    SEL_TRACE(2);

    if (warp == kSWarps - 1) {
        // =============================== producer ===============================
        if (lane == 0) {
            const uint32_t pbar = smem_u32(&sh.bars[2 * kSStages]);
            mbar_expect_tx(pbar, L.G * D * 2 + C::PB);
            bulk_g2s(smem_u32(prm_raw), q + size_t(u) * L.G * D, L.G * D * 2, pbar);  // units are b-major
            bulk_g2s(smem_u32(prm_raw + C::QB), L.scales + size_t(u) * D, D * 4, pbar);
            bulk_g2s(smem_u32(prm_raw + C::QB + D * 4), L.zps + size_t(u) * D, D * 4, pbar);
            for (uint32_t c = 0; c < n_chunks; ++c) {
                const uint32_t stg = c % stages;
                if (c >= stages) mbar_wait(smem_u32(&sh.bars[kSStages + stg]), ((c / stages) - 1) & 1);
                const uint32_t rows = min(uint32_t(kSRows), ns - c * kSRows);
                const uint32_t bar = smem_u32(&sh.bars[stg]);
                mbar_expect_tx(bar, rows * C::ROWB);
                bulk_g2s(smem_u32(ring + size_t(stg) * C::STAGEB), L.codes + (du.seg + s0 + c * kSRows) * W,
                         rows * C::ROWB, bar);
            }
        }
        __syncwarp();
    } else {
        // =============================== consumers ==============================
        mbar_wait(smem_u32(&sh.bars[2 * kSStages]), 0);
        SEL_TRACE(3);
        const bool asym = L.mode == ABSP_QUANT_ASYM;
        // Every warp derives the weights itself (identical arithmetic, no CTA barrier):
        // lane owns channels lane + 32 j. q_c = left-to-right fp32 group sum (score.cu).
        constexpr int CPL = D / 32;
        const uint32_t G = L.G;
        auto qsum = [&](uint32_t c) {
            float qg[8];
#pragma unroll
            for (int g = 0; g < 8; ++g) qg[g] = uint32_t(g) < G ? bf16f(qrows[g * D + c]) : 0.0f;  // independent loads
            float qc = qg[0];
#pragma unroll
            for (int g = 1; g < 8; ++g)
                if (uint32_t(g) < G) qc = __fadd_rn(qc, qg[g]);
            return qc;
        };
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
        auto& hlw = sh.hlw;  // this warp's h and l per channel
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
            hlw[warp][0][c] = int8_t(h);
            hlw[warp][1][c] = int8_t(l);
            resid += fabsf(wv[j] - sigma * (float(h) + float(l) * 0.00390625f)) + fabsf(wv[j]) * 0x1p-23f;
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            resid += __shfl_xor_sync(0xffffffffu, resid, off);
            M += __shfl_xor_sync(0xffffffffu, M, off);
        }
        const float E = M * 0x1p-14f + 15.0f * resid * 1.01f;
        const uint32_t e_int = sigma > 0.0f ? uint32_t(fminf(ceilf(E * 256.0f * inv), 1.0e9f)) + 2u : 0xffffffffu;
        if (tid == 0) {
            sh.st[0] = e_int;
            if (diag_err && r == 0) diag_err[u] = E;
        }
        __syncwarp();
        // B fragments (column n = lane / 4 of the m16n8k32 tile), group G, word j = 4G + t4:
        //   col 0: h of the even channels 8j + 0,2,4,6   col 1: l of them
        //   col 2: h of the odd channels (their codes arrive x16, so col 2 sums 16 x h . code)
        //   col 3: l of the odd channels                  cols 4-7: zero
        const uint32_t gq = lane >> 2, t4 = lane & 3;
        uint32_t bfr[NG][2];
#pragma unroll
        for (int G = 0; G < NG; ++G) {
            const uint32_t j = 4 * G + t4;
            uint32_t v = 0;
            if (gq < 4) {
                const int8_t* src = hlw[warp][gq & 1];
                const uint32_t odd = gq >> 1;
#pragma unroll
                for (int bb = 0; bb < 4; ++bb) v |= uint32_t(uint8_t(src[8 * j + 2 * bb + odd])) << (8 * bb);
            }
            bfr[G][0] = gq < 2 ? v : 0u;
            bfr[G][1] = (gq >= 2 && gq < 4) ? v : 0u;
        }
        // exact product table (for the refine): this warp's 16 channels x 16 codes
        {
            constexpr uint32_t CPT = 16 * D / 8 / 32;  // codes per lane
            const uint32_t c = warp * (D / 8) + (lane % (D / 8)), code0 = (lane / (D / 8)) * CPT;
            const float qc = qsum(c), sc = scl[c], zp = zps[c], fc0 = float(code0);
#pragma unroll
            for (uint32_t k = 0; k < CPT; ++k) {
                const float fc = fc0 + float(k);  // exact small integers
                const float deq = asym ? __fadd_rn(zp, __fmul_rn(fc, sc)) : __fmul_rn(fc - 7.0f, sc);
                tbl[c * 16 + code0 + k] = __fmul_rn(qc, deq);
            }
        }
        SEL_TRACE(4);

        // ---- filter: exact integer scores I_i of the slice on the tensor cores ----
        uint32_t kmin = 0xffffffffu, kmax = 0u;
        const float a_scale = sigma * 0.00390625f;
        for (uint32_t c = 0; c < n_chunks; ++c) {
            const uint32_t stg = c % stages;
            mbar_wait(smem_u32(&sh.bars[stg]), (c / stages) & 1);
            const uint32_t sbase = smem_u32(ring + size_t(stg) * C::STAGEB);
            for (uint32_t tile = warp; tile < uint32_t(kSRows / 16); tile += kSCons / 32) {
                const uint32_t row0 = c * kSRows + tile * 16;  // slice-relative
                if (row0 >= ns) break;
                int acc[4] = {0, 0, 0, 0};
                // ldmatrix.x4: lanes 8m.. address matrix m: rows (m & 1) * 8 + 0..7, group 2gp + (m >> 1)
                const uint32_t mi = lane >> 3, rr = (lane & 7) + (mi & 1) * 8;
                const uint32_t rkey = code_row_key(s0 + row0 + rr, W);
                const uint32_t raddr = sbase + (tile * 16 + rr) * C::ROWB;
#pragma unroll
                for (int gp = 0; gp < NG / 2; ++gp) {
                    const uint32_t grp = 2 * gp + (mi >> 1);
                    uint32_t x0, x1, x2, x3;  // rows g / g+8 of groups 2gp / 2gp+1, word t4
                    ldsm_x4(raddr + ((grp ^ rkey) << 4), x0, x1, x2, x3);
                    constexpr uint32_t LO = 0x0F0F0F0Fu, HI = 0xF0F0F0F0u;
                    imma(acc, x0 & LO, x1 & LO, x0 & HI, x1 & HI, bfr[2 * gp][0], bfr[2 * gp][1]);
                    imma(acc, x2 & LO, x3 & LO, x2 & HI, x3 & HI, bfr[2 * gp + 1][0], bfr[2 * gp + 1][1]);
                }
                // t4 = 0 holds (even h, even l), t4 = 1 (16 x odd h, 16 x odd l), rows g and g+8
                const int o0 = __shfl_down_sync(0xffffffffu, acc[0], 1), o1 = __shfl_down_sync(0xffffffffu, acc[1], 1);
                const int o2 = __shfl_down_sync(0xffffffffu, acc[2], 1), o3 = __shfl_down_sync(0xffffffffu, acc[3], 1);
                if (t4 == 0) {
                    const int I0 = (acc[0] + (o0 >> 4)) * 256 + acc[1] + (o1 >> 4);
                    const int I1 = (acc[2] + (o2 >> 4)) * 256 + acc[3] + (o3 >> 4);
                    const uint32_t ra = row0 + gq, rb = ra + 8;
                    if (ra < ns) {
                        const uint32_t k = uint32_t(I0) ^ 0x80000000u;
                        keys[ra] = k;
                        kmin = min(kmin, k);
                        kmax = max(kmax, k);
                        if (diag_approx) diag_approx[du.seg + s0 + ra] = float(I0) * a_scale;
                    }
                    if (rb < ns) {
                        const uint32_t k = uint32_t(I1) ^ 0x80000000u;
                        keys[rb] = k;
                        kmin = min(kmin, k);
                        kmax = max(kmax, k);
                        if (diag_approx) diag_approx[du.seg + s0 + rb] = float(I1) * a_scale;
                    }
                }
            }
            if (!resident) {
                __syncwarp();
                if (lane == 0) mbar_arrive(smem_u32(&sh.bars[kSStages + stg]));
            }
        }
        SEL_TRACE(5);
        // ---- local lower bound t_r of the k_r-th largest: 1024 bins of the key range ----
        uint32_t t_r = 0u;
        const uint32_t kr = (K - 1 + Cn - 1) / Cn;
        if (!all && K > 1 && ns >= kr) {
            kmin = __reduce_min_sync(0xffffffffu, kmin);
            kmax = __reduce_max_sync(0xffffffffu, kmax);
            if (lane == 0) {
                sh.red[0][warp] = __uint_as_float(kmin);
                sh.red[1][warp] = __uint_as_float(kmax);
            }
            cons_sync();
            kmin = 0xffffffffu;
            kmax = 0u;
#pragma unroll
            for (int i = 0; i < kSCons / 32; ++i) {
                kmin = min(kmin, __float_as_uint(sh.red[0][i]));
                kmax = max(kmax, __float_as_uint(sh.red[1][i]));
            }
            const uint32_t span = kmax - kmin;  // bins: (key - kmin) >> shift < 1024
            const uint32_t shift = span < uint32_t(kBins) ? 0u : 32u - __clz(span) - 10u;
            for (uint32_t i = tid; i < ns; i += kSCons) atomicAdd(&sh.hist[(keys[i] - kmin) >> shift], 1u);
            cons_sync();
            if (warp == 0) {  // bin holding the kr-th largest, counted from the top
                constexpr int PER = kBins / 32;
                uint32_t tot = 0;
#pragma unroll 8
                for (int j = 0; j < PER; ++j) tot += sh.hist[kBins - 1 - (lane * PER + j)];
                uint32_t incl = tot;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= uint32_t(o)) incl += v;
                }
                uint32_t cum = incl - tot;
                if (cum < kr && kr <= incl) {
                    for (int j = 0; j < PER; ++j) {
                        const uint32_t b = kBins - 1 - (lane * PER + j);
                        cum += sh.hist[b];
                        if (cum >= kr) {  // every key of bin b and above is >= its lower edge
                            sh.st[1] = kmin + (b << shift);
                            break;
                        }
                    }
                }
            }
            cons_sync();
            t_r = sh.st[1];
        }
        SEL_TRACE(6);
        if (tid == 0) sh.st[5] = t_r;
    }
    __syncthreads();
    cluster_wait();  // every CTA of the cluster is initialised (phase 0)
    if (tid < Cn) st_cluster_u32(dsmem(&sh.slot[r], tid), sh.st[5]);  // every CTA gets every t_r
    cluster_sync();  // #1: slices scored, bounds exchanged, product table complete
    SEL_TRACE(7);

    // ---- candidates of this slice, exact scores, composites to the leader ----
    if (r == 0 && trailing && tid == kSThreads - 1) sh.st[3] = order_key(exact_row<W>(trail, tbl));
    const uint32_t e_int = sh.st[0];
    uint32_t thr = 0u;
    if (!all && K > 1) {
        uint32_t T = 0xffffffffu;
        for (uint32_t i = 0; i < Cn; ++i) T = min(T, sh.slot[i]);
        thr = (e_int == 0xffffffffu || T < 2ull * e_int) ? 0u : T - 2u * e_int;
    }
    if (warp < kSCons / 32 && (all || K > 1)) {
        for (uint32_t b0 = warp * 32; b0 < ns; b0 += kSCons) {  // warp-uniform trip count
            const uint32_t i = b0 + lane;
            const bool cnd = i < ns && keys[i] >= thr;
            const uint32_t m = __ballot_sync(0xffffffffu, cnd);
            uint32_t base = 0;
            if (lane == 0 && m) base = atomicAdd(&sh.local_cnt, __popc(m));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (cnd) {
                const uint32_t p = base + __popc(m & ((1u << lane) - 1u));
                if (p < cand_cap) list[p] = i;
            }
        }
    }
    __syncthreads();
    const uint32_t nl = sh.local_cnt;
    const uint32_t leader_cnt = dsmem(&sh.cand_cnt, 0), leader_of = dsmem(&sh.overflow, 0);
    if (nl > cand_cap) {
        if (tid == 0) red_or_cluster(leader_of, 1u);
    } else if (nl > 0) {
        if (tid == 0) sh.st[2] = atom_add_cluster(leader_cnt, nl);
        __syncthreads();
        const uint32_t pos0 = sh.st[2];
        if (pos0 + nl > cand_cap) {
            if (tid == 0) red_or_cluster(leader_of, 1u);
        } else {
            for (uint32_t j = tid; j < nl; j += kSThreads) {
                const uint32_t i = list[j];
                uint32_t wd[W];
                if (resident) {
                    const unsigned char* src = ring + size_t(i / kSRows) * C::STAGEB + (i % kSRows) * C::ROWB;
                    const uint32_t key = code_row_key(s0 + i, W);
#pragma unroll
                    for (int g = 0; g < W / 4; ++g) {
                        const uint4 v = *reinterpret_cast<const uint4*>(src + ((g ^ key) << 4));
                        wd[4 * g] = v.x;
                        wd[4 * g + 1] = v.y;
                        wd[4 * g + 2] = v.z;
                        wd[4 * g + 3] = v.w;
                    }
                } else {
                    load_row_global<W>(L.codes, du.seg + s0 + i, s0 + i, wd);
                }
                const float x = exact_row<W>(wd, tbl);
                const unsigned long long comp = (uint64_t(order_key(x)) << 32) | uint32_t(~(s0 + i));
                st_cluster_u64(dsmem(&cand[pos0 + j], 0), comp);
            }
        }
    }
    SEL_TRACE(8);
    cluster_sync();  // #2: every composite has landed in the leader
    SEL_TRACE(9);
    if (r != 0) return;

    // ================================ leader ===================================
    const unsigned long long ct = trailing ? (uint64_t(sh.st[3]) << 32) | uint32_t(~(N - 1)) : 0ull;
    const uint32_t n = sh.cand_cnt;
    const uint32_t K1 = trailing ? K - 1 : n;
    SEL_TRACE(10);
    if (trailing && (K > 1) && (sh.overflow || n < K1)) {  // mass ties: exact fallback
        exact_fallback<W>(L, du, sh, tbl, K, ct);
        publish_selection(L, du, u, sh.outs, K, blocks, stride, counts, pages, ready);
        SEL_TRACE(12);
        return;
    }
    // Order and publish in one pass: the rank of a candidate among the candidates is its
    // output position (composites are distinct); the trailing block goes after every
    // winner above it. The thread that ranks a winner writes its block id and resolves
    // its pages straight into the attention producer's page list.
    const uint32_t n_sel = trailing ? K : n;
    const uint32_t ppb = du.block / L.P;
    const uint32_t* pt = L.page_table + size_t(du.seq) * L.max_pages;
    const uint32_t head_base = du.head * uint32_t(L.pool_pages);
    const size_t pbase = pages.page ? size_t(pages.chunk_base[u]) * pages.ns : 0;
    auto emit = [&](uint32_t p, uint32_t blk) {
        blocks[size_t(u) * stride + p] = blk;
        if (!pages.page) return;
        if (trailing && blk == N - 1) {  // resolved at the start
            for (uint32_t pp = 0; pp < ppb; ++pp) {
                pages.page[pbase + size_t(p) * ppb + pp] = sh.tpg[pp];
                pages.valid[pbase + size_t(p) * ppb + pp] = uint16_t(sh.tvl[pp]);
            }
            return;
        }
        for (uint32_t pp = 0; pp < ppb; ++pp) {
            const uint32_t t0 = blk * du.block + pp * L.P;
            uint32_t v = 0, page = 0;
            if (t0 < du.n_tokens) {
                v = min(L.P, du.n_tokens - t0);
                page = head_base + __ldg(pt + t0 / L.P);
            }
            pages.page[pbase + size_t(p) * ppb + pp] = page;
            pages.valid[pbase + size_t(p) * ppb + pp] = uint16_t(v);
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
            emit(rank + (trailing && ct > me ? 1u : 0u), ~uint32_t(me));
        }
    } else {  // large candidate sets (large budgets): sort, then emit by position
        sort_desc(cand, n);
        for (uint32_t p = tid; p < K1; p += kSThreads) {
            const unsigned long long me = cand[p];
            if (trailing && me > ct) atomicAdd(&sh.nsel, 1u);
            emit(p + (trailing && ct > me ? 1u : 0u), ~uint32_t(me));
        }
    }
    SEL_TRACE(11);
    uint32_t n_above = __syncthreads_count(above);
    if (n > uint32_t(kSThreads)) n_above = sh.nsel;  // (set before the barrier above)
    if (trailing && tid == 0) emit(n_above, N - 1);
    if (pages.page) {  // the rest of the unit's last attention chunk: empty slots
        const uint32_t E = kAttnChunkRows / du.block;
        const uint32_t slot_end = ((n_sel + E - 1) / E * E) * ppb;
        for (uint32_t s = n_sel * ppb + tid; s < slot_end; s += kSThreads) {
            pages.page[pbase + s] = 0u;
            pages.valid[pbase + s] = 0u;
        }
    }
    if (tid == 0) counts[u] = n_sel;
    __syncthreads();
    if (ready && tid == 0)  // release: cumulative over the CTA's writes ordered by the barrier
        asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(ready + u), "r"(1u) : "memory");
    SEL_TRACE(12);
}

}  // namespace

#ifdef ABSP_ATTN_TRACE
cudaError_t debug_select_trace(void* dst, size_t bytes) { return cudaMemcpyFromSymbol(dst, g_sel_trace, bytes); }
#endif

bool select_fused_supported(const LayerView& L) {
    return L.bits == 4 && L.method == ABSP_CENTROID_MEAN && (L.D == 64 || L.D == 128) && L.G <= 8;
}

// Cluster size and shared-memory plan of a layer: enough CTAs per unit to cover the SMs
// (cfg3 on 1 GPU: 128 units x 2; its 8-GPU shard: 16 units x 8), the key slice for the
// largest unit at capacity, 4 ring stages when they fit (2 CTAs per SM if possible).
SelectPlan plan_select(uint32_t units, uint32_t max_cap_blocks, uint32_t max_budget, uint32_t D, int num_sms) {
    SelectPlan p{};
    p.cluster = 1;
    while (p.cluster < 8 && units * p.cluster < uint32_t(num_sms)) p.cluster <<= 1;
    p.cand_cap = 512;  // a power of two (bitonic sort in place), >= K
    while (p.cand_cap < kCandCapMax && p.cand_cap < 4 * max_budget) p.cand_cap <<= 1;
    p.slice_cap = (max_cap_blocks + p.cluster - 1) / p.cluster + 1;
    for (p.stages = kSStages; p.stages > 2; --p.stages)
        if (select_fused_smem(D, p.stages, p.slice_cap, p.cand_cap) <= 227 * 1024) break;
    p.ok = select_fused_smem(D, p.stages, p.slice_cap, p.cand_cap) <= 227 * 1024;
    return p;
}

size_t select_fused_smem(uint32_t D, uint32_t stages, uint32_t slice_cap, uint32_t cand_cap) {
    return D == 64 ? SelLayout<64>(stages, slice_cap, cand_cap).total : SelLayout<128>(stages, slice_cap, cand_cap).total;
}

cudaError_t init_select_attributes() {
    cudaError_t e = cudaFuncSetAttribute(k_select<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_select<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_select<64>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(k_select<128>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
}

cudaError_t launch_select_fused(const LayerView& L, const uint16_t* q, const SelectPlan& plan, uint32_t* blocks,
                                uint32_t stride, uint32_t* counts, const PageList& pages, uint32_t* ready,
                                float* diag_approx, float* diag_err, cudaStream_t s, int* launches) {
    const uint32_t cluster = plan.cluster;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(L.units * cluster);
    cfg.blockDim = dim3(kSThreads);
    cfg.dynamicSmemBytes = select_fused_smem(L.D, plan.stages, plan.slice_cap, plan.cand_cap);
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = cluster;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    cudaError_t e;
    if (L.D == 64)
        e = cudaLaunchKernelEx(&cfg, k_select<64>, L, q, plan.stages, plan.slice_cap, plan.cand_cap, blocks, stride,
                               counts, pages, ready, diag_approx, diag_err);
    else
        e = cudaLaunchKernelEx(&cfg, k_select<128>, L, q, plan.stages, plan.slice_cap, plan.cand_cap, blocks, stride,
                               counts, pages, ready, diag_approx, diag_err);
    ++*launches;
    return e == cudaSuccess ? cudaGetLastError() : e;
}

}  // namespace absp

// Fused decode-step selection (sm_100a): estimate_scores + select_topk +
// populate_page_spans (engine.cpp:34-97, 119-178, 271-283) for INT4 mean stores in
// ONE kernel, one thread-block cluster of C CTAs per (sequence, KV head) unit, with
// the same ordered block lists the reference computes (bit-exact), but without the
// serial fp32 score of every centroid.
//
//   stream  : the producer warp bulk-copies (TMA) the CTA's slice of the unit's packed
//             code rows into a 4-stage ring, plus q and the unit's scale / zero point.
//   filter  : consumers compute, per centroid, the exact integer
//                 I_i = sum_c (256 h_c + l_c) code_ic            (IDP4A, codes 0..15)
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

template <int D>
struct SelCfg {
    static constexpr int W = D / 8;        // int4 words per code row
    static constexpr int U = W / 4;        // 16-byte groups per row
    static constexpr int ROWB = W * 4;
    static constexpr int STAGEB = kSRows * ROWB;
    static constexpr int RING = kSStages * STAGEB;
    static constexpr int QB = 8 * D * 2;   // q rows (G <= 8)
    static constexpr int PB = 2 * D * 4;   // scales + zero points
    static constexpr int TBL = D * 16 * 4; // exact product table
};

// Fixed-size part of the shared memory; the candidate arrays follow it:
//   cand [cand_cap] u64 (leader: composites), list / outs [cand_cap] u32 (this CTA's
//   candidate indices, then the leader's ordered selection).
struct SelHead {
    unsigned long long bars[2 * kSStages + 1];  // full[NS], empty[NS], params
    __align__(16) uint32_t wts[4 * 16];  // packed int8 weights: [word][HE, HO, LE, LO] (W <= 16)
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

template <int D>
__global__ void __launch_bounds__(kSThreads, 2) k_select(LayerView L, const uint16_t* __restrict__ q, uint32_t stages,
                                                       uint32_t slice_cap, uint32_t cand_cap, uint32_t* blocks,
                                                       uint32_t stride, uint32_t* counts, PageList pages,
                                                       uint32_t* ready, float* diag_approx, float* diag_err) {
    using C = SelCfg<D>;
    constexpr int W = C::W, U = C::U;
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

    if (tid == 0) {
        sh.cand = reinterpret_cast<unsigned long long*>(smem + lay.cand);
        sh.list = reinterpret_cast<uint32_t*>(smem + lay.list);
        sh.outs = sh.list;  // the candidate list is dead once the composites are in
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
    }
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
    cluster_sync();  // every CTA's shared memory is initialised before any DSMEM access

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
        // exact product table (score.cu) and the group-summed query
        for (uint32_t e = tid; e < uint32_t(D * 16); e += kSCons) {
            const uint32_t c = e >> 4, code = e & 15u;
            float qc = bf16f(qrows[c]);
            for (uint32_t g = 1; g < L.G; ++g) qc = __fadd_rn(qc, bf16f(qrows[g * D + c]));
            const float deq = L.mode == ABSP_QUANT_ASYM ? __fadd_rn(zps[c], __fmul_rn(float(code), scl[c]))
                                                        : __fmul_rn(float(int(code) - 7), scl[c]);
            tbl[e] = __fmul_rn(qc, deq);
        }
        // weights w_c = fl(q_c s_c) -> sigma (h + l / 256)
        float w = 0.0f, qc = 0.0f;
        if (tid < uint32_t(D)) {
            qc = bf16f(qrows[tid]);
            for (uint32_t g = 1; g < L.G; ++g) qc = __fadd_rn(qc, bf16f(qrows[g * D + tid]));
            w = __fmul_rn(qc, scl[tid]);
        }
        float wmax = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(fabsf(w))));
        if (lane == 0) sh.red[0][warp] = wmax;
        cons_sync();
        wmax = 0.0f;
        for (int i = 0; i < kSCons / 32; ++i) wmax = fmaxf(wmax, sh.red[0][i]);
        const float sigma = wmax / 127.0f;
        float resid = 0.0f, pmax = 0.0f;
        int h = 0, l = 0;
        if (tid < uint32_t(D)) {
            if (sigma > 0.0f) {
                h = __float2int_rn(w / sigma);
                h = h > 127 ? 127 : (h < -127 ? -127 : h);
                l = __float2int_rn((w - float(h) * sigma) * 256.0f / sigma);
                l = l > 127 ? 127 : (l < -127 ? -127 : l);
            }
            resid = fabsf(w - sigma * (float(h) + float(l) * 0.00390625f)) + fabsf(w) * 0x1p-23f;
            for (int code = 0; code < 16; ++code) pmax = fmaxf(pmax, fabsf(tbl[tid * 16 + code]));
        }
        // packed weights: word j, byte b <- channel 8j + 2b (even) / 8j + 2b + 1 (odd)
        if (tid < uint32_t(D)) {
            const uint32_t j = tid >> 3, k = tid & 7u, b = k >> 1, odd = k & 1u;
            unsigned char* wb = reinterpret_cast<unsigned char*>(sh.wts);
            wb[(j * 4 + odd) * 4 + b] = uint8_t(int8_t(h));
            wb[(j * 4 + 2 + odd) * 4 + b] = uint8_t(int8_t(l));
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            resid += __shfl_xor_sync(0xffffffffu, resid, off);
            pmax += __shfl_xor_sync(0xffffffffu, pmax, off);
        }
        if (lane == 0) {
            sh.red[1][warp] = resid;
            sh.red[2][warp] = pmax;
        }
        cons_sync();
        float R = 0.0f, M = 0.0f;
        for (int i = 0; i < kSCons / 32; ++i) {
            R += sh.red[1][i];
            M += sh.red[2][i];
        }
        const float E = M * 0x1p-14f + 15.0f * R * 1.01f;
        const uint32_t e_int = sigma > 0.0f ? uint32_t(fminf(ceilf(E * 256.0f / sigma), 1.0e9f)) + 2u : 0xffffffffu;
        if (tid == 0) {
            sh.st[0] = e_int;
            if (diag_err && r == 0) diag_err[u] = E;
        }
        const uint4* wq = reinterpret_cast<const uint4*>(sh.wts);  // [word] {HE, HO, LE, LO}, broadcast loads

        // ---- filter: integer scores of the slice -> keys (order-preserving u32) ----
        uint32_t kmin = 0xffffffffu, kmax = 0u;
        for (uint32_t c = 0; c < n_chunks; ++c) {
            const uint32_t stg = c % stages;
            mbar_wait(smem_u32(&sh.bars[stg]), (c / stages) & 1);
            const uint32_t row = c * kSRows + tid;
            if (row < ns) {
                const unsigned char* src = ring + size_t(stg) * C::STAGEB + tid * C::ROWB;
                const uint32_t key = code_row_key(s0 + row, W);
                int sh_ = 0, sl_ = 0;
#pragma unroll
                for (int g = 0; g < U; ++g) {
                    const uint4 v = *reinterpret_cast<const uint4*>(src + ((g ^ key) << 4));
                    const uint32_t wd[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        const uint4 wj = wq[4 * g + t];
                        const int lo = int(wd[t] & 0x0F0F0F0Fu), hi = int((wd[t] >> 4) & 0x0F0F0F0Fu);
                        sh_ = __dp4a(lo, int(wj.x), sh_);
                        sh_ = __dp4a(hi, int(wj.y), sh_);
                        sl_ = __dp4a(lo, int(wj.z), sl_);
                        sl_ = __dp4a(hi, int(wj.w), sl_);
                    }
                }
                const int I = sh_ * 256 + sl_;
                const uint32_t k = uint32_t(I) ^ 0x80000000u;
                keys[row] = k;
                kmin = min(kmin, k);
                kmax = max(kmax, k);
                if (diag_approx) diag_approx[du.seg + s0 + row] = float(I) * (sigma * 0.00390625f);
            }
            if (!resident) {
                __syncwarp();
                if (lane == 0) mbar_arrive(smem_u32(&sh.bars[kSStages + stg]));
            }
        }
        kmin = __reduce_min_sync(0xffffffffu, kmin);
        kmax = __reduce_max_sync(0xffffffffu, kmax);
        if (lane == 0) {
            sh.red[0][warp] = __uint_as_float(kmin);
            sh.red[1][warp] = __uint_as_float(kmax);
        }
        for (uint32_t i = tid; i < uint32_t(kBins); i += kSCons) sh.hist[i] = 0u;
        cons_sync();
        kmin = 0xffffffffu;
        kmax = 0u;
        for (int i = 0; i < kSCons / 32; ++i) {
            kmin = min(kmin, __float_as_uint(sh.red[0][i]));
            kmax = max(kmax, __float_as_uint(sh.red[1][i]));
        }
        // ---- local lower bound of the k_r-th largest (1024-bin histogram) ----
        uint32_t t_r = 0u;
        if (!all && K > 1) {
            const uint32_t kr = (K - 1 + Cn - 1) / Cn;
            if (ns >= kr) {
                const uint64_t R64 = uint64_t(kmax - kmin) + 1;
                for (uint32_t i = tid; i < ns; i += kSCons)
                    atomicAdd(&sh.hist[uint32_t((uint64_t(keys[i] - kmin) * kBins) / R64)], 1u);
                cons_sync();
                if (tid < 32) {  // bin holding the kr-th largest, counted from the top
                    constexpr int PER = kBins / 32;
                    uint32_t tot = 0;
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
                            if (cum >= kr) {  // lower edge: the smallest key mapping to bin b
                                sh.st[1] = kmin + uint32_t((uint64_t(b) * R64 + kBins - 1) / kBins);
                                break;
                            }
                        }
                    }
                }
                cons_sync();
                t_r = sh.st[1];
            }
        }
        if (tid < Cn) st_cluster_u32(dsmem(&sh.slot[r], tid), t_r);  // every CTA gets every t_r
    }
    cluster_sync();  // #1: slices scored, bounds exchanged

    // ---- candidates of this slice, exact scores, composites to the leader ----
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
            const bool cand = i < ns && keys[i] >= thr;
            const uint32_t m = __ballot_sync(0xffffffffu, cand);
            uint32_t base = 0;
            if (lane == 0 && m) base = atomicAdd(&sh.local_cnt, __popc(m));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (cand) {
                const uint32_t p = base + __popc(m & ((1u << lane) - 1u));
                if (p < cand_cap) sh.list[p] = i;
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
                const uint32_t i = sh.list[j];
                uint32_t wd[W];
                if (resident) {
                    const unsigned char* src = ring + size_t(i / kSRows) * C::STAGEB + (i % kSRows) * C::ROWB;  // resident: stage i / rows
                    const uint32_t key = code_row_key(s0 + i, W);
#pragma unroll
                    for (int g = 0; g < U; ++g) {
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
                st_cluster_u64(dsmem(&sh.cand[pos0 + j], 0), comp);
            }
        }
    }
    cluster_sync();  // #2: every composite has landed in the leader
    if (r != 0) return;

    // ================================ leader ===================================
    unsigned long long ct = 0ull;
    if (!all) {  // the trailing block's exact score (forced into the selection)
        if (tid == 0) {
            uint32_t wd[W];
            load_row_global<W>(L.codes, du.seg + N - 1, N - 1, wd);
            const float x = exact_row<W>(wd, tbl);
            sh.st[3] = order_key(x);
        }
        __syncthreads();
        ct = (uint64_t(sh.st[3]) << 32) | uint32_t(~(N - 1));
    }
    uint32_t n_sel;
    if (!all && K == 1) {
        if (tid == 0) sh.outs[0] = N - 1;
        n_sel = 1;
    } else if (!all && (sh.overflow || sh.cand_cnt < K - 1)) {
        exact_fallback<W>(L, du, sh, tbl, K, ct);  // (all: N <= K <= cand_cap never overflows)
        n_sel = K;
    } else {
        n_sel = order_selection(sh, sh.cand_cnt, K, !all, ct, N);
    }
    publish_selection(L, du, u, sh.outs, n_sel, blocks, stride, counts, pages, ready);
}

}  // namespace

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

// Decode-step selection: tensor-core filter + exact refine (sm_100a).
//
// Computes exactly what score.cu + topk.cu compute — the reference's
// estimate_scores + select_topk (engine.cpp:34-97, 119-178) on the group-summed
// query, bit-exact ordered block lists — without evaluating the serial fp32
// score of every centroid:
//
//   k_score_approx : streams the packed INT4 code rows (TMA bulk copies, as the
//                    exact scorer) and computes A_i = sum_c w_c * code_ic + alpha,
//                    the score with the dequantisation linearised, on the integer
//                    tensor cores: w_c = q_c * s_c ~ sigma * (h_c + l_c / 256) with
//                    int8 h, l, and the u8 codes taken straight from the packed words
//                    (mma.sync m16n8k32 u8 x s8 -> s32, exact). Per unit
//                    |A_i - S_i| <= E_u = 2^-14 * sum_c |q_c| (|zp_c| + 15 |s_c|)
//                                        + 15 * sum_c |w_c - sigma (h_c + l_c/256)|:
//                    the first term has a 7x margin over the serial fp32 sum
//                    (~130u) plus the approximation's own roundings (~15u), the
//                    second is the weight quantisation exactly (codes <= 15).
//   k_select_refine: one CTA per unit. a = (K-1)-th largest A over blocks
//                    [0, N-1); every block of the exact top-(K-1) has
//                    S >= tau >= a - E, hence A >= a - 2E: the candidates
//                    {A_i >= a - 2E} (typically K-1 plus a few) are re-scored with
//                    the reference's exact serial arithmetic (product table), and
//                    the exact top-(K-1) by (score desc, index asc) plus the
//                    trailing block N-1 is taken among them, ordered, published and
//                    resolved to pages. Degenerate inputs with more candidates than
//                    fit (mass near-ties) re-score every block instead.
//
// Opt-in for absp_decode_step on INT4 mean stores (ABSP_FAST_SELECT=1): parity-green,
// but on B200 at cfg3 it is not yet faster than score.cu + topk.cu end to end (its
// refine phase is a chain of short latency-bound steps); absp_select always keeps
// the full exact scores, the reference's estimate_scores output.
#include "absp_internal.cuh"
#include "common.cuh"
#include "ptx.cuh"

#include <math.h>

namespace absp {
namespace {

// Optional timeline instrumentation (debug builds with -DABSP_ATTN_TRACE): per unit
// CTA of k_select_refine, globaltimer stamps at its phase boundaries.
#ifdef ABSP_ATTN_TRACE
constexpr int kRefineTraceSlots = 8;
__device__ unsigned long long g_refine_trace[1024 * kRefineTraceSlots];
#define REFINE_TRACE(slot)                                                                        \
    do {                                                                                          \
        if (threadIdx.x == 0 && blockIdx.x < 1024) {                                              \
            unsigned long long t_;                                                                \
            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_));                                 \
            g_refine_trace[blockIdx.x * kRefineTraceSlots + (slot)] = t_;                         \
        }                                                                                         \
    } while (0)
__device__ uint32_t g_refine_cand[1024];
#else
#define REFINE_TRACE(slot) do {} while (0)
#endif

// ============================ phase 1: approximate scores ============================
constexpr int kAThreads = 256;            // consumer threads: 8 warps x 32 rows per chunk
constexpr int kAWarps = kAThreads / 32;
constexpr int kABlock = kAThreads + 32;   // + producer warp
constexpr int kAChunk = kAThreads;        // rows per stage (2 m16 tiles per warp)
constexpr int kANS = 4;                   // ring stages

template <int D>
struct ApproxCfg {
    static constexpr int W = D / 8;        // int4: words per code row
    static constexpr int U = W / 4;        // 16-byte groups per row
    static constexpr int KS = D / 32;      // k32 integer mma steps
    static constexpr int ROWB = W * 4;
    static constexpr int STAGEB = kAChunk * ROWB;
    static constexpr int QB = 8 * D * 2;   // q rows of a unit (G <= 8)
    static constexpr int PB = 2 * D * 4;   // scales + zps
    static constexpr int SLOTB = QB + PB;
    static constexpr int WB = D * 4 + 2 * D;  // fp32 weights + int8 hi + int8 lo
    static constexpr int RB = 32 * 4;         // per-warp reduction partials
    static constexpr size_t SMEM = size_t(kANS) * STAGEB + 2 * SLOTB + 2 * (WB + RB) + (2 * kANS + 4) * 8;
};

__device__ __forceinline__ void consumers_sync() {  // named barrier 1: the 8 consumer warps
    asm volatile("bar.sync 1, %0;\n" ::"n"(kAThreads) : "memory");
}

// Integer MMA: D[16x8] (s32) += A[16x32] (u8, row) * B[32x8] (s8, col), exact.
__device__ __forceinline__ void imma(int* c, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                     uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// Logical k of an m16n8k32 step ks -> channel. The A fragment byte group
// gamma = k / 4 of a row is one masked word of packed codes: word
// 4ks + (gamma & 3) / 2 + 2 * (gamma >= 4), its even (gamma odd: odd) nibbles, so a
// register of four u8 codes is one LOP3 (plus a shift for odd nibbles). The
// weights (B) are laid out with the same permutation; the sum over k is unchanged.
__device__ __forceinline__ uint32_t imma_channel(uint32_t ks, uint32_t k) {
    const uint32_t gamma = k >> 2, b = k & 3u;
    const uint32_t word = 4 * ks + ((gamma & 3u) >> 1) + ((gamma >> 2) << 1);
    return 8 * word + (gamma & 1u) + 2 * b;
}

template <int D, bool ASYM>
__global__ void __launch_bounds__(kABlock, kScoreCtasPerSm) k_score_approx(LayerView L, const uint16_t* __restrict__ q,
                                                                           ScoreWork work, float* __restrict__ approx,
                                                                           float* __restrict__ err) {
    using C = ApproxCfg<D>;
    constexpr int W = C::W, U = C::U, KS = C::KS;
    static_assert(W % 4 == 0, "whole 16-byte groups per code row");
    extern __shared__ __align__(1024) unsigned char smem[];
    unsigned char* ring = smem;
    unsigned char* slots = smem + size_t(kANS) * C::STAGEB;
    unsigned char* wbase = slots + 2 * C::SLOTB;  // [2][weights | partials]
    unsigned long long* bars = reinterpret_cast<unsigned long long*>(wbase + 2 * (C::WB + C::RB));
    // bars: full[NS], empty[NS], slot_full[2], slot_empty[2]
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t it0 = work.item_begin[blockIdx.x], it1 = work.item_begin[blockIdx.x + 1];
    if (it0 >= it1) {
        griddep_wait();
        griddep_launch_dependents();
        return;
    }
    if (tid == 0) {
        for (int i = 0; i < kANS; ++i) {
            mbar_init(smem_u32(&bars[i]), 1);
            mbar_init(smem_u32(&bars[kANS + i]), kAWarps);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(smem_u32(&bars[2 * kANS + i]), 1);
            mbar_init(smem_u32(&bars[2 * kANS + 2 + i]), kAWarps);
        }
        mbar_fence_init();
    }
    __syncthreads();
    griddep_wait();  // q and the score buffers are step data
    // only now may the refine kernel start: it reads q before its own wait
    griddep_launch_dependents();

    if (warp == kAWarps) {
        // ================================ producer ================================
        if (lane != 0) return;
        uint32_t chunk = 0;
        for (uint32_t k = it0; k < it1; ++k) {
            const ScoreItem it = work.items[k];
            const uint32_t u = it.unit;
            const uint64_t seg = L.desc[u].seg;
            const uint32_t sl_i = (k - it0) & 1;
            if (k >= it0 + 2) mbar_wait(smem_u32(&bars[2 * kANS + 2 + sl_i]), (((k - it0) >> 1) - 1) & 1);
            {
                unsigned char* sl = slots + sl_i * C::SLOTB;
                const uint32_t bar = smem_u32(&bars[2 * kANS + sl_i]);
                const uint32_t qbytes = L.G * D * 2;
                mbar_expect_tx(bar, qbytes + C::PB);
                bulk_g2s(smem_u32(sl), q + size_t(u) * L.G * D, qbytes, bar);  // units are b-major
                float* prm = reinterpret_cast<float*>(sl + C::QB);
                bulk_g2s(smem_u32(prm), L.scales + size_t(u) * D, D * 4, bar);
                bulk_g2s(smem_u32(prm + D), L.zps + size_t(u) * D, D * 4, bar);
            }
            for (uint32_t pos = it.start; pos < it.end; pos += kAChunk, ++chunk) {
                const uint32_t st = chunk % kANS;
                if (chunk >= uint32_t(kANS)) mbar_wait(smem_u32(&bars[kANS + st]), ((chunk / kANS) - 1) & 1);
                const uint32_t n = min(uint32_t(kAChunk), it.end - pos);
                const uint32_t bar = smem_u32(&bars[st]);
                mbar_expect_tx(bar, n * C::ROWB);
                bulk_g2s(smem_u32(ring + size_t(st) * C::STAGEB), L.codes + (seg + pos) * W, n * C::ROWB, bar);
            }
        }
        return;
    }

    // ================================ consumers =================================
    // per item: w_c = q_c * s_c as sigma * (h_c + l_c / 256), h, l int8 (B operand,
    // column 0 = h, column 1 = l); per 16-row tile: 4 bytes of u8 codes per register
    // straight from the packed words, D/32 integer MMAs, exact int32 sums
    const uint32_t g = lane >> 2, t4 = lane & 3;
    const uint32_t odd = t4 & 1u, wsel = t4 >> 1;
    const int mid = 7;
    uint32_t chunk = 0;
    for (uint32_t k = it0; k < it1; ++k) {
        const ScoreItem it = work.items[k];
        const UnitDesc du = L.desc[it.unit];
        const uint32_t buf = (k - it0) & 1;
        mbar_wait(smem_u32(&bars[2 * kANS + buf]), ((k - it0) >> 1) & 1);
        const unsigned char* sl = slots + buf * C::SLOTB;
        const uint16_t* qrows = reinterpret_cast<const uint16_t*>(sl);
        const float* prm = reinterpret_cast<const float*>(sl + C::QB);
        unsigned char* wb = wbase + buf * (C::WB + C::RB);
        float* wf = reinterpret_cast<float*>(wb);
        int8_t* wh = reinterpret_cast<int8_t*>(wb + D * 4);
        int8_t* wl = wh + D;
        float* rd = reinterpret_cast<float*>(wb + C::WB);  // [0,8) max|w|, [8,16) alpha, [16,24) bound, [24,32) residual
        float qc = 0.0f, sc = 0.0f, zp = 0.0f, w = 0.0f;
        if (tid < uint32_t(D)) {
            qc = bf16f(qrows[tid]);  // left-to-right fp32 group sum (as the exact scorer)
            for (uint32_t gg = 1; gg < L.G; ++gg) qc = __fadd_rn(qc, bf16f(qrows[gg * D + tid]));
            sc = prm[tid];
            zp = prm[D + tid];
            w = qc * sc;
            wf[tid] = w;
        }
        // |w| as bits orders like the floats (non-negative)
        const float wmax = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(fabsf(w))));
        if (lane == 0) rd[warp] = wmax;
        consumers_sync();
        float smax = 0.0f;
#pragma unroll
        for (int i = 0; i < kAWarps; ++i) smax = fmaxf(smax, rd[i]);
        const float sigma = smax / 127.0f;
        float alpha_c = 0.0f, bound_c = 0.0f, res_c = 0.0f;
        if (tid < uint32_t(D)) {
            int h = 0, l = 0;
            if (sigma > 0.0f) {
                h = __float2int_rn(w / sigma);
                h = h > 127 ? 127 : (h < -127 ? -127 : h);
                l = __float2int_rn((w - float(h) * sigma) * 256.0f / sigma);
                l = l > 127 ? 127 : (l < -127 ? -127 : l);
            }
            wh[tid] = int8_t(h);
            wl[tid] = int8_t(l);
            res_c = fabsf(w - sigma * (float(h) + float(l) * 0.00390625f));
            alpha_c = ASYM ? qc * zp : -float(mid) * w;
            bound_c = fabsf(qc) * (fabsf(zp) + 15.0f * fabsf(sc));
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            alpha_c += __shfl_xor_sync(0xffffffffu, alpha_c, off);
            bound_c += __shfl_xor_sync(0xffffffffu, bound_c, off);
            res_c += __shfl_xor_sync(0xffffffffu, res_c, off);
        }
        if (lane == 0) {
            rd[8 + warp] = alpha_c;
            rd[16 + warp] = bound_c;
            rd[24 + warp] = res_c;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&bars[2 * kANS + 2 + buf]));  // slot read
        consumers_sync();
        float alpha = 0.0f, bound = 0.0f, res = 0.0f;
#pragma unroll
        for (int i = 0; i < kAWarps; ++i) {
            alpha += rd[8 + i];
            bound += rd[16 + i];
            res += rd[24 + i];
        }
        // |approx - exact| <= 2^-14 sum |q|(|zp| + 15|s|) + 15 sum |w - sigma (h + l/256)|.
        // First term: the exact score's serial fp32 sum of 128 rounded products deviates
        // from the real-valued sum by <= ~130u sum |q|(|zp| + 15|s|) (u = 2^-24), and the
        // approximation's own roundings (w = q s, alpha's tree sum, the int -> float
        // conversions, sigma scaling, + alpha) by <= ~15u of the same sum: 145u ~ 2^-16.8,
        // so 2^-14 keeps a 7x margin. Second term: the weight quantisation, exactly
        // (codes <= 15; 1.01 covers the rounding of res itself).
        if (tid == 0) err[it.unit] = bound * 0x1p-14f + 15.0f * res * 1.01f;  // same in every CTA of the unit
        // B fragments: b0 = logical k 4t4..4t4+3, b1 = 16 + 4t4.., column g (0: h, 1: l)
        uint32_t bfr[KS][2];
#pragma unroll
        for (int ks = 0; ks < KS; ++ks)
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
                uint32_t v = 0;
                if (g < 2) {
                    const int8_t* src = g == 0 ? wh : wl;
#pragma unroll
                    for (int b = 0; b < 4; ++b)
                        v |= uint32_t(uint8_t(src[imma_channel(ks, 16 * hf + 4 * t4 + b)])) << (8 * b);
                }
                bfr[ks][hf] = v;
            }

        float* out = approx + du.seg;
        for (uint32_t pos = it.start; pos < it.end; pos += kAChunk, ++chunk) {
            const uint32_t st = chunk % kANS;
            const uint32_t n = min(uint32_t(kAChunk), it.end - pos);
            mbar_wait(smem_u32(&bars[st]), (chunk / kANS) & 1);
            const unsigned char* stage = ring + size_t(st) * C::STAGEB;
#pragma unroll
            for (int mt = 0; mt < 2; ++mt) {
                const uint32_t tile = warp * 32 + mt * 16;
                if (tile >= n) break;
                uint32_t rw[2][W];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const uint32_t r = tile + g + 8 * h;
                    const uint32_t key = code_row_key(pos + r, W);
                    const unsigned char* row = stage + r * C::ROWB;
#pragma unroll
                    for (int gr = 0; gr < U; ++gr) {
                        const uint4 v = *reinterpret_cast<const uint4*>(row + ((gr ^ key) << 4));
                        rw[h][4 * gr] = v.x;
                        rw[h][4 * gr + 1] = v.y;
                        rw[h][4 * gr + 2] = v.z;
                        rw[h][4 * gr + 3] = v.w;
                    }
                }
                int acc[4] = {0, 0, 0, 0};
#pragma unroll
                for (int ks = 0; ks < KS; ++ks) {
                    uint32_t a[4];
#pragma unroll
                    for (int q4 = 0; q4 < 4; ++q4) {  // a0: row g, a1: row g+8, a2/a3: groups +4
                        const int wi = 4 * ks + ((q4 >> 1) << 1);  // compile-time register index
                        const uint32_t word = wsel ? rw[q4 & 1][wi + 1] : rw[q4 & 1][wi];
                        a[q4] = (odd ? (word >> 4) : word) & 0x0F0F0F0Fu;
                    }
                    imma(acc, a[0], a[1], a[2], a[3], bfr[ks][0], bfr[ks][1]);
                }
                if (t4 == 0) {
                    const uint32_t r0 = tile + g, r1 = r0 + 8;
                    if (r0 < n) out[pos + r0] = sigma * (float(acc[0]) + float(acc[1]) * 0.00390625f) + alpha;
                    if (r1 < n) out[pos + r1] = sigma * (float(acc[2]) + float(acc[3]) * 0.00390625f) + alpha;
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&bars[kANS + st]));
        }
    }
}

// ============================ phase 2: exact refine ============================
constexpr int kRThreads = 512;
constexpr int kRWarps = kRThreads / 32;
constexpr uint32_t kKeyCap = 32768;  // max N per unit (keys in shared memory)
constexpr uint32_t kCandCap = 4096;  // max candidates re-scored exactly
constexpr uint32_t kRankCap = 1024;  // candidates ordered by rank counting (else bitonic)
constexpr int kHistBits = 9;  // histogram / sample scratch: 512 entries

template <int D>
struct RefineCfg {
    static constexpr size_t KEYS = size_t(kKeyCap) * 4;
    static constexpr size_t COMP = size_t(kCandCap) * 8;
    static constexpr size_t CIDX = size_t(kCandCap) * 4;
    static constexpr size_t TBL = size_t(D) * 16 * 4;
    static constexpr size_t OUT = 2048 * 4;
    static constexpr size_t HIST = (size_t(1) << kHistBits) * 4;
    static constexpr size_t SMEM = KEYS + COMP + CIDX + TBL + OUT + D * 4 + HIST + 64 * 4;
};

// Among the bins [0, nbins) of hist, counted from the top, the bin holding the
// rem-th key: st[2] = bin, st[3] = keys in higher bins. Warp 0 only.
__device__ __forceinline__ void find_bin(const uint32_t* hist, uint32_t nbins, uint32_t rem, uint32_t* st) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t per = (nbins + 31) / 32;  // lane l covers bins top - l*per - [0, per)
    uint32_t tot = 0;
    for (uint32_t j = 0; j < per; ++j) {
        const uint32_t b = lane * per + j;
        tot += b < nbins ? hist[nbins - 1 - b] : 0u;
    }
    uint32_t incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= uint32_t(o)) incl += v;
    }
    uint32_t cum = incl - tot;
    if (cum < rem && rem <= incl) {
        for (uint32_t j = 0; j < per; ++j) {
            const uint32_t b = lane * per + j;
            const uint32_t c = b < nbins ? hist[nbins - 1 - b] : 0u;
            if (cum + c >= rem) {
                st[2] = nbins - 1 - b;
                st[3] = cum;
                break;
            }
            cum += c;
        }
    }
}

// A lower bound on the k-th largest of keys[0, n) (1 <= k <= n). The filter only
// needs a bound — a lower one just widens the candidate set — and a valid one is
// cheap: warp w of 16 takes a slice of the keys and finds its m-th largest x_w,
// m = ceil(k / 16), so at least 16 m >= k keys are >= min_w x_w. Each lane keeps its
// L largest keys sorted in registers (insertion, fixed indices), the warp pops the
// largest head m times (__reduce_max_sync). No atomics, one CTA barrier. Returns 0
// (no bound: every key a candidate) when m > L.
template <int L>
__device__ uint32_t warp_slice_kth(const uint32_t* keys, uint32_t lo, uint32_t hi, uint32_t m) {
    const uint32_t lane = threadIdx.x & 31;
    uint32_t top[L];
#pragma unroll
    for (int j = 0; j < L; ++j) top[j] = 0u;
    for (uint32_t i = lo + lane; i < hi; i += 32) {
        uint32_t x = keys[i];
#pragma unroll
        for (int j = 0; j < L; ++j) {  // insert: top stays descending
            const uint32_t hiv = max(top[j], x);
            x = min(top[j], x);
            top[j] = hiv;
        }
    }
    uint32_t x = 0;
    for (uint32_t r = 0; r < m; ++r) {
        x = __reduce_max_sync(0xffffffffu, top[0]);
        const uint32_t owner = __ffs(__ballot_sync(0xffffffffu, top[0] == x)) - 1;
        if (lane == owner) {
#pragma unroll
            for (int j = 0; j < L - 1; ++j) top[j] = top[j + 1];
            top[L - 1] = 0u;
        }
    }
    return x;
}

__device__ uint32_t kth_lower_bound(const uint32_t* keys, uint32_t n, uint32_t k, uint32_t* st) {
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t m = (k + kRWarps - 1) / kRWarps;
    const uint32_t lo = uint32_t((uint64_t(warp) * n) / kRWarps), hi = uint32_t((uint64_t(warp + 1) * n) / kRWarps);
    uint32_t x = 0;
    if (m <= 8) x = warp_slice_kth<8>(keys, lo, hi, m);
    else if (m <= 16) x = warp_slice_kth<16>(keys, lo, hi, m);
    else if (m <= 32) x = warp_slice_kth<32>(keys, lo, hi, m);
    if (lane == 0) st[16 + warp] = x;
    __syncthreads();
    uint32_t b = 0xffffffffu;
    for (int w = 0; w < kRWarps; ++w) b = min(b, st[16 + w]);
    __syncthreads();
    return b;
}

// Exact k-th largest of keys[0, n) (MSB-first radix, 8-bit digits): st[0] = tau,
// st[1] = number of keys > tau. Used only when the filter degenerates.
__device__ void radix_kth(const uint32_t* keys, uint32_t n, uint32_t k, uint32_t* hist, uint32_t* st) {
    const uint32_t tid = threadIdx.x;
    uint32_t prefix = 0, mask = 0, rem = k, gt = 0;
    for (int shift = 24; shift >= 0; shift -= 8) {
        for (uint32_t i = tid; i < 256; i += kRThreads) hist[i] = 0u;
        __syncthreads();
        for (uint32_t i = tid; i < n; i += kRThreads) {
            const uint32_t key = keys[i];
            if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
        }
        __syncthreads();
        if (tid < 32) find_bin(hist, 256, rem, st);
        __syncthreads();
        prefix |= st[2] << shift;
        mask |= 255u << shift;
        gt += st[3];
        rem -= st[3];
        __syncthreads();
    }
    if (tid == 0) {
        st[0] = prefix;
        st[1] = gt;
    }
    __syncthreads();
}

// Bitonic sort of comp[0, n) descending (n <= kCandCap; padded with zeros).
__device__ void sort_desc(unsigned long long* comp, uint32_t n) {
    uint32_t sp = 1;
    while (sp < n) sp <<= 1;
    for (uint32_t i = n + threadIdx.x; i < sp; i += kRThreads) comp[i] = 0ull;
    __syncthreads();
    for (uint32_t k = 2; k <= sp; k <<= 1)
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t i = threadIdx.x; i < sp; i += kRThreads) {
                const uint32_t ixj = i ^ j;
                if (ixj > i) {
                    const unsigned long long a = comp[i], b = comp[ixj];
                    if (((i & k) == 0) ? (a < b) : (a > b)) {
                        comp[i] = b;
                        comp[ixj] = a;
                    }
                }
            }
            __syncthreads();
        }
}

__device__ __forceinline__ float key_to_float(uint32_t k) {
    return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

template <int D, bool ASYM>
__global__ void __launch_bounds__(kRThreads, 1) k_select_refine(LayerView L, const uint16_t* __restrict__ q,
                                                                const float* __restrict__ approx,
                                                                const float* __restrict__ err, uint32_t* blocks,
                                                                uint32_t stride, uint32_t* counts, PageList pages,
                                                                uint32_t* ready) {
    using C = RefineCfg<D>;
    constexpr int W = D / 8, U = W / 4, LV = 16;
    extern __shared__ __align__(1024) unsigned char smem[];
    uint32_t* keys = reinterpret_cast<uint32_t*>(smem);
    unsigned long long* comp = reinterpret_cast<unsigned long long*>(smem + C::KEYS);
    uint32_t* cidx = reinterpret_cast<uint32_t*>(smem + C::KEYS + C::COMP);
    float* tbl = reinterpret_cast<float*>(smem + C::KEYS + C::COMP + C::CIDX);
    uint32_t* outs = reinterpret_cast<uint32_t*>(smem + C::KEYS + C::COMP + C::CIDX + C::TBL);
    float* qs = reinterpret_cast<float*>(outs + 2048);
    uint32_t* hist = reinterpret_cast<uint32_t*>(qs + D);
    uint32_t* st = hist + (1u << kHistBits);  // [0..15] scalars, [16..47] warp partials

    const uint32_t u = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const UnitDesc du = L.desc[u];
    const uint32_t N = du.n_blocks, K = du.budget;
    const bool all = N <= K;
    const uint32_t K1 = all ? N : K - 1, n = all ? N : N - 1;  // ranked blocks: [0, n)
    REFINE_TRACE(0);
    griddep_launch_dependents();
    // Before the wait: the exact product table of the reference's serial score (as
    // k_score_tbl). q is safe to read here: k_score_approx triggers this launch only
    // after its own wait, i.e. once q's producer has completed; the store is immutable.
    for (uint32_t c = tid; c < uint32_t(D); c += kRThreads) {
        const uint16_t* qb = q + size_t(u) * L.G * D + c;  // units are b-major
        float acc = bf16f(qb[0]);
        for (uint32_t g = 1; g < L.G; ++g) acc = __fadd_rn(acc, bf16f(qb[size_t(g) * D]));
        qs[c] = acc;
    }
    if (tid == 0) st[4] = 0u;  // candidate count
    __syncthreads();
    const int mid = 7;
    for (uint32_t e = tid; e < uint32_t(D * LV); e += kRThreads) {
        const uint32_t c = e / LV, code = e % LV;
        const float sc = __ldg(L.scales + size_t(u) * D + c), zp = __ldg(L.zps + size_t(u) * D + c);
        const float deq = ASYM ? __fadd_rn(zp, __fmul_rn(float(code), sc)) : __fmul_rn(float(int(code) - mid), sc);
        tbl[e] = __fmul_rn(qs[c], deq);
    }
    griddep_wait();  // approximate scores and bounds come from k_score_approx
    REFINE_TRACE(1);
    if (!all) {
        const float* ap = approx + du.seg;
        for (uint32_t i = tid; i < n; i += kRThreads) keys[i] = order_key(__ldcg(ap + i));
    }
    __syncthreads();
    REFINE_TRACE(2);
    const uint32_t* codes = L.codes + du.seg * W;
    auto exact = [&](uint32_t i) -> float {  // the reference's serial fp32 score of block i
        uint32_t wd[W];
        const uint4* row = reinterpret_cast<const uint4*>(codes + size_t(i) * W);
        const uint32_t key = code_row_key(i, W);
#pragma unroll
        for (int gr = 0; gr < U; ++gr) {
            const uint4 v = __ldg(row + (gr ^ key));
            wd[4 * gr] = v.x;
            wd[4 * gr + 1] = v.y;
            wd[4 * gr + 2] = v.z;
            wd[4 * gr + 3] = v.w;
        }
        const char* tb = reinterpret_cast<const char*>(tbl);
        float acc = 0.0f;
#pragma unroll
        for (int w = 0; w < W; ++w) {
            const CodeOffsets<4> co(wd[w]);
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
                acc = __fadd_rn(acc, *reinterpret_cast<const float*>(tb + (w * 8 + kk) * LV * 4 + co(kk)));
        }
        return acc;
    };
    auto comp_of = [](float s, uint32_t i) -> unsigned long long {
        return (static_cast<unsigned long long>(order_key(s)) << 32) | uint32_t(~i);
    };

    // ---- candidates: every block that can belong to the exact top-K1 ----
    uint32_t Cn;  // candidates, in cidx[0, Cn)
    if (all) {
        Cn = n;
        for (uint32_t i = tid; i < n; i += kRThreads) cidx[i] = i;
    } else if (K1 == 0) {
        Cn = 0;
    } else {
        const uint32_t ak = kth_lower_bound(keys, n, K1, st);
        REFINE_TRACE(3);
        // threshold a' - 2E, rounded down; a bin edge below -inf (NaN images) keeps all
        const float e2 = 2.0f * __ldcg(err + u) * 1.0001f + 1e-30f;
        const uint32_t thr = ak < 0x007fffffu ? 0u : order_key(__fsub_rd(key_to_float(ak), e2));
        for (uint32_t i = tid; i < n; i += kRThreads)
            if (keys[i] >= thr) {
                const uint32_t j = atomicAdd(&st[4], 1u);
                if (j < kCandCap) cidx[j] = i;
            }
        __syncthreads();
        Cn = st[4];
    }
    __syncthreads();  // table complete
    REFINE_TRACE(4);

    if (Cn < kCandCap) {
        // exact scores of the candidates, and of the trailing block in the last slot
        const uint32_t tail = all ? 0u : 1u;
        for (uint32_t j = tid; j < Cn + tail; j += kRThreads) {
            const uint32_t i = j < Cn ? cidx[j] : N - 1;
            comp[j < Cn ? j : kCandCap - 1] = comp_of(exact(i), i);
        }
        __syncthreads();
        const unsigned long long ct = all ? 0ull : comp[kCandCap - 1];
        REFINE_TRACE(5);
        if (Cn <= kRankCap) {
            // position = rank among the candidates (composites are distinct), shifted by
            // one past the trailing block when it ranks higher
            // Placement by rank: tpc adjacent lanes share an element (each counts a strided
            // share with four independent partial counts); the cost is m^2 / 32 shared loads.
            auto place = [&](const unsigned long long* arr, uint32_t m) {
                if (tid == 0) st[5] = 0u;
                __syncthreads();
                const uint32_t tpc = m <= kRThreads / 8 ? 8u : m <= kRThreads / 4 ? 4u : m <= kRThreads / 2 ? 2u : 1u;
                const uint32_t part = tid % tpc;
                for (uint32_t jb = 0; jb < m * tpc; jb += kRThreads) {  // uniform trip count
                    const uint32_t jj = (jb + tid) / tpc;
                    const bool live = jb + tid < m * tpc;
                    const unsigned long long me = live ? arr[jj] : ~0ull;
                    uint32_t r0 = 0, r1 = 0, r2 = 0, r3 = 0;
                    uint32_t o = part;
                    for (; o + 3 * tpc < m; o += 4 * tpc) {
                        r0 += arr[o] > me;
                        r1 += arr[o + tpc] > me;
                        r2 += arr[o + 2 * tpc] > me;
                        r3 += arr[o + 3 * tpc] > me;
                    }
                    for (; o < m; o += tpc) r0 += arr[o] > me;
                    uint32_t rank = r0 + r1 + r2 + r3;
                    for (uint32_t off = 1; off < tpc; off <<= 1) rank += __shfl_xor_sync(0xffffffffu, rank, off);
                    if (live && part == 0 && rank < K1) {
                        const bool below = ct > me;
                        outs[rank + (below ? 1u : 0u)] = ~uint32_t(me);
                        if (!below && !all) atomicAdd(&st[5], 1u);
                    }
                }
                __syncthreads();
            };
            place(comp, Cn);
            if (tid == 0 && !all) outs[st[5]] = N - 1;
        } else {
            sort_desc(comp, Cn);
            for (uint32_t j = tid; j < K1; j += kRThreads) outs[j + (ct > comp[j] ? 1u : 0u)] = ~uint32_t(comp[j]);
            if (warp == 0 && !all) {
                uint32_t above = 0;
                for (uint32_t j = lane; j < K1; j += 32) above += comp[j] > ct;
                above = __reduce_add_sync(0xffffffffu, above);
                if (lane == 0) outs[above] = N - 1;
            }
        }
    } else {
        // mass near-ties: exact scores of every block, exact radix select, ties at the
        // threshold to the lowest indices (index-ordered scan)
        for (uint32_t i = tid; i < n; i += kRThreads) keys[i] = order_key(exact(i));
        __syncthreads();
        radix_kth(keys, n, K1, hist, st);
        const uint32_t tau = st[0], need_eq = K1 - st[1];
        if (tid == 0) st[5] = 0u;
        __syncthreads();
        for (uint32_t i = tid; i < n; i += kRThreads)
            if (keys[i] > tau) comp[atomicAdd(&st[5], 1u)] = (static_cast<unsigned long long>(keys[i]) << 32) | uint32_t(~i);
        __syncthreads();
        uint32_t taken = 0;
        for (uint32_t base = 0; base < n && taken < need_eq; base += kRThreads) {
            const uint32_t i = base + tid;
            const bool eq = i < n && keys[i] == tau;
            const uint32_t bal = __ballot_sync(0xffffffffu, eq);
            if (lane == 0) hist[warp] = __popc(bal);
            __syncthreads();
            uint32_t before = 0, total = 0;
            for (uint32_t w = 0; w < uint32_t(kRWarps); ++w) {
                before += w < warp ? hist[w] : 0u;
                total += hist[w];
            }
            const uint32_t rank = taken + before + __popc(bal & ((1u << lane) - 1u));
            if (eq && rank < need_eq)
                comp[K1 - need_eq + rank] = (static_cast<unsigned long long>(tau) << 32) | uint32_t(~i);
            taken += total;
            __syncthreads();
        }
        sort_desc(comp, K1);
        if (tid == 0) comp[kCandCap - 1] = comp_of(exact(N - 1), N - 1);
        __syncthreads();
        const unsigned long long ct = comp[kCandCap - 1];
        for (uint32_t j = tid; j < K1; j += kRThreads) outs[j + (ct > comp[j] ? 1u : 0u)] = ~uint32_t(comp[j]);
        if (warp == 0) {
            uint32_t above = 0;
            for (uint32_t j = lane; j < K1; j += 32) above += comp[j] > ct;
            above = __reduce_add_sync(0xffffffffu, above);
            if (lane == 0) outs[above] = N - 1;
        }
    }
    const uint32_t sel_total = all ? N : K;
    __syncthreads();
    REFINE_TRACE(6);
    publish_selection(L, du, u, outs, sel_total, blocks, stride, counts, pages, ready);
    REFINE_TRACE(7);
#ifdef ABSP_ATTN_TRACE
    if (tid == 0 && blockIdx.x < 1024) g_refine_cand[blockIdx.x] = Cn;
#endif
}

template <int D, bool ASYM>
cudaError_t attrs_d() {
    cudaError_t e = cudaFuncSetAttribute(k_score_approx<D, ASYM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(ApproxCfg<D>::SMEM));
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(k_select_refine<D, ASYM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                int(RefineCfg<D>::SMEM));
}

template <int D, bool ASYM>
cudaError_t launch_d(const LayerView& L, const uint16_t* q, const ScoreWork& w, float* approx, float* err,
                     uint32_t* blocks, uint32_t stride, uint32_t* counts, const PageList& pages, uint32_t* ready,
                     cudaStream_t s) {
    cudaError_t e = launch_pdl(k_score_approx<D, ASYM>, dim3(w.grid), dim3(kABlock), ApproxCfg<D>::SMEM, s, L, q, w,
                               approx, err);
    if (e != cudaSuccess) return e;
    return launch_pdl(k_select_refine<D, ASYM>, dim3(L.units), dim3(kRThreads), RefineCfg<D>::SMEM, s, L, q,
                      static_cast<const float*>(approx), static_cast<const float*>(err), blocks, stride, counts, pages,
                      ready);
}

}  // namespace

#ifdef ABSP_ATTN_TRACE
cudaError_t debug_refine_trace(void* dst, size_t bytes, void* cand, size_t cbytes) {
    cudaError_t e = cudaMemcpyFromSymbol(dst, g_refine_trace, bytes);
    if (e == cudaSuccess) e = cudaMemcpyFromSymbol(cand, g_refine_cand, cbytes);
    return e;
}
#endif

bool select_fast_supported(const LayerView& L, uint32_t max_nblocks, uint32_t max_budget) {
    return L.bits == 4 && L.method == ABSP_CENTROID_MEAN && (L.D == 64 || L.D == 128) &&
           max_nblocks <= kKeyCap && max_budget <= 2048u;
}

cudaError_t init_select_attributes() {
    cudaError_t e = attrs_d<64, false>();
    if (e == cudaSuccess) e = attrs_d<64, true>();
    if (e == cudaSuccess) e = attrs_d<128, false>();
    if (e == cudaSuccess) e = attrs_d<128, true>();
    return e;
}

cudaError_t launch_select_fast(const LayerView& L, const uint16_t* q, const ScoreWork& work, float* approx, float* err,
                               uint32_t* blocks, uint32_t stride, uint32_t* counts, const PageList& pages,
                               uint32_t* ready, cudaStream_t s, int* launches) {
    *launches += 2;
    const bool asym = L.mode == ABSP_QUANT_ASYM;
    cudaError_t e;
    if (L.D == 64)
        e = asym ? launch_d<64, true>(L, q, work, approx, err, blocks, stride, counts, pages, ready, s)
                 : launch_d<64, false>(L, q, work, approx, err, blocks, stride, counts, pages, ready, s);
    else
        e = asym ? launch_d<128, true>(L, q, work, approx, err, blocks, stride, counts, pages, ready, s)
                 : launch_d<128, false>(L, q, work, approx, err, blocks, stride, counts, pages, ready, s);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

}  // namespace absp

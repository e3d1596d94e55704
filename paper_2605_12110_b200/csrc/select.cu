// Fused decode-step selection (sm_100a): estimate_scores + select_topk +
// populate_page_spans (engine.cpp:34-97, 119-178, 271-283) for INT4 mean stores,
// with the same ordered block lists the reference computes (bit-exact), but without
// the serial fp32 score of every centroid.
//
// Work is cut into SLICES of at most S consecutive centroids of one (sequence, KV
// head) unit (S picked per layout so that the slices fill about two CTAs per SM), one
// CTA per slice, slices in unit order: every CTA streams about the same number of code
// bytes whatever the block sizes, and the last slice of a unit to finish completes
// its selection (no cluster, no inter-CTA waiting):
//
//   stream  : the producer warp bulk-copies (TMA) the slice's packed code rows into a
//             4-stage ring, plus q and the unit's scale / zero point.
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
//             E_int = ceil(E 256 / sigma) + 2. Every slice derives the same weights.
//   bound   : each slice r of the unit's C slices finds a lower bound t_r of the
//             ceil((K-1)/C)-th largest I of its rows (a 1024-bin histogram) and writes
//             its keys and t_r to global memory; T = min_r t_r is a lower bound of the
//             (K-1)-th largest I of the unit. Any block of the exact top-(K-1) has
//             I >= T - 2 E_int (else K-1 blocks score strictly higher), so the
//             candidates {I_i >= T - 2 E_int} (typically K-1 plus a few) contain it.
//   finalize: the slice CTA that arrives last on the unit's counter (acq_rel) scans the
//             unit's keys (L2), scores the candidates with the reference's exact serial
//             fp32 arithmetic (product table, score.cu), ranks the composites
//             (key << 32 | ~index), keeps the top K-1, inserts the trailing block N-1
//             (forced, exactly where its exact score ranks), and publishes blocks,
//             counts, the page list and the unit's ready flag for the attention
//             producer (common.cuh).
//   fallback: more candidates than fit (mass ties) -> the finalizing CTA scores every
//             block exactly into the scores buffer and runs an exact radix select
//             (slow, rare, identical result).
#include "select_core.cuh"

namespace absp {
namespace {

using namespace selcore;

template <int D>
__global__ void __launch_bounds__(kSThreads, 2) k_select(LayerView L, const uint16_t* __restrict__ q, SelectPlan plan,
                                                       SelectWork sw, uint32_t* blocks, uint32_t stride,
                                                       uint32_t* counts, PageList pages, uint32_t* ready,
                                                       float* diag_approx, float* diag_err,
                                                       uint16_t* __restrict__ q_copy) {
    using C = SelCfg<D>;
    constexpr int W = C::W, NG = D / 32;  // code words per row, 16-byte groups (32 channels) per row
    extern __shared__ __align__(1024) unsigned char smem[];
    const uint32_t stages = plan.stages, cand_cap = plan.cand_cap;
    const SelLayout<D> lay(stages, cand_cap, plan.pg_cap, plan.rows);
    uint32_t* slk = reinterpret_cast<uint32_t*>(smem + lay.slk);
    unsigned char* ring = smem;
    float* tbl = reinterpret_cast<float*>(smem + lay.tbl);          // [D][16]
    unsigned char* prm_raw = smem + lay.prm;                         // q rows | scales | zps
    SelHead& sh = *reinterpret_cast<SelHead*>(smem + lay.head);
    const uint16_t* qrows = reinterpret_cast<const uint16_t*>(prm_raw);
    const float* scl = reinterpret_cast<const float*>(prm_raw + C::QB);
    const float* zps = scl + D;
    unsigned long long* cand = reinterpret_cast<unsigned long long*>(smem + lay.cand);  // finalize (ring)
    uint32_t* list = reinterpret_cast<uint32_t*>(smem + lay.list);
    uint32_t* cpg = reinterpret_cast<uint32_t*>(smem + lay.cpg);                        // finalize (ring)

    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const SliceDesc sd = sw.slices[blockIdx.x];
    const uint32_t u = sd.unit, r = sd.r, Cn = sd.n;
    const UnitDesc du = L.desc[u];
    const uint32_t N = du.n_blocks, K = du.budget;
    const bool all = N <= K;               // every block selected (ordered)
    const uint32_t nd = all ? N : N - 1;   // candidate domain [0, nd)
    const uint32_t s0 = uint32_t((uint64_t(r) * nd) / Cn), s1 = uint32_t((uint64_t(r + 1) * nd) / Cn);
    const uint32_t ns = s1 - s0;
    const uint32_t n_chunks = (ns + kSRows - 1) / kSRows;
    uint32_t* gkeys = sw.keys + du.seg;
    // a unit whose keys need several finalize batches: each slice bounds its own
    // ceil((K-1)/C)-th largest key, and the finalize takes T = min over the slices
    // (one pass over the unit's keys instead of two histogram passes and a compaction)
    const bool big = !all && K > 1 && Cn > 1 && nd > kFinKeys;

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
        mbar_init(smem_u32(&sh.bars[2 * kSStages + 1]), 1);
        mbar_fence_init();
        sh.local_cnt = 0u;
        sh.cand_cnt = 0u;
        sh.overflow = 0u;
        sh.nsel = 0u;
        sh.st[1] = 0u;
    }
    for (uint32_t i = tid; i < uint32_t(kBins); i += kSThreads) sh.hist[i] = 0u;
    if (r + 1 == Cn) {  // the page resolution of the finalize reads the sequence's page-table row: warm L2
        const uint32_t row_pages = (du.n_tokens + L.P - 1) / L.P;
        const uint32_t* pt = L.page_table + size_t(du.seq) * L.max_pages;
        for (uint32_t p = tid * 32; p < row_pages; p += kSThreads * 32) asm volatile("prefetch.global.L2 [%0];" ::"l"(pt + p));
    }
    __syncthreads();
    griddep_wait();  // codes / params (appends) and q are written by earlier kernels
    // The attention kernel may be scheduled now: every CTA of this grid is past its wait,
    // i.e. the previous step's attention has completed (its merges re-armed the ready flags).
    griddep_launch_dependents();
    SEL_TRACE(1);

    const uint32_t G = L.G;
    // q_c = left-to-right fp32 group sum (score.cu)
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
    const bool asym = L.mode == ABSP_QUANT_ASYM;

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
        if (lane == 0) mbar_wait(smem_u32(&sh.bars[2 * kSStages]), 0);  // parameters landed (finalize reads them)
        __syncwarp();
    } else {
        // =============================== consumers ==============================
        mbar_wait(smem_u32(&sh.bars[2 * kSStages]), 0);
        SEL_TRACE(3);
        // Every warp derives the weights itself (identical arithmetic, no CTA barrier).
        float E = 0.0f, sigma = 0.0f;
        const uint32_t e_int = unit_weights<D>(qrows, scl, zps, G, asym, lane, sh.hlw[warp], &E, &sigma);
        auto& hlw = sh.hlw;  // this warp's h and l per channel
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
                        __stcg(gkeys + s0 + ra, k);
                        if (big) slk[ra] = k;
                        kmin = min(kmin, k);
                        kmax = max(kmax, k);
                        if (diag_approx) diag_approx[du.seg + s0 + ra] = float(I0) * a_scale;
                    }
                    if (rb < ns) {
                        const uint32_t k = uint32_t(I1) ^ 0x80000000u;
                        __stcg(gkeys + s0 + rb, k);
                        if (big) slk[rb] = k;
                        kmin = min(kmin, k);
                        kmax = max(kmax, k);
                        if (diag_approx) diag_approx[du.seg + s0 + rb] = float(I1) * a_scale;
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&sh.bars[kSStages + stg]));
        }
        SEL_TRACE(5);
        // ---- the slice's key range for the unit's finalize ----
        kmin = __reduce_min_sync(0xffffffffu, kmin);
        kmax = __reduce_max_sync(0xffffffffu, kmax);
        if (lane == 0) {
            sh.red[0][warp] = __uint_as_float(kmin);
            sh.red[1][warp] = __uint_as_float(kmax);
        }
        cons_sync();
        if (tid == 0) {
            kmin = 0xffffffffu;
            kmax = 0u;
#pragma unroll
            for (int i = 0; i < kSCons / 32; ++i) {
                kmin = min(kmin, __float_as_uint(sh.red[0][i]));
                kmax = max(kmax, __float_as_uint(sh.red[1][i]));
            }
            __stcg(sw.slot + 4 * blockIdx.x, kmin);
            __stcg(sw.slot + 4 * blockIdx.x + 1, kmax);
            sh.st[10] = kmin;
            sh.st[11] = kmax;
        }
        if (big) {  // this slice's bound t_r <= its kr-th largest key (0: none)
            const uint32_t kr = (K - 1 + Cn - 1) / Cn;
            uint32_t t_r = 0u;
            cons_sync();
            if (ns >= kr) {
                const uint32_t smin = sh.st[10], span = sh.st[11] - smin;
                const uint32_t shift = span < uint32_t(kBins) ? 0u : 32u - __clz(span) - 10u;
#pragma unroll 4
                for (uint32_t i = tid; i < ns; i += kSCons) atomicAdd(&sh.hist[(slk[i] - smin) >> shift], 1u);
                cons_sync();
                if (warp == 0) find_bin_desc(sh.hist, kr, lane, &sh.st[12], &sh.st[13]);
                cons_sync();
                t_r = smin + (sh.st[12] << shift);
            }
            if (tid == 0) __stcg(sw.slot + 4 * blockIdx.x + 2, t_r);
        }
        SEL_TRACE(6);
    }
    __syncthreads();
    // the last slice of the unit to arrive finalizes it (acq_rel: every slice's keys and
    // bound, published before its arrival, are visible after ours)
    if (tid == 0) {
        uint32_t old;
        asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;\n" : "=r"(old) : "l"(sw.arrive + u) : "memory");
        sh.st[6] = old + 1 == Cn;
        if (sh.st[6]) sw.arrive[u] = 0u;  // re-armed for the next step (every slice has arrived)
    }
    __syncthreads();
    SEL_TRACE(7);
    if (!sh.st[6]) return;
    __threadfence();

    FinIn<D> fin;
    fin.L = L;
    fin.u = u;
    fin.du = du;
    fin.first = sd.first;
    fin.Cn = Cn;
    fin.plan = plan;
    fin.sw = sw;
    fin.blocks = blocks;
    fin.stride = stride;
    fin.counts = counts;
    fin.pages = pages;
    fin.ready = ready;
    fin.q_copy = q_copy;
    fin.cand = cand;
    fin.list = list;
    fin.cpg = cpg;
    fin.skeys = reinterpret_cast<uint32_t*>(smem + lay.fkeys);
    fin.tbl = tbl;
    fin.qrows = qrows;
    fin.scl = scl;
    fin.zps = zps;
    finalize_unit<D>(fin, sh);
}

}  // namespace

#ifdef ABSP_ATTN_TRACE
cudaError_t debug_select_trace(void* dst, size_t bytes) { return cudaMemcpyFromSymbol(dst, g_sel_trace, bytes); }
#endif

bool select_fused_supported(const LayerView& L) {
    return L.bits == 4 && L.method == ABSP_CENTROID_MEAN && (L.D == 64 || L.D == 128) && L.G <= 8;
}

size_t select_fused_smem(uint32_t D, uint32_t stages, uint32_t cand_cap, uint32_t pg_cap, uint32_t rows) {
    return D == 64 ? SelLayout<64>(stages, cand_cap, pg_cap, rows).total
                   : SelLayout<128>(stages, cand_cap, pg_cap, rows).total;
}

// Slices of a layout: the smallest slice size S (a multiple of 256 rows, at most 4096)
// that keeps the layer within about two resident CTAs per SM (cfg3 on one GPU: S = 2304,
// 320 slices; its 8-GPU shard: S = 512), the unit's candidate domain cut evenly into
// ceil(nd / S) slices, in unit order. Ring stages: 4 when they fit (2 CTAs per SM).
SelectPlan plan_select(const std::vector<UnitDesc>& desc, uint32_t max_budget, uint32_t D, int num_sms,
                       std::vector<SliceDesc>* slices) {
    SelectPlan p{};
    auto nd_of = [](const UnitDesc& d) { return d.n_blocks <= d.budget ? d.n_blocks : d.n_blocks - 1; };
    auto count = [&](uint32_t S) {
        uint64_t c = 0;
        for (const UnitDesc& d : desc) c += std::max(1u, (nd_of(d) + S - 1) / S);
        return c;
    };
    p.rows = kSliceMin;
    while (p.rows < kSliceMax && count(p.rows) > uint64_t(2 * num_sms)) p.rows += kSliceMin;
    p.cand_cap = 512;  // a power of two (bitonic sort in place), >= K
    while (p.cand_cap < kCandCapMax && p.cand_cap < 4 * max_budget) p.cand_cap <<= 1;
    p.pg_cap = 4096;
    for (p.stages = kSStages; p.stages > 2; --p.stages)
        if (select_fused_smem(D, p.stages, p.cand_cap, p.pg_cap, p.rows) * 2 + 2048 <= 228 * 1024) break;
    p.ok = select_fused_smem(D, p.stages, p.cand_cap, p.pg_cap, p.rows) <= 227 * 1024;
    if (slices) {
        slices->clear();
        for (uint32_t u = 0; u < desc.size(); ++u) {
            const uint32_t n = std::max(1u, (nd_of(desc[u]) + p.rows - 1) / p.rows);
            const uint32_t first = uint32_t(slices->size());
            for (uint32_t r = 0; r < n; ++r) slices->push_back(SliceDesc{u, r, n, first});
        }
    }
    p.n_slices = slices ? uint32_t(slices->size()) : uint32_t(count(p.rows));
    return p;
}

// Slices a unit can ever need (reservation at bind: every unit at capacity, S = 256).
uint64_t select_slices_bound(const std::vector<UnitDesc>& desc) {
    uint64_t c = 0;
    for (const UnitDesc& d : desc) c += std::max<uint64_t>(1, (uint64_t(std::max(d.n_blocks, d.cap)) + kSliceMin - 1) / kSliceMin);
    return c;
}

cudaError_t init_select_attributes() {
    cudaError_t e = cudaFuncSetAttribute(k_select<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(k_select<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
}

cudaError_t launch_select_fused(const LayerView& L, const uint16_t* q, const SelectPlan& plan, const SelectWork& work,
                                uint32_t* blocks, uint32_t stride, uint32_t* counts, const PageList& pages,
                                uint32_t* ready, float* diag_approx, float* diag_err, uint16_t* q_copy, cudaStream_t s,
                                int* launches) {
    const size_t smem = select_fused_smem(L.D, plan.stages, plan.cand_cap, plan.pg_cap, plan.rows);
    cudaError_t e;
    if (L.D == 64)
        e = launch_pdl(k_select<64>, dim3(plan.n_slices), dim3(kSThreads), smem, s, L, q, plan, work, blocks, stride,
                       counts, pages, ready, diag_approx, diag_err, q_copy);
    else
        e = launch_pdl(k_select<128>, dim3(plan.n_slices), dim3(kSThreads), smem, s, L, q, plan, work, blocks,
                       stride, counts, pages, ready, diag_approx, diag_err, q_copy);
    ++*launches;
    return e == cudaSuccess ? cudaGetLastError() : e;
}

}  // namespace absp

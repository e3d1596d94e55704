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
#include "ptx.cuh"
#include "common.cuh"

namespace absp {
namespace {

constexpr int kThreads = 256;

// Optional timeline instrumentation (debug builds with -DABSP_ATTN_TRACE): per CTA,
// globaltimer stamps at start, after each item's table and at the end.
#ifdef ABSP_ATTN_TRACE
constexpr int kScoreTraceSlots = 16;
__device__ unsigned long long g_score_trace[320 * kScoreTraceSlots];
__device__ __forceinline__ void score_trace(int slot) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    if (blockIdx.x < 320 && slot < kScoreTraceSlots) g_score_trace[blockIdx.x * kScoreTraceSlots + slot] = t;
}
#define SCORE_TRACE(slot) do { if (threadIdx.x == 0) score_trace(slot); } while (0)
#else
#define SCORE_TRACE(slot) do {} while (0)
#endif

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

// Table path (bits in {2, 4}; MAXMIN doubles the tables and code streams).
//
// Work: CTA c scores items [item_begin[c], item_begin[c+1]) — an equal share of
// the layer's flattened centroids cut at unit boundaries — in chunks of
// kChunkRows rows. Warp-specialised:
//   producer warp : drives the TMA bulk-copy engine. Each chunk's packed code rows
//                   (contiguous per unit) are one cp.async.bulk into an NS-stage
//                   ring (full/empty mbarriers); each item's G query rows and
//                   (scale, zp) vectors are bulk-copied into a double-buffered slot.
//   8 consumer warps: per item, build the exact product table (double-buffered,
//                   one named barrier per item); per chunk, each thread reads its
//                   rows with conflict-free 16-byte loads (rows are XOR-swizzled,
//                   code_word_pos) and runs the serial exact sum. Warps whose rows
//                   lie past the end of a partial chunk skip it.
// Consumers never wait on a global load and never synchronise per chunk.
constexpr int kConsumerWarps = kThreads / 32;
constexpr int kTblThreads = kThreads + 32;
constexpr int kRowsPerThread = 1;
constexpr int kChunkRows = kThreads * kRowsPerThread;

template <int D, int BITS, bool MAXMIN>
struct TblCfg {
    static constexpr int LV = 1 << BITS;
    static constexpr int W = D * BITS / 32;   // words per code row
    static constexpr int U = W / 4;           // 16-byte groups per row
    static constexpr int CPW = 32 / BITS;     // codes per word
    static constexpr int NT = MAXMIN ? 2 : 1;  // code arrays / tables
    static constexpr int ROWB = W * 4;
    static constexpr int STAGEB = kChunkRows * ROWB;  // per array
    static constexpr int NS = MAXMIN ? 3 : 4;         // ring stages
    static constexpr int QB = 8 * D * 2;              // q rows of a unit (G <= 8)
    static constexpr int PB = NT * 2 * D * 4;         // scales + zps (+ min arrays)
    static constexpr int SLOTB = QB + PB;
    static constexpr size_t RING = size_t(NS) * NT * STAGEB;
    static constexpr size_t SMEM = RING + 2 * SLOTB + (2 * NS + 4) * 8;  // + static tables (2 x TBLB)
};

__device__ __forceinline__ void consumers_sync() {  // named barrier 1: the 8 consumer warps
    asm volatile("bar.sync 1, %0;\n" ::"n"(kThreads) : "memory");
}

// Scores this thread's rows of one staged chunk against table `tbl` (a static
// shared array, so each lookup is LDS [code offset + immediate]).
template <class C, int BITS, bool MAXMIN>
__device__ __forceinline__ void score_rows(const float* tbl, const unsigned char* stage, uint32_t pos, uint32_t n,
                                           float* out) {
    constexpr int LV = C::LV, W = C::W, U = C::U, CPW = C::CPW, NT = C::NT;
    constexpr int D = W * 32 / BITS;
    const uint32_t tid = threadIdx.x, lane = tid & 31;
#pragma unroll
    for (int j = 0; j < kRowsPerThread; ++j) {
        const uint32_t r = tid + j * kThreads;
        if (r - lane >= n) break;  // the warp's 32 rows lie past the chunk's end
        const uint32_t key = code_row_key(pos + r, W);
        uint32_t wd[NT][W];
#pragma unroll
        for (int a = 0; a < NT; ++a) {
            const unsigned char* row = stage + size_t(a) * C::STAGEB + r * C::ROWB;
#pragma unroll
            for (int g = 0; g < U; ++g) {
                const uint4 v = *reinterpret_cast<const uint4*>(row + ((g ^ key) << 4));
                wd[a][4 * g] = v.x;
                wd[a][4 * g + 1] = v.y;
                wd[a][4 * g + 2] = v.z;
                wd[a][4 * g + 3] = v.w;
            }
        }
        const char* tb = reinterpret_cast<const char*>(tbl);
        float acc = 0.0f;
#pragma unroll
        for (int w = 0; w < W; ++w) {
            const CodeOffsets<BITS> hi(wd[0][w]);
            const CodeOffsets<BITS> lo(MAXMIN ? wd[NT - 1][w] : 0u);
#pragma unroll
            for (int kk = 0; kk < CPW; ++kk) {
                const char* trow = tb + (w * CPW + kk) * LV * 4;
                float p = *reinterpret_cast<const float*>(trow + hi(kk));
                if (MAXMIN) p = ref_max(p, *reinterpret_cast<const float*>(trow + D * LV * 4 + lo(kk)));
                acc = __fadd_rn(acc, p);
            }
        }
        if (r < n) out[pos + r] = acc;
    }
}

template <int D, int BITS, bool ASYM, bool MAXMIN>
__global__ void __launch_bounds__(kTblThreads, kScoreCtasPerSm) k_score_tbl(LayerView L, const uint16_t* __restrict__ q,
                                                                            ScoreWork work) {
    using C = TblCfg<D, BITS, MAXMIN>;
    constexpr int LV = C::LV, W = C::W, NT = C::NT, NS = C::NS;
    extern __shared__ __align__(1024) unsigned char smem[];
    // Product tables at static shared addresses: every table load is then a single
    // LDS [offset register + immediate] (a dynamic base would add an IADD per code).
    __shared__ __align__(16) float tbl_buf[2][NT * D * LV];
    unsigned char* ring = smem;
    unsigned char* slots = smem + C::RING;
    unsigned long long* bars = reinterpret_cast<unsigned long long*>(slots + 2 * C::SLOTB);
    // bars: full[NS], empty[NS], slot_full[2], slot_empty[2]
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t it0 = work.item_begin[blockIdx.x], it1 = work.item_begin[blockIdx.x + 1];
    griddep_launch_dependents();
    if (it0 >= it1) return;
    SCORE_TRACE(0);
    if (tid == 0) {
        for (int i = 0; i < NS; ++i) {
            mbar_init(smem_u32(&bars[i]), 1);
            mbar_init(smem_u32(&bars[NS + i]), kConsumerWarps);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(smem_u32(&bars[2 * NS + i]), 1);
            mbar_init(smem_u32(&bars[2 * NS + 2 + i]), kConsumerWarps);
        }
        mbar_fence_init();
    }
    __syncthreads();
    griddep_wait();  // q and the scores buffer are step data

    if (warp == kConsumerWarps) {
        // ================================ producer ================================
        // Besides the copies, the producer publishes progress: when the last chunk of
        // an item has been consumed (its stage released by every consumer warp, after
        // their score stores), the item's centroids are added to scored[unit] behind a
        // fence, so the top-k of a unit can start as soon as its last item is done.
        if (lane != 0) return;
        uint32_t pub_unit[NS], pub_len[NS];
#pragma unroll
        for (int i = 0; i < NS; ++i) pub_len[i] = 0u;
        auto publish = [&](uint32_t st) {
#pragma unroll
            for (int i = 0; i < NS; ++i)
                if (uint32_t(i) == st && pub_len[i]) {
                    // the consumers' score stores happen-before this (their mbarrier
                    // arrive releases, the producer's wait acquires, CTA scope); the
                    // gpu-scope release reduction publishes them cumulatively
                    asm volatile("red.release.gpu.global.add.u32 [%0], %1;\n" ::"l"(work.scored + pub_unit[i]),
                                 "r"(pub_len[i])
                                 : "memory");
                    pub_len[i] = 0u;
                }
        };
        uint32_t chunk = 0;
        ScoreItem nxt = work.items[it0];
        for (uint32_t k = it0; k < it1; ++k) {
            const ScoreItem it = nxt;
            if (k + 1 < it1) nxt = work.items[k + 1];
            const uint32_t u = it.unit;
            const uint64_t seg = L.desc[u].seg;
            // item slot (k - it0) & 1 is free once every consumer warp built item k-2's table
            if (k >= it0 + 2) mbar_wait(smem_u32(&bars[2 * NS + 2 + ((k - it0) & 1)]), (((k - it0) >> 1) - 1) & 1);
            {
                unsigned char* sl = slots + ((k - it0) & 1) * C::SLOTB;
                const uint32_t bar = smem_u32(&bars[2 * NS + ((k - it0) & 1)]);
                const uint32_t qbytes = L.G * D * 2;
                mbar_expect_tx(bar, qbytes + C::PB);
                bulk_g2s(smem_u32(sl), q + size_t(u) * L.G * D, qbytes, bar);  // units are b-major
                float* prm = reinterpret_cast<float*>(sl + C::QB);
                bulk_g2s(smem_u32(prm), L.scales + size_t(u) * D, D * 4, bar);
                bulk_g2s(smem_u32(prm + D), L.zps + size_t(u) * D, D * 4, bar);
                if (MAXMIN) {
                    bulk_g2s(smem_u32(prm + 2 * D), L.scales_min + size_t(u) * D, D * 4, bar);
                    bulk_g2s(smem_u32(prm + 3 * D), L.zps_min + size_t(u) * D, D * 4, bar);
                }
            }
            for (uint32_t pos = it.start; pos < it.end; pos += kChunkRows, ++chunk) {
                const uint32_t st = chunk % NS;
                if (chunk >= uint32_t(NS)) {
                    mbar_wait(smem_u32(&bars[NS + st]), ((chunk / NS) - 1) & 1);
                    if (work.scored) publish(st);
                } else if (chunk == 2) {
                    // ramp-up: the rest of the ring is requested once the first chunk has
                    // landed — the kernel-start burst of every CTA's first two chunks then
                    // clears sooner (the scorer is LDS-bound; two stages ahead suffice)
                    mbar_wait(smem_u32(&bars[0]), 0);
                }
                const uint32_t n = min(uint32_t(kChunkRows), it.end - pos);
                const uint32_t bar = smem_u32(&bars[st]);
                mbar_expect_tx(bar, NT * n * C::ROWB);
                bulk_g2s(smem_u32(ring + size_t(st * NT) * C::STAGEB), L.codes + (seg + pos) * W, n * C::ROWB, bar);
                if (MAXMIN)
                    bulk_g2s(smem_u32(ring + size_t(st * NT + 1) * C::STAGEB), L.codes_min + (seg + pos) * W,
                             n * C::ROWB, bar);
#pragma unroll
                for (int i = 0; i < NS; ++i)
                    if (uint32_t(i) == st) {
                        pub_unit[i] = u;
                        pub_len[i] = pos + n >= it.end ? it.end - it.start : 0u;
                    }
            }
        }
        if (work.scored)  // the chunks still in flight
            for (uint32_t j = chunk > uint32_t(NS) ? chunk - NS : 0u; j < chunk; ++j) {
                mbar_wait(smem_u32(&bars[NS + j % NS]), (j / NS) & 1);
                publish(j % NS);
            }
        return;
    }

    // ================================ consumers =================================
    const int mid = (1 << (BITS - 1)) - 1;
    uint32_t chunk = 0;
    ScoreItem nxt = work.items[it0];
    for (uint32_t k = it0; k < it1; ++k) {
        const ScoreItem it = nxt;
        if (k + 1 < it1) nxt = work.items[k + 1];
        const uint64_t seg = L.desc[it.unit].seg;
        // table k (buffer (k - it0) & 1) from the item slot; the buffer was last read in
        // item k-2, finished by every warp before the barrier that ended item k-1's build
        mbar_wait(smem_u32(&bars[2 * NS + ((k - it0) & 1)]), ((k - it0) >> 1) & 1);
        const unsigned char* sl = slots + ((k - it0) & 1) * C::SLOTB;
        const uint16_t* qrows = reinterpret_cast<const uint16_t*>(sl);
        const float* prm = reinterpret_cast<const float*>(sl + C::QB);
        const uint32_t buf = (k - it0) & 1;
        float* tbl = tbl_buf[buf];
        for (uint32_t e = tid; e < uint32_t(NT * D * LV); e += kThreads) {
            const uint32_t t = e / (D * LV), c = (e / LV) % D, code = e % LV;
            float qc = bf16f(qrows[c]);  // left-to-right fp32 group sum
            for (uint32_t g = 1; g < L.G; ++g) qc = __fadd_rn(qc, bf16f(qrows[g * D + c]));
            const float sc = prm[t * 2 * D + c], zp = prm[t * 2 * D + D + c];
            const float deq = ASYM ? __fadd_rn(zp, __fmul_rn(float(code), sc))
                                   : __fmul_rn(float(int(code) - mid), sc);
            tbl[e] = __fmul_rn(qc, deq);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&bars[2 * NS + 2 + ((k - it0) & 1)]));  // slot read
        consumers_sync();
        SCORE_TRACE(2 + int(k - it0));

        float* out = L.scores + seg;
        for (uint32_t pos = it.start; pos < it.end; pos += kChunkRows, ++chunk) {
            const uint32_t st = chunk % NS;
            const uint32_t n = min(uint32_t(kChunkRows), it.end - pos);
            mbar_wait(smem_u32(&bars[st]), (chunk / NS) & 1);
            const unsigned char* stage = ring + size_t(st * NT) * C::STAGEB;
            if (buf) score_rows<C, BITS, MAXMIN>(tbl_buf[1], stage, pos, n, out);
            else score_rows<C, BITS, MAXMIN>(tbl_buf[0], stage, pos, n, out);
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&bars[NS + st]));
        }
    }
    SCORE_TRACE(1);
}

// Direct path for int8 codes (a 256-entry table per channel would not fit).
template <int D, bool ASYM, bool MAXMIN>
__global__ void __launch_bounds__(kThreads) k_score_int8(LayerView L, const uint16_t* q, ScoreWork work) {
    constexpr int W = D / 4;
    __shared__ float qs[D];
    __shared__ float prm[4][D];
    griddep_launch_dependents();
    griddep_wait();
    const uint32_t it_end = work.item_begin[blockIdx.x + 1];
    for (uint32_t it_i = work.item_begin[blockIdx.x]; it_i < it_end; ++it_i) {
        const ScoreItem it = work.items[it_i];
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
        for (uint32_t i = it.start + threadIdx.x; i < it.end; i += kThreads) {
            float acc = 0.0f;
            for (int w = 0; w < W; ++w) {
                const size_t at = size_t(i) * W + code_word_pos(i, w, W);
                const uint32_t word = __ldg(codes + at);
                const uint32_t wlo = MAXMIN ? __ldg(codes_lo + at) : 0u;
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
        __syncthreads();
    }
}

// Full-precision store (EngineConfig::quant == nullopt): engine.cpp:21-32.
template <int D, bool MAXMIN>
__global__ void __launch_bounds__(kThreads) k_score_f32(LayerView L, const uint16_t* q, ScoreWork work) {
    __shared__ float qs[D];
    griddep_launch_dependents();
    griddep_wait();
    const uint32_t it_end = work.item_begin[blockIdx.x + 1];
    for (uint32_t it_i = work.item_begin[blockIdx.x]; it_i < it_end; ++it_i) {
        const ScoreItem it = work.items[it_i];
        const UnitDesc du = L.desc[it.unit];
        load_query<D>(L, du, q, qs);
        __syncthreads();
        for (uint32_t i = it.start + threadIdx.x; i < it.end; i += kThreads) {
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
        __syncthreads();
    }
}

template <int D, int BITS, bool ASYM, bool MAXMIN>
void launch_tbl(const LayerView& L, const uint16_t* q, const ScoreWork& w, cudaStream_t s) {
    launch_pdl(k_score_tbl<D, BITS, ASYM, MAXMIN>, dim3(w.grid), dim3(kTblThreads), TblCfg<D, BITS, MAXMIN>::SMEM, s,
               L, q, w);
}

template <int D, int BITS, bool ASYM, bool MAXMIN>
cudaError_t tbl_attr() {
    return cudaFuncSetAttribute(k_score_tbl<D, BITS, ASYM, MAXMIN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                int(TblCfg<D, BITS, MAXMIN>::SMEM));
}

template <int D, int BITS>
cudaError_t tbl_attrs() {
    cudaError_t e = tbl_attr<D, BITS, false, false>();
    if (e == cudaSuccess) e = tbl_attr<D, BITS, false, true>();
    if (e == cudaSuccess) e = tbl_attr<D, BITS, true, false>();
    if (e == cudaSuccess) e = tbl_attr<D, BITS, true, true>();
    return e;
}

template <int D>
cudaError_t score_d(const LayerView& L, const uint16_t* q, const ScoreWork& w, cudaStream_t s) {
    const bool asym = L.mode == ABSP_QUANT_ASYM;
    const bool mm = L.method == ABSP_CENTROID_MAXMIN;
#define ABSP_SCORE(KERNEL, ...) launch_pdl(KERNEL<__VA_ARGS__>, dim3(w.grid), dim3(kThreads), 0, s, L, q, w)
#define ABSP_TBL(...) launch_tbl<__VA_ARGS__>(L, q, w, s)
    if (L.bits == 0) {
        if (mm) ABSP_SCORE(k_score_f32, D, true);
        else ABSP_SCORE(k_score_f32, D, false);
    } else if (L.bits == 8) {
        if (asym) { if (mm) ABSP_SCORE(k_score_int8, D, true, true); else ABSP_SCORE(k_score_int8, D, true, false); }
        else      { if (mm) ABSP_SCORE(k_score_int8, D, false, true); else ABSP_SCORE(k_score_int8, D, false, false); }
    } else if (L.bits == 4) {
        if (asym) { if (mm) ABSP_TBL(D, 4, true, true); else ABSP_TBL(D, 4, true, false); }
        else      { if (mm) ABSP_TBL(D, 4, false, true); else ABSP_TBL(D, 4, false, false); }
    } else {
        if (asym) { if (mm) ABSP_TBL(D, 2, true, true); else ABSP_TBL(D, 2, true, false); }
        else      { if (mm) ABSP_TBL(D, 2, false, true); else ABSP_TBL(D, 2, false, false); }
    }
#undef ABSP_TBL
#undef ABSP_SCORE
    return cudaGetLastError();
}

}  // namespace

#ifdef ABSP_ATTN_TRACE
cudaError_t debug_score_trace(void* dst, size_t bytes) {
    return cudaMemcpyFromSymbol(dst, g_score_trace, bytes);
}
#endif

cudaError_t init_score_attributes() {
    cudaError_t e = tbl_attrs<64, 2>();
    if (e == cudaSuccess) e = tbl_attrs<64, 4>();
    if (e == cudaSuccess) e = tbl_attrs<128, 2>();
    if (e == cudaSuccess) e = tbl_attrs<128, 4>();
    return e;
}

cudaError_t launch_score(const LayerView& L, const uint16_t* q, const ScoreWork& work, cudaStream_t s,
                         int* launches) {
    ++*launches;
    if (L.D == 64) return score_d<64>(L, q, work, s);
    return score_d<128>(L, q, work, s);
}

}  // namespace absp

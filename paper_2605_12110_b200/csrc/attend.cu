// Kernel 3: variable-block-size sparse paged flash-decoding with split-KV
// partials and a fused log-sum-exp merge (sm_100a).
//
// Reference: sparse_attention / attend_rows (engine.cpp:180-210, 285-327):
// softmax(q . k / sqrt(d)) . v over the rows of the selected blocks, rows
// resolved through the page table (block_to_pages, kv_cache.cpp:118-138). The
// PageSpan objects of populate_page_spans (engine.cpp:271-283) become the page
// list the top-k kernel resolves; no gather copy, no per-step allocation.
//
// Work: the selection of unit u = (b, h) is cut into chunks of E = 128/B
// consecutive entries (128 rows = 128/P whole pages). All chunks of all units form
// one list; a persistent grid (one CTA per SM) takes contiguous ranges of it, so
// every SM streams the same number of KV bytes whatever the block sizes.
//
// CTA = 8 consumer warps + 2 or 4 producer warps, 3-stage mbarrier ring of 64 KB stages:
//   producers: lane s handles page slot s of the chunk two ahead (page list
//              prefetched with independent loads); even warps issue one cp.async.bulk
//              per page for K, odd warps for V (4 warps for pages of <= 4 rows: each
//              pair over half of the slots) — the TMA bulk-copy engine, 1 instruction
//              per 1-4 KB page — and warp 0 one for the unit's G query rows, all
//              completing on the stage's full barrier. In the decode step a unit is started as soon
//              as its selection is published (per-unit ready flag, acquire), not
//              when the whole top-k grid has finished. (A copy-only probe of this pipeline streams
//              scattered 4 KB pages at 97% of measured HBM bandwidth.)
//   consumers: warp w owns rows [16w, 16w+16) of every chunk and is an independent
//              split with its own fp32 online-softmax state: S^T = K Q^T on
//              mma.m16n8k16 (M = 16 KV rows, N = 8 query heads of the GQA group,
//              K = d), P through a per-warp smem tile (bf16 hi + bf16 residual,
//              ~16 mantissa bits), O^T += V^T P^T (M = 16 channels x d/16 tiles,
//              N = 8 heads, K = the warp's 16 rows). A warp takes its fragments
//              into registers and releases the stage before the softmax/PV math, so
//              a stage is held only for QK + ldmatrix. At the end of a run of chunks
//              of one unit (a unit boundary in the CTA's range, or the range's end)
//              the 8 warps combine their online-softmax states in shared memory (max
//              rescale, then each thread sums the 8 warps' o values of its columns)
//              into ONE partial (m, l, o[G][d]) per (unit, CTA run), written to global
//              memory; the CTA completing a unit (acq_rel counter) queues its LSE merge
//              over the unit's R runs (R <= 16: one L2 round trip), done after the
//              chunk loop (one warp per (unit, head)).
//
// Bank conflicts without TMA swizzle: a page lands contiguously in smem, so rows
// of one page are 256 B apart (same banks). Page slots are staggered by 16 B and
// logical row i of a chunk is (slot i % NS, row i / NS), NS = 128/P: the 8 rows of
// an ldmatrix phase come from 8 different slots, i.e. 8 distinct 16 B bank groups
// (P <= 16). Softmax is permutation-invariant over rows and P uses the same
// permutation, so the result is unchanged.
#include "absp_internal.cuh"
#include "ptx.cuh"

#include <math.h>

namespace absp {
namespace {

constexpr int kRows = kAttnChunkRows;    // 128 rows per chunk / stage
constexpr int kWarps = kAttnSplits;      // consumer warps = splits per chunk (8)
constexpr int kConsumers = 32 * kWarps;
// Producer warps per CTA (a template parameter chosen at launch from the page size,
// attend_producers): even warps issue the K copies, odd ones the V copies. Two warps
// while a stage is at most 32 bulk copies (pages of >= 8 rows); smaller pages take 4,
// each pair over half of the page slots.
__host__ __device__ constexpr int attend_producers(uint32_t P) { return 2 * (kRows / P) <= 32 ? 2 : 4; }
constexpr int kStages = 3;
constexpr int kWarpRows = kRows / kWarps;  // 16
constexpr int kPStride = kWarpRows + 8;    // bf16 row stride of a P tile (bank-conflict free)
constexpr int kMaxSlots = kRows;           // P >= 1
constexpr int kMaxPend = 32;               // units completed by one CTA

// Optional timeline instrumentation (debug builds with -DABSP_ATTN_TRACE): per CTA,
// globaltimer stamps of the producer's issues, warp 0's data arrivals / releases,
// flushes and merges. Read back with absp_debug_attn_trace.
#ifdef ABSP_ATTN_TRACE
constexpr int kTraceSlots = 256;
__device__ unsigned long long g_attn_trace[160 * kTraceSlots];
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define ATTN_TRACE(slot) \
    do { if (blockIdx.x < 160 && (slot) < kTraceSlots) g_attn_trace[blockIdx.x * kTraceSlots + (slot)] = gtime(); } while (0)
#else
#define ATTN_TRACE(slot) do {} while (0)
#endif

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ uint32_t atom_add_acq_rel(uint32_t* p, uint32_t v) {
    uint32_t old;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;\n" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}

__device__ __forceinline__ void consumer_sync() {  // named barrier 1: consumer warps only
    asm volatile("bar.sync 1, %0;\n" ::"n"(kConsumers) : "memory");
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& a0, uint32_t& a1, uint32_t& a2,
                                        uint32_t& a3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3)
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& a0, uint32_t& a1, uint32_t& a2,
                                          uint32_t& a3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3)
                 : "r"(addr));
}
__device__ __forceinline__ void mma_bf16(float* c, uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};\n"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint16_t f2bf(float f) {
    uint32_t u = __float_as_uint(f);
    u += 0x7fffu + ((u >> 16) & 1u);
    return uint16_t(u >> 16);
}

struct StageMeta {
    __align__(16) uint16_t q[8 * 128];  // the chunk's unit's G query rows (bf16)
    uint32_t unit;
    uint32_t chunk;             // bit 31: some row of the chunk carries no token
    __align__(4) uint8_t valid[kMaxSlots];   // valid rows per page slot (0..P; P <= 128)
};

template <int D>
struct SmemHead {  // fixed-size part after the stage tiles
    unsigned long long full[kStages];
    unsigned long long empty[kStages];
    StageMeta meta[kStages];
    uint32_t npend;          // units this CTA completed (merged after the chunk loop)
    uint32_t merge_now;      // a completed unit that did not fit the queue
    uint32_t pend[kMaxPend];
    uint16_t p[kWarps][2][8 * kPStride];  // per-warp P tile: bf16 hi + bf16 residual
    float2 cm[kWarps][8];    // run combine: per-warp (m, l) per head
    // then (dynamic): float red[kWarps][HP][D], the run combine's o staging, HP heads a pass
};

__host__ __device__ constexpr uint32_t tile_bytes(uint32_t D, uint32_t P) {
    return ((kRows * D * 2 + (kRows / P) * 16) + 127) / 128 * 128;
}

// CTA c owns work items [c*W/C, (c+1)*W/C).
__device__ __forceinline__ uint32_t range_begin(uint32_t c, uint32_t W, uint32_t C) {
    return uint32_t((uint64_t(c) * W) / C);
}

template <int D, int NPROD>
__global__ void __launch_bounds__(kConsumers + 32 * NPROD, 1) k_attn(LayerView L, const uint16_t* __restrict__ q,
                                                      PageList pages, uint32_t* __restrict__ ready,
                                                      const uint32_t* __restrict__ chunk_unit,
                                                      const uint32_t* __restrict__ chunk_idx,
                                                      const uint32_t* __restrict__ chunk_base,
                                                      const uint32_t* __restrict__ unit_run,
                                                      uint32_t n_work, uint32_t max_runs, uint32_t hp,
                                                      float* __restrict__ part_o,
                                                      float* __restrict__ part_ml,
                                                      uint32_t* __restrict__ unit_done,
                                                      float* __restrict__ out) {
    constexpr int MT = D / 16;  // 16-channel PV m-tiles (each warp covers every channel)
    extern __shared__ __align__(1024) unsigned char smem[];
    const uint32_t P = L.P;
    const uint32_t NS = kRows / P;  // page slots per chunk
    const uint32_t TB = tile_bytes(D, P);
    const uint32_t slot_stride = P * D * 2 + 16;
    SmemHead<D>& sh = *reinterpret_cast<SmemHead<D>*>(smem + kStages * 2 * TB);
    float* red = reinterpret_cast<float*>(smem + kStages * 2 * TB + ((sizeof(SmemHead<D>) + 15) & ~size_t(15)));
    const uint32_t smem_base = smem_u32(smem);

    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    static_assert(NPROD == 2 || NPROD == 4, "producer warps come in K / V pairs");
    constexpr uint32_t nprod = NPROD;
    const uint32_t w_begin = range_begin(blockIdx.x, n_work, gridDim.x);
    const uint32_t w_end = range_begin(blockIdx.x + 1, n_work, gridDim.x);
    // the producer's first 32 chunk descriptors (layout data, written before any step):
    // loaded before anything else so no fetch waits on them
    uint32_t cu_pre = 0, ci_pre = 0;
    if (warp >= kWarps && w_begin + lane < w_end) {
        cu_pre = __ldg(chunk_unit + w_begin + lane);
        ci_pre = __ldg(chunk_idx + w_begin + lane);
    }

    if (tid == 0) {
        sh.npend = 0u;
        for (int s = 0; s < kStages; ++s) {
            mbar_init(smem_u32(&sh.full[s]), nprod);  // one arrive (+ expect_tx) per producer warp
            mbar_init(smem_u32(&sh.empty[s]), kWarps);  // every consumer warp
        }
        mbar_fence_init();
    }
    if (tid == 0) ATTN_TRACE(0);
    griddep_launch_dependents();
    __syncthreads();
    // Page lists, q, partial buffers and unit counters are step data. In the decode step
    // the per-unit ready flags order this kernel after its predecessors (a flag is
    // raised after the top-k kernel's own wait); otherwise wait for the previous grid.
    if (!ready) griddep_wait();

    if (warp >= kWarps) {
        // ============================ producers ===============================
        // NPROD warps walk the same chunks: warp 0 writes the stage meta and issues the
        // q copy, even warps the K copies, odd warps the V copies of their slot group.
        // Bulk copies are issued one lane at a time, so one warp issuing a whole stage
        // caps small pages (P = 4: 64 copies of 1 KB per stage) at ~3.3 TB/s; two warps
        // reach ~5.9 TB/s (tools/bw_probe.cu, profiles/r2/bw_probe_producers.txt).
        const uint32_t pw = warp - kWarps;
        const bool kw = pw == 0, vw = (pw & 1) != 0;
        constexpr uint32_t groups = nprod / 2;
        const uint32_t grp = pw >> 1;  // slot group: slots s with s % groups == grp (groups: 1 or 2)
        // The page list (resolved by the top-k kernel, laid out by global chunk index)
        // of chunk w+2 is fetched while chunk w waits for a free stage: one round trip
        // of independent loads, two chunks ahead of the copy issue. Lane k*32+l owns
        // page slot k*32+l (NS <= 128 slots -> up to 4 per lane).
        constexpr int SPL = kMaxSlots / 32;
        struct Pref {
            uint32_t u, c, gp[SPL], vl[SPL];
        };
        uint32_t pu = 0xffffffffu;  // last unit whose ready flag was acquired
        auto fetch = [&](uint32_t w, Pref& f) {
            if (w >= w_end) return;
            if (w - w_begin < 32u) {
                f.u = __shfl_sync(0xffffffffu, cu_pre, w - w_begin);
                f.c = __shfl_sync(0xffffffffu, ci_pre, w - w_begin);
            } else {
                f.u = __ldg(chunk_unit + w);
                f.c = __ldg(chunk_idx + w);
            }
            if (ready && f.u != pu) {  // decode step: the unit's page list must be published
                pu = f.u;
                for (uint32_t ns = 32; ld_acquire(ready + size_t(pu) * kReadyStride) == 0u; ns = min(2 * ns, 256u))
                    __nanosleep(ns);
                // the unit's q rows may have been written by the selection with generic
                // stores (host-resident q, select.cu q_copy): order them before our TMA reads
                asm volatile("fence.proxy.async.global;\n" ::: "memory");
            }
            const size_t base = size_t(w) * NS;
#pragma unroll
            for (int k = 0; k < SPL; ++k) {
                const uint32_t s = k * 32 + lane;
                f.gp[k] = s < NS ? __ldcg(pages.page + base + s) : 0u;
                f.vl[k] = s < NS ? __ldcg(pages.valid + base + s) : 0u;
            }
        };
        Pref f0{}, f1{};
        fetch(w_begin, f0);
        fetch(w_begin + 1, f1);
        uint32_t stage = 0, phase = 0;
        for (uint32_t w = w_begin; w < w_end; ++w) {
            const uint32_t u = f0.u, c = f0.c;
            uint32_t gp[SPL], vl[SPL];
#pragma unroll
            for (int k = 0; k < SPL; ++k) {
                gp[k] = f0.gp[k];
                vl[k] = f0.vl[k];
            }
            f0 = f1;
            fetch(w + 2, f1);  // its loads fly while this chunk waits for a free stage
            mbar_wait(smem_u32(&sh.empty[stage]), phase ^ 1);
            StageMeta& mt = sh.meta[stage];
            const uint32_t kdst = smem_base + stage * 2 * TB;
            const uint32_t full = smem_u32(&sh.full[stage]);
            uint32_t bytes = 0, invalid = 0;
            if (!kw) {  // K or V copies of this warp's slot group only
#pragma unroll
                for (int k = 0; k < SPL; ++k) {
                    const bool mine = vl[k] && ((k * 32 + lane) & (groups - 1)) == grp;
                    bytes += __reduce_add_sync(0xffffffffu, mine ? P * D * 2 : 0u);
                }
                if (lane == 0) mbar_expect_tx(full, bytes);
                __syncwarp();
                const uint32_t dst0 = kdst + (vw ? TB : 0u);
                const uint16_t* pool = vw ? L.v_pool : L.k_pool;
#pragma unroll
                for (int k = 0; k < SPL; ++k) {
                    const uint32_t s = k * 32 + lane;
                    if (s < NS && vl[k] && (s & (groups - 1)) == grp)
                        bulk_g2s(dst0 + s * slot_stride, pool + size_t(gp[k]) * P * D, P * D * 2, full);
                }
                if (++stage == kStages) {
                    stage = 0;
                    phase ^= 1;
                }
                continue;
            }
#pragma unroll
            for (int k = 0; k < SPL; ++k) {
                const uint32_t s = k * 32 + lane;
                bytes += __reduce_add_sync(0xffffffffu, vl[k] && (s & (groups - 1)) == 0 ? P * D * 2 : 0u);
                invalid |= __ballot_sync(0xffffffffu, s < NS && vl[k] < P);
                // valid[] is stored by lane 0, the thread whose arrive on `full` (release)
                // publishes the stage: 4 slots per word, gathered by shuffles
#pragma unroll
                for (int m = 0; m < 8; ++m) {
                    if (k * 32 + 4 * m >= int(NS)) break;  // warp-uniform
                    uint32_t wv = 0;
#pragma unroll
                    for (int e = 0; e < 4; ++e) wv |= __shfl_sync(0xffffffffu, vl[k], 4 * m + e) << (8 * e);
                    if (lane == 0) reinterpret_cast<uint32_t*>(mt.valid)[k * 8 + m] = wv;
                }
            }
            if (lane == 0) {
                mt.unit = u;
                mt.chunk = c | (invalid ? 0x80000000u : 0u);
                // the unit's G query rows ride along (units are b-major: the q row block
                // of unit u = b*H + h starts at u * G * D)
                mbar_expect_tx(full, bytes + L.G * D * 2);
                bulk_g2s(smem_u32(mt.q), q + size_t(u) * L.G * D, L.G * D * 2, full);
            }
            __syncwarp();
#pragma unroll
            for (int k = 0; k < SPL; ++k) {
                const uint32_t s = k * 32 + lane;
                if (s < NS && vl[k] && (s & (groups - 1)) == 0)  // gp = head * pool_pages + page
                    bulk_g2s(kdst + s * slot_stride, L.k_pool + size_t(gp[k]) * P * D, P * D * 2, full);
            }
            if (lane == 0) ATTN_TRACE(1 + (w - w_begin));  // producer issued chunk
            if (++stage == kStages) {
                stage = 0;
                phase ^= 1;
            }
        }
        return;
    }

    // ============================== consumers =================================
    const uint32_t g = lane >> 2, t4 = lane & 3;
    const uint32_t G = L.G;
    const float scale_log2 = rsqrtf(float(D)) * 1.4426950408889634f;
    const uint32_t ns_log = 31 - __clz(NS);  // NS = 128 / P is a power of two
    // logical row i of a chunk -> byte offset inside a tile
    auto row_off = [&](uint32_t i) -> uint32_t {
        return (i & (NS - 1)) * slot_stride + (i >> ns_log) * (D * 2);
    };
    const uint32_t row0 = warp * kWarpRows;
    // per-thread smem offsets, identical for every chunk:
    //   QK  A = K rows (ldmatrix): lanes 0-15 rows 0-15 at k-chunk 0, lanes 16-31 at chunk 1
    //   PV  A = V^T (ldmatrix.trans): lanes 0-7 rows 0-7 ch 0, 8-15 rows 0-7 ch 8,
    //       16-23 rows 8-15 ch 0, 24-31 rows 8-15 ch 8
    const uint32_t qk_off = row_off(row0 + (lane & 7) + ((lane >> 3) & 1) * 8) + (lane >> 4) * 16;
    const uint32_t pv_off = row_off(row0 + (lane & 7) + ((lane >> 4) & 1) * 8) + ((lane >> 3) & 1) * 16;
    uint32_t rv_slot[2], rv_row[2];
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
        const uint32_t row = row0 + g + hh * 8;
        rv_slot[hh] = row & (NS - 1);
        rv_row[hh] = row >> ns_log;
    }
    uint16_t* pt0 = sh.p[warp][0];
    uint16_t* pt1 = sh.p[warp][1];

    uint32_t cur_u = 0xffffffffu, seg_first = 0, seg_last = 0;
    float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.0f, 0.0f};
    float o[MT][4];
    uint32_t qb[D / 16][2];

    // Partial slot of (unit, run): a run is the part of a unit's chunks one CTA processes
    // (CTA ranges are contiguous, so run r of unit u belongs to CTA first_cta(u) + r).
    // part_o [slot][8][D] (heads < G used), part_ml [slot][8] x (m, l).
    auto slot_of = [&](uint32_t unit, uint32_t run) -> size_t { return size_t(unit) * max_runs + run; };

    // LSE merge of the R run partials of unit mu for query head h into `out` (one warp).
    // Every slot of the unit's runs is written each step; with R <= 16 all loads are
    // issued before any is used (one L2 round trip). Lanes own D/32 contiguous channels.
    auto merge = [&](uint32_t mu, uint32_t h) {
        constexpr int PER = D / 32;
        const uint32_t R = unit_run[mu] >> 16;
        const float* mlu = part_ml + slot_of(mu, 0) * 16 + h * 2;
        const float* pou = part_o + (slot_of(mu, 0) * 8 + h) * D + lane * PER;
        float acc[PER];
#pragma unroll
        for (int i = 0; i < PER; ++i) acc[i] = 0.0f;
        float lpart = 0.0f, M = -INFINITY;
        for (uint32_t base = 0; base < R; base += 16) {
            const uint32_t n = min(16u, R - base);
            float v[16][PER];
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const float* src = pou + size_t(base + j) * 8 * D;
                if (uint32_t(j) < n) {
                    if (PER == 4) {
                        const float4 t = __ldcg(reinterpret_cast<const float4*>(src));
                        v[j][0] = t.x; v[j][1] = t.y; v[j][2 % PER] = t.z; v[j][3 % PER] = t.w;
                    } else {
                        const float2 t = __ldcg(reinterpret_cast<const float2*>(src));
                        v[j][0] = t.x; v[j][1 % PER] = t.y;
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < PER; ++i) v[j][i] = 0.0f;
                }
            }
            const float mv = lane < n ? __ldcg(mlu + (base + lane) * 16) : -INFINITY;
            const float lv = lane < n ? __ldcg(mlu + (base + lane) * 16 + 1) : 0.0f;
            float Mw = mv;
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) Mw = fmaxf(Mw, __shfl_xor_sync(0xffffffffu, Mw, off));
            const float Mn = fmaxf(M, Mw);
            if (Mn == -INFINITY) continue;  // nothing live so far (warp-uniform)
            const float r = M == -INFINITY ? 0.0f : exp2f(M - Mn);
            lpart *= r;
#pragma unroll
            for (int i = 0; i < PER; ++i) acc[i] *= r;
            M = Mn;
            const float wl = mv == -INFINITY ? 0.0f : exp2f(mv - M);  // weight of slot base + lane
            lpart += wl * lv;
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const float wj = __shfl_sync(0xffffffffu, wl, j);
#pragma unroll
                for (int i = 0; i < PER; ++i) acc[i] += wj * v[j][i];
            }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) lpart += __shfl_xor_sync(0xffffffffu, lpart, off);
        const float inv = lpart > 0.0f ? 1.0f / lpart : 0.0f;  // an empty (rejected) selection writes zeros
        float* dst = out + (size_t(mu) * G + h) * D + lane * PER;  // out is [b][h*G + g][d], u = b*H + h
        if (PER == 4)
            *reinterpret_cast<float4*>(dst) = make_float4(acc[0] * inv, acc[1 % PER] * inv, acc[2 % PER] * inv,
                                                          acc[3 % PER] * inv);
        else
            *reinterpret_cast<float2*>(dst) = make_float2(acc[0] * inv, acc[1 % PER] * inv);
        if (ready && h == 0 && lane == 0) ready[size_t(mu) * kReadyStride] = 0u;  // every producer is past mu: re-arm
    };

    // End of a run: the 8 warps combine their states into the run's single partial
    // (shared memory, consumer barriers only), the CTA counts the run, and the CTA
    // completing the unit queues its merge for after the chunk loop.
    auto flush = [&]() {
        float lsum[2] = {l_run[0], l_run[1]};
#pragma unroll
        for (int hc = 0; hc < 2; ++hc)
#pragma unroll
            for (int off = 4; off < 32; off <<= 1) lsum[hc] += __shfl_xor_sync(0xffffffffu, lsum[hc], off);
        if (g == 0) {
            sh.cm[warp][2 * t4] = make_float2(m_run[0], lsum[0]);
            sh.cm[warp][2 * t4 + 1] = make_float2(m_run[1], lsum[1]);
        }
        consumer_sync();
        // every warp rescales its o to the run maximum M of each of its heads
#pragma unroll
        for (int hc = 0; hc < 2; ++hc) {
            const uint32_t h = 2 * t4 + hc;
            float M = -INFINITY;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) M = fmaxf(M, sh.cm[w][h].x);
            const float sc = (m_run[hc] == -INFINITY || M == -INFINITY) ? 0.0f : exp2f(m_run[hc] - M);
#pragma unroll
            for (int m = 0; m < MT; ++m) {
                o[m][hc] *= sc;
                o[m][2 + hc] *= sc;
            }
        }
        const size_t slot = slot_of(cur_u, blockIdx.x - (unit_run[cur_u] & 0xffffu));
        if (tid < G) {  // the run's (M, L) per head
            float M = -INFINITY, Lr = 0.0f;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) M = fmaxf(M, sh.cm[w][tid].x);
#pragma unroll
            for (int w = 0; w < kWarps; ++w) {
                const float2 c = sh.cm[w][tid];
                if (c.x != -INFINITY) Lr += c.y * exp2f(c.x - M);
            }
            part_ml[slot * 16 + tid * 2] = M;
            part_ml[slot * 16 + tid * 2 + 1] = Lr;
        }
        // o: HP heads per pass through red[warp][HP][D]; each thread then sums the 8 warps
        // of its columns and stores them
        float* po = part_o + slot * 8 * D;
        for (uint32_t h0 = 0; h0 < G; h0 += hp) {
#pragma unroll
            for (int m = 0; m < MT; ++m) {
                const uint32_t c0 = m * 16 + g;
#pragma unroll
                for (int hc = 0; hc < 2; ++hc) {
                    const uint32_t h = 2 * t4 + hc;
                    if (h >= h0 && h < h0 + hp && h < G) {
                        float* dst = red + ((warp * hp) + (h - h0)) * D;
                        dst[c0] = o[m][hc];
                        dst[c0 + 8] = o[m][2 + hc];
                    }
                }
            }
            consumer_sync();
            const uint32_t nh = min(hp, G - h0);
            for (uint32_t e = tid; e < nh * D; e += kConsumers) {
                float acc = 0.0f;
#pragma unroll
                for (int w = 0; w < kWarps; ++w) acc += red[(w * hp) * D + e];
                po[size_t(h0) * D + e] = acc;  // [h][d] rows of heads h0.. are contiguous
            }
            consumer_sync();
        }
        // run completion: the barrier orders every thread's partial stores before the
        // release; the acquire of the completing CTA makes all runs' partials visible
        if (tid == 0) {
            uint32_t now = 0xffffffffu;
            const uint32_t runs = unit_run[cur_u] >> 16;
            const uint32_t done = atom_add_acq_rel(unit_done + cur_u, 1u) + 1u;
            if (done == runs) {
                unit_done[cur_u] = 0u;  // re-arm for the next step
                if (sh.npend < uint32_t(kMaxPend)) sh.pend[sh.npend++] = cur_u;
                else now = cur_u;  // queue full: merged right away
            }
            sh.merge_now = now;
        }
        consumer_sync();
        const uint32_t now = sh.merge_now;
        if (now != 0xffffffffu)
            for (uint32_t h = warp; h < G; h += kWarps) merge(now, h);
    };

    uint32_t stage = 0, phase = 0, nflush = 0;
    (void)nflush;
    for (uint32_t w = w_begin; w < w_end; ++w) {
        mbar_wait(smem_u32(&sh.full[stage]), phase);
        if (tid == 0) ATTN_TRACE(64 + (w - w_begin));  // data arrived (warp 0)
        const StageMeta& mt = sh.meta[stage];
        const uint32_t u = mt.unit;
        const uint32_t chunk = mt.chunk & 0x7fffffffu;
        const bool new_unit = u != cur_u;
        const uint32_t k_base = smem_base + stage * 2 * TB;
        const uint32_t v_base = k_base + TB;
        const bool any_invalid = (mt.chunk >> 31) != 0;
        if (any_invalid) {
            // zero this warp's V rows that carry no token: stale or uninitialised smem
            // could hold NaN/Inf, and 0 * NaN would poison the PV product
            for (uint32_t e = lane; e < kWarpRows * (D / 8); e += 32) {
                const uint32_t row = row0 + e / (D / 8), ch = e % (D / 8);
                if ((row >> ns_log) >= mt.valid[row & (NS - 1)]) {
                    unsigned char* p = smem + stage * 2 * TB + TB + row_off(row) + ch * 16;
                    *reinterpret_cast<uint4*>(p) = make_uint4(0u, 0u, 0u, 0u);
                }
            }
            __syncwarp();
        }

        // On a unit change the new unit's Q^T fragments (B operand) come from the q rows
        // staged with the chunk: b0 = Q[g][16ks+2t..], b1 = Q[g][16ks+8+2t..]. The old
        // unit's flush below needs only o / m / l, so qb can be replaced right away.
        if (new_unit) {
            const uint16_t* qrow = mt.q + g * D;
#pragma unroll
            for (int ks = 0; ks < D / 16; ++ks) {
                qb[ks][0] = g < G ? *reinterpret_cast<const uint32_t*>(qrow + ks * 16 + 2 * t4) : 0u;
                qb[ks][1] = g < G ? *reinterpret_cast<const uint32_t*>(qrow + ks * 16 + 8 + 2 * t4) : 0u;
            }
        }
        // S^T = K Q^T over the warp's 16 rows straight from the stage (two accumulator
        // chains, even / odd ks); then the V fragments go to registers and the stage is
        // released: softmax, PV and any flush of the previous unit run on registers
        // while the producer refills it, so a stage is held only for QK + ldmatrix.
        float s[4] = {0.0f, 0.0f, 0.0f, 0.0f}, s2[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks) {
            uint32_t a0, a1, a2, a3;
            ldsm_x4(k_base + qk_off + ks * 32, a0, a1, a2, a3);
            mma_bf16((ks & 1) ? s2 : s, a0, a1, a2, a3, qb[ks][0], qb[ks][1]);
        }
        uint32_t vf[MT][4];
#pragma unroll
        for (int m = 0; m < MT; ++m) ldsm_x4_t(v_base + pv_off + m * 32, vf[m][0], vf[m][1], vf[m][2], vf[m][3]);
        bool rv[2];
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) rv[hh] = !any_invalid || rv_row[hh] < mt.valid[rv_slot[hh]];
#pragma unroll
        for (int i = 0; i < 4; ++i) s[i] += s2[i];
        // the fragments must have left shared memory before the stage is released:
        // empty asms consuming S and every V fragment register make the warp wait
        asm volatile("" ::"f"(s[0]), "f"(s[1]), "f"(s[2]), "f"(s[3]) : "memory");
#pragma unroll
        for (int m = 0; m < MT; ++m)
            asm volatile("" ::"r"(vf[m][0]), "r"(vf[m][1]), "r"(vf[m][2]), "r"(vf[m][3]) : "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&sh.empty[stage]));
        if (tid == 0) ATTN_TRACE(128 + (w - w_begin));  // stage released (warp 0)

        if (new_unit) {
            if (tid == 0) ATTN_TRACE(192 + 2 * (nflush & 3));
            if (cur_u != 0xffffffffu) flush();
            if (tid == 0) ATTN_TRACE(193 + 2 * (nflush & 3));
            ++nflush;
            cur_u = u;
            seg_first = chunk;
            m_run[0] = m_run[1] = -INFINITY;
            l_run[0] = l_run[1] = 0.0f;
#pragma unroll
            for (int m = 0; m < MT; ++m) o[m][0] = o[m][1] = o[m][2] = o[m][3] = 0.0f;
        }
        seg_last = chunk;

        // warp-local online softmax: this warp is its own split
        float mnew[2];
#pragma unroll
        for (int hc = 0; hc < 2; ++hc) {
            float mx = fmaxf(rv[0] ? s[hc] : -INFINITY, rv[1] ? s[2 + hc] : -INFINITY);
#pragma unroll
            for (int off = 4; off < 32; off <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
            mnew[hc] = fmaxf(m_run[hc], mx * scale_log2);
            const float alpha = mnew[hc] == -INFINITY ? 1.0f : exp2f(m_run[hc] - mnew[hc]);
            m_run[hc] = mnew[hc];
            l_run[hc] *= alpha;
#pragma unroll
            for (int m = 0; m < MT; ++m) {
                o[m][hc] *= alpha;
                o[m][2 + hc] *= alpha;
            }
        }
#pragma unroll
        for (int hc = 0; hc < 2; ++hc) {
            const float p0 = rv[0] ? exp2f(fmaf(s[hc], scale_log2, -mnew[hc])) : 0.0f;
            const float p1 = rv[1] ? exp2f(fmaf(s[2 + hc], scale_log2, -mnew[hc])) : 0.0f;
            l_run[hc] += p0 + p1;
            const int h = 2 * t4 + hc;
            const uint16_t h0 = f2bf(p0), h1 = f2bf(p1);
            pt0[h * kPStride + g] = h0;
            pt0[h * kPStride + g + 8] = h1;
            pt1[h * kPStride + g] = f2bf(p0 - __uint_as_float(uint32_t(h0) << 16));
            pt1[h * kPStride + g + 8] = f2bf(p1 - __uint_as_float(uint32_t(h1) << 16));
        }
        __syncwarp();
        // O^T += V^T P^T, K = the warp's 16 rows: b0 = P[head g][rows 2t..], b1 = rows 8+2t..
        const uint32_t b00 = *reinterpret_cast<const uint32_t*>(pt0 + g * kPStride + 2 * t4);
        const uint32_t b01 = *reinterpret_cast<const uint32_t*>(pt0 + g * kPStride + 8 + 2 * t4);
        const uint32_t b10 = *reinterpret_cast<const uint32_t*>(pt1 + g * kPStride + 2 * t4);
        const uint32_t b11 = *reinterpret_cast<const uint32_t*>(pt1 + g * kPStride + 8 + 2 * t4);
        __syncwarp();  // P tile reads done before the next chunk overwrites it
#pragma unroll
        for (int m = 0; m < MT; ++m) {
            mma_bf16(o[m], vf[m][0], vf[m][1], vf[m][2], vf[m][3], b00, b01);
            mma_bf16(o[m], vf[m][0], vf[m][1], vf[m][2], vf[m][3], b10, b11);
        }
        if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
        }
    }
    if (tid == 0) ATTN_TRACE(240);
    if (cur_u != 0xffffffffu) flush();
    if (tid == 0) ATTN_TRACE(241);
    consumer_sync();
    // pending merges: warp w takes (unit, head) pairs w, w + 8, ...
    const uint32_t npend = min(sh.npend, uint32_t(kMaxPend));
    for (uint32_t j = warp; j < npend * G; j += kWarps) merge(sh.pend[j / G], j % G);
    if (lane == 0) ATTN_TRACE(242 + warp);  // per-warp end (merges done)
    if (ready) griddep_wait();  // complete only after the selection grid (clean ordering downstream)
}

}  // namespace

#ifdef ABSP_ATTN_TRACE
cudaError_t debug_attn_trace(void* dst, size_t bytes) {
    return cudaMemcpyFromSymbol(dst, g_attn_trace, bytes);
}
#endif

// Shared memory of one CTA: the stage tiles, the fixed head, and the run combine's
// staging for hp heads at a time (hp <= G, as many as fit in 227 KB).
static size_t attend_smem(uint32_t D, uint32_t P, uint32_t hp) {
    const size_t head = D == 64 ? sizeof(SmemHead<64>) : sizeof(SmemHead<128>);
    return size_t(kStages) * 2 * tile_bytes(D, P) + ((head + 15) & ~size_t(15)) + size_t(kWarps) * hp * D * 4;
}
static uint32_t attend_hp(uint32_t D, uint32_t P, uint32_t G) {
    uint32_t hp = G < 4 ? G : 4;
    while (hp > 1 && attend_smem(D, P, hp) > 227 * 1024) --hp;
    return hp;
}

size_t attend_smem_bytes(uint32_t D, uint32_t P) { return attend_smem(D, P, attend_hp(D, P, 8)); }

cudaError_t init_attend_attributes() {
    for (const void* f : {reinterpret_cast<const void*>(k_attn<64, 2>), reinterpret_cast<const void*>(k_attn<64, 4>),
                          reinterpret_cast<const void*>(k_attn<128, 2>), reinterpret_cast<const void*>(k_attn<128, 4>)}) {
        const cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

cudaError_t launch_attend(const LayerView& L, const uint16_t* q, const PageList& pages, uint32_t* ready,
                          const AttendWork& wk, float* part_o, float* part_ml, float* out, cudaStream_t s,
                          int* launches) {
    const uint32_t hp = attend_hp(L.D, L.P, L.G);
    const size_t smem = attend_smem(L.D, L.P, hp);
    if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
    const uint32_t grid = wk.grid;  // = min(n_work, SMs): the CTA runs in unit_run assume it
    if (grid == 0) return cudaSuccess;
    auto go = [&](auto kern, int nprod) {
        launch_pdl(kern, dim3(grid), dim3(kConsumers + 32 * nprod), smem, s, L, q, pages, ready, wk.chunk_unit,
                   wk.chunk_idx, wk.chunk_base, wk.unit_run, wk.n_work, wk.max_runs, hp, part_o, part_ml, wk.unit_done,
                   out);
    };
    const int np = attend_producers(L.P);
    if (L.D == 64) {
        if (np == 2) go(k_attn<64, 2>, 2);
        else go(k_attn<64, 4>, 4);
    } else {
        if (np == 2) go(k_attn<128, 2>, 2);
        else go(k_attn<128, 4>, 4);
    }
    ++*launches;
    return cudaGetLastError();
}

}  // namespace absp

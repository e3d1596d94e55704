// Kernel 3: variable-block-size sparse paged flash-decoding with split-KV
// partials and a log-sum-exp merge (sm_100a).
//
// Reference: sparse_attention / attend_rows (engine.cpp:180-210, 285-327):
// softmax(q . k / sqrt(d)) . v over the rows of the selected blocks, rows
// resolved through the page table (block_to_pages, kv_cache.cpp:118-138). The
// PageSpan objects of populate_page_spans (engine.cpp:271-283) are replaced by
// index arithmetic: block j of head h covers page-table entries
// [j*B/P, (j+1)*B/P) — no gather copy, no per-step allocation.
//
// Work decomposition: unit u = (b, h) owns its G query heads and its selection.
// The selection list is cut into chunks of E = 128/B consecutive entries
// (<= 128 rows). A grid of (nsplit, units) 128-thread CTAs walks the chunks
// (split s takes chunks s, s+nsplit, ...) with an online softmax, and writes an
// unnormalised partial (m, l, o[G][d]); k_merge combines the splits of a unit
// with the usual LSE rescaling. For a full-budget decode step nsplit equals the
// chunk count, so every CTA handles exactly one chunk.
//
// Inside a chunk: all K and V rows are requested at once with 16-byte
// cp.async (zero-filled for rows past the sequence end), written into an
// XOR-swizzled tile (16 B chunk c of row r stored at c ^ (r & 7)) so the
// ldmatrix reads below are bank-conflict free. The GQA group is a dense tile:
//   S^T = K . Q^T      mma.m16n8k16 (M = 16 KV rows, N = 8 query heads, K = d)
//   O^T = V^T . P^T    mma.m16n8k16 (M = 16 channels, N = 8 heads, K = rows)
// with P materialised in shared memory as a bf16 hi/lo pair (two MMAs share the
// V fragments), so P carries ~16 mantissa bits into the PV product.
// Accumulation is fp32 throughout; tolerance vs the fp32 reference is
// 1e-3 abs + 1e-2 rel.
#include "absp_internal.cuh"

#include <math.h>

namespace absp {
namespace {

constexpr int kRows = kAttnChunkRows;  // 128
constexpr int kThreads = 128;
constexpr int kPStride = kRows + 8;    // bf16 row stride of P (bank-conflict free)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint32_t src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src),
                 "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
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

template <int D>
struct __align__(16) AttnSmem {
    uint16_t k[kRows * D];
    uint16_t v[kRows * D];
    uint16_t p[2][8 * kPStride];  // P as bf16 hi + bf16 residual (~16 mantissa bits)
    int64_t row_off[kRows];  // element offset of the row in the pool, -1 = masked
    float red[2][4][8];      // per-warp max / sum per head
};

template <int D>
__global__ void __launch_bounds__(kThreads) k_attn(LayerView L, const uint16_t* __restrict__ q,
                                                   const uint32_t* __restrict__ blocks,
                                                   uint32_t stride,
                                                   const uint32_t* __restrict__ counts,
                                                   float* __restrict__ part_o,
                                                   float* __restrict__ part_ml) {
    constexpr int CPR = D / 8;  // 16 B chunks per row
    constexpr int MT = D / 64;  // 16-channel PV m-tiles per warp
    extern __shared__ __align__(128) unsigned char smem_raw[];
    AttnSmem<D>& sm = *reinterpret_cast<AttnSmem<D>*>(smem_raw);

    const uint32_t u = blockIdx.y;
    const uint32_t split = blockIdx.x;
    const uint32_t nsplit = gridDim.x;
    const UnitDesc du = L.desc[u];
    const uint32_t B = du.block;
    const uint32_t E = B >= kRows ? 1u : kRows / B;  // selection entries per chunk
    const uint32_t cnt = counts[u];
    const uint32_t G = L.G;
    float* ml = part_ml + (size_t(u) * nsplit + split) * 16;
    if (split * E >= cnt) {  // no chunk for this split: neutral partial
        if (threadIdx.x < 8) {
            ml[threadIdx.x * 2] = -INFINITY;
            ml[threadIdx.x * 2 + 1] = 0.0f;
        }
        return;
    }
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t g = lane >> 2, t4 = lane & 3;
    const uint32_t k_base = smem_u32(sm.k), v_base = smem_u32(sm.v);
    const float scale_log2 = rsqrtf(float(D)) * 1.4426950408889634f;

    // Q^T fragments (B operand of S^T = K Q^T): b0 = Q[g][16ks+2t..], b1 = Q[g][16ks+8+2t..]
    uint32_t qb[D / 16][2];
    {
        const uint16_t* qrow = q + (size_t(du.seq) * L.H * G + size_t(du.head) * G + g) * D;
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks) {
            qb[ks][0] = g < G ? *reinterpret_cast<const uint32_t*>(qrow + ks * 16 + 2 * t4) : 0u;
            qb[ks][1] = g < G ? *reinterpret_cast<const uint32_t*>(qrow + ks * 16 + 8 + 2 * t4) : 0u;
        }
    }

    // running state for this thread's head columns h = 2*t4 + {0,1}
    float m_run[2] = {-INFINITY, -INFINITY};  // log2-scaled running max (block-uniform per head)
    float l_run[2] = {0.0f, 0.0f};            // this thread's share of the denominators
    float o[MT][4];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) o[mt][0] = o[mt][1] = o[mt][2] = o[mt][3] = 0.0f;

    for (uint32_t chunk = split; chunk * E < cnt; chunk += nsplit) {
        const uint32_t j0 = chunk * E;
        const uint32_t ne = min(E, cnt - j0);
        __syncthreads();  // previous chunk's smem reads are done
        {   // row table: pool element offset of each of the kRows rows (-1 = masked)
            const uint32_t r = tid;
            int64_t off = -1;
            const uint32_t e = r / B, w = r % B;
            if (e < ne) {
                const uint32_t blk = blocks[size_t(u) * stride + j0 + e];
                const uint32_t t = blk * B + w;
                if (t < du.n_tokens) {
                    const uint32_t page = L.page_table[size_t(du.seq) * L.max_pages + t / L.P];
                    off = int64_t(((size_t(du.head) * L.pool_pages + page) * L.P + t % L.P) * D);
                }
            }
            sm.row_off[r] = off;
        }
        __syncthreads();
#pragma unroll 4
        for (uint32_t idx = tid; idx < kRows * CPR; idx += kThreads) {
            const uint32_t r = idx / CPR, c = idx % CPR;
            const int64_t off = sm.row_off[r];
            cp_async16(k_base + (r * D + ((c ^ (r & 7)) * 8)) * 2, L.k_pool + (off < 0 ? 0 : off) + c * 8,
                       off < 0 ? 0u : 16u);
        }
        cp_async_commit();
#pragma unroll 4
        for (uint32_t idx = tid; idx < kRows * CPR; idx += kThreads) {
            const uint32_t r = idx / CPR, c = idx % CPR;
            const int64_t off = sm.row_off[r];
            cp_async16(v_base + (r * D + ((c ^ (r & 7)) * 8)) * 2, L.v_pool + (off < 0 ? 0 : off) + c * 8,
                       off < 0 ? 0u : 16u);
        }
        cp_async_commit();
        cp_async_wait<1>();
        __syncthreads();

        // S^T = K Q^T: warp w owns rows [32w, 32w+32)
        float s[2][4];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
            s[mt][0] = s[mt][1] = s[mt][2] = s[mt][3] = 0.0f;
            const uint32_t row = warp * 32 + mt * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
#pragma unroll
            for (int ks = 0; ks < D / 16; ++ks) {
                const uint32_t ch = ks * 2 + (lane >> 4);
                uint32_t a0, a1, a2, a3;
                ldsm_x4(k_base + (row * D + ((ch ^ (row & 7)) * 8)) * 2, a0, a1, a2, a3);
                mma_bf16(s[mt], a0, a1, a2, a3, qb[ks][0], qb[ks][1]);
            }
        }
        // this thread's rows: 32w + 16mt + g (+8); heads 2t4, 2t4+1
        bool rv[2][2];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
            rv[mt][0] = sm.row_off[warp * 32 + mt * 16 + g] >= 0;
            rv[mt][1] = sm.row_off[warp * 32 + mt * 16 + g + 8] >= 0;
        }
        float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int hc = 0; hc < 2; ++hc) {
                if (rv[mt][0]) mx[hc] = fmaxf(mx[hc], s[mt][hc]);
                if (rv[mt][1]) mx[hc] = fmaxf(mx[hc], s[mt][2 + hc]);
            }
#pragma unroll
        for (int hc = 0; hc < 2; ++hc)
#pragma unroll
            for (int off = 4; off < 32; off <<= 1)
                mx[hc] = fmaxf(mx[hc], __shfl_xor_sync(0xffffffffu, mx[hc], off));
        if (g == 0) {
            sm.red[0][warp][2 * t4] = mx[0];
            sm.red[0][warp][2 * t4 + 1] = mx[1];
        }
        __syncthreads();
        float mnew[2], alpha[2];
#pragma unroll
        for (int hc = 0; hc < 2; ++hc) {
            const int h = 2 * t4 + hc;
            const float cm = fmaxf(fmaxf(sm.red[0][0][h], sm.red[0][1][h]),
                                   fmaxf(sm.red[0][2][h], sm.red[0][3][h]));
            mnew[hc] = fmaxf(m_run[hc], cm * scale_log2);
            alpha[hc] = mnew[hc] == -INFINITY ? 1.0f : exp2f(m_run[hc] - mnew[hc]);
            m_run[hc] = mnew[hc];
            l_run[hc] *= alpha[hc];
        }
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
            o[mt][0] *= alpha[0];
            o[mt][1] *= alpha[1];
            o[mt][2] *= alpha[0];
            o[mt][3] *= alpha[1];
        }
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
            const uint32_t r0 = warp * 32 + mt * 16 + g;
#pragma unroll
            for (int hc = 0; hc < 2; ++hc) {
                const float p0 = rv[mt][0] ? exp2f(fmaf(s[mt][hc], scale_log2, -mnew[hc])) : 0.0f;
                const float p1 = rv[mt][1] ? exp2f(fmaf(s[mt][2 + hc], scale_log2, -mnew[hc])) : 0.0f;
                l_run[hc] += p0 + p1;
                const int h = 2 * t4 + hc;
                const uint16_t h0 = f2bf(p0), h1 = f2bf(p1);
                sm.p[0][h * kPStride + r0] = h0;
                sm.p[0][h * kPStride + r0 + 8] = h1;
                sm.p[1][h * kPStride + r0] = f2bf(p0 - __uint_as_float(uint32_t(h0) << 16));
                sm.p[1][h * kPStride + r0 + 8] = f2bf(p1 - __uint_as_float(uint32_t(h1) << 16));
            }
        }
        cp_async_wait<0>();
        __syncthreads();

        // O^T += V^T P^T: warp w owns channels [w*D/4, (w+1)*D/4)
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
            const uint32_t cbase = warp * (D / 4) + mt * 16;
#pragma unroll
            for (int ks = 0; ks < kRows / 16; ++ks) {
                const uint32_t row = ks * 16 + (lane & 7) + ((lane >> 4) & 1) * 8;
                const uint32_t ch = cbase / 8 + ((lane >> 3) & 1);
                uint32_t a0, a1, a2, a3;
                ldsm_x4_t(v_base + (row * D + ((ch ^ (row & 7)) * 8)) * 2, a0, a1, a2, a3);
#pragma unroll
                for (int part = 0; part < 2; ++part) {
                    const uint16_t* pp = sm.p[part] + g * kPStride + ks * 16 + 2 * t4;
                    mma_bf16(o[mt], a0, a1, a2, a3, *reinterpret_cast<const uint32_t*>(pp),
                             *reinterpret_cast<const uint32_t*>(pp + 8));
                }
            }
        }
    }

    // ---- partial (m, l, o) of this split ------------------------------------
#pragma unroll
    for (int hc = 0; hc < 2; ++hc)
#pragma unroll
        for (int off = 4; off < 32; off <<= 1) l_run[hc] += __shfl_xor_sync(0xffffffffu, l_run[hc], off);
    __syncthreads();
    if (g == 0) {
        sm.red[1][warp][2 * t4] = l_run[0];
        sm.red[1][warp][2 * t4 + 1] = l_run[1];
        if (warp == 0) {
            sm.red[0][0][2 * t4] = m_run[0];
            sm.red[0][0][2 * t4 + 1] = m_run[1];
        }
    }
    float* po = part_o + (size_t(u) * nsplit + split) * 8 * D;
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
        const uint32_t c0 = warp * (D / 4) + mt * 16 + g;
#pragma unroll
        for (int hc = 0; hc < 2; ++hc) {
            const uint32_t h = 2 * t4 + hc;
            if (h < G) {
                po[h * D + c0] = o[mt][hc];
                po[h * D + c0 + 8] = o[mt][2 + hc];
            }
        }
    }
    __syncthreads();
    if (tid < 8) {
        const int h = tid;
        ml[h * 2] = sm.red[0][0][h];
        ml[h * 2 + 1] = sm.red[1][0][h] + sm.red[1][1][h] + sm.red[1][2][h] + sm.red[1][3][h];
    }
}

// LSE merge of the chunk partials of one unit: one warp per query head.
template <int D>
__global__ void __launch_bounds__(256) k_merge(LayerView L, uint32_t nchunks,
                                               const float* __restrict__ part_o,
                                               const float* __restrict__ part_ml,
                                               float* __restrict__ out) {
    const uint32_t u = blockIdx.x;
    const uint32_t h = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (h >= L.G) return;
    const UnitDesc du = L.desc[u];
    const float* ml = part_ml + size_t(u) * nchunks * 16;
    float M = -INFINITY;
    for (uint32_t c = 0; c < nchunks; ++c) M = fmaxf(M, ml[c * 16 + h * 2]);
    constexpr int PER = D / 32;
    float acc[PER];
#pragma unroll
    for (int i = 0; i < PER; ++i) acc[i] = 0.0f;
    float lsum = 0.0f;
    for (uint32_t c = 0; c < nchunks; ++c) {
        const float m = ml[c * 16 + h * 2];
        if (m == -INFINITY) continue;
        const float w = exp2f(m - M);
        lsum += w * ml[c * 16 + h * 2 + 1];
        const float* po = part_o + ((size_t(u) * nchunks + c) * 8 + h) * D;
#pragma unroll
        for (int i = 0; i < PER; ++i) acc[i] += w * po[lane + 32 * i];
    }
    const float inv = 1.0f / lsum;
    float* dst = out + (size_t(du.seq) * L.H * L.G + size_t(du.head) * L.G + h) * D;
#pragma unroll
    for (int i = 0; i < PER; ++i) dst[lane + 32 * i] = acc[i] * inv;
}

template <int D>
cudaError_t attend_d(const LayerView& L, const uint16_t* q, const uint32_t* blocks,
                     uint32_t stride, const uint32_t* counts, uint32_t chunks, float* part_o,
                     float* part_ml, float* out, cudaStream_t s, int* launches) {
    const size_t smem = sizeof(AttnSmem<D>);
    k_attn<D><<<dim3(chunks, L.units), kThreads, smem, s>>>(L, q, blocks, stride, counts, part_o,
                                                            part_ml);
    k_merge<D><<<L.units, 256, 0, s>>>(L, chunks, part_o, part_ml, out);
    *launches += 2;
    return cudaGetLastError();
}

}  // namespace

cudaError_t init_attend_attributes() {
    cudaError_t e = cudaFuncSetAttribute(k_attn<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(sizeof(AttnSmem<64>)));
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(k_attn<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                int(sizeof(AttnSmem<128>)));
}

cudaError_t launch_attend(const LayerView& L, const uint16_t* q, const uint32_t* blocks,
                          uint32_t stride, const uint32_t* counts, uint32_t chunks_per_unit,
                          float* part_o, float* part_ml, float* out, cudaStream_t s,
                          int* launches) {
    if (L.D == 64)
        return attend_d<64>(L, q, blocks, stride, counts, chunks_per_unit, part_o, part_ml, out, s,
                            launches);
    return attend_d<128>(L, q, blocks, stride, counts, chunks_per_unit, part_o, part_ml, out, s,
                         launches);
}

}  // namespace absp

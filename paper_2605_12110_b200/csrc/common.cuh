// Device helpers shared by the scoring, selection and fused-select kernels.
#pragma once

#include <stdint.h>

#include "absp_internal.cuh"

namespace absp {

__device__ __forceinline__ float bf16f(uint16_t x) { return __uint_as_float(uint32_t(x) << 16); }

// std::max(a, b) as the reference writes it ((a < b) ? b : a), NaN behaviour included.
__device__ __forceinline__ float ref_max(float a, float b) { return (a < b) ? b : a; }

// Order-preserving u32 image of a score: larger score -> larger key; -0.0 == +0.0
// (the reference compares scores with !=, engine.cpp:123-128).
__device__ __forceinline__ uint32_t order_key(float f) {
    uint32_t u = __float_as_uint(f);
    if ((u & 0x7fffffffu) == 0u) u = 0u;
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// Byte offset (code * 4) of nibble/crumb k of a packed code word, for a 4-byte
// table entry. 4-bit: two masked copies hold the even / odd nibbles pre-scaled by 4
// in their bytes, and one PRMT per code extracts a byte (1.5 ALU ops per code).
template <int BITS>
struct CodeOffsets {
    uint32_t a, b, w;
    __device__ __forceinline__ explicit CodeOffsets(uint32_t word) : w(word) {
        if (BITS == 4) {
            a = (word << 2) & 0x3c3c3c3cu;  // nibbles 0,2,4,6 (x4) in bytes 0..3
            b = (word >> 2) & 0x3c3c3c3cu;  // nibbles 1,3,5,7 (x4)
        }
    }
    __device__ __forceinline__ uint32_t operator()(int k) const {
        if (BITS == 4) return __byte_perm((k & 1) ? b : a, 0u, 0x4440u | uint32_t(k >> 1));
        return ((w >> (k * BITS)) & ((1u << BITS) - 1u)) << 2;
    }
};

// Page-list slot of page pp of selection entry e: a 128-row attention chunk holds
// E = floor(128 / B) whole blocks of ppb = B / P pages in its NS = 128 / P slots, so
// entry e sits in chunk e / E at slot (e % E) * ppb + pp (the chunk's last
// NS - E * ppb slots stay empty when B does not divide 128). When B divides 128 this
// is e * ppb + pp.
__host__ __device__ __forceinline__ uint32_t page_slot(uint32_t e, uint32_t pp, uint32_t E, uint32_t ppb,
                                                       uint32_t ns) {
    return (e / E) * ns + (e % E) * ppb + pp;
}

// Resolve the ordered selection `out` (global or shared) of unit u to pool pages
// for the attention producer (the reference's populate_page_spans,
// engine.cpp:271-283): every slot of the unit's chunks is written (page_slot), empty
// ones with valid = 0. Starts with a CTA barrier so `out` written by this CTA is
// visible.
__device__ __forceinline__ void resolve_pages(const LayerView& L, const UnitDesc& du, uint32_t u,
                                              uint32_t sel_total, const uint32_t* out,
                                              const PageList& pages) {
    if (!pages.page) return;
    const uint32_t ppb = du.block / L.P;
    const uint32_t E = kAttnChunkRows / du.block;
    const uint32_t ns = pages.ns;
    const uint32_t slot_end = ((sel_total + E - 1) / E) * ns;
    const uint32_t* pt = L.page_table + size_t(du.seq) * L.max_pages;
    const uint32_t head_base = du.head * uint32_t(L.pool_pages);
    const size_t base = size_t(pages.chunk_base[u]) * ns;
    uint32_t* pg = pages.page + base;
    uint16_t* vl = pages.valid + base;
    __syncthreads();
    for (uint32_t s = threadIdx.x; s < slot_end; s += blockDim.x) {
        const uint32_t w = s % ns, ein = w / ppb, pp = w % ppb;
        const uint32_t e = (s / ns) * E + ein;
        uint32_t v = 0, page = 0;
        if (ein < E && e < sel_total) {
            const uint32_t t0 = out[e] * du.block + pp * L.P;
            if (t0 < du.n_tokens) {
                v = min(L.P, du.n_tokens - t0);
                page = head_base + __ldg(pt + t0 / L.P);
            }
        }
        pg[s] = page;
        vl[s] = uint16_t(v);
    }
}

// Publishes unit u's ordered selection `outs` (shared memory): blocks / counts, the
// page list for the attention producer and, in the decode step, the unit's ready
// flag (CTA barrier, then a gpu-scope release store by thread 0: release is
// cumulative over the CTA's writes ordered before it by the barrier, so no separate
// fence is needed — the same pattern as CUTLASS's semaphore release).
__device__ __forceinline__ void publish_selection(const LayerView& L, const UnitDesc& du, uint32_t u,
                                                  const uint32_t* outs, uint32_t n, uint32_t* blocks, uint32_t stride,
                                                  uint32_t* counts, const PageList& pages, uint32_t* ready) {
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) blocks[size_t(u) * stride + i] = outs[i];
    if (threadIdx.x == 0) counts[u] = n;
    resolve_pages(L, du, u, n, outs, pages);
    if (!ready) return;
    __syncthreads();
    if (threadIdx.x == 0)
        asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(ready + size_t(u) * kReadyStride), "r"(1u) : "memory");
}

}  // namespace absp

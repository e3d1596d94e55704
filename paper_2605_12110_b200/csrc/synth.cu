// Deterministic synthetic bf16 data (benchmark/test inputs). Integer-only up to
// one fp32 multiply, so the host twin (oracle/synth.py) produces the same bytes.
#include "absp_internal.cuh"

namespace absp {
namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

__global__ void k_fill_synth(uint16_t* dst, uint64_t count, uint64_t seed, uint64_t stream_id) {
    const uint64_t base = stream_id << 40;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < count;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t z = splitmix64(seed + 0x9e3779b97f4a7c15ull * (base + i + 1));
        const int32_t s = int32_t(z & 0xffff) + int32_t((z >> 16) & 0xffff) +
                          int32_t((z >> 32) & 0xffff) + int32_t(z >> 48) - 131070;
        const float f = __fmul_rn(float(s), 2.6429e-05f);  // ~1/37837: unit variance
        uint32_t u = __float_as_uint(f);
        u += 0x7fffu + ((u >> 16) & 1u);
        dst[i] = uint16_t(u >> 16);
    }
}

}  // namespace

cudaError_t launch_fill_synth(uint16_t* dst, uint64_t count, uint64_t seed, uint64_t stream_id,
                              cudaStream_t s) {
    if (count == 0) return cudaSuccess;
    const uint64_t blocks = (count + 255) / 256;
    k_fill_synth<<<unsigned(blocks < 148 * 64 ? blocks : 148 * 64), 256, 0, s>>>(dst, count, seed,
                                                                                  stream_id);
    return cudaGetLastError();
}

}  // namespace absp

// Instruction-fetch probe (tooling, not product): a straight-line block of ~N_INS
// independent integer instructions executed twice in a row by one warp; the first pass
// runs on a cold instruction cache (code fetched from L2 / HBM), the second warm.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/icache_probe.cu -o /tmp/icache_probe
#include <cstdio>
#include <cstdint>

#define R8(x) x x x x x x x x
#define R64(x) R8(R8(x))

__global__ void k_ic(long long* out, uint32_t seed, int flush_first) {
    if (threadIdx.x >= 32) return;
    uint32_t a = seed + threadIdx.x, b = a * 3u, c = a ^ 7u, d = a + 11u;
    long long t[3];
#pragma unroll 1
    for (int pass = 0; pass < 2; ++pass) {
        t[pass] = clock64();
        // 4 x 64 x 8 = 2048 dependent-free ALU ops (about 32 KB of SASS)
        R64(R8(a = a * 5u + b; b = b ^ (c + 3u); c = c + (d << 1); d = d * 7u + a;))
        asm volatile("" ::"r"(a), "r"(b), "r"(c), "r"(d));
    }
    t[2] = clock64();
    if (threadIdx.x == 0) {
        out[0] = t[1] - t[0];
        out[1] = t[2] - t[1];
        out[2] = a + b + c + d;
    }
}

int main() {
    long long* dv;
    cudaMalloc(&dv, 64);
    char* junk;
    const size_t jb = size_t(512) << 20;
    cudaMalloc(&junk, jb);
    for (int rep = 0; rep < 4; ++rep) {
        if (rep >= 2) cudaMemset(junk, rep, jb);  // evict L2 (code included) before the launch
        k_ic<<<1, 32>>>(dv, rep, 0);
        long long h[3];
        cudaMemcpy(h, dv, 24, cudaMemcpyDeviceToHost);
        printf("%s: first pass %lld cycles, second pass %lld cycles (%s)\n", rep >= 2 ? "L2 flushed" : "L2 warm   ",
               h[0], h[1], cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}

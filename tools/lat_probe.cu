// Latency probe (tooling, not product): dependent chains of warp shuffles, warp
// reductions (redux.sync), shared-memory loads and ballots on one warp of a 288-thread
// CTA (the finalize's shape), SM clock cycles per operation.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/lat_probe.cu -o /tmp/lat_probe
#include <cstdio>
#include <cstdint>

constexpr int kN = 256;

__global__ void k_lat(long long* out, uint32_t seed) {
    __shared__ uint32_t s[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = (i * 7 + 1) & 1023;
    __syncthreads();
    if (threadIdx.x >= 32) return;
    const uint32_t lane = threadIdx.x;
    uint32_t v = seed + lane;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < kN; ++i) v = __shfl_xor_sync(0xffffffffu, v, 1 + (i & 15)) + 1;
    long long t1 = clock64();
#pragma unroll 1
    for (int i = 0; i < kN; ++i) v = __shfl_down_sync(0xffffffffu, v, 1) + lane;
    long long t2 = clock64();
#pragma unroll 1
    for (int i = 0; i < kN; ++i) v = __reduce_add_sync(0xffffffffu, v) + lane;
    long long t3 = clock64();
    uint32_t p = v & 1023;
#pragma unroll 1
    for (int i = 0; i < kN; ++i) p = s[p];
    long long t4 = clock64();
#pragma unroll 1
    for (int i = 0; i < kN; ++i) v = __ballot_sync(0xffffffffu, (v >> (lane & 7)) & 1) + lane;
    long long t5 = clock64();
#pragma unroll 1
    for (int i = 0; i < kN; ++i) v = v * 3u + 1u;
    long long t6 = clock64();
    if (lane == 0) {
        out[0] = (t1 - t0) / kN;
        out[1] = (t2 - t1) / kN;
        out[2] = (t3 - t2) / kN;
        out[3] = (t4 - t3) / kN;
        out[4] = (t5 - t4) / kN;
        out[5] = (t6 - t5) / kN;
        out[6] = v + p;
    }
}

int main() {
    long long* d;
    cudaMalloc(&d, 8 * 8);
    for (int rep = 0; rep < 3; ++rep) {
        k_lat<<<1, 288>>>(d, rep);
        long long h[8];
        cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
        printf("cycles/op: shfl.bfly %lld  shfl.down %lld  redux.add %lld  lds(chase) %lld  ballot %lld  imad %lld  (%s)\n",
               h[0], h[1], h[2], h[3], h[4], h[5], cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}

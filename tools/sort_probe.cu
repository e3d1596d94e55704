// Micro-benchmark (tooling, not product): the finalize's register bitonic sort
// (select_core.cuh sortreg_desc) alone in one CTA of the selection's shape, clock64 cycles.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include
//        -I paper_2605_12110_b200/csrc tools/sort_probe.cu -o /tmp/sort_probe
#include <cstdio>
#include <vector>

#define SORT_PROBE
__device__ long long g_sort_clk[16];
#include "select_core.cuh"

using namespace absp::selcore;

template <int R>
__global__ void k_probe(const unsigned long long* in, unsigned long long* out, uint32_t n, long long* cyc) {
    __shared__ unsigned long long a[256 * R];
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) a[i] = in[i];
    __syncthreads();
    const long long t0 = clock64();
    sortreg_desc<R>(a, n);
    const long long t1 = clock64();
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) out[i] = a[i];
    if (threadIdx.x == 0) {
        *cyc = t1 - t0;
        for (int i = 1; i < 12; ++i) cyc[i] = g_sort_clk[i] ? g_sort_clk[i] - t0 : -1;
    }
}

int main() {
    for (int R : {4, 8}) {
        const uint32_t n = R == 4 ? 1000 : 2000;
        std::vector<unsigned long long> h(n);
        uint64_t x = 88172645463325252ull;
        for (auto& e : h) {
            x ^= x << 13; x ^= x >> 7; x ^= x << 17;
            e = x | 1ull;
        }
        unsigned long long *din, *dout;
        long long* dc;
        cudaMalloc(&din, n * 8);
        cudaMalloc(&dout, n * 8);
        cudaMalloc(&dc, 12 * 8);
        cudaMemcpy(din, h.data(), n * 8, cudaMemcpyHostToDevice);
        for (int rep = 0; rep < 3; ++rep) {
            if (R == 4) k_probe<4><<<1, kSThreads>>>(din, dout, n, dc);
            else k_probe<8><<<1, kSThreads>>>(din, dout, n, dc);
            long long cc[12];
            cudaMemcpy(cc, dc, 12 * 8, cudaMemcpyDeviceToHost);
            const long long c = cc[0];
            printf("   k-stage start cycles:");
            for (int i = 1; i < 12; ++i) printf(" %lld", cc[i]);
            printf("\n");
            std::vector<unsigned long long> o(n);
            cudaMemcpy(o.data(), dout, n * 8, cudaMemcpyDeviceToHost);
            bool ok = true;
            for (uint32_t i = 1; i < n; ++i) ok &= o[i - 1] >= o[i];
            printf("R=%d n=%u rep %d: %lld cycles (%.2f us at 1.965 GHz) sorted=%d err=%s\n", R, n, rep, c, c / 1965.0, ok,
                   cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}

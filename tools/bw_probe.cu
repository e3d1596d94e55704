// Bandwidth probe (tooling, not product): how fast can one CTA per SM stream
// scattered KV pages into shared memory?
//   mode 0: cp.async.bulk of `page` bytes per instruction into an S-stage ring of
//           `stage` bytes (producer warp issues, consumer warps only wait/arrive)
//   mode 1: plain 16 B vector loads (LDG.128) of the same pages, all warps
//   mode 2: cp.async (LDGSTS) 16 B into the same ring layout
// Pages are visited in a random permutation (like a sparse selection) over a
// 4 GiB pool. Prints GB/s. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n\t}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}

constexpr int kConsumerWarps = 4;

__global__ void k_bulk(const char* pool, const uint32_t* perm, uint32_t n_pages, uint32_t page, uint32_t stage,
                       uint32_t stages, unsigned long long* sink, long long hold_cycles) {
    extern __shared__ __align__(1024) unsigned char smem[];
    unsigned long long* full = reinterpret_cast<unsigned long long*>(smem + stages * stage);
    unsigned long long* empty = full + stages;
    const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const uint32_t per_stage = stage / page;
    const uint32_t n_chunks = n_pages / per_stage;
    const uint32_t c0 = uint64_t(blockIdx.x) * n_chunks / gridDim.x, c1 = uint64_t(blockIdx.x + 1) * n_chunks / gridDim.x;
    if (threadIdx.x == 0) {
        for (uint32_t s = 0; s < stages; ++s) {
            mbar_init(smem_u32(&full[s]), 1);
            mbar_init(smem_u32(&empty[s]), kConsumerWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    if (warp == kConsumerWarps) {
        uint32_t st = 0, ph = 0;
        for (uint32_t c = c0; c < c1; ++c) {
            mbar_wait(smem_u32(&empty[st]), ph ^ 1);
            if (lane == 0) mbar_expect_tx(smem_u32(&full[st]), stage);
            __syncwarp();
            for (uint32_t p = lane; p < per_stage; p += 32) {
                const uint32_t pg = perm[c * per_stage + p];
                bulk_g2s(smem_u32(smem + st * stage + p * page), pool + size_t(pg) * page, page, smem_u32(&full[st]));
            }
            if (++st == stages) { st = 0; ph ^= 1; }
        }
        return;
    }
    uint32_t st = 0, ph = 0;
    unsigned long long acc = 0;
    for (uint32_t c = c0; c < c1; ++c) {
        mbar_wait(smem_u32(&full[st]), ph);
        acc += smem[st * stage + threadIdx.x * 16];
        if (hold_cycles) {  // emulate consumer compute holding the stage
            const long long t0 = clock64();
            while (clock64() - t0 < hold_cycles) {}
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&empty[st]));
        if (++st == stages) { st = 0; ph ^= 1; }
    }
    if (acc == 12345) sink[0] = acc;
}

__global__ void k_ldg(const char* pool, const uint32_t* perm, uint32_t n_pages, uint32_t page, unsigned long long* sink) {
    const uint32_t p0 = uint64_t(blockIdx.x) * n_pages / gridDim.x, p1 = uint64_t(blockIdx.x + 1) * n_pages / gridDim.x;
    uint4 acc = make_uint4(0, 0, 0, 0);
    const uint32_t vec_per_page = page / 16;
    for (uint32_t p = p0; p < p1; ++p) {
        const uint4* src = reinterpret_cast<const uint4*>(pool + size_t(perm[p]) * page);
#pragma unroll 4
        for (uint32_t i = threadIdx.x; i < vec_per_page; i += blockDim.x) {
            const uint4 v = __ldcs(src + i);
            acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
        }
    }
    if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678u) sink[0] = 1;
}

int main(int argc, char** argv) {
    const size_t pool_bytes = size_t(4) << 30;
    char* pool;
    cudaMalloc(&pool, pool_bytes);
    cudaMemset(pool, 1, pool_bytes);
    unsigned long long* sink;
    cudaMalloc(&sink, 8);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t read_bytes = size_t(1) << 30;  // bytes moved per run
    struct Cfg { uint32_t page, stage, stages, run; };  // run: consecutive pages per random start
    std::vector<Cfg> cfgs = {{4096, 65536, 3, 1}, {2048, 65536, 3, 1}, {1024, 65536, 3, 1},
                             {1024, 65536, 3, 4}, {1024, 65536, 3, 16}, {2048, 65536, 3, 8}};
    const long long holds[] = {0, 2000};  // SM cycles (~0.5 ns each)
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (const Cfg& c : cfgs) {
        const uint32_t n_pages = uint32_t(read_bytes / c.page);
        const uint32_t pool_pages = uint32_t(pool_bytes / c.page);
        std::vector<uint32_t> perm(n_pages);
        srand(1);
        for (uint32_t i = 0; i < n_pages; i += c.run) {
            const uint32_t start = uint32_t((uint64_t(rand()) * 65536 + rand()) % (pool_pages - c.run));
            for (uint32_t j = 0; j < c.run && i + j < n_pages; ++j) perm[i + j] = start + j;
        }
        uint32_t* dperm;
        cudaMalloc(&dperm, n_pages * 4);
        cudaMemcpy(dperm, perm.data(), n_pages * 4, cudaMemcpyHostToDevice);
        const size_t smem = size_t(c.stages) * c.stage + 2 * c.stages * 8;
        cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        for (long long hold : holds) {
            float best = 1e30f;
            for (int rep = 0; rep < 4; ++rep) {
                cudaEventRecord(e0);
                k_bulk<<<sms, (kConsumerWarps + 1) * 32, smem>>>(pool, dperm, n_pages, c.page, c.stage, c.stages, sink, hold);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (rep) best = ms < best ? ms : best;
            }
            cudaError_t err = cudaGetLastError();
            printf("bulk page=%5u run=%2u stage=%6u stages=%2u hold=%5lld cyc : %7.1f GB/s %s\n", c.page, c.run, c.stage,
                   c.stages, hold, read_bytes / (best * 1e-3) / 1e9, err ? cudaGetErrorString(err) : "");
        }
        cudaFree(dperm);
    }
    return 0;
}

// Bandwidth probe (tooling, not product): how fast can one CTA per SM stream
// scattered KV pages into shared memory?
//   k_bulk   : cp.async.bulk of `page` bytes per instruction into an S-stage ring of
//              `stage` bytes (1 or 2 producer warps issue, consumer warps only wait/arrive)
//   k_cpasync: cp.async (LDGSTS) 16 B pieces into the same ring, 1/2/4 producer warps
//   k_ldg    : plain 16 B vector loads (LDG.128) of the same pages (not run by main)
// Finding (profiles/r2/bw_probe_producers.txt): 1 KB bulk copies from one warp cap at
// ~3.3 TB/s, from two warps ~5.9 TB/s — the per-lane issue of the copies, not the
// copy engine, is the limit; LDGSTS needs 4 warps to approach the same rates.
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
    if (warp >= kConsumerWarps) {
        const uint32_t pw = warp - kConsumerWarps, np = (blockDim.x / 32 - kConsumerWarps) * 32;
        uint32_t st = 0, ph = 0;
        for (uint32_t c = c0; c < c1; ++c) {
            mbar_wait(smem_u32(&empty[st]), ph ^ 1);
            if (pw == 0 && lane == 0) mbar_expect_tx(smem_u32(&full[st]), stage);
            asm volatile("bar.sync 1, %0;\n" ::"r"(np) : "memory");  // expect_tx before any copy lands
            for (uint32_t p = pw * 32 + lane; p < per_stage; p += np) {
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

// mode 2: the producer warp copies each page with 16-byte cp.async (LDGSTS) pieces and
// signals the stage's full barrier with cp.async.mbarrier.arrive (no TMA)
__global__ void k_cpasync(const char* pool, const uint32_t* perm, uint32_t n_pages, uint32_t page, uint32_t stage,
                          uint32_t stages, unsigned long long* sink, long long hold_cycles, uint32_t pwarps) {
    extern __shared__ __align__(1024) unsigned char smem[];
    unsigned long long* full = reinterpret_cast<unsigned long long*>(smem + stages * stage);
    unsigned long long* empty = full + stages;
    const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const uint32_t per_stage = stage / page;
    const uint32_t n_chunks = n_pages / per_stage;
    const uint32_t c0 = uint64_t(blockIdx.x) * n_chunks / gridDim.x, c1 = uint64_t(blockIdx.x + 1) * n_chunks / gridDim.x;
    if (threadIdx.x == 0) {
        for (uint32_t s = 0; s < stages; ++s) {
            mbar_init(smem_u32(&full[s]), pwarps * 32);
            mbar_init(smem_u32(&empty[s]), kConsumerWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    if (warp >= kConsumerWarps) {
        const uint32_t pw = warp - kConsumerWarps, pt = pw * 32 + lane, np = pwarps * 32;
        (void)pt; (void)np;
        uint32_t st = 0, ph = 0;
        for (uint32_t c = c0; c < c1; ++c) {
            mbar_wait(smem_u32(&empty[st]), ph ^ 1);
            // one warp instruction = 512 contiguous bytes of one page; page ids loaded once
            // per stage (lane l: pages l, l + 32) and broadcast by shuffles
            const uint32_t pg0 = lane < per_stage ? perm[c * per_stage + lane] : 0u;
            const uint32_t pg1 = lane + 32 < per_stage ? perm[c * per_stage + lane + 32] : 0u;
            for (uint32_t p = pw; p < per_stage; p += pwarps) {
                const uint32_t pg = __shfl_sync(0xffffffffu, p < 32 ? pg0 : pg1, p & 31);
                const char* src = pool + size_t(pg) * page + lane * 16;
                const uint32_t dst = smem_u32(smem + st * stage + p * page + lane * 16);
                for (uint32_t k = 0; k < page; k += 512)
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst + k), "l"(src + k) : "memory");
            }
            asm volatile("cp.async.mbarrier.arrive.noinc.shared.b64 [%0];\n" ::"r"(smem_u32(&full[st])) : "memory");
            if (++st == stages) { st = 0; ph ^= 1; }
        }
        return;
    }
    uint32_t st = 0, ph = 0;
    unsigned long long acc = 0;
    for (uint32_t c = c0; c < c1; ++c) {
        mbar_wait(smem_u32(&full[st]), ph);
        acc += smem[st * stage + threadIdx.x * 16];
        if (hold_cycles) {
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
        for (uint32_t bw : {1u, 2u})
        for (long long hold : holds) {
            float best = 1e30f;
            for (int rep = 0; rep < 4; ++rep) {
                cudaEventRecord(e0);
                k_bulk<<<sms, (kConsumerWarps + bw) * 32, smem>>>(pool, dperm, n_pages, c.page, c.stage, c.stages, sink, hold);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (rep) best = ms < best ? ms : best;
            }
            cudaError_t err = cudaGetLastError();
            printf("bulk page=%5u run=%2u stage=%6u stages=%2u pwarps=%u hold=%5lld cyc : %7.1f GB/s %s\n", c.page, c.run, c.stage,
                   c.stages, bw, hold, read_bytes / (best * 1e-3) / 1e9, err ? cudaGetErrorString(err) : "");
        }
        cudaFuncSetAttribute(k_cpasync, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        for (uint32_t pw : {1u, 2u, 4u})
            for (long long hold : holds) {
                float best = 1e30f;
                for (int rep = 0; rep < 4; ++rep) {
                    cudaEventRecord(e0);
                    k_cpasync<<<sms, (kConsumerWarps + pw) * 32, smem>>>(pool, dperm, n_pages, c.page, c.stage, c.stages,
                                                                         sink, hold, pw);
                    cudaEventRecord(e1);
                    cudaEventSynchronize(e1);
                    float ms;
                    cudaEventElapsedTime(&ms, e0, e1);
                    if (rep) best = ms < best ? ms : best;
                }
                cudaError_t err = cudaGetLastError();
                printf("cp.async page=%5u run=%2u stage=%6u stages=%2u pwarps=%u hold=%5lld cyc : %7.1f GB/s %s\n", c.page,
                       c.run, c.stage, c.stages, pw, hold, read_bytes / (best * 1e-3) / 1e9,
                       err ? cudaGetErrorString(err) : "");
            }
        cudaFree(dperm);
    }
    return 0;
}

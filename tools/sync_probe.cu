// Host round-trip probe (tooling, not product): wall time per call of a one-kernel CUDA
// graph, (a) launch + cudaStreamSynchronize, (b) launch + host spin on a pinned flag the
// kernel writes (system-scope release), (c) as (b) then cudaStreamSynchronize.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/sync_probe.cu -o /tmp/sync_probe
#include <chrono>
#include <cstdio>
#include <cstdint>

__global__ void k_flag(volatile uint32_t* flag, uint32_t v) {
    if (threadIdx.x == 0) {
        __threadfence_system();
        *flag = v;
    }
}

int main() {
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    uint32_t* flag;
    cudaHostAlloc(&flag, 64, cudaHostAllocMapped);
    *flag = 0;
    uint32_t* dflag;
    cudaHostGetDevicePointer(&dflag, flag, 0);
    uint32_t* dval;
    cudaMalloc(&dval, 4);
    // graph: one kernel writing flag = *val (the value set by a memset node before it)
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    k_flag<<<1, 32, 0, s>>>(dflag, 1u);
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    auto now = [] { return std::chrono::steady_clock::now(); };
    const int reps = 2000;
    for (int mode = 0; mode < 3; ++mode) {
        double best = 1e30;
        for (int trial = 0; trial < 3; ++trial) {
            auto t0 = now();
            for (int i = 0; i < reps; ++i) {
                *reinterpret_cast<volatile uint32_t*>(flag) = 0;
                cudaGraphLaunch(ge, s);
                if (mode == 0) {
                    cudaStreamSynchronize(s);
                } else {
                    while (*reinterpret_cast<volatile uint32_t*>(flag) == 0) {
                    }
                    if (mode == 2) cudaStreamSynchronize(s);
                }
            }
            cudaStreamSynchronize(s);
            const double us = std::chrono::duration<double, std::micro>(now() - t0).count() / reps;
            best = us < best ? us : best;
        }
        printf("%s: %.2f us per call\n",
               mode == 0 ? "launch + cudaStreamSynchronize" : mode == 1 ? "launch + spin on pinned flag" : "launch + spin + cudaStreamSynchronize",
               best);
    }
    return 0;
}

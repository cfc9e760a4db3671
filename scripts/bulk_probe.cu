// bulk_probe.cu — microbenchmark: sustained L2 -> shared memory bandwidth per SM
// with cp.async.bulk (the ring GEMM's producer path), for several copy sizes
// and numbers of copies in flight.  Source data is L2-resident (a 24 MiB
// window re-read by every CTA at staggered offsets).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 bulk_probe.cu -o bulk_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(32, 1) probe(const uint8_t* src, size_t window, int copy_bytes, int copies_per_stage,
                                               int stages, int iters, unsigned long long* cycles) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ __align__(8) uint64_t bar[8];
    if (threadIdx.x != 0) return;
    for (int s = 0; s < stages; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    const int stage_bytes = copy_bytes * copies_per_stage;
    size_t off = ((size_t)blockIdx.x * 1315423911ull) % (window - stage_bytes);
    off &= ~(size_t)1023;
    long long t0 = clock64();
    uint32_t ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int it = 0; it < iters + stages; ++it) {
        const int s = it % stages;
        if (it >= stages) {  // wait for the copy issued `stages` iterations ago
            asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W;}"
                         :: "r"(smem_u32(&bar[s])), "r"(ph[s]));
            ph[s] ^= 1;
        }
        if (it < iters) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(&bar[s])), "r"(stage_bytes));
            for (int c = 0; c < copies_per_stage; ++c) {
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             :: "r"(smem_u32(sm + s * stage_bytes + c * copy_bytes)), "l"(src + off + (size_t)c * copy_bytes),
                                "r"(copy_bytes), "r"(smem_u32(&bar[s])) : "memory");
            }
            off += stage_bytes;
            if (off + stage_bytes > window) off = 0;
        }
    }
    long long t1 = clock64();
    atomicAdd(cycles, (unsigned long long)(t1 - t0));
}

int main() {
    const size_t window = 24ull << 20;
    uint8_t* src;
    cudaMalloc(&src, window);
    cudaMemset(src, 1, window);
    unsigned long long* dc;
    cudaMalloc(&dc, 8);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    struct Cfg { int copy, per, stages; } cfgs[] = {
        {2048, 1, 4}, {4096, 1, 4}, {16384, 1, 4}, {32768, 1, 4}, {32768, 1, 6}, {24576, 2, 4}, {4096, 8, 4},
        {2048, 16, 4}, {49152, 1, 4}, {16384, 3, 4}, {8192, 6, 4}};
    for (auto c : cfgs) {
        const int iters = 400;
        for (int rep = 0; rep < 2; ++rep) {
            cudaMemset(dc, 0, 8);
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaEventRecord(e0);
            probe<<<148, 32, 200 * 1024>>>(src, window, c.copy, c.per, c.stages, iters, dc);
            cudaEventRecord(e1);
            cudaError_t err = cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            unsigned long long cyc; cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
            const double bytes = (double)c.copy * c.per * iters;
            if (rep == 1)
                printf("copy %6d x %2d per stage, %d stages: err=%d  %6.1f B/clk/SM   chip %6.2f TB/s\n", c.copy, c.per,
                       c.stages, (int)err, bytes / ((double)cyc / 148), bytes * 148 / (ms * 1e-3) / 1e12);
        }
    }
    return 0;
}

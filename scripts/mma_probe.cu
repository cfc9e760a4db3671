// mma_probe.cu — microbenchmark: sustained tcgen05.mma kind::i8 rate from
// shared memory (SS operands) for the tile shapes the ring GEMM could use.
// No global traffic: every CTA re-issues MMAs on fixed smem tiles.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 mma_probe.cu -o mma_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a) {
    return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)8 << 16) | ((uint64_t)16 << 32) | (1ull << 46);
}

template <int CG, int M, int N>
__global__ void __launch_bounds__(128, 1) probe(int iters, unsigned long long* cycles, const uint8_t* gsrc, int copy_bytes) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t bar;
    const int warp = threadIdx.x >> 5;
    constexpr uint32_t idesc = (2u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    uint32_t rank = 0;
    if (CG == 2) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (warp == 1) {
        if (CG == 1) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(smem_u32(&slot)));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(smem_u32(&slot)));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    if (CG == 2) asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;");
    else __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = slot;
    __shared__ __align__(8) uint64_t cbar;
    __shared__ volatile int stop;
    if (threadIdx.x == 0) { stop = 0; asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&cbar))); }
    __syncwarp();
    if (warp == 2 && threadIdx.x == 64 && copy_bytes > 0) {
        // concurrent L2 -> smem bulk copies (producer-like traffic) into bytes [96K, 96K+copy_bytes)
        uint32_t ph = 0;
        size_t off = (size_t)blockIdx.x * 65536;
        for (int it = 0; it < 1000000 && !stop; ++it) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(&cbar)), "r"(copy_bytes));
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         :: "r"(smem_u32(sm + 96 * 1024)), "l"(gsrc + off), "r"(copy_bytes), "r"(smem_u32(&cbar)) : "memory");
            asm volatile("{.reg .pred p; WB: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra WB;}" :: "r"(smem_u32(&cbar)), "r"(ph));
            ph ^= 1;
            off = (off + copy_bytes) % (16u << 20);
        }
    }
    if (warp == 0 && threadIdx.x == 0 && rank == 0) {
        const uint32_t a = smem_u32(sm), b = a + 64 * 1024;
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const uint32_t d = tm + (uint32_t)((j * N) % 512);
                if (CG == 1)
                    asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;}"
                                 :: "r"(d), "l"(desc(a + j * 4096)), "l"(desc(b + j * 4096)), "r"(idesc), "r"(1));
                else
                    asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;}"
                                 :: "r"(d), "l"(desc(a + j * 4096)), "l"(desc(b + j * 4096)), "r"(idesc), "r"(1));
            }
        }
        if (CG == 1)
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&bar)));
        else
            asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                         :: "r"(smem_u32(&bar)), "h"((uint16_t)3));
        asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0; @!p bra W;}" :: "r"(smem_u32(&bar)));
        long long t1 = clock64();
        atomicAdd(cycles, (unsigned long long)(t1 - t0));
    }
    if (threadIdx.x == 0) stop = 1;
    if (CG == 2 && rank == 1 && threadIdx.x == 0)
        asm volatile("{.reg .pred p; W2: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0; @!p bra W2;}" :: "r"(smem_u32(&bar)));
    __syncwarp();
    asm volatile("tcgen05.fence::before_thread_sync;");
    if (CG == 2) asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;");
    else __syncthreads();
    if (warp == 1) {
        if (CG == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tm));
        else asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" :: "r"(tm));
    }
}

template <int CG, int M, int N>
void run(const char* name, const uint8_t* gsrc = nullptr, int copy_bytes = 0, int iters_ = 2000) {
    auto k = probe<CG, M, N>;
    const int smem = 160 * 1024;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (CG == 2) cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 0);
    unsigned long long* dc;
    cudaMalloc(&dc, 8);
    const int iters = iters_;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(148);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CG; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    for (int rep = 0; rep < 2; ++rep) {
        cudaMemset(dc, 0, 8);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        cudaLaunchKernelEx(&cfg, k, iters, dc, gsrc, copy_bytes);
        cudaEventRecord(e1);
        cudaError_t err = cudaEventSynchronize(e1);
        float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
        unsigned long long cyc = 0; cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
        const int issuers = 148 / CG;
        const double cyc_per_mma = (double)cyc / issuers / (iters * 8.0);
        const double macs = (double)M * N * 32;
        const double tops = 2.0 * macs * iters * 8 * issuers / (ms * 1e-3) / 1e12;
        if (rep == 1 && name[0])
            printf("%-28s err=%d  cycles/MMA=%7.2f  MAC/clk/SM=%7.0f  chip=%7.0f TOPS (%.3f ms)\n", name, (int)err,
                   cyc_per_mma, macs / cyc_per_mma / CG, tops, ms);
    }
    cudaFree(dc);
}

int main(int argc, char** argv) {
    if (argc > 1) {   // sustained mode: the GEMM's MMA shape back-to-back for ~4 s
        const int reps = 40;
        for (int r = 0; r < reps; ++r) run<2, 256, 128>(r + 1 == reps ? "cg2 M256 N128 sustained" : "", nullptr, 0, 60000);
        return 0;
    }
    uint8_t* g; cudaMalloc(&g, 32u << 20); cudaMemset(g, 1, 32u << 20);
    run<2, 256, 128>("cg2 M256 N128 +copy 32K", g, 32768);
    run<2, 256, 128>("cg2 M256 N128 +copy 48K", g, 49152);
    run<1, 128, 128>("cg1 M128 N128 +copy 32K", g, 32768);
    run<2, 256, 256>("cg2 M256 N256 +copy 32K", g, 32768);
    run<1, 128, 64>("cg1 M128 N64");
    run<1, 128, 128>("cg1 M128 N128");
    run<1, 128, 256>("cg1 M128 N256");
    run<2, 256, 64>("cg2 M256 N64");
    run<2, 256, 128>("cg2 M256 N128");
    run<2, 256, 256>("cg2 M256 N256");
    return 0;
}

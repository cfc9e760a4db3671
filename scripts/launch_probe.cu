// launch_probe.cu — fixed cost of launching a ring_gemm-shaped kernel on B200:
// 2-CTA clusters, 384 threads, ~197 KB dynamic smem, optional TMEM alloc/dealloc,
// grid = G clusters.  Times N back-to-back launches with CUDA events, with and
// without a CUDA graph.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o launch_probe launch_probe.cu && ./launch_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(384, 1) probe_kernel(int tmem, int* sink) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t slot;
    if (tmem && threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;"
                     :: "r"((uint32_t)__cvta_generic_to_shared(&slot)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (threadIdx.x == 0 && smem[0] == 123) sink[0] = 1;
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (tmem && threadIdx.x < 32)
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" :: "r"(slot), "r"(512));
}

__global__ void plain_kernel(int* sink) {
    if (threadIdx.x == 0 && blockIdx.x == 100000) sink[0] = 1;
}

int main() {
    int* sink;
    cudaMalloc(&sink, 4);
    const int smem = 4 * 48 * 1024 + 1024 + 256;
    cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaStream_t st;
    cudaStreamCreate(&st);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int n = 200;
    struct Cfg { int clusters, smem, tmem; } cfgs[] = {
        {74, smem, 1}, {74, smem, 0}, {74, 0, 0}, {13, smem, 1}, {1, smem, 1}, {74, 100 * 1024, 1}};
    for (auto c : cfgs) {
        for (int graph = 0; graph < 2; ++graph) {
            cudaGraphExec_t ge = nullptr;
            auto body = [&] {
                for (int i = 0; i < n; ++i) probe_kernel<<<2 * c.clusters, 384, c.smem, st>>>(c.tmem, sink);
            };
            if (graph) {
                cudaGraph_t g;
                cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
                body();
                cudaStreamEndCapture(st, &g);
                cudaGraphInstantiate(&ge, g, 0);
                cudaGraphLaunch(ge, st);
            } else {
                body();
            }
            cudaStreamSynchronize(st);
            cudaEventRecord(a, st);
            if (graph) cudaGraphLaunch(ge, st); else body();
            cudaEventRecord(b, st);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            printf("clusters %3d smem %6d tmem %d graph %d: %.2f us per launch (%s)\n", c.clusters, c.smem, c.tmem,
                   graph, ms * 1e3 / n, cudaGetErrorString(cudaGetLastError()));
        }
    }
    for (int graph = 0; graph < 2; ++graph) {
        cudaEventRecord(a, st);
        for (int i = 0; i < n; ++i) plain_kernel<<<1184, 256, 0, st>>>(sink);
        cudaEventRecord(b, st);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("plain 1184x256: %.2f us per launch\n", ms * 1e3 / n);
    }
    return 0;
}

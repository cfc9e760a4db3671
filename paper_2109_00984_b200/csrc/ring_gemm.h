// ring_gemm.h — host interface of the tcgen05 limb-plane ring GEMM (internal).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace mpc {

struct RingGemmSegment {
    const uint8_t* A;        // left limb planes  (rows = M), Layout::Left
    const uint8_t* B;        // right limb planes (rows = N), Layout::Right
    int kb;                  // number of 32-K blocks of this segment (both operands)
    int64_t party_stride_A;  // bytes between parties' A planes (0 = shared, e.g. eps)
    int64_t party_stride_B;
    int64_t batch_stride_A;  // bytes between batch elements' planes (batched GEMM; 0 when batch = 1)
    int64_t batch_stride_B;
};

// 2-D tensor maps (rows of 256 B over a whole plane buffer) of the two segments' left /
// right planes, one per super-pass width (8 or 6 planes per 32-K block); filled by
// ring_gemm_launch for the 2-CTA kernel's tensor-TMA producer.
struct RingGemmTma {
    CUtensorMap a[2][2];                // [segment][pass]
    CUtensorMap b[2][2];
};

struct RingGemmParams {
    RingGemmSegment seg[2];
    int nseg;
    int64_t M, N;                       // logical output size
    const uint64_t* C;                  // optional addend [party][M][N] (Beaver c_p)
    uint64_t* Z;                        // output [party][M][N]
    int64_t party_stride_c, party_stride_z;  // elements
    int trunc_bits;                     // 0 = none; else per-share round-half-up division (R10)
    int kc;                             // 32-K blocks per accumulation unit (<= ring_gemm_max_kc())
    unsigned long long* dbg;            // optional (MPC_GEMM_DEBUG): [0..3] stall cycles (producer empty, MMA
                                        // tempty, MMA full, MMA total); [4..7] globaltimer: first entry, last
                                        // setup done, last MMA issue end, last epilogue end
    int splits;                         // K ranges per output tile (split-K); 0/1 = none.  Set by the launcher.
    uint64_t* partials;                 // split-K slabs [splits][parties][M][N] (workspace,
                                        // ring_gemm_partials_bytes); unused when splits <= 1
    int64_t partial_stride;             // elements per slab (parties * M * N)
    int max_clusters;                   // 0: all SMs; else at most this many 2-CTA clusters (SMs left
                                        // to NCCL while a reveal overlaps the GEMM)
    int transpose_out;                  // 1: the GEMM computes Z^T (M, N are its own sizes, i.e. the
                                        // caller's N, M); element (m, n) is stored at Z[n * M + m] (and
                                        // C is read there).  Used for small caller M (fewer padded rows).
    int64_t out_hw;                     // > 0 (overrides transpose_out): row m = b * out_hw + s of the GEMM
                                        // goes to Z[(b * N + n) * out_hw + s] — the NCHW output of a
                                        // convolution whose im2col rows are (b, pixel s).  C likewise.
    int small;                          // 1: stacked-plane kernel (M <= 32, planes in Layout::Small)
    int group_m;                        // row tiles per scheduling group of the 2-CTA kernel (0: default 4)
    int serpentine;                     // set by the launcher: alternate K direction per wave (MPC_GEMM_SERPENTINE)
    int party_major;                    // set by the launcher: tile order instance-major (MPC_GEMM_PARTY_MAJOR)
    int batch;                          // independent GEMMs of the same shape (0/1 = one); instance
                                        // (b, p) reads planes at b * batch_stride_A/B + p * party_stride_A/B
    int64_t batch_stride_c, batch_stride_z;  // elements between batch elements of C / Z (and the partials)
    int partials_evict_first;           // experiment (MPC_PARTIALS_EVICT_FIRST=1): split-K partials stored
                                        // evict-first like z; default evict-last, so finalize reads them from L2
    int fault_inject;                   // test hook (MPC_GEMM_FAULT_INJECT=1): drop one stage's copies, so the
                                        // pipeline stalls and the mbarrier watchdog must trap
    int tma_l2;                         // L2 policy of the TMA operand loads: 0 evict_normal, 1 evict_last,
                                        // 2 evict_first, 3 no hint (MPC_GEMM_TMA_L2; experiment)
    RingGemmTma tma;                    // set by the launcher (2-CTA kernel, MPC_GEMM_TMA != 0)
};

// Two kernels: the 2-CTA 256 x 128 kernel (planes in Layout::Left / Right) and
// the stacked-plane kernel of ring_gemm_small.cu (32 x 32 tiles, for few rows)
// (both operands in Layout::Small) — RingGemmParams::small picks it; the caller
// wrote the planes in the matching layout.  Tensor-time model (SM-cycles, both
// kernels as launched, split-K included) used to choose kernel and orientation:
double ring_gemm_model_cycles(int parties, int64_t M, int64_t N, int tkb, int64_t max_clusters, bool small);
// split-K factor the launcher uses (1 without a partials buffer)
int ring_gemm_splits(int parties, int64_t M, int64_t N, int tkb, int64_t max_clusters, bool small);
size_t ring_gemm_small_smem_bytes();
cudaError_t ring_gemm_small_launch(const RingGemmParams& q, int parties, int64_t max_ctas, cudaStream_t stream);
constexpr int kSmallRows = 32;                     // output rows of one stacked-plane tile
constexpr int kSmallMaxRows = 256;                 // GEMM rows up to which the stacked kernel is considered

// Largest unit length (32-K blocks) for which every s32 accumulator stays exact.
int ring_gemm_max_kc();
// Unit length used for a fused reduction of `total_kb` blocks (L2-window sized).
int ring_gemm_default_kc(int total_kb);
size_t ring_gemm_smem_bytes();
int ring_gemm_choose_splits(int64_t tiles, int tkb, int64_t clusters);
// workspace for the split-K partial sums of a GEMM with these sizes (0 if no split)
size_t ring_gemm_partials_bytes(int parties, int64_t M, int64_t N, int total_kb, int max_clusters = 0,
                                bool small = false);
int64_t ring_gemm_out_elems(const RingGemmParams& q, int parties);
cudaError_t ring_gemm_finalize(const RingGemmParams& q, int parties, cudaStream_t stream);
cudaError_t ring_gemm_launch(const RingGemmParams& p, int parties, cudaStream_t stream);

// The fused 2-party Beaver matmul for M <= 32, N <= 32 with both parties on this GPU
// (ring_gemm_fused.cu): mask, local reveal, limb split and limb GEMM in one kernel,
// reading the u64 shares once; split-K slabs added by ring_gemm_finalize.
struct FusedSmallParams {
    const uint64_t *x, *a;              // [2][M][K] row-major (party stride M*K)
    const uint64_t *y, *b;              // [2][K][N] row-major (party stride K*N)
    const uint64_t* C;                  // [2][M][N] Beaver c_p (may be null)
    uint64_t* Z;                        // [2][M][N]
    int64_t M, K, N;
    int trunc_bits;                     // 0 or the per-share truncation (P <= 2, R10)
    uint64_t* partials;                 // fused_small_partials_bytes (null when 0)
    int unit;                           // set by the launcher: 32-K blocks per drained TMEM unit
    int pf_mode;                        // set by the launcher: L2 prefetch of the x / a rows (0 none,
                                        // 1 line prefetches, 2 one bulk prefetch per row; MPC_FUSED_PF)
    int pf_dist;                        // set by the launcher: blocks the L2 prefetch runs ahead
    int cyclic;                         // set by the launcher: 32-K blocks dealt to the CTAs round-robin
    unsigned long long* dbg;            // MPC_FUSED_DEBUG: [0] MMA full-wait, [1] MMA total, [2] converter
                                        // empty-wait, [3] converter total cycles (summed over CTAs / warps)
    // set by the launcher for the TMA-staged kernel: 3-D maps over x, a ([2][M][K], boxes of 16 K x
    // 32 rows, 128-byte swizzle) and y, b ([2][K][N], boxes of N x 32 K rows)
    CUtensorMap tm_x, tm_a, tm_y, tm_b;
};
size_t fused_small_smem_bytes();
int fused_small_ctas(int64_t K, int sms);
size_t fused_small_partials_bytes(int64_t M, int64_t K, int64_t N);
cudaError_t fused_small_launch(const FusedSmallParams& p, cudaStream_t stream);

}  // namespace mpc

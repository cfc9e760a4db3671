// ring_gemm_small.cu — the stacked-plane ring GEMM (tcgen05, sm_100a), for
// outputs with few rows: in 32 x 32 output tiles, the limb planes of the left
// operand's 32 rows are STACKED along the UMMA M dimension instead of padding
// the rows to a 256-row tile.
//
// Same product as ring_gemm.cu (Z_p = [C_p] + sum_seg L @ R^T mod 2^64 from
// u8 limb planes, L = sum_i 2^(8i) L_i, R = sum_j 2^(8j) R_j), computed as
//     L @ R^T = sum_i sum_{j <= 7-i} 2^(8(i+j)) L_i @ R_j^T      (mod 2^64)
// with the 32 rows of the 8 planes L_0..L_7 stacked into two 128-row MMA
// operands: A_lo = [L_0; L_1; L_2; L_3] and A_hi = [L_4; L_5; L_6; L_7]
// (rows 32 i' + r), and the 8 right planes stacked along N (the 32 rows of
// R_0..R_7 of one 32-K block are 8 KiB contiguous in Layout::Small: one
// 256-row B operand).  Two tcgen05.mma.cta_group::1.kind::i8 per 32-K block:
//     A_lo @ [R_0..R_7]^T (N = 256) -> columns 32 j + c: L_i' @ R_j^T,
//     A_hi @ [R_0..R_3]^T (N = 128) -> columns 128 + 32 j + c: L_{4+i'} @ R_j^T,
// so TMEM lane 32 i' + r, column block j holds shift i' + j from both (A_hi's
// block j + 4 has shift 4 + i' + j = i' + (j + 4)).  Each epilogue thread owns
// TMEM lane 32 i' + r and adds
//     run[c] += D[lane][32 j + c] << 8(i' + j)        (read as u32, i' + j <= 7)
// into u64 running sums; at the tile end the four planes of a row are summed
// through shared memory and c_p / the truncation applied (the store mapping,
// split-K slabs and finalize are those of ring_gemm.cu).  Round 1 issued 12 MMAs
// (one per right plane, N = 32) into 12 accumulators; the stacked B operand
// reads the A stacks 2 instead of 12 times per block.
//
// Exactness: an entry with shift i' + j <= 3 is a single limb product sum
// (no A_hi term there), D <= K_r * 255^2, so the s32 accumulator read as u32 is
// exact for K_r <= 66052 (2064 32-K blocks, the unit length cap); for shifts
// >= 4 only D mod 2^(64-8(i+j)) matters.
//
// Why: a 256 x 128 tile holding 32 x 32 useful outputs (the 32 x 519,820 x 32
// text matmul) wastes 31/32 of the tensor work; stacking wastes
// only the plane pairs with i + j >= 8 (28 of the 64 plane products issued per
// 32-K block).
//
// Operands in Layout::Small (common.cuh): one 32-K block of the 32 rows of all
// 8 planes is 8 KiB contiguous, so a stage is two bulk copies (16 x 1 KiB
// copies from the 128/64-row layouts ran at a third of this speed: the copy
// engine is message-rate bound for small copies).
//
// Warp roles (384 threads): warp 0 producer (two 8 KiB bulk copies per
// 32-K block), warp 1 MMA
// issuer, warp 2 TMEM allocator, warps 4..11 epilogue (two per TMEM lane
// quadrant, 16 columns each).
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#include "common.cuh"
#include "ring_gemm.h"
#include "tcgen05.cuh"

namespace mpc {
namespace gemm_small {
using namespace tc;

constexpr int kRows = 32;                         // output rows per tile (stacked per plane)
constexpr int kTileN = 32;                        // output columns per tile (UMMA N)
constexpr int kChunk = 1024;                      // 32 rows x 32 K bytes of one plane (4 core-matrix row groups)
constexpr int kStageBytes = 16 * kChunk;          // A: 8 planes, B: 8 planes
constexpr int kStages = 8;
constexpr int kEpiWarps = 8;
constexpr int kThreads = 128 + 32 * kEpiWarps;
constexpr int kTmemCols = 512;                    // 256 columns used (8 column blocks of 32)
constexpr int kMaxUnit = 2048;                    // 32-K blocks per accumulation unit (<= 2064)
// instruction descriptor: D S32; A, B unsigned 8-bit; M = 128; N = 8 right planes x 32
// columns (A_lo against R_0..R_7) or 4 x 32 (A_hi against R_0..R_3)
constexpr uint32_t idesc_n(int n) { return (2u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24); }
constexpr uint32_t kIdescLo = idesc_n(8 * kTileN), kIdescHi = idesc_n(4 * kTileN);

__device__ __forceinline__ void mma_u8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
        :: "r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate) : "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}"
        :: "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void epi_sync() {           // the 8 epilogue warps only
    asm volatile("bar.sync 1, %0;" :: "n"(32 * kEpiWarps) : "memory");
}

// work item w -> (party, 32-row tile, 32-column tile, K block range) — all warps
// compute the same values; the split-K ranges of one tile are consecutive items
struct Items {
    int parties, mt, nt, tkb, splits;
    __device__ int count() const { return parties * mt * nt * splits; }
    __device__ void decode(int w, int& party, int& m, int& n, int& klo, int& khi) const {
        const int t = w / splits, s = w % splits;
        party = t % parties;
        m = (t / parties) % mt;
        n = t / (parties * mt);
        klo = (int)((int64_t)tkb * s / splits);
        khi = (int)((int64_t)tkb * (s + 1) / splits);
    }
};

__global__ void __launch_bounds__(kThreads, 1) ring_gemm_small_kernel(const __grid_constant__ RingGemmParams p,
                                                                     int parties) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    if (threadIdx.x == 0) asm volatile("griddepcontrol.launch_dependents;");
    uint64_t* red = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);      // [4][32][32] u64 = 32 KiB
    uint64_t* full = red + 4 * kRows * kTileN;
    uint64_t* empty = full + kStages;
    uint64_t* tfull = empty + kStages;
    uint64_t* tempty = tfull + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    Items it{parties * (p.batch > 1 ? p.batch : 1), (int)((p.M + kRows - 1) / kRows), (int)((p.N + kTileN - 1) / kTileN),
             p.seg[0].kb + (p.nseg > 1 ? p.seg[1].kb : 0), p.splits < 1 ? 1 : p.splits};
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        mbar_init(tfull, 1);
        mbar_init(tempty, kEpiWarps);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                     :: "r"(smem_u32(tmem_slot)), "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ------------------------------------------------ producer
        asm volatile("griddepcontrol.wait;" ::: "memory");        // planes written by the split kernel
        int s = 0; uint32_t ph = 0;
        for (int w = blockIdx.x; w < it.count(); w += gridDim.x) {
            int party, m, n, klo, khi;
            it.decode(w, party, m, n, klo, khi);
            const int bi = party / parties;                        // instance -> (batch element, party)
            party -= bi * parties;
            for (int kt = klo; kt < khi; ++kt) {
                const int sg = (kt < p.seg[0].kb) ? 0 : 1;
                const RingGemmSegment& S = p.seg[sg];
                const int64_t kb = kt - (sg ? p.seg[0].kb : 0);
                // Layout::Small: (32-row block, 32-K block) of all 8 planes = 8 KiB contiguous
                const uint8_t* srcA = S.A + party * S.party_stride_A + bi * S.batch_stride_A +
                                      ((int64_t)m * S.kb + kb) * (8 * kChunk);
                const uint8_t* srcB = S.B + party * S.party_stride_B + bi * S.batch_stride_B +
                                      ((int64_t)n * S.kb + kb) * (8 * kChunk);
                mbar_wait(&empty[s], ph ^ 1);
                uint8_t* st = smem + s * kStageBytes;
                if (elect_one()) {
                    mbar_expect_tx(&full[s], kStageBytes);
                    bulk_g2s(st, srcA, 8 * kChunk, &full[s]);
                    bulk_g2s(st + 8 * kChunk, srcB, 8 * kChunk, &full[s]);
                }
                __syncwarp();
                if (++s == kStages) { s = 0; ph ^= 1; }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer
        int s = 0; uint32_t ph = 0; uint32_t u = 0;
        for (int w = blockIdx.x; w < it.count(); w += gridDim.x) {
            int party, m, n, klo, khi;
            it.decode(w, party, m, n, klo, khi);
            const int bi = party / parties;                        // instance -> (batch element, party)
            party -= bi * parties;
            for (int k0 = klo; k0 < khi; k0 += kMaxUnit, ++u) {
                const int k1 = min(khi, k0 + kMaxUnit);
                mbar_wait(tempty, (u & 1) ^ 1);                     // the epilogue drained the last unit
                tc_fence_after();
                for (int kt = k0; kt < k1; ++kt) {
                    mbar_wait(&full[s], ph);
                    tc_fence_after();
                    const uint64_t da = smem_desc(smem_u32(smem + s * kStageBytes));
                    const uint64_t db = da + ((8 * kChunk) >> 4);
                    const uint32_t acc = kt == k0 ? 0u : 1u;
                    // the 8 right planes of a 32-K block are 8 KiB contiguous (Layout::Small): one
                    // 256-row B operand.  A_lo x R_0..7 -> columns 32 j (shift i' + j), A_hi x R_0..3
                    // -> columns 128 + 32 j (shift 4 + i' + j: the same as A_lo's there), 2 MMAs
                    mma_u8(tmem_base, da, db, kIdescLo, acc);
                    mma_u8(tmem_base + 4 * kTileN, da + (uint64_t)((4 * kChunk) >> 4), db, kIdescHi, 1u);
                    tc_commit(&empty[s]);
                    if (++s == kStages) { s = 0; ph ^= 1; }
                }
                tc_commit(tfull);
            }
        }
    } else if (warp >= 4) {
        // ------------------------------------------------ epilogue
        // reads C / writes Z: ordered after the previous kernel even when no K block
        // (and so no producer wait) precedes the first tile end (K == 0)
        asm volatile("griddepcontrol.wait;" ::: "memory");
        const int q = warp & 3;                                    // TMEM lane quadrant = plane i' (i = i' or 4 + i')
        const int h = (warp - 4) >> 2;                             // column half
        const uint32_t tq = tmem_base + ((uint32_t)(q * 32) << 16) + h * 16;
        const int et = threadIdx.x - 128;                          // 0..255
        uint32_t u = 0;
        for (int w = blockIdx.x; w < it.count(); w += gridDim.x) {
            int party, m, n, klo, khi;
            it.decode(w, party, m, n, klo, khi);
            const int bi = party / parties;                        // instance -> (batch element, party)
            party -= bi * parties;
            uint64_t run[16];
#pragma unroll
            for (int c = 0; c < 16; ++c) run[c] = 0;
            for (int k0 = klo; k0 < khi; k0 += kMaxUnit, ++u) {
                mbar_wait(tfull, u & 1);
                tc_fence_after();
#pragma unroll
                for (int a = 0; a < 8; ++a) {
                    const int sh = q + a;                           // lane group i' = q, column block j = a
                    if (sh > 7) continue;                           // warp-uniform (q is per warp)
                    uint32_t v[16];
                    tmem_ld16(tq + a * kTileN, v);
                    tmem_wait_ld();
#pragma unroll
                    for (int c = 0; c < 16; ++c) run[c] += (uint64_t)v[c] << (8 * sh);
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(tempty);
            }
            // sum the four planes of each row (TMEM quadrants) through shared memory
            uint64_t* mine = red + ((int64_t)q * kRows + lane) * kTileN + h * 16;
#pragma unroll
            for (int c = 0; c < 16; c += 2) *reinterpret_cast<ulonglong2*>(mine + c) = make_ulonglong2(run[c], run[c + 1]);
            epi_sync();
            const int64_t row0 = (int64_t)m * kRows;
            const int64_t hw = p.out_hw > 0 ? p.out_hw : (p.transpose_out ? p.M : 0);
            const bool tr = hw > 0;
            const bool split = it.splits > 1;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int idx = e * 256 + et;                        // consecutive threads: consecutive columns
                const int r = idx / kTileN, col = idx % kTileN;
                const int64_t gc = (int64_t)n * kTileN + col;
                const int64_t gr = row0 + r;
                if (gr >= p.M || gc >= p.N) continue;
                uint64_t v = 0;
#pragma unroll
                for (int qq = 0; qq < 4; ++qq) v += red[((int64_t)qq * kRows + r) * kTileN + col];
                const int64_t off = tr ? (gr / hw) * p.N * hw + gr % hw + gc * hw : gr * p.N + gc;
                if (split) {
                    const int sidx = w % it.splits;
                    p.partials[(int64_t)sidx * p.partial_stride + party * p.party_stride_z + bi * p.batch_stride_z +
                               off] = v;
                } else {
                    if (p.C) v += p.C[party * p.party_stride_c + bi * p.batch_stride_c + off];
                    if (p.trunc_bits) v = div_pow2_round(v, p.trunc_bits);
                    p.Z[party * p.party_stride_z + bi * p.batch_stride_z + off] = v;
                }
            }
            epi_sync();                                              // red is reused by the next item
        }
    }
    __syncwarp();
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem_base), "r"(kTmemCols));
    }
}

}  // namespace gemm_small

size_t ring_gemm_small_smem_bytes() {
    return (size_t)gemm_small::kStages * gemm_small::kStageBytes + 4 * 32 * 32 * 8 + 1024 /*align*/ + 256;
}

namespace {
int64_t waves(int64_t items, int64_t slots) { return (items + slots - 1) / slots; }
int small_splits(int64_t tiles, int tkb, int64_t ctas) {
    if (tiles <= 0 || tiles >= ctas) return 1;
    int64_t s = ctas / tiles;
    if (s > 64) s = 64;
    if (s > tkb / 8) s = tkb / 8;
    return s < 1 ? 1 : (int)s;
}
}  // namespace

int64_t small_tiles(int parties, int64_t M, int64_t N) {
    return (int64_t)parties * ((M + gemm_small::kRows - 1) / gemm_small::kRows) *
           ((N + gemm_small::kTileN - 1) / gemm_small::kTileN);
}

int ring_gemm_splits(int parties, int64_t M, int64_t N, int tkb, int64_t max_clusters, bool small) {
    if (small) return small_splits(small_tiles(parties, M, N), tkb, 2 * max_clusters);
    const int64_t tiles = (int64_t)parties * (pad_rows<Layout::Left>(M) / 256) * (pad_rows<Layout::Right>(N) / 128);
    return ring_gemm_choose_splits(tiles, tkb, max_clusters);
}

// The 2-CTA kernel issues 36 MMAs of 64 cycles per 256 x 128 tile and 32-K
// block on a CTA pair.  The stacked one is costed at 576 cycles per 32 x 32 tile
// and block on one SM — the round-1 figure (12 N = 32 MMAs of ~48 cycles): its
// two stacked MMAs now take ~192, but a tile then needs its 16 KiB of planes
// every ~200 cycles, more than the L2 -> SM feed gives one SM (~36-70 B/clk), so
// the old figure stays as the conservative cost that selected the shapes it wins.
// A split-K launch also pays its partial-sum stores and the finalize pass: ~12000 cycles
// (≈ 7 µs: measured per-layer, the stacked kernel without split-K beats the 2-CTA kernel
// with it on exactly the ResNet-50 shapes where this term flips the choice — 3136 x 576 x 64
// 59.6 -> 49.6 us, 196 x 1024 x 256 30.8 -> 24.6 us — and loses everywhere it does not;
// MPC_SPLIT_PENALTY overrides, 0 restores the MMA-only model).
double ring_gemm_model_cycles(int parties, int64_t M, int64_t N, int tkb, int64_t max_clusters, bool small) {
    static const double pen = getenv("MPC_SPLIT_PENALTY") ? atof(getenv("MPC_SPLIT_PENALTY")) : 12000.0;
    const int s = ring_gemm_splits(parties, M, N, tkb, max_clusters, small);
    const double split_cost = s > 1 ? pen : 0.0;
    if (small)
        return (double)waves(small_tiles(parties, M, N) * s, 2 * max_clusters) * ((tkb + s - 1) / s) * 12.0 * 48.0 +
               split_cost;
    const int64_t tiles = (int64_t)parties * (pad_rows<Layout::Left>(M) / 256) * (pad_rows<Layout::Right>(N) / 128);
    return (double)waves(tiles * s, max_clusters) * ((tkb + s - 1) / s) * 2304.0 + split_cost;
}

cudaError_t ring_gemm_small_launch(const RingGemmParams& q, int parties, int64_t max_ctas, cudaStream_t stream) {
    static int attr_dev = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    const size_t smem = ring_gemm_small_smem_bytes();
    if (attr_dev != dev) {
        cudaError_t e = cudaFuncSetAttribute(gemm_small::ring_gemm_small_kernel,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr_dev = dev;
    }
    const int64_t items = small_tiles(parties * (q.batch > 1 ? q.batch : 1), q.M, q.N) * (q.splits < 1 ? 1 : q.splits);
    if (items >= (int64_t)1 << 31) return cudaErrorInvalidValue;
    int64_t ctas = items < max_ctas ? items : max_ctas;
    if (ctas < 1) ctas = 1;
    return launch_pdl(gemm_small::ring_gemm_small_kernel, dim3((unsigned)ctas), dim3(gemm_small::kThreads), smem,
                      stream, q, parties);
}

}  // namespace mpc

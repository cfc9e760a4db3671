// ring_gemm.cu — the mod-2^64 ring GEMM on tcgen05 int8 tensor cores (sm_100a).
//
// Computes, per party p:
//     Z_p = [C_p] + sum_seg  L_seg,p @ R_seg,p^T      (mod 2^64)
// where every u64 operand is given as 8 u8 limb planes (common.cuh layout),
// L = sum_i 2^(8i) L_i, R = sum_j 2^(8j) R_j, so
//     L @ R^T = sum_{s=0..7} 2^(8s) acc_s,  acc_s = sum_{i+j=s} L_i @ R_j^T  (mod 2^64)
// — 36 u8 x u8 -> s32 limb products; pairs with i+j >= 8 vanish mod 2^64.
// For the Beaver matmul (R7/R8) the host passes two
// segments: (a_p, delta) and (eps, b_p + [p=0] delta), i.e.
//     z_p = c_p + a_p @ delta + eps @ b'_p.
//
// Exactness: acc_s <= (s+1) * K_r * 255^2.  The s32
// accumulator wraps mod 2^32 (no .sat), so reading it as u32 is exact while
// acc_s < 2^32; for s >= 4 only acc_s mod 2^(64-8s) <= 2^32 matters, so the
// wrap is harmless.  The host splits K into chunks of at most
// floor((2^32-1) / ((s+1) * 65025)) for the low shift s of each pass and the
// epilogue drains every chunk into the u64 result.
//
// Schedule.  A cluster of 2 CTAs (one per SM of a TPC) computes a 256 x 256
// output tile with tcgen05.mma.cta_group::2 (UMMA M = 256, N = 256, K = 32):
// CTA r holds rows 128r..128r+127 of the left planes and rows 128r..+127 of
// the right planes of the tile in its shared memory, and its half of the
// accumulator (128 TMEM lanes) — each CTA moves half the operand bytes of a
// 1-CTA 128 x 256 tile for twice the MACs.  The 36 limb products are issued as
// 4 passes q = 0..3, each accumulating the shift pair {q, 7-q} (q+1 + 8-q = 9
// MMAs per 32-K block) into two 256-column TMEM accumulators (all 512
// columns); a pass needs only limb planes 0..7-q.  The kernel is persistent:
// 74 clusters walk the tiles in a grouped order (parties and 4 row tiles
// innermost) so concurrently running clusters share operand planes in L2.
//
// Warp roles (256 threads per CTA): warp 0 = bulk-copy producer (both CTAs),
// warp 1 = MMA issuer (leader CTA) / stage relay (peer CTA), warp 2 = TMEM
// allocator, warps 4..7 = epilogue (one TMEM lane = one output row per thread).
#include <cstdint>
#include <cuda_runtime.h>
#include "common.cuh"
#include "ring_gemm.h"

namespace mpc {
namespace gemm {

constexpr int kTileM = 256;              // UMMA M (cta_group::2): 128 rows per CTA
constexpr int kTileN = 256;              // UMMA N: 128 right-operand rows per CTA
constexpr int kHalfBytes = 8 * kPlaneTileBytes;        // 8 planes x (128 rows x 32 K) = 32 KiB
constexpr int kStageBytes = 2 * kHalfBytes;            // A + B planes of one 32-K block = 64 KiB
constexpr int kStages = 3;
constexpr int kThreads = 256;
constexpr int kTmemCols = 512;
constexpr int kGroupM = 4;               // row tiles per scheduling group
constexpr uint32_t kIdesc = (2u << 4)            // D format: S32
                          | (0u << 7)            // A: unsigned 8-bit
                          | (0u << 10)           // B: unsigned 8-bit
                          | ((uint32_t)(kTileN >> 3) << 17)
                          | ((uint32_t)(kTileM >> 4) << 24);

// ----------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cluster_id() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t nclusters() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
    return r;
}
// shared::cluster address of the same smem offset in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa(uint32_t saddr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// arrive on the barrier at cluster address `caddr` (possibly in the peer CTA)
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t caddr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" :: "r"(caddr) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}"
        :: "r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAITC_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAITC_%=;\n\t}"
        :: "r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// commit all prior MMAs of this thread; arrive on `bar` (same offset) in both CTAs
__device__ __forceinline__ void tc_commit_both(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 :: "r"(smem_u32(bar)), "h"((uint16_t)0x3) : "memory");
}
// SWIZZLE_NONE K-major descriptor: LBO = 128 B (K halves), SBO = 256 B (8-row groups), version 1
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(128u >> 4) << 16) | ((uint64_t)(256u >> 4) << 32)
         | (1ull << 46);
}
__device__ __forceinline__ void mma_u8_2cta(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}"
        :: "r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(kIdesc), "r"(accumulate) : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// Tile t -> (party, m tile, n tile) in the grouped order: groups of kGroupM row
// tiles; inside a group, n tiles outer, then row tiles, then parties.
struct TileMap {
    int parties, mt, nt;
    __device__ void decode(int t, int& party, int& m, int& n) const {
        const int per_group_full = kGroupM * nt * parties;
        const int g = t / per_group_full;
        const int r = t % per_group_full;
        const int gm = min(kGroupM, mt - g * kGroupM);        // row tiles in this group
        const int per_n = gm * parties;
        n = r / per_n;
        const int r2 = r % per_n;
        m = g * kGroupM + r2 / parties;
        party = r2 % parties;
    }
};

__device__ __forceinline__ int total_kb(const RingGemmParams& p) { return p.seg[0].kb + (p.nseg > 1 ? p.seg[1].kb : 0); }

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
ring_gemm_kernel(const __grid_constant__ RingGemmParams p, int parties) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* stage_base = smem;
    uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
    uint64_t* empty_bar = full_bar + kStages;
    uint64_t* tfull_bar = empty_bar + kStages;
    uint64_t* tempty_bar = tfull_bar + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const bool leader = (rank == 0);
    const TileMap tm{parties, (int)(pad_rows(p.M) / kTileM), (int)(pad_rows(p.N) / kTileN)};
    const int ntiles = tm.parties * tm.mt * tm.nt;
    const int tkb = total_kb(p);
    int nunits = 0;
    for (int q = 0; q < 4; ++q) nunits += (tkb + p.kb_chunk[q] - 1) / p.kb_chunk[q];

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) { mbar_init(&full_bar[s], leader ? 2 : 1); mbar_init(&empty_bar[s], 1); }
        mbar_init(tfull_bar, 1);
        mbar_init(tempty_bar, 8);          // 4 epilogue warps x 2 CTAs (leader's copy is the one used)
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;"
                     :: "r"(smem_u32(tmem_slot)), "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ------------------------------------------------ producer (both CTAs: own halves)
        if (lane == 0) {
            int s = 0; uint32_t ph = 0;
            for (int t = cluster_id(); t < ntiles; t += nclusters()) {
                int party, m, n;
                tm.decode(t, party, m, n);
                const int64_t rtA = (int64_t)m * 2 + rank, rtB = (int64_t)n * 2 + rank;
                for (int q = 0; q < 4; ++q) {
                    const uint32_t bytes = (uint32_t)(8 - q) * kPlaneTileBytes;
                    for (int kt = 0; kt < tkb; ++kt) {
                        const int sg = (kt < p.seg[0].kb) ? 0 : 1;
                        const RingGemmSegment& S = p.seg[sg];
                        const int kb = kt - (sg ? p.seg[0].kb : 0);
                        const uint8_t* srcA = S.A + party * S.party_stride_A + (rtA * S.kb + kb) * kHalfBytes;
                        const uint8_t* srcB = S.B + party * S.party_stride_B + (rtB * S.kb + kb) * kHalfBytes;
                        mbar_wait(&empty_bar[s], ph ^ 1);
                        mbar_expect_tx(&full_bar[s], 2 * bytes);
                        uint8_t* st = stage_base + s * kStageBytes;
                        bulk_g2s(st, srcA, bytes, &full_bar[s]);
                        bulk_g2s(st + kHalfBytes, srcB, bytes, &full_bar[s]);
                        if (++s == kStages) { s = 0; ph ^= 1; }
                    }
                }
            }
        }
    } else if (warp == 1 && !leader) {
        // ------------------------------------------------ peer: relay "stage full" to the leader
        if (lane == 0) {
            int s = 0; uint32_t ph = 0;
            const uint32_t leader_full0 = mapa(smem_u32(&full_bar[0]), 0);
            for (int t = cluster_id(); t < ntiles; t += nclusters())
                for (int i = 0; i < 4 * tkb; ++i) {
                    mbar_wait(&full_bar[s], ph);
                    mbar_arrive_cluster(leader_full0 + s * 8);
                    if (++s == kStages) { s = 0; ph ^= 1; }
                }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ leader: MMA issuer (one thread)
        if (lane == 0) {
            int s = 0; uint32_t ph = 0; uint32_t uph = 0;
            const uint32_t d_lo = tmem_base;             // shift q
            const uint32_t d_hi = tmem_base + 256;       // shift 7-q
            for (int t = cluster_id(); t < ntiles; t += nclusters()) {
                for (int q = 0; q < 4; ++q) {
                    const int chunk = p.kb_chunk[q];
                    for (int c0 = 0; c0 < tkb; c0 += chunk) {
                        const int c1 = min(tkb, c0 + chunk);
                        mbar_wait_cluster(tempty_bar, uph ^ 1);      // both epilogues drained TMEM
                        uph ^= 1;
                        tc_fence_after();
                        for (int kt = c0; kt < c1; ++kt) {
                            mbar_wait_cluster(&full_bar[s], ph);
                            tc_fence_after();
                            const uint32_t a0 = smem_u32(stage_base + s * kStageBytes);
                            const uint32_t b0 = a0 + kHalfBytes;
                            const uint32_t first = (kt == c0);
                            for (int i = 0; i <= q; ++i)
                                mma_u8_2cta(d_lo, smem_desc(a0 + i * kPlaneTileBytes),
                                            smem_desc(b0 + (q - i) * kPlaneTileBytes), !(first && i == 0));
                            for (int i = 0; i <= 7 - q; ++i)
                                mma_u8_2cta(d_hi, smem_desc(a0 + i * kPlaneTileBytes),
                                            smem_desc(b0 + (7 - q - i) * kPlaneTileBytes), !(first && i == 0));
                            tc_commit_both(&empty_bar[s]);
                            if (++s == kStages) { s = 0; ph ^= 1; }
                        }
                        tc_commit_both(tfull_bar);
                    }
                }
            }
        }
    } else if (warp >= 4) {
        // ------------------------------------------------ epilogue (both CTAs, own 128 rows)
        const int wq = warp & 3;
        const int row = wq * 32 + lane;
        const uint32_t tempty_leader = mapa(smem_u32(tempty_bar), 0);
        const bool vec = (p.N & 1) == 0;
        uint32_t uph = 0;
        for (int t = cluster_id(); t < ntiles; t += nclusters()) {
            int party, m, n;
            tm.decode(t, party, m, n);
            const int64_t grow = (int64_t)m * kTileM + rank * 128 + row;
            const bool row_ok = grow < p.M;
            uint64_t* zrow = p.Z + party * p.party_stride_z + grow * p.N;
            const uint64_t* crow = p.C ? p.C + party * p.party_stride_c + grow * p.N : nullptr;
            const int64_t col0 = (int64_t)n * kTileN;
            int unit = 0;
            for (int q = 0; q < 4; ++q) {
                const int chunk = p.kb_chunk[q];
                for (int c0 = 0; c0 < tkb; c0 += chunk, ++unit) {
                    const bool first_unit = (unit == 0), last_unit = (unit == nunits - 1);
                    mbar_wait(tfull_bar, uph);
                    uph ^= 1;
                    tc_fence_after();
                    const uint32_t t_lo = tmem_base + ((uint32_t)(wq * 32) << 16);
                    const uint32_t t_hi = t_lo + 256;
                    for (int cc = 0; cc < kTileN; cc += 32) {
                        uint32_t lo[32], hi[32];
                        tmem_ld32(t_lo + cc, lo);
                        tmem_ld32(t_hi + cc, hi);
                        tmem_wait_ld();
                        if (!row_ok) continue;
                        const int64_t gc0 = col0 + cc;
                        if (vec && gc0 + 32 <= p.N) {
#pragma unroll
                            for (int j = 0; j < 32; j += 2) {
                                const uint64_t v0 = ((uint64_t)lo[j] << (8 * q)) + ((uint64_t)hi[j] << (8 * (7 - q)));
                                const uint64_t v1 = ((uint64_t)lo[j + 1] << (8 * q)) + ((uint64_t)hi[j + 1] << (8 * (7 - q)));
                                ulonglong2 cur;
                                if (first_unit) {
                                    cur = crow ? *reinterpret_cast<const ulonglong2*>(crow + gc0 + j) : make_ulonglong2(0, 0);
                                } else {
                                    cur = *reinterpret_cast<const ulonglong2*>(zrow + gc0 + j);
                                }
                                cur.x += v0; cur.y += v1;
                                if (last_unit && p.trunc_bits) {
                                    cur.x = div_pow2_round(cur.x, p.trunc_bits);
                                    cur.y = div_pow2_round(cur.y, p.trunc_bits);
                                }
                                *reinterpret_cast<ulonglong2*>(zrow + gc0 + j) = cur;
                            }
                        } else {
#pragma unroll
                            for (int j = 0; j < 32; ++j) {
                                const int64_t gc = gc0 + j;
                                if (gc < p.N) {
                                    const uint64_t v = ((uint64_t)lo[j] << (8 * q)) + ((uint64_t)hi[j] << (8 * (7 - q)));
                                    uint64_t cur = first_unit ? (crow ? crow[gc] : 0ull) : zrow[gc];
                                    cur += v;
                                    if (last_unit && p.trunc_bits) cur = div_pow2_round(cur, p.trunc_bits);
                                    zrow[gc] = cur;
                                }
                            }
                        }
                    }
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive_cluster(tempty_leader);
                }
            }
            if (nunits == 0 && row_ok) {       // K == 0: Z = C (then truncated)
                for (int j = 0; j < kTileN; ++j) {
                    const int64_t gc = col0 + j;
                    if (gc < p.N) {
                        uint64_t cur = crow ? crow[gc] : 0ull;
                        if (p.trunc_bits) cur = div_pow2_round(cur, p.trunc_bits);
                        zrow[gc] = cur;
                    }
                }
            }
        }
    }
    __syncwarp();
    tc_fence_before();
    cluster_sync();
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" :: "r"(tmem_base), "r"(kTmemCols));
    }
}

}  // namespace gemm

int ring_gemm_kb_chunk(int q) {
    // largest K_r with (q+1) * K_r * 255^2 <= 2^32 - 1, in 32-K blocks
    const uint64_t lim = 0xFFFFFFFFull / ((uint64_t)(q + 1) * 65025ull);
    return (int)(lim / kKBlock);
}

size_t ring_gemm_smem_bytes() {
    return (size_t)gemm::kStages * gemm::kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
}

cudaError_t ring_gemm_launch(const RingGemmParams& prm, int parties, cudaStream_t stream) {
    static int attr_dev = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    const size_t smem = ring_gemm_smem_bytes();
    if (attr_dev != dev) {
        cudaError_t e = cudaFuncSetAttribute(gemm::ring_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr_dev = dev;
    }
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t tiles = (int64_t)parties * (pad_rows(prm.M) / gemm::kTileM) * (pad_rows(prm.N) / gemm::kTileN);
    int64_t clusters = sms / 2;
    if (tiles < clusters) clusters = tiles;
    if (clusters < 1) clusters = 1;
    gemm::ring_gemm_kernel<<<(unsigned)(clusters * 2), gemm::kThreads, smem, stream>>>(prm, parties);
    return cudaGetLastError();
}

}  // namespace mpc

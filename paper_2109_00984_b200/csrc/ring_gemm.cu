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
// Exactness: acc_s <= (s+1) * K_r * 255^2 where K_r is
// the reduction length of one accumulation unit.  The s32 accumulator wraps
// mod 2^32 (no .sat), so reading it as u32 is exact while acc_s < 2^32, i.e.
// K_r <= 16512 for s = 3; for s >= 4 only acc_s mod 2^(64-8s) <= 2^32 matters,
// so the wrap is harmless.  Every unit covers at most ring_gemm_max_kc() 32-K
// blocks and is drained into a u64 running sum.
//
// Schedule.  A cluster of 2 CTAs (one TPC) computes a 256 x 128 output tile
// with tcgen05.mma.cta_group::2 (UMMA M = 256, N = 128, K = 32): CTA r holds
// rows 128r..128r+127 of the left planes (4 KiB per plane and 32-K block) and
// rows 64r..64r+63 of the right planes (2 KiB) in shared memory, and its
// 128-lane half of the accumulators.  TMEM (512 columns) holds 4 accumulators
// of 128 columns, so the 8 shifts run as 2 super-passes per K chunk:
// {0, 7, 1, 6} (18 MMAs per 32-K block, limb planes 0..7) and {2, 5, 3, 4}
// (18 MMAs, planes 0..5) — 14 plane loads per 32-K block instead of the 26 a
// 2-accumulator schedule needs, which keeps the per-SM L2->SM feed at about
// 36 B/clk for 8192 MAC/clk.  Units (K chunk, super-pass) are ordered chunk
// major so the second super-pass re-reads a K window still resident in L2.
// The u64 running sum of a tile lives in the registers of 8 epilogue warps
// (64 columns x 1 row per thread; setmaxnreg gives them 216 registers) and is
// written once, with the Beaver c_p addend and the fused truncation, at the
// tile end.  The kernel is persistent: 74 clusters walk the tiles in a grouped
// order (4 row tiles x all column tiles x parties per group).
//
// Warp roles (384 threads per CTA): warp 0 = producer (both CTAs: 2-CTA tensor
// TMA completing the leader's stage barrier, or — MPC_GEMM_TMA=0 / fault
// injection — bulk copies), warp 1 = MMA issuer (leader CTA) / stage relay
// (peer CTA, bulk-copy producer only), warp 2 = TMEM
// allocator, warps 4..11 = epilogue.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include "common.cuh"
#include "ring_gemm.h"
#include "tcgen05.cuh"

namespace mpc {
namespace gemm {

using GL = PlaneGeom<Layout::Left>;
using GR = PlaneGeom<Layout::Right>;
constexpr int kTileM = 256;                       // UMMA M (cta_group::2): 128 rows per CTA
constexpr int kTileN = 128;                       // UMMA N: 64 right-operand rows per CTA
constexpr int kAStage = 8 * GL::kBlock;           // 32 KiB
constexpr int kBStage = 8 * GR::kBlock;           // 16 KiB
constexpr int kStageBytes = kAStage + kBStage;    // 48 KiB
constexpr int kStages = 4;
constexpr int kEpiWarps = 8;
constexpr int kThreads = 128 + 32 * kEpiWarps;    // 384
constexpr int kTmemCols = 512;
constexpr int kGroupM = 4;                        // row tiles per scheduling group (MPC_GEMM_GROUPM overrides)
constexpr int kPasses = 2;                        // super-passes of 4 shifts each
constexpr uint32_t kIdesc = (2u << 4)             // D format: S32
                          | (0u << 7)             // A: unsigned 8-bit
                          | (0u << 10)            // B: unsigned 8-bit
                          | ((uint32_t)(kTileN >> 3) << 17)
                          | ((uint32_t)(kTileM >> 4) << 24);

// ----------------------------------------------------------------- PTX helpers (tcgen05.cuh)
using namespace tc;
__device__ __forceinline__ void mma_u8_2cta(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}"
        :: "r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(kIdesc), "r"(accumulate) : "memory");
}

// Tile t -> (party, m tile, n tile) in the grouped order: groups of kGroupM row
// tiles; inside a group, n tiles outer, then row tiles, then parties.
struct TileMap {
    int parties, mt, nt, gmax;                       // gmax: row tiles per group
    int party_major;                                 // 1: instance outermost, then the grouped (m, n) order
    __device__ void decode(int t, int& party, int& m, int& n) const {
        if (party_major) {
            // one instance's tiles at a time: a wave then shares its party-specific operand strips
            // (a_p, b'_p) across more tiles (R-less L2 traffic when the party operands dominate)
            const int per_inst = mt * nt;
            party = t / per_inst;
            const int r0 = t - party * per_inst;
            const int per_group_full = gmax * nt;
            const int g = r0 / per_group_full;
            const int r = r0 % per_group_full;
            const int gm = min(gmax, mt - g * gmax);
            n = r / gm;
            m = g * gmax + r % gm;
            return;
        }
        const int per_group_full = gmax * nt * parties;
        const int g = t / per_group_full;
        const int r = t % per_group_full;
        const int gm = min(gmax, mt - g * gmax);              // row tiles in this group
        const int per_n = gm * parties;
        n = r / per_n;
        const int r2 = r % per_n;
        m = g * gmax + r2 / parties;
        party = r2 % parties;
    }
};

// Work item w -> (tile, K range): `splits` contiguous ranges of the fused
// 32-K block sequence per tile (split-K for shapes with few tiles); the
// ranges of one tile are consecutive items, so they run concurrently.
struct WorkMap {
    TileMap tm;                                      // tm.parties = instances = parties x batch
    int tkb, kc, splits;
    int nparties;                                    // parties per batch element
    __device__ int items() const { return tm.parties * tm.mt * tm.nt * splits; }
    // 32-bit arithmetic only (the launcher uses splits > 1 only for tkb < 2^24),
    // and results broadcast from lane 0: the role loops must stay provably
    // warp-uniform for the MMA descriptors to live in uniform registers.
    __device__ void decode(int w, int& party, int& m, int& n, int& klo, int& khi) const {
        const int t = w / splits, s = w % splits;
        tm.decode(t, party, m, n);
        klo = (int)((unsigned)tkb * (unsigned)s / (unsigned)splits);
        khi = (int)((unsigned)tkb * (unsigned)(s + 1) / (unsigned)splits);
        party = __shfl_sync(0xffffffffu, party, 0);
        m = __shfl_sync(0xffffffffu, m, 0);
        n = __shfl_sync(0xffffffffu, n, 0);
        klo = __shfl_sync(0xffffffffu, klo, 0);
        khi = __shfl_sync(0xffffffffu, khi, 0);
    }
    __device__ int item_kb(int w) const {
        const int s = w % splits;
        const int kb = (int)((unsigned)tkb * (unsigned)(s + 1) / (unsigned)splits) -
                       (int)((unsigned)tkb * (unsigned)s / (unsigned)splits);
        return __shfl_sync(0xffffffffu, kb, 0);
    }
};

struct Bars {
    uint8_t* stage_base;
    uint64_t *full, *empty, *tfull, *tempty;
};

// Super-pass g accumulates 4 shifts into TMEM slots 0..3 (128 columns each):
// g = 0: shifts {0, 7, 1, 6} (1+8+2+7 = 18 MMAs per 32-K block, planes 0..7)
// g = 1: shifts {2, 5, 3, 4} (3+6+4+5 = 18 MMAs per 32-K block, planes 0..5)
__host__ __device__ constexpr int slot_shift(int g, int a) {
    return g == 0 ? ((a & 1) ? 7 - (a >> 1) : (a >> 1)) : ((a & 1) ? 5 - (a >> 1) : 2 + (a >> 1));
}
__device__ __forceinline__ int pass_planes(int g) { return g == 0 ? 8 : 6; }

// The limb MMAs of TMEM slots A0 and A0+1 (one release group) for one 32-K
// block of super-pass G, fully unrolled (9 MMAs): every descriptor is the
// stage's base descriptor plus a compile-time offset (A plane i at +4 KiB * i,
// B plane j at +2 KiB * j; the 14-bit address field never carries for smem
// addresses < 256 KiB).  FIRST: the block starts a unit, so the first product
// of each shift overwrites its accumulator.
template <int G, bool FIRST, int A0>
__device__ __forceinline__ void issue_slots(uint64_t da, uint64_t db, uint32_t tmem_base) {
#pragma unroll
    for (int a = A0; a < A0 + 2; ++a) {
        const int sh = slot_shift(G, a);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (i <= sh)
                mma_u8_2cta(tmem_base + a * 128, da + (uint64_t)(i * (GL::kBlock >> 4)),
                            db + (uint64_t)((sh - i) * (GR::kBlock >> 4)), (FIRST && i == 0) ? 0u : 1u);
        }
    }
}
template <int G>
__device__ __forceinline__ void issue_kblock(uint64_t da, uint64_t db, uint32_t tmem_base) {
    issue_slots<G, false, 0>(da, db, tmem_base);
    issue_slots<G, false, 2>(da, db, tmem_base);
}

// ---------------------------------------------------------------- control warpgroup
// FAULT: the fault-injection instantiation (MPC_GEMM_FAULT_INJECT, watchdog test).  A
// compile-time switch: a runtime check in the producer's copy loop cost the
// 8192^3 GEMMs 8-10% (measured: 108 vs 117-121 ms for 4-party 8192^3).
template <bool FAULT, bool TMA, bool SERP>
__device__ __forceinline__ void control_roles(const RingGemmParams& p, const WorkMap& wm, int warp, int lane,
                                              uint32_t rank, uint32_t tmem_base, const Bars& B) {
    const bool leader = rank == 0;
    const int kc = wm.kc;
    if (warp == 0) {
        // ------------------------------------------------ producer (both CTAs: own halves)
        // the tensor maps are kernel parameters: fetch their descriptors before the wait
        // (the first TMA of every CTA otherwise pays the descriptor miss after it)
        if (TMA && lane < 8 && (lane >> 1 & 1) < p.nseg) {
            const CUtensorMap* m = lane < 4 ? &p.tma.a[lane >> 1 & 1][lane & 1] : &p.tma.b[lane >> 1 & 1][lane & 1];
            asm volatile("prefetch.tensormap [%0];" :: "l"(reinterpret_cast<uint64_t>(m)) : "memory");
        }
        // launched as a programmatic dependent of the limb-split kernel: the
        // prologue overlapped its tail; the planes are read only after it completed
        asm volatile("griddepcontrol.wait;" ::: "memory");
        int s = 0; uint32_t ph = 0;
        long long st_empty = 0;
        int item_no = 0;                                 // this cluster's items so far (K-serpentine parity)
        const uint64_t l2pol = l2_policy(p.tma_l2);
        for (int w = cluster_id(); w < wm.items(); w += nclusters()) {
            int party, m, n, klo, khi;
            wm.decode(w, party, m, n, klo, khi);
            const int bi = party / wm.nparties;              // instance -> (batch element, party)
            party -= bi * wm.nparties;
            const int64_t rbA = (int64_t)m * 2 + rank;       // 128-row left block
            const int64_t rbB = (int64_t)n * 2 + rank;       // 64-row right block
            // this item's block-0 addresses of both segments (the copy loop is latency-critical:
            // per block only a select and one add remain)
            const int kb0 = p.seg[0].kb;
            const RingGemmSegment& S0 = p.seg[0];
            const RingGemmSegment& S1 = p.seg[p.nseg > 1 ? 1 : 0];
            const uint8_t* a0 = S0.A + party * S0.party_stride_A + bi * S0.batch_stride_A + rbA * S0.kb * (8 * GL::kBlock);
            const uint8_t* b0 = S0.B + party * S0.party_stride_B + bi * S0.batch_stride_B + rbB * S0.kb * (8 * GR::kBlock);
            const uint8_t* a1 = S1.A + party * S1.party_stride_A + bi * S1.batch_stride_A + rbA * S1.kb * (8 * GL::kBlock) -
                                (int64_t)kb0 * (8 * GL::kBlock);
            const uint8_t* b1 = S1.B + party * S1.party_stride_B + bi * S1.batch_stride_B + rbB * S1.kb * (8 * GR::kBlock) -
                                (int64_t)kb0 * (8 * GR::kBlock);
            const bool rev = SERP && (item_no++ & 1);
            const int kstep = rev ? -kc : kc;
            for (int k0 = rev ? klo + (khi - klo - 1) / kc * kc : klo; rev ? k0 >= klo : k0 < khi; k0 += kstep) {
                const int k1 = min(khi, k0 + kc);
                for (int g = 0; g < kPasses; ++g) {
                    const uint32_t bytesA = (uint32_t)pass_planes(g) * GL::kBlock;
                    const uint32_t bytesB = (uint32_t)pass_planes(g) * GR::kBlock;
                    for (int kt = k0; kt < k1; ++kt) {
                        const bool second = kt >= kb0;
                        const uint8_t* srcA = (second ? a1 : a0) + (int64_t)kt * (8 * GL::kBlock);
                        const uint8_t* srcB = (second ? b1 : b0) + (int64_t)kt * (8 * GR::kBlock);
                        if (p.dbg) { const long long w0 = clock64(); mbar_wait(&B.empty[s], ph ^ 1); st_empty += clock64() - w0; }
                        else mbar_wait(&B.empty[s], ph ^ 1);
                        if (TMA) {
                            // both CTAs: own half by 2-CTA tensor TMA, completing the LEADER's
                            // barrier, which expects both halves' bytes (rows of 2 KiB; the maps
                            // start at the segment's plane buffer)
                            if (elect_one()) {
                                if (leader) mbar_expect_tx(&B.full[s], 2 * (bytesA + bytesB));
                                const uint32_t fb = mapa(smem_u32(&B.full[s]), 0);
                                const uint8_t* st = B.stage_base + s * kStageBytes;
                                const RingGemmSegment& Sx = second ? S1 : S0;
                                if (p.tma_l2 == 3) {
                                    tma_load_2d_2sm(smem_u32(st), &p.tma.a[second ? 1 : 0][g], 0,
                                                    (int)((srcA - Sx.A) >> 11), fb);
                                    tma_load_2d_2sm(smem_u32(st + kAStage), &p.tma.b[second ? 1 : 0][g], 0,
                                                    (int)((srcB - Sx.B) >> 11), fb);
                                } else {
                                    tma_load_2d_2sm_hint(smem_u32(st), &p.tma.a[second ? 1 : 0][g], 0,
                                                         (int)((srcA - Sx.A) >> 11), fb, l2pol);
                                    tma_load_2d_2sm_hint(smem_u32(st + kAStage), &p.tma.b[second ? 1 : 0][g], 0,
                                                         (int)((srcB - Sx.B) >> 11), fb, l2pol);
                                }
                            }
                            __syncwarp();
                            if (++s == kStages) { s = 0; ph ^= 1; }
                            continue;
                        }
                        const bool drop = FAULT && kt == klo && w == (int)cluster_id();
                        if (elect_one()) {
                            mbar_expect_tx(&B.full[s], bytesA + bytesB);
                            uint8_t* st = B.stage_base + s * kStageBytes;
                            if (!drop) {
                                bulk_g2s(st, srcA, bytesA, &B.full[s]);
                                bulk_g2s(st + kAStage, srcB, bytesB, &B.full[s]);
                            }
                        }
                        __syncwarp();
                        if (++s == kStages) { s = 0; ph ^= 1; }
                    }
                }
            }
        }
        if (p.dbg && lane == 0) atomicAdd(&p.dbg[0], (unsigned long long)st_empty);
    } else if (warp == 1 && !leader) {
        // ------------------------------------------------ peer: relay "stage full" to the leader
        // (bulk-copy producer only; 2-CTA TMA completes the leader's barrier directly)
        if (!TMA) {
            int s = 0; uint32_t ph = 0;
            const uint32_t leader_full0 = mapa(smem_u32(&B.full[0]), 0);
            for (int w = cluster_id(); w < wm.items(); w += nclusters())
                for (int i = 0; i < kPasses * wm.item_kb(w); ++i) {
                    mbar_wait(&B.full[s], ph);
                    if (elect_one()) mbar_arrive_cluster(leader_full0 + s * 8);
                    __syncwarp();
                    if (++s == kStages) { s = 0; ph ^= 1; }
                }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ leader: MMA issuer (one elected lane)
        int s = 0; uint32_t ph = 0; uint32_t u = 0;
        int item_no = 0;
        long long st_tempty = 0, st_full = 0;
        const long long t_start = clock64();
        for (int w = cluster_id(); w < wm.items(); w += nclusters()) {
            int party, m, n, klo, khi;
            wm.decode(w, party, m, n, klo, khi);
            const bool rev = SERP && (item_no++ & 1);
            const int kstep = rev ? -kc : kc;
            for (int k0 = rev ? klo + (khi - klo - 1) / kc * kc : klo; rev ? k0 >= klo : k0 < khi; k0 += kstep) {
                const int k1 = min(khi, k0 + kc);
                for (int g = 0; g < kPasses; ++g, ++u) {
                    for (int kt = k0; kt < k1; ++kt) {
                        {
                            const long long w0 = p.dbg ? clock64() : 0;
                            mbar_wait_cluster(&B.full[s], ph);
                            if (p.dbg) st_full += clock64() - w0;
                        }
                        tc_fence_after();
                        const uint64_t da = smem_desc(smem_u32(B.stage_base + s * kStageBytes));
                        const uint64_t db = da + (kAStage >> 4);
                        if (kt == k0) {
                            // first block of the unit: each slot pair may be overwritten once both
                            // epilogues have drained it (the pair-1 drain overlaps pair-0 MMAs)
                            const long long w0 = p.dbg ? clock64() : 0;
                            mbar_wait_cluster(&B.tempty[0], (u & 1) ^ 1);
                            if (p.dbg) st_tempty += clock64() - w0;
                            tc_fence_after();
                            if (g == 0) issue_slots<0, true, 0>(da, db, tmem_base); else issue_slots<1, true, 0>(da, db, tmem_base);
                            const long long w1 = p.dbg ? clock64() : 0;
                            mbar_wait_cluster(&B.tempty[1], (u & 1) ^ 1);
                            if (p.dbg) st_tempty += clock64() - w1;
                            tc_fence_after();
                            if (g == 0) issue_slots<0, true, 2>(da, db, tmem_base); else issue_slots<1, true, 2>(da, db, tmem_base);
                        } else {
                            if (g == 0) issue_kblock<0>(da, db, tmem_base); else issue_kblock<1>(da, db, tmem_base);
                        }
                        tc_commit_both(&B.empty[s]);
                        if (++s == kStages) { s = 0; ph ^= 1; }
                    }
                    tc_commit_both(B.tfull);
                }
            }
        }
        if (p.dbg && lane == 0) {
            atomicAdd(&p.dbg[1], (unsigned long long)st_tempty);
            atomicAdd(&p.dbg[2], (unsigned long long)st_full);
            atomicAdd(&p.dbg[3], (unsigned long long)(clock64() - t_start));
        }
    }
}

// ---------------------------------------------------------------- epilogue warpgroups
// run[j] += acc_S[j] * 2^(8S) + acc_{7-S}[j] * 2^(8(7-S))  (mod 2^64) for the 64
// columns of this thread, with acc read as u32.  Compile-time S: the two 32-bit
// halves of the contribution are built with constant shifts (the 7-S term only
// touches the high word), then one 64-bit add.
template <int S>
__device__ __forceinline__ void drain_pair(uint64_t (&run)[64], uint32_t t_lo, uint32_t t_hi) {
#pragma unroll
    for (int cc = 0; cc < 64; cc += 16) {
        uint32_t a[16], b[16];
        tmem_ld16(t_lo + cc, a);
        tmem_ld16(t_hi + cc, b);
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const uint32_t lo32 = a[j] << (8 * S);
            const uint32_t hi32 = (S == 0 ? 0u : (a[j] >> (32 - 8 * S))) + (b[j] << (24 - 8 * S));
            run[cc + j] += ((uint64_t)hi32 << 32) | lo32;
        }
    }
}

__device__ __forceinline__ void epilogue_role(const RingGemmParams& p, const WorkMap& wm, int warp, int lane,
                                              uint32_t rank, uint32_t tmem_base, const Bars& B) {
    const int wq = warp & 3;                       // TMEM lane quadrant of this warp
    const int half = (warp - 4) >> 2;              // column half: 64 columns each
    const int row = wq * 32 + lane;
    const uint32_t tempty_leader = mapa(smem_u32(B.tempty), 0);   // [0] slots 0-1, [1] slots 2-3
    // full-sector (32-byte) accesses when every row start is 32-byte aligned
    const bool vec = (p.N & 3) == 0 && (p.party_stride_z & 3) == 0 && (p.party_stride_c & 3) == 0 &&
                     (p.partial_stride & 3) == 0 && (reinterpret_cast<uintptr_t>(p.Z) & 31) == 0 &&
                     (reinterpret_cast<uintptr_t>(p.C) & 31) == 0 && (reinterpret_cast<uintptr_t>(p.partials) & 31) == 0;
    const uint64_t pol = evict_first_policy();
    const uint32_t tbase = tmem_base + ((uint32_t)(wq * 32) << 16) + half * 64;
    // the epilogue reads C and writes Z: order it after the previous kernel (PDL) itself,
    // not only through the producer -> MMA chain, which is empty when K == 0
    asm volatile("griddepcontrol.wait;" ::: "memory");
    uint32_t u = 0;
    for (int w = cluster_id(); w < wm.items(); w += nclusters()) {
        int party, m, n, klo, khi;
        wm.decode(w, party, m, n, klo, khi);
        const int bi = party / wm.nparties;                  // instance -> (batch element, party)
        party -= bi * wm.nparties;
        uint64_t run[64];
#pragma unroll
        for (int j = 0; j < 64; ++j) run[j] = 0;
        for (int k0 = klo; k0 < khi; k0 += wm.kc) {
            for (int g = 0; g < kPasses; ++g, ++u) {
                mbar_wait(B.tfull, u & 1);
                tc_fence_after();
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    // slot pair h of super-pass g holds shifts (S, 7-S) with S = 2g + h
                    const uint32_t tl = tbase + (2 * h) * 128, th = tl + 128;
                    switch (2 * g + h) {
                        case 0: drain_pair<0>(run, tl, th); break;
                        case 1: drain_pair<1>(run, tl, th); break;
                        case 2: drain_pair<2>(run, tl, th); break;
                        default: drain_pair<3>(run, tl, th); break;
                    }
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive_cluster(tempty_leader + h * 8);   // release this slot pair
                }
            }
        }
        // tile end: z = trunc(c + sum of all units) — one write per element.
        // Element (grow, gc) of the GEMM's output sits at base + gc * cs: row-major
        // normally; column-major (i.e. the caller's row-major z, with the GEMM
        // computing z^T) when transpose_out is set, and per-image column-major
        // (NCHW conv output) with out_hw — then the 32 lanes of a warp (32
        // consecutive rows) touch up to 256 contiguous bytes per column.
        const int64_t grow = (int64_t)m * kTileM + rank * 128 + row;
        const int64_t gc0 = (int64_t)n * kTileN + half * 64;
        const int64_t hw = p.out_hw > 0 ? p.out_hw : (p.transpose_out ? p.M : 0);
        const bool tr = hw > 0;
        const int64_t cs = tr ? hw : 1;
        const int64_t off = (tr ? (grow / hw) * p.N * hw + grow % hw : grow * p.N) + gc0 * cs;
        const bool full = !tr && vec && gc0 + 64 <= p.N;
        if (grow < p.M && wm.splits > 1) {
            // split-K: store this K range's partial sum in its own slab of the
            // partials buffer (same element layout as z); ring_gemm_finalize adds
            // the slabs (ring addition commutes, any order is exact), c_p, and
            // applies the truncation.
            const int s = w % wm.splits;
            uint64_t* pb = p.partials + (int64_t)s * p.partial_stride + party * p.party_stride_z +
                           bi * p.batch_stride_z + off;
            if (full) {
                const uint64_t ppol = p.partials_evict_first ? pol : evict_last_policy();
#pragma unroll
                for (int j = 0; j < 64; j += 4) st_stream4(pb + j, &run[j], ppol);
            } else {
#pragma unroll
                for (int j = 0; j < 64; ++j)
                    if (gc0 + j < p.N) pb[j * cs] = run[j];
            }
        } else if (grow < p.M) {
            // z = trunc(c + run).  z may alias c (in-place second phase): each
            // element is read before it is written by the same thread.  Batches of
            // 16 columns: all loads of a batch are issued before its stores, so a
            // row costs 4 memory round trips, not 32.
            uint64_t* zb = p.Z + party * p.party_stride_z + bi * p.batch_stride_z + off;
            const uint64_t* cb = p.C ? p.C + party * p.party_stride_c + bi * p.batch_stride_c + off : nullptr;
#pragma unroll
            for (int jb = 0; jb < 64; jb += 16) {
                uint64_t v[16];
                if (full) {
#pragma unroll
                    for (int q = 0; q < 16; q += 4) {
                        if (cb) ld_stream4(cb + jb + q, pol, &v[q]);
                        else v[q] = v[q + 1] = v[q + 2] = v[q + 3] = 0ull;
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < 16; ++j) v[j] = (cb && gc0 + jb + j < p.N) ? cb[(jb + j) * cs] : 0ull;
                }
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    v[j] += run[jb + j];
                    if (p.trunc_bits) v[j] = div_pow2_round(v[j], p.trunc_bits);
                }
                if (full) {
#pragma unroll
                    for (int q = 0; q < 16; q += 4) st_stream4(zb + jb + q, &v[q], pol);
                } else {
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        if (gc0 + jb + j < p.N) zb[(jb + j) * cs] = v[j];
                }
            }
        }
    }
}

template <bool FAULT, bool TMA, bool SERP = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
ring_gemm_kernel(const __grid_constant__ RingGemmParams p, int parties) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    if (p.dbg && threadIdx.x == 0) atomicMin(&p.dbg[4], globaltimer());      // timeline (debug mode)
    if (threadIdx.x == 0) asm volatile("griddepcontrol.launch_dependents;");  // the split-K finalize may launch
    Bars B;
    B.stage_base = smem;
    B.full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
    B.empty = B.full + kStages;
    B.tfull = B.empty + kStages;
    B.tempty = B.tfull + 1;           // [2]: TMEM slots 0-1 / 2-3 drained
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(B.tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const bool leader = (rank == 0);
    WorkMap wm;
    wm.tm = TileMap{parties * (p.batch > 1 ? p.batch : 1), (int)(pad_rows<Layout::Left>(p.M) / kTileM),
                    (int)(pad_rows<Layout::Right>(p.N) / kTileN), p.group_m > 0 ? p.group_m : kGroupM,
                    p.party_major};
    wm.nparties = parties;
    wm.tkb = p.seg[0].kb + (p.nseg > 1 ? p.seg[1].kb : 0);
    wm.kc = p.kc;
    wm.splits = p.splits < 1 ? 1 : p.splits;

    if (threadIdx.x == 0) {
        // full: the leader's own copies (+ the peer's relay without TMA; with 2-CTA TMA the
        // peer's bytes complete the leader's barrier directly)
        for (int s = 0; s < kStages; ++s) { mbar_init(&B.full[s], (leader && !TMA) ? 2 : 1); mbar_init(&B.empty[s], 1); }
        mbar_init(B.tfull, 1);
        for (int h = 0; h < 2; ++h) mbar_init(&B.tempty[h], 2 * kEpiWarps);   // both CTAs' epilogue warps (leader's copy)
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
    if (p.dbg && threadIdx.x == 0) atomicMax(&p.dbg[5], globaltimer());
    // register budget: the control warpgroup needs few, the epilogue holds 64 u64 sums per thread
    if (warp < 4) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 64;");
        control_roles<FAULT, TMA, SERP>(p, wm, warp, lane, rank, tmem_base, B);
        if (p.dbg && warp == 1 && lane == 0 && rank == 0) atomicMax(&p.dbg[6], globaltimer());
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 216;");
        epilogue_role(p, wm, warp, lane, rank, tmem_base, B);
        if (p.dbg && lane == 0) atomicMax(&p.dbg[7], globaltimer());
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

int ring_gemm_max_kc() {
    // largest K_r with 4 * K_r * 255^2 <= 2^32 - 1 (shift 3, the tightest exact one), in 32-K blocks
    const uint64_t lim = 0xFFFFFFFFull / (4ull * 65025ull);
    return (int)(lim / kKBlock);
}

int ring_gemm_default_kc(int total_kb) {
    // 64 blocks = 2048 K per unit: long enough that the TMEM drain between units
    // costs ~2% of the MMA time, short enough that the concurrent clusters' K
    // window stays in L2 for the second super-pass.  Short reductions run as
    // one chunk.  MPC_GEMM_KC overrides (tuning experiments).
    static int env_kc = -1;
    if (env_kc < 0) {
        const char* e = getenv("MPC_GEMM_KC");
        env_kc = e ? atoi(e) : 0;
    }
    int kc = env_kc > 0 ? env_kc : 64;
    if (total_kb <= kc + kc / 2) kc = total_kb;
    if (kc > ring_gemm_max_kc()) kc = ring_gemm_max_kc();
    return kc < 1 ? 1 : kc;
}

size_t ring_gemm_smem_bytes() {
    return (size_t)gemm::kStages * gemm::kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
}

// Tensor maps of the 2-CTA kernel's operands: each segment's plane buffer as a 2-D
// tensor of 256-byte rows (every block offset, party and batch stride is a multiple
// of 256 B), boxes of one super-pass's planes (8 or 6) of one 32-K block.
static PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
    static const PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult qr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &qr) != cudaSuccess ||
            qr != cudaDriverEntryPointSuccess)
            f = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    }();
    return fn;
}
static CUtensorMapL2promotion tma_promotion() {
    static const int v = getenv("MPC_GEMM_TMA_PROMO") ? atoi(getenv("MPC_GEMM_TMA_PROMO")) : 3;   // tuning knob
    return v == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE : v == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
         : v == 2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
}
constexpr int kTmaRow = 2048;                     // bytes per tensor-map row: 256 x 8-byte elements
static bool encode_rows(CUtensorMap* m, const void* base, uint64_t bytes, uint32_t box_rows) {
    const PFN_cuTensorMapEncodeTiled_v12000 enc = tmap_encoder();
    if (!enc || !base || bytes < kTmaRow || (bytes % kTmaRow) || (reinterpret_cast<uintptr_t>(base) & 15)) return false;
    const cuuint64_t dims[2] = {kTmaRow / 8, bytes / kTmaRow};
    const cuuint64_t strides[1] = {kTmaRow};
    const cuuint32_t box[2] = {kTmaRow / 8, box_rows};
    const cuuint32_t es[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, const_cast<void*>(base), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, tma_promotion(),
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// Bytes of every operand plane buffer a launch reads (both segments, all instances).
static uint64_t ring_gemm_plane_bytes(const RingGemmParams& q, int parties) {
    const int64_t nb = q.batch > 1 ? q.batch : 1;
    const int64_t rbA = pad_rows<Layout::Left>(q.M) / gemm::GL::kRows, rbB = pad_rows<Layout::Right>(q.N) / gemm::GR::kRows;
    uint64_t tot = 0;
    for (int sg = 0; sg < q.nseg && sg < 2; ++sg) {
        const RingGemmSegment& S = q.seg[sg];
        const uint64_t ia = (uint64_t)rbA * S.kb * 8 * gemm::GL::kBlock, ib = (uint64_t)rbB * S.kb * 8 * gemm::GR::kBlock;
        tot += ia * ((S.party_stride_A ? parties : 1) * (S.batch_stride_A ? nb : 1));
        tot += ib * ((S.party_stride_B ? parties : 1) * (S.batch_stride_B ? nb : 1));
    }
    return tot;
}
static bool fill_tma(RingGemmParams& q, int parties) {
    const int64_t nb = q.batch > 1 ? q.batch : 1;
    const int64_t rbA = pad_rows<Layout::Left>(q.M) / gemm::GL::kRows, rbB = pad_rows<Layout::Right>(q.N) / gemm::GR::kRows;
    for (int sg = 0; sg < q.nseg && sg < 2; ++sg) {
        const RingGemmSegment& S = q.seg[sg];
        const uint64_t instA = (uint64_t)rbA * S.kb * 8 * gemm::GL::kBlock;
        const uint64_t instB = (uint64_t)rbB * S.kb * 8 * gemm::GR::kBlock;
        const uint64_t extA = instA + (uint64_t)(parties - 1) * S.party_stride_A + (uint64_t)(nb - 1) * S.batch_stride_A;
        const uint64_t extB = instB + (uint64_t)(parties - 1) * S.party_stride_B + (uint64_t)(nb - 1) * S.batch_stride_B;
        if ((S.party_stride_A | S.party_stride_B | S.batch_stride_A | S.batch_stride_B) % kTmaRow) return false;
        for (int g = 0; g < gemm::kPasses; ++g) {
            const int planes = g == 0 ? 8 : 6;
            if (!encode_rows(&q.tma.a[sg][g], S.A, extA, planes * gemm::GL::kBlock / kTmaRow) ||
                !encode_rows(&q.tma.b[sg][g], S.B, extB, planes * gemm::GR::kBlock / kTmaRow))
                return false;
        }
    }
    return true;
}

cudaError_t ring_gemm_launch(const RingGemmParams& prm, int parties, cudaStream_t stream) {
    static int attr_dev = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    const size_t smem = ring_gemm_smem_bytes();
    if (attr_dev != dev) {
        cudaError_t e = cudaSuccess;
        for (auto k : {gemm::ring_gemm_kernel<false, true>, gemm::ring_gemm_kernel<false, true, true>,
                       gemm::ring_gemm_kernel<false, false>, gemm::ring_gemm_kernel<false, false, true>,
                       gemm::ring_gemm_kernel<true, false>})
            if (e == cudaSuccess) e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr_dev = dev;
    }
    if (prm.kc < 1 || prm.kc > ring_gemm_max_kc()) return cudaErrorInvalidValue;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int inst = parties * (prm.batch > 1 ? prm.batch : 1);       // GEMM instances (batch x parties)
    const int64_t tiles = (int64_t)inst * (pad_rows<Layout::Left>(prm.M) / gemm::kTileM) *
                          (pad_rows<Layout::Right>(prm.N) / gemm::kTileN);
    int64_t max_clusters = sms / 2;
    if (prm.max_clusters > 0 && prm.max_clusters < max_clusters) max_clusters = prm.max_clusters;
    const int tkb = prm.seg[0].kb + (prm.nseg > 1 ? prm.seg[1].kb : 0);
    RingGemmParams q = prm;
    static const int env_group = getenv("MPC_GEMM_GROUPM") ? atoi(getenv("MPC_GEMM_GROUPM")) : 0;
    if (q.group_m <= 0) q.group_m = env_group;
    static const int env_pm = getenv("MPC_GEMM_PARTY_MAJOR") ? atoi(getenv("MPC_GEMM_PARTY_MAJOR")) : -1;
    q.party_major = env_pm > 0 ? 1 : 0;
    static const int env_fault = getenv("MPC_GEMM_FAULT_INJECT") ? atoi(getenv("MPC_GEMM_FAULT_INJECT")) : 0;
    q.fault_inject = env_fault;
    static const int env_pef = getenv("MPC_PARTIALS_EVICT_FIRST") ? atoi(getenv("MPC_PARTIALS_EVICT_FIRST")) : 0;
    q.partials_evict_first = env_pef;
    q.splits = prm.partials ? ring_gemm_splits(inst, prm.M, prm.N, tkb, max_clusters, prm.small != 0) : 1;
    if (prm.small) {
        if (q.splits > 1) q.partial_stride = ring_gemm_out_elems(q, parties);
        cudaError_t e = ring_gemm_small_launch(q, parties, 2 * max_clusters, stream);
        if (e != cudaSuccess || q.splits <= 1) return e;
        return ring_gemm_finalize(q, parties, stream);
    }
    if (q.splits > 1) {
        // split-K: partial sums go to per-split slabs, then finalize adds them, c_p, truncates
        q.partial_stride = ring_gemm_out_elems(q, parties);
        const int64_t kc_split = (tkb + q.splits - 1) / q.splits;
        if (kc_split < q.kc) q.kc = (int)kc_split;
    }
    int64_t clusters = tiles * q.splits < max_clusters ? tiles * q.splits : max_clusters;
    if (clusters < 1) clusters = 1;
    static const bool debug = getenv("MPC_GEMM_DEBUG") != nullptr;
    void (*dbg_kern)(const RingGemmParams, int) = nullptr;
    {
        // Producer: 2-CTA tensor TMA (no relay hop; measured 2-3% faster at 4096^3 over
        // 50-200 step runs and 1-4% on the model chains), except for GEMMs whose operand
        // planes exceed 2 GiB: there the TMA-fed kernel reads far more DRAM (4-party
        // 8192^3: 276 vs 100 GB per launch; faster alone under ncu, 3% slower in a
        // power-capped run).  In some GPU calls the TMA producer also read 1.5-1.8x the
        // DRAM bytes at 4096^3.  MPC_GEMM_TMA=0 / 1 forces either; fault
        // injection uses the bulk path.
        static const int env_tma = getenv("MPC_GEMM_TMA") ? atoi(getenv("MPC_GEMM_TMA")) : -1;
        const uint64_t plane_bytes = ring_gemm_plane_bytes(q, parties);
        const bool want_tma = env_tma < 0 ? plane_bytes <= (2ull << 30) : env_tma != 0;
        // Launches over more than 2 GiB of operand planes (configs[4]) use 32-block units:
        // the concurrent clusters' K window then stays in L2 (4-party 8192^3: DRAM reads
        // 106 -> 68 GB per launch, ncu 101.7 -> 95.3 ms; 16 / 24 blocks no better), while
        // 4096^3 keeps 64 (32: 5.90 -> 6.01 ms, the drain between units costs more).
        if (plane_bytes > (2ull << 30) && !getenv("MPC_GEMM_KC") && q.kc > 32) q.kc = 32;
        // ... and take the tiles one instance (party) at a time in groups of 8 row tiles: a wave of 74
        // tiles then reads 8 row strips of (a_p, eps) and ~9 column strips of (delta, b'_p) instead of
        // 4 x (4 a_p + eps) and ~5 x (delta + 4 b'_p) — 4-party 8192^3 DRAM reads 68.5 -> 55.3 GB per
        // launch, GEMM 102.4 -> 101.3 ms (profiles/r02/tile_order.txt); 4096^3 unchanged either way
        if (plane_bytes > (2ull << 30) && env_pm < 0) {
            q.party_major = 1;
            if (prm.group_m <= 0 && env_group <= 0) q.group_m = 8;
        }
        // Every launch walks K in alternate directions on a cluster's consecutive items: a wave
        // ends with the last K units of its row strips in L2, and the next wave (same row tiles,
        // the next column tiles) starts there.  DRAM reads per launch: 4-party 8192^3 55.3 -> 53.0 GB,
        // 8-party 111 -> 107 GB (time unchanged); 2-party 4096^3 7.25 -> 6.6 GB, 100-step bench
        // 6.50 -> 6.46 ms (lower power under the cap).  One-item-per-cluster launches (small layers)
        // are unaffected.  MPC_GEMM_SERPENTINE=0 disables it.
        static const int env_serp = getenv("MPC_GEMM_SERPENTINE") ? atoi(getenv("MPC_GEMM_SERPENTINE")) : 1;
        q.serpentine = env_serp != 0 ? 1 : 0;
        const bool tma = want_tma && !q.fault_inject && fill_tma(q, parties);
        static const int env_l2 = getenv("MPC_GEMM_TMA_L2") ? atoi(getenv("MPC_GEMM_TMA_L2")) : 3;
        q.tma_l2 = env_l2;
        auto kern = q.fault_inject             ? gemm::ring_gemm_kernel<true, false>
                  : tma && q.serpentine        ? gemm::ring_gemm_kernel<false, true, true>
                  : tma                        ? gemm::ring_gemm_kernel<false, true>
                  : q.serpentine               ? gemm::ring_gemm_kernel<false, false, true>
                                               : gemm::ring_gemm_kernel<false, false>;
        if (!debug) {
            cudaError_t e = launch_pdl(kern, dim3((unsigned)(clusters * 2)), dim3(gemm::kThreads), smem, stream, q, parties);
            if (e != cudaSuccess || q.splits <= 1) return e;
            return ring_gemm_finalize(q, parties, stream);
        }
        dbg_kern = kern;
    }
    // diagnostic mode (the same kernel variant, launched without PDL): stall-cycle attribution of the
    // producer and MMA threads and a globaltimer timeline
    unsigned long long h[8] = {0, 0, 0, 0, ~0ull, 0, 0, 0};
    cudaMalloc(&q.dbg, sizeof(h));
    cudaMemcpyAsync(q.dbg, h, sizeof(h), cudaMemcpyHostToDevice, stream);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0, stream);
    dbg_kern<<<(unsigned)(clusters * 2), gemm::kThreads, smem, stream>>>(q, parties);
    cudaEventRecord(e1, stream);
    cudaError_t e = cudaGetLastError();
    cudaMemcpyAsync(h, q.dbg, sizeof(h), cudaMemcpyDeviceToHost, stream);
    cudaStreamSynchronize(stream);
    float kms = 0.f;
    cudaEventElapsedTime(&kms, e0, e1);
    cudaEventDestroy(e0); cudaEventDestroy(e1);
    cudaFree(q.dbg);
    const double n = (double)clusters;
    fprintf(stderr, "[ring_gemm] M=%lld N=%lld kb=%d kc=%d splits=%d clusters=%lld  per MMA thread: total %.0f cyc, "
            "wait tempty %.1f%%, wait full %.1f%%; producer wait empty %.0f cyc | event %.1f us, timeline us: "
            "setup done %.1f, MMA issue end %.1f, epilogue end %.1f\n",
            (long long)prm.M, (long long)prm.N, tkb, q.kc, q.splits, (long long)clusters, h[3] / n,
            100.0 * h[1] / h[3], 100.0 * h[2] / h[3], h[0] / (2 * n), kms * 1e3, (h[5] - h[4]) * 1e-3,
            (h[6] - h[4]) * 1e-3, (h[7] - h[4]) * 1e-3);
    q.dbg = nullptr;
    if (e != cudaSuccess || q.splits <= 1) return e;
    return ring_gemm_finalize(q, parties, stream);
}

// Split-K factor: minimise (waves of work items) x (blocks per item), with at
// least 8 blocks per item; ties keep fewer splits (the finalize pass costs an
// extra read/write of z).
int ring_gemm_choose_splits(int64_t tiles, int tkb, int64_t clusters) {
    static const int env = getenv("MPC_GEMM_SPLITS") ? atoi(getenv("MPC_GEMM_SPLITS")) : 0;
    if (env > 0) return tkb >= env ? env : (tkb > 0 ? tkb : 1);
    static const int env_minkb = getenv("MPC_GEMM_MINKB") ? atoi(getenv("MPC_GEMM_MINKB")) : 0;
    // items of at least 8 blocks; a reduction of under 16 blocks may split into items of 4
    // (784 x 128 x 512: 30.8 -> 26.7 us per layer; MPC_GEMM_MINKB forces one length everywhere)
    const int minkb = env_minkb > 0 ? env_minkb : (tkb < 16 ? 4 : 8);
    if (tiles <= 0 || tkb < 2 * minkb || tiles >= clusters) return 1;
    int best = 1;
    double best_cost = 1e30;
    for (int s = 1; s <= tkb / minkb && s <= 64; ++s) {
        const int64_t waves = (tiles * s + clusters - 1) / clusters;
        const double cost = (double)waves * ((tkb + s - 1) / s) * 1.0 + (s > 1 ? 2.0 : 0.0);
        if (cost < best_cost - 1e-9) { best_cost = cost; best = s; }
    }
    return best;
}

size_t ring_gemm_partials_bytes(int parties, int64_t M, int64_t N, int total_kb, int max_clusters, bool small) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t tiles = (int64_t)parties * (pad_rows<Layout::Left>(M) / gemm::kTileM) *
                          (pad_rows<Layout::Right>(N) / gemm::kTileN);
    int64_t clusters = sms / 2;
    if (max_clusters > 0 && max_clusters < clusters) clusters = max_clusters;
    (void)tiles;
    const int s = ring_gemm_splits(parties, M, N, total_kb, clusters, small);
    return s > 1 ? (size_t)s * parties * M * N * sizeof(uint64_t) : 0;
}

namespace gemm {
__global__ void finalize_kernel(uint64_t* z, const uint64_t* c, const uint64_t* __restrict__ part, int splits,
                                int64_t n, int bits) {
    asm volatile("griddepcontrol.wait;" ::: "memory");     // programmatic dependent of the GEMM
    asm volatile("griddepcontrol.launch_dependents;");      // the next split kernel may be scheduled
    const bool vec = (n & 1) == 0 && ((reinterpret_cast<uintptr_t>(z) | reinterpret_cast<uintptr_t>(part) |
                                       (c ? reinterpret_cast<uintptr_t>(c) : 0)) & 15) == 0;
    if (vec) {
        // two elements per thread (16-byte accesses) and four slabs' loads in flight per step
        // (ring addition: any grouping is exact); z may alias c — each pair is read first
        const int64_t n2 = n / 2;
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2; i += (int64_t)gridDim.x * blockDim.x) {
            ulonglong2 v = c ? reinterpret_cast<const ulonglong2*>(c)[i] : make_ulonglong2(0ull, 0ull);
            int s = 0;
            for (; s + 4 <= splits; s += 4) {
                ulonglong2 t[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) t[q] = __ldcs(reinterpret_cast<const ulonglong2*>(part + (int64_t)(s + q) * n) + i);
#pragma unroll
                for (int q = 0; q < 4; ++q) { v.x += t[q].x; v.y += t[q].y; }
            }
            for (; s < splits; ++s) {
                const ulonglong2 t = __ldcs(reinterpret_cast<const ulonglong2*>(part + (int64_t)s * n) + i);
                v.x += t.x; v.y += t.y;
            }
            if (bits) { v.x = div_pow2_round(v.x, bits); v.y = div_pow2_round(v.y, bits); }
            reinterpret_cast<ulonglong2*>(z)[i] = v;
        }
        return;
    }
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t v = c ? c[i] : 0ull;
        for (int s = 0; s < splits; ++s) v += part[(int64_t)s * n + i];
        z[i] = bits ? div_pow2_round(v, bits) : v;
    }
}
}  // namespace gemm

// z = trunc(z + c) over all parties after a split-K GEMM (party buffers contiguous).
int64_t ring_gemm_out_elems(const RingGemmParams& q, int parties) {
    const int64_t per_party = (q.batch > 1 ? q.batch : 1) * q.M * q.N;
    return parties > 1 ? (int64_t)parties * q.party_stride_z : per_party;
}

cudaError_t ring_gemm_finalize(const RingGemmParams& q, int parties, cudaStream_t stream) {
    const int64_t n = ring_gemm_out_elems(q, parties);
    const int64_t per_party = (q.batch > 1 ? q.batch : 1) * q.M * q.N;
    if ((parties > 1 && (q.party_stride_z != per_party || (q.C && q.party_stride_c != q.party_stride_z))) ||
        (q.batch > 1 && (q.batch_stride_z != q.M * q.N || (q.C && q.batch_stride_c != q.batch_stride_z))))
        return cudaErrorInvalidValue;                   // the finalize pass needs z (and c) contiguous
    int64_t blocks = ((n % 2 == 0 ? n / 2 : n) + 255) / 256;     // element pairs when n is even
    if (blocks > 148 * 8) blocks = 148 * 8;
    if (blocks < 1) blocks = 1;
    return launch_pdl(gemm::finalize_kernel, dim3((unsigned)blocks), dim3(256), 0, stream, q.Z, q.C,
                      (const uint64_t*)q.partials, q.splits, n, q.trunc_bits);
}

}  // namespace mpc

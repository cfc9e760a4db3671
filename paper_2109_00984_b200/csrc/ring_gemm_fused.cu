// ring_gemm_fused.cu — the whole 2-party Beaver private matmul of a small output
// (M <= 32, N <= 32, both parties on this GPU) in one tcgen05 kernel: mask, local
// reveal, limb split and the limb GEMM, with the u64 shares read from HBM once.
//
// The planes-based path (split kernel -> limb planes in HBM -> ring GEMM) reads
// the four u64 share inputs, writes six plane sets (eps, a_0, a_1, delta, b'_0,
// b'_1) and reads them back: for the wide-K text matmul (32 x 519,820 x 32, P:397-
// 410) that is 1.9 GB + 0.8 GB against the 1.06 GB the protocol
// must read.  Here each CTA takes a K range of the one 32 x 32 output tile and,
// per 32-K block, its converter warps load x_p, a_p (32 x 32 each) and y_p, b_p
// (32 x 32 each) straight into registers, form (R7/R8)
//     eps = sum_p (x_p - a_p),   delta = sum_p (y_p - b_p),   b'_0 = b_0 + delta,
// and write the u8 limb planes of eps, a_0, a_1, delta, b'_0, b'_1 into a shared-
// memory stage in the UMMA canonical K-major layout; one thread issues
//     z_p = c_p + a_p @ delta + eps @ b'_p          (mod 2^64, p = 0, 1)
// as stacked-plane MMAs: A_lo / A_hi = left planes 0-3 / 4-7 stacked along M
// (M = 128: lanes 32 i' + r) and B = all 8 planes of a right operand stacked
// along N (N = 256: column 32 j + n), so ONE MMA forms every plane product
// L_i' @ R_j of a stack; party p owns 256 TMEM columns (both parties: all 512):
//   A_lo x R (N = 256)  -> columns 32 j + n,         lane group i' shift i' + j
//   A_hi x R_0..3 (N = 128) -> columns 128 + 32 j + n, lane group i' shift 4 + i' + j
// — the same shift per (lane, column) for both, so they share the accumulator —
// for eps @ b'_p and a_p @ delta: 4 MMAs per party and 32-K block (8 in all)
// instead of 36 plane-pair MMAs (ring_gemm_small.cu issues 12 per party with N =
// 32); products with i + j >= 8 are computed and ignored (64 issued, 36 needed).
// Exactness: an entry with shift <= 3 sums <= 2 products per K (no A_hi term),
// so reading it as u32 is exact for units of <= 1032 32-K blocks; shifts >= 4
// only need the entry mod 2^(64 - 8s) (<= 2^32).
//
// Split-K over the CTAs (one per SM), the 32-K blocks dealt round-robin so the
// CTAs stream neighbouring 256-byte row pieces of x / a through DRAM together;
// slab g of the partials buffer holds CTA g's [2][M][N] sum, and
// ring_gemm_finalize adds the slabs, c_p and the per-share truncation (P <= 2,
// R10).  Bit-identical to the planes-based path: the same ring sums, and
// unsigned addition commutes.
//
// Warps: 0 = TMEM allocator and MMA issuer (one thread), 1..3 idle, then NG (1 by
// default) groups of 8 converter warps taking alternate blocks: in each group 4
// warps for x / a rows (8 rows each) and 4 for y / b columns (8 columns each).
// A converter prefetches its next block into L2; group 0 also drains TMEM at unit
// ends into shared-memory output sums (a warp reads the TMEM lane quadrant
// warp % 4; its warps 4..7 hold party 0, 8..11 party 1) and writes the slab.
//
// Two kernels.  The register path (any K, N) is described above; the TMA-staged one
// (K and N even: 16-byte tensor-map strides) lets one producer thread bring each
// block's shares into shared memory by TMA (x / a in 128-byte-swizzled boxes) and
// the converters read them from there — the default where it applies.
//
// Measured (text 32 x 519,820 x 32, one B200; scripts/gpu/fused*.sh,
// profiles/r02/fused_small/): planes-based path 0.49 ms; register path 0.271 ms;
// TMA-staged 0.193 ms = 0.86 of the HBM floor (kernel 174 µs under ncu: 1.065 GB
// DRAM = the algorithmic bytes at 6.1 TB/s).  The register path's converters
// wait on scattered global loads (long-scoreboard) whose fills share the L1TEX
// data path with the plane stores and the tensor core's operand reads; with 36
// N = 32/64 plane-pair MMAs per block (before the stacked B operand) that path
// ran 0.286 ms (LSU 68% + tensor core 35% of the L1TEX wavefronts).  Knobs:
// MPC_FUSED_TMA=0 (register path), MPC_FUSED_GROUPS=2 (register path: two
// converter groups on alternate blocks), MPC_FUSED_PFD / MPC_FUSED_PF (its L2
// prefetch), MPC_FUSED_CYCLIC=0 (contiguous K ranges); dropped: two blocks of
// loads in flight per thread (setmaxnreg), L1::no_allocate loads (2x slower).
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "ring_gemm.h"
#include "tcgen05.cuh"

namespace mpc {
namespace gemm_fused {
using namespace tc;

constexpr int kRows = 32;                         // output rows and columns of the tile
constexpr int kPlane = 1024;                      // one limb plane of 32 rows x 32 K
constexpr int kSet = 8 * kPlane;                  // the 8 planes of one operand
// stage: [eps][a_0][a_1][delta][b'_0][b'_1] plane sets (plane j of a set at j KiB: the 8 planes of a
// right operand form one 256-row B operand, planes 0..3 / 4..7 of a left one the A_lo / A_hi stacks)
constexpr int kOffEps = 0, kOffA0 = kSet, kOffDelta = 3 * kSet, kOffB0 = 4 * kSet;
constexpr int kStageBytes = 6 * kSet;             // 48 KiB
constexpr int kStages = 4;
// warp 0: TMEM allocator + MMA issuer; 1..3 idle; 4..: NG groups of 8 converter warps
__host__ __device__ constexpr int kThreadsOf(int ng) { return 128 + 256 * ng; }
constexpr int kTmemCols = 512;
constexpr int kMaxUnit = 1032;                    // 32-K blocks per accumulation unit (exact, see above)
constexpr int kPrefetch = 1;                      // blocks (of a converter group) the L2 prefetch runs ahead
__host__ __device__ constexpr uint32_t idesc(int n) {
    return (2u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);   // S32 <- u8 x u8, M = 128
}

__device__ __forceinline__ void mma_u8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t id, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
        :: "r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(id), "r"(acc) : "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                 :: "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void conv_sync() {            // the 8 warps of converter group 0
    asm volatile("bar.sync 1, 256;" ::: "memory");
}
// bulk L2 prefetch of [p, p + bytes): the instruction takes a 16-byte aligned start and size
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(p), a0 = a & ~uintptr_t(15);
    const uint32_t n = (uint32_t)((a + bytes - a0 + 15) & ~uintptr_t(15));
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(a0), "r"(n) : "memory");
}
__device__ __forceinline__ void prefetch_l2_line(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" :: "l"(p));
}

// 8 consecutive-k values of one row -> byte l of each into plane l (8 bytes at
// `off` inside every plane of the set; planes `pstride` bytes apart)
__device__ __forceinline__ void st_planes8(uint8_t* set, uint32_t off, int pstride, const uint64_t (&v)[8]) {
    uint32_t w[8][2];
#pragma unroll
    for (int g = 0; g < 2; ++g) {
        uint32_t lo[4], hi[4];
        transpose4x4((uint32_t)v[4 * g], (uint32_t)v[4 * g + 1], (uint32_t)v[4 * g + 2], (uint32_t)v[4 * g + 3], lo);
        transpose4x4((uint32_t)(v[4 * g] >> 32), (uint32_t)(v[4 * g + 1] >> 32), (uint32_t)(v[4 * g + 2] >> 32),
                     (uint32_t)(v[4 * g + 3] >> 32), hi);
#pragma unroll
        for (int l = 0; l < 4; ++l) { w[l][g] = lo[l]; w[4 + l][g] = hi[l]; }
    }
#pragma unroll
    for (int l = 0; l < 8; ++l)
        *reinterpret_cast<uint2*>(set + off + l * pstride) = make_uint2(w[l][0], w[l][1]);
}

// (row, 8-K quarter kq) -> byte offset of its 8-byte run inside a 32-row plane
__device__ __forceinline__ uint32_t plane_off(int row, int kq) {
    return (uint32_t)((row >> 3) * 256 + (kq >> 1) * 128 + (row & 7) * 16 + (kq & 1) * 8);
}

// 8 consecutive u64 of one row of a row-major matrix (0 past `left` valid values)
__device__ __forceinline__ void load_row8(const uint64_t* __restrict__ src, int64_t left, bool vec, uint64_t (&v)[8]) {
    if (vec && left >= 8) {
        const ulonglong2* s2 = reinterpret_cast<const ulonglong2*>(src);
#pragma unroll
        for (int m = 0; m < 4; ++m) { const ulonglong2 t = __ldg(s2 + m); v[2 * m] = t.x; v[2 * m + 1] = t.y; }
    } else {
#pragma unroll
        for (int m = 0; m < 8; ++m) v[m] = m < left ? __ldg(src + m) : 0ull;
    }
}

template <int NG>
__global__ void __launch_bounds__(kThreadsOf(NG), 1) fused_small_kernel(const __grid_constant__ FusedSmallParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    if (threadIdx.x == 0) asm volatile("griddepcontrol.launch_dependents;");   // the finalize may launch
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes + 2 * kRows * kRows * 8);
    uint64_t* empty = full + kStages;
    uint64_t* tfull = empty + kStages;
    uint64_t* tempty = tfull + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t M = p.M, K = p.K, N = p.N;
    const int KB = (int)num_kb(K);
    const int g = blockIdx.x, G = gridDim.x;
    // this CTA's 32-K blocks: i -> g + i * G (block-cyclic: at any moment the CTAs read neighbouring
    // blocks of the same rows, so the 256-byte row pieces of x / a stream through DRAM pages in order),
    // or a contiguous range (MPC_FUSED_CYCLIC=0)
    const int kb0 = (int)((int64_t)KB * g / G);
    const int nblk = p.cyclic ? (KB > g ? (KB - g + G - 1) / G : 0) : (int)((int64_t)KB * (g + 1) / G) - kb0;
    auto kt_of = [&](int i) { return p.cyclic ? g + i * G : kb0 + i; };
    const int U = p.unit;                                                    // even when NG == 2 (launcher)
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) { mbar_init(&full[s], 8); mbar_init(&empty[s], 1); }
        mbar_init(tfull, 1);
        mbar_init(tempty, 8);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                     :: "r"(smem_u32(tmem_slot)), "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const int64_t sMK = M * K, sKN = K * N;

    if (warp == 0) {
        // ------------------------------------------------ MMA issuer (one thread)
        if (lane == 0) {
            int s = 0; uint32_t ph = 0; uint32_t u = 0;
            long long dbg_full = 0;
            const long long t_mma0 = clock64();
            for (int k0 = 0; k0 < nblk; k0 += U, ++u) {
                const int k1 = min(nblk, k0 + U);
                mbar_wait(tempty, (u & 1) ^ 1);                               // last unit drained
                tc_fence_after();
                for (int kt = k0; kt < k1; ++kt) {
                    const long long w0 = p.dbg ? clock64() : 0;
                    mbar_wait(&full[s], ph);
                    if (p.dbg) dbg_full += clock64() - w0;
                    tc_fence_after();
                    // every operand address from two per-block base values, re-read through an opaque
                    // move so the compiler does not hoist 36 addresses out of the loop
                    uint32_t st = smem_u32(smem + s * kStageBytes), tb = tmem_base;
                    asm volatile("mov.b32 %0, %0;" : "+r"(st));
                    asm volatile("mov.b32 %0, %0;" : "+r"(tb));
                    const uint64_t d0 = smem_desc(st);                       // eps set; +offset>>4 for the rest
                    const uint32_t first = kt == k0 ? 0u : 1u;
                    // party q's accumulator: 256 TMEM columns (column 32 j + n holds right plane j).
                    // Per party 4 MMAs: A_lo (planes 0-3) against all 8 right planes (N = 256) and
                    // A_hi (planes 4-7) against right planes 0-3 into columns 128.. (N = 128), for
                    // eps @ b'_q and a_q @ delta; the first one opens the party's accumulator
#pragma unroll
                    for (int q = 0; q < 2; ++q) {
                        const uint32_t dq = tb + q * 256;
                        const uint64_t dB = d0 + (uint64_t)((kOffB0 + q * kSet) >> 4);
                        const uint64_t dA = d0 + (uint64_t)((kOffA0 + q * kSet) >> 4);
                        const uint64_t dD = d0 + (uint64_t)(kOffDelta >> 4);
                        mma_u8(dq, d0, dB, idesc(256), first);
                        mma_u8(dq + 128, d0 + (uint64_t)((4 * kPlane) >> 4), dB, idesc(128), 1u);
                        mma_u8(dq, dA, dD, idesc(256), 1u);
                        mma_u8(dq + 128, dA + (uint64_t)((4 * kPlane) >> 4), dD, idesc(128), 1u);
                    }
                    tc_commit(&empty[s]);
                    if (++s == kStages) { s = 0; ph ^= 1; }
                }
                tc_commit(tfull);
            }
            if (p.dbg) {
                atomicAdd(&p.dbg[0], (unsigned long long)dbg_full);
                atomicAdd(&p.dbg[1], (unsigned long long)(clock64() - t_mma0));
            }
        }
        __syncwarp();
    } else if (warp >= 4) {
        // ------------------------------------------------ converters (NG groups of 8 warps on alternate
        // blocks, so one group's loads are in flight while the other converts), then the TMEM drain
        asm volatile("griddepcontrol.wait;" ::: "memory");                  // shares written by earlier kernels
        const int cw = warp - 4, cg = cw >> 3, w8 = cw & 7;                  // group, warp in the group
        const bool left = w8 < 4;
        const int grp = w8 & 3;                                              // 8-row (left) / 8-column (right) group
        const int idx = grp * 8 + (lane & 7);                                // row of x / a, or column of y / b
        const int kq = lane >> 3;                                            // 8-K quarter of the 32-K block
        const bool vec = ((K & 1) == 0) && ((reinterpret_cast<uintptr_t>(p.x) | reinterpret_cast<uintptr_t>(p.a)) & 15) == 0;
        const uint32_t poff = plane_off(idx, kq);
        const int q4 = warp & 3;                                             // TMEM lane quadrant = plane group i'
        const int party = w8 >> 2;                                           // drain (group 0): this warp's party
        // L2 prefetch of a later block: a left lane's own 64-byte runs of x_p, a_p; one lane of each
        // right warp the whole 32 x N run of one of y_0, b_0, y_1, b_1 (contiguous)
        auto prefetch = [&](int i) {
            if (i >= nblk || p.pf_mode == 0) return;
            const int kt = kt_of(i);
            const int64_t kbase = (int64_t)kt * 32 + kq * 8;
            if (left) {
                if (idx < M && kbase < K) {
                    const int64_t o = idx * K + kbase;
                    if (p.pf_mode == 1) {
                        prefetch_l2_line(p.x + o); prefetch_l2_line(p.a + o);
                        prefetch_l2_line(p.x + sMK + o); prefetch_l2_line(p.a + sMK + o);
                    } else if (kq == 0) {                                    // one bulk prefetch per row
                        const uint32_t nb = (uint32_t)(8 * (K - kbase < 32 ? K - kbase : 32));
                        prefetch_l2(p.x + o, nb); prefetch_l2(p.a + o, nb);
                        prefetch_l2(p.x + sMK + o, nb); prefetch_l2(p.a + sMK + o, nb);
                    }
                }
            } else if (lane == 0) {
                const int64_t k0 = (int64_t)kt * 32, kl = K - k0 < 32 ? K - k0 : 32;
                const uint64_t* base = ((grp & 1) ? p.b : p.y) + (grp >> 1) * sKN + k0 * N;
                prefetch_l2(base, (uint32_t)(kl * N * 8));
            }
        };
        // TMEM drain target (group 0): the output sums [party][row][32] in shared memory, added to by
        // the four lane-group warps of each party (shared-memory atomics; once per unit)
        unsigned long long* runb = reinterpret_cast<unsigned long long*>(smem + kStages * kStageBytes);
        unsigned long long* mine = runb + ((int64_t)party * kRows + lane) * kRows;
        if (cg == 0) {
            for (int i = threadIdx.x - 128; i < 2 * kRows * kRows; i += 256) runb[i] = 0ull;
            conv_sync();
        }
        int s = cg; uint32_t ph = 0; uint32_t u = 0;                        // block i uses stage i % kStages
        long long dbg_empty = 0;
        const long long t_conv0 = clock64();
        for (int j = 0; j < p.pf_dist; ++j) prefetch(cg + NG * j);
        for (int i = cg; i < nblk; i += NG) {
            prefetch(i + NG * p.pf_dist);
            // this thread's 8 K values of its row / column from the four share inputs
            uint64_t v0[8], v1[8], v2[8], v3[8];
            const int64_t kbase = (int64_t)kt_of(i) * 32 + kq * 8;
            if (left) {
                if (idx < M) {
                    const int64_t o = idx * K + kbase, lft = K - kbase;
                    load_row8(p.x + o, lft, vec, v0);
                    load_row8(p.a + o, lft, vec, v1);
                    load_row8(p.x + sMK + o, lft, vec, v2);
                    load_row8(p.a + sMK + o, lft, vec, v3);
                } else {
#pragma unroll
                    for (int m = 0; m < 8; ++m) v0[m] = v1[m] = v2[m] = v3[m] = 0ull;
                }
            } else {
                const uint64_t* py = p.y + kbase * N + idx;
                const uint64_t* pb = p.b + kbase * N + idx;
                const int lim = idx < N ? (int)(K - kbase < 8 ? K - kbase : 8) : 0;   // valid K rows
#pragma unroll
                for (int m = 0; m < 8; ++m) {
                    const bool ok = m < lim;
                    v0[m] = ok ? __ldg(py + m * N) : 0ull;
                    v1[m] = ok ? __ldg(pb + m * N) : 0ull;
                    v2[m] = ok ? __ldg(py + sKN + m * N) : 0ull;
                    v3[m] = ok ? __ldg(pb + sKN + m * N) : 0ull;
                }
            }
            // mask + local reveal: v0 <- sum_p (plus_p - minus_p)
#pragma unroll
            for (int m = 0; m < 8; ++m) v0[m] = v0[m] - v1[m] + v2[m] - v3[m];
            const long long w0 = p.dbg ? clock64() : 0;
            mbar_wait(&empty[s], ph ^ 1);
            if (p.dbg) dbg_empty += clock64() - w0;
            uint8_t* st = smem + s * kStageBytes;
            if (left) {
                st_planes8(st + kOffEps, poff, kPlane, v0);                 // eps
                st_planes8(st + kOffA0, poff, kPlane, v1);                  // a_0
                st_planes8(st + kOffA0 + kSet, poff, kPlane, v3);           // a_1
            } else {
#pragma unroll
                for (int m = 0; m < 8; ++m) v1[m] += v0[m];                 // b'_0 = b_0 + delta (R8)
                st_planes8(st + kOffDelta, poff, kPlane, v0);               // delta
                st_planes8(st + kOffB0, poff, kPlane, v1);                  // b'_0
                st_planes8(st + kOffB0 + kSet, poff, kPlane, v3);           // b'_1
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> tensor core
            __syncwarp();
            if (lane == 0) mbar_arrive(&full[s]);
            s += NG;
            if (s >= kStages) { s -= kStages; ph ^= 1; }
            // group 0 drains each unit after its own last block of the unit (every unit starts at an
            // even block, so group 0 has one); tfull follows the unit's last MMA, whichever group fed it
            if (cg != 0) continue;
            const int uend = min((i / U + 1) * U, nblk);
            if (i + NG < uend) continue;
            // lane group i' = q4 of D_j holds shift q4 + j (> 7 vanishes mod 2^64)
            mbar_wait(tfull, u & 1);
            tc_fence_after();
            const uint32_t tq = tmem_base + ((uint32_t)(q4 * 32) << 16) + party * 256;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                uint64_t run[16];
#pragma unroll
                for (int c = 0; c < 16; ++c) run[c] = 0ull;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    if (q4 + j > 7) continue;                                // warp-uniform
                    uint32_t a[16];
                    tmem_ld16(tq + j * 32 + 16 * h, a);
                    tmem_wait_ld();
                    const int sh = 8 * (q4 + j);
#pragma unroll
                    for (int c = 0; c < 16; ++c) run[c] += (uint64_t)a[c] << sh;
                }
#pragma unroll
                for (int c = 0; c < 16; ++c) atomicAdd(mine + 16 * h + c, (unsigned long long)run[c]);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(tempty);
            ++u;
        }
        if (p.dbg && lane == 0) {
            atomicAdd(&p.dbg[2], (unsigned long long)dbg_empty);
            atomicAdd(&p.dbg[3], (unsigned long long)(clock64() - t_conv0));
        }
        if (cg == 0) {
            conv_sync();                                                     // every drain has added
            const int et = threadIdx.x - 128;
            const bool split = G > 1;
            for (int e = et; e < 2 * kRows * kRows; e += 256) {
                const int pq = e >> 10, r = (e >> 5) & 31, col = e & 31;
                if (r >= M || col >= N) continue;
                uint64_t v = runb[((int64_t)pq * kRows + r) * kRows + col];
                const int64_t o = (int64_t)pq * M * N + r * N + col;
                if (split) {
                    p.partials[(int64_t)g * 2 * M * N + o] = v;
                } else {
                    if (p.C) v += p.C[o];
                    p.Z[o] = p.trunc_bits ? div_pow2_round(v, p.trunc_bits) : v;
                }
            }
        }
    }
    __syncwarp();
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem_base), "r"(kTmemCols));
    }
}

// ---------------------------------------------------------------- TMA-staged variant
// The same product, the shares brought into shared memory by the tensor-memory
// accelerator instead of the converters' own loads: one producer thread issues, per
// 32-K block, 8 boxes of 16 K x 32 rows of x_p / a_p (128-byte swizzle, so the
// converters' 16-byte reads of one row piece per lane hit distinct banks) and 4
// boxes of N x 32 K rows of y_p / b_p into a raw stage (64 KiB, 2 stages; rows past
// M / K are zero-filled by the TMA); the converters read their 8 K values of each
// input from shared memory, free the raw stage, and write the planes into a plane
// stage (48 KiB, 2 stages) as before.  The MMAs and the drain are the register
// path's; the drained sums stay in registers and are summed across lane groups in
// a raw stage at the end.  Needs K and N even (16-byte tensor-map strides).
constexpr int kRawStages = 2, kPlaneStages = 2;
constexpr int kRawBytes = 64 * 1024;                 // 4 x 8 KiB left boxes, 4 x (32 N 8 B) right boxes
constexpr int kRawRight = 32 * 1024;
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* m, int c0, int c1, int c2, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
        :: "r"(dst), "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)) : "memory");
}

__global__ void __launch_bounds__(384, 1) fused_small_tma_kernel(const __grid_constant__ FusedSmallParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    if (threadIdx.x == 0) asm volatile("griddepcontrol.launch_dependents;");   // the finalize may launch
    uint8_t* planes = smem;                                                    // [kPlaneStages][48 KiB]
    uint8_t* raw = smem + kPlaneStages * kStageBytes;                          // [kRawStages][64 KiB]
    uint64_t* pfull = reinterpret_cast<uint64_t*>(raw + kRawStages * kRawBytes);
    uint64_t* pempty = pfull + kPlaneStages;
    uint64_t* rfull = pempty + kPlaneStages;
    uint64_t* rempty = rfull + kRawStages;
    uint64_t* tfull = rempty + kRawStages;
    uint64_t* tempty = tfull + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t M = p.M, K = p.K, N = p.N;
    const int KB = (int)num_kb(K);
    const int g = blockIdx.x, G = gridDim.x;
    const int nblk = KB > g ? (KB - g + G - 1) / G : 0;                       // blocks g, g + G, ...
    const int U = p.unit;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kPlaneStages; ++s) { mbar_init(&pfull[s], 8); mbar_init(&pempty[s], 1); }
        for (int s = 0; s < kRawStages; ++s) { mbar_init(&rfull[s], 1); mbar_init(&rempty[s], 8); }
        mbar_init(tfull, 1);
        mbar_init(tempty, 8);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                     :: "r"(smem_u32(tmem_slot)), "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ------------------------------------------------ MMA issuer (one thread)
        if (lane == 0) {
            int s = 0; uint32_t ph = 0; uint32_t u = 0;
            for (int k0 = 0; k0 < nblk; k0 += U, ++u) {
                const int k1 = min(nblk, k0 + U);
                mbar_wait(tempty, (u & 1) ^ 1);
                tc_fence_after();
                for (int kt = k0; kt < k1; ++kt) {
                    mbar_wait(&pfull[s], ph);
                    tc_fence_after();
                    uint32_t st = smem_u32(planes + s * kStageBytes), tb = tmem_base;
                    asm volatile("mov.b32 %0, %0;" : "+r"(st));
                    asm volatile("mov.b32 %0, %0;" : "+r"(tb));
                    const uint64_t d0 = smem_desc(st);
                    const uint32_t first = kt == k0 ? 0u : 1u;
#pragma unroll
                    for (int q = 0; q < 2; ++q) {
                        const uint32_t dq = tb + q * 256;
                        const uint64_t dB = d0 + (uint64_t)((kOffB0 + q * kSet) >> 4);
                        const uint64_t dA = d0 + (uint64_t)((kOffA0 + q * kSet) >> 4);
                        const uint64_t dD = d0 + (uint64_t)(kOffDelta >> 4);
                        mma_u8(dq, d0, dB, idesc(256), first);
                        mma_u8(dq + 128, d0 + (uint64_t)((4 * kPlane) >> 4), dB, idesc(128), 1u);
                        mma_u8(dq, dA, dD, idesc(256), 1u);
                        mma_u8(dq + 128, dA + (uint64_t)((4 * kPlane) >> 4), dD, idesc(128), 1u);
                    }
                    tc_commit(&pempty[s]);
                    if (++s == kPlaneStages) { s = 0; ph ^= 1; }
                }
                tc_commit(tfull);
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ------------------------------------------------ TMA producer (one thread)
        asm volatile("griddepcontrol.wait;" ::: "memory");                  // shares written by earlier kernels
        if (lane == 0) {
            int s = 0; uint32_t ph = 0;
            const uint32_t bytes = 8 * 4096 + 4 * (uint32_t)(32 * N * 8);
            for (int i = 0; i < nblk; ++i) {
                const int k0 = (g + i * G) * 32;
                mbar_wait(&rempty[s], ph ^ 1);
                mbar_expect_tx(&rfull[s], bytes);
                const uint32_t dst = smem_u32(raw + s * kRawBytes);
#pragma unroll
                for (int src = 0; src < 4; ++src) {                          // x_0, a_0, x_1, a_1
                    const CUtensorMap* m = (src & 1) ? &p.tm_a : &p.tm_x;
                    tma_load_3d(dst + src * 8192, m, k0, 0, src >> 1, &rfull[s]);
                    tma_load_3d(dst + src * 8192 + 4096, m, k0 + 16, 0, src >> 1, &rfull[s]);
                }
#pragma unroll
                for (int src = 0; src < 4; ++src) {                          // y_0, b_0, y_1, b_1
                    const CUtensorMap* m = (src & 1) ? &p.tm_b : &p.tm_y;
                    tma_load_3d(dst + kRawRight + src * (uint32_t)(32 * N * 8), m, 0, k0, src >> 1, &rfull[s]);
                }
                if (++s == kRawStages) { s = 0; ph ^= 1; }
            }
        }
        __syncwarp();
    } else if (warp >= 4) {
        // ------------------------------------------------ converters (shared memory -> planes), drain
        const int w8 = warp - 4;
        const bool left = w8 < 4;
        const int grp = w8 & 3;
        const int idx = grp * 8 + (lane & 7);
        const int kq = lane >> 3;
        const uint32_t poff = plane_off(idx, kq);
        const int q4 = warp & 3;
        const int party = w8 >> 2;
        uint64_t run[32];
#pragma unroll
        for (int c = 0; c < 32; ++c) run[c] = 0ull;
        int rs = 0, ps = 0; uint32_t rph = 0, pph = 0, u = 0;
        for (int i = 0; i < nblk; ++i) {
            uint64_t v0[8], v1[8], v2[8], v3[8];
            mbar_wait(&rfull[rs], rph);
            const uint8_t* rb = raw + rs * kRawBytes;
            if (left) {
                // row idx, K values 8 kq .. 8 kq + 7: half kq >> 1, 16-byte chunks (kq & 1) * 4 + j,
                // stored at chunk ^ (row & 7) (128-byte swizzle)
                const uint8_t* hb = rb + (kq >> 1) * 4096 + idx * 128;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int ch = (((kq & 1) * 4 + j) ^ (idx & 7)) * 16;
                    const ulonglong2 t0 = *reinterpret_cast<const ulonglong2*>(hb + ch);
                    const ulonglong2 t1 = *reinterpret_cast<const ulonglong2*>(hb + 8192 + ch);
                    const ulonglong2 t2 = *reinterpret_cast<const ulonglong2*>(hb + 16384 + ch);
                    const ulonglong2 t3 = *reinterpret_cast<const ulonglong2*>(hb + 24576 + ch);
                    v0[2 * j] = t0.x; v0[2 * j + 1] = t0.y; v1[2 * j] = t1.x; v1[2 * j + 1] = t1.y;
                    v2[2 * j] = t2.x; v2[2 * j + 1] = t2.y; v3[2 * j] = t3.x; v3[2 * j + 1] = t3.y;
                }
            } else {
                const uint64_t* r0 = reinterpret_cast<const uint64_t*>(rb + kRawRight);
                const int64_t sstride = 32 * N;                              // elements per right box
                const bool ok = idx < N;
#pragma unroll
                for (int m = 0; m < 8; ++m) {
                    const int64_t o = (int64_t)(kq * 8 + m) * N + idx;
                    v0[m] = ok ? r0[o] : 0ull;
                    v1[m] = ok ? r0[sstride + o] : 0ull;
                    v2[m] = ok ? r0[2 * sstride + o] : 0ull;
                    v3[m] = ok ? r0[3 * sstride + o] : 0ull;
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&rempty[rs]);                         // this warp is done reading
            if (++rs == kRawStages) { rs = 0; rph ^= 1; }
#pragma unroll
            for (int m = 0; m < 8; ++m) v0[m] = v0[m] - v1[m] + v2[m] - v3[m];
            mbar_wait(&pempty[ps], pph ^ 1);
            uint8_t* st = planes + ps * kStageBytes;
            if (left) {
                st_planes8(st + kOffEps, poff, kPlane, v0);
                st_planes8(st + kOffA0, poff, kPlane, v1);
                st_planes8(st + kOffA0 + kSet, poff, kPlane, v3);
            } else {
#pragma unroll
                for (int m = 0; m < 8; ++m) v1[m] += v0[m];                 // b'_0 = b_0 + delta (R8)
                st_planes8(st + kOffDelta, poff, kPlane, v0);
                st_planes8(st + kOffB0, poff, kPlane, v1);
                st_planes8(st + kOffB0 + kSet, poff, kPlane, v3);
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&pfull[ps]);
            if (++ps == kPlaneStages) { ps = 0; pph ^= 1; }
            if ((i + 1) % U != 0 && i + 1 != nblk) continue;
            mbar_wait(tfull, u & 1);
            tc_fence_after();
            const uint32_t tq = tmem_base + ((uint32_t)(q4 * 32) << 16) + party * 256;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                if (q4 + j > 7) continue;
                uint32_t a[16], b[16];
                tmem_ld16(tq + j * 32, a);
                tmem_ld16(tq + j * 32 + 16, b);
                tmem_wait_ld();
                const int sh = 8 * (q4 + j);
#pragma unroll
                for (int c = 0; c < 16; ++c) { run[c] += (uint64_t)a[c] << sh; run[16 + c] += (uint64_t)b[c] << sh; }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(tempty);
            ++u;
        }
        // every TMA write has landed (each was waited on) and every MMA completed: the raw stages are
        // free; sum the four lane groups of each output row there
        uint64_t* red = reinterpret_cast<uint64_t*>(raw);                    // [party][i'][row][32]
        uint64_t* mine = red + (((int64_t)party * 4 + q4) * kRows + lane) * kRows;
#pragma unroll
        for (int c = 0; c < 32; c += 2) *reinterpret_cast<ulonglong2*>(mine + c) = make_ulonglong2(run[c], run[c + 1]);
        conv_sync();
        asm volatile("griddepcontrol.wait;" ::: "memory");                  // C / Z / partials after the predecessor
        for (int e = threadIdx.x - 128; e < 2 * kRows * kRows; e += 256) {
            const int pq = e >> 10, r = (e >> 5) & 31, col = e & 31;
            if (r >= M || col >= N) continue;
            uint64_t v = 0;
#pragma unroll
            for (int qq = 0; qq < 4; ++qq) v += red[(((int64_t)pq * 4 + qq) * kRows + r) * kRows + col];
            const int64_t o = (int64_t)pq * M * N + r * N + col;
            if (G > 1) {
                p.partials[(int64_t)g * 2 * M * N + o] = v;
            } else {
                if (p.C) v += p.C[o];
                p.Z[o] = p.trunc_bits ? div_pow2_round(v, p.trunc_bits) : v;
            }
        }
    }
    __syncwarp();
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem_base), "r"(kTmemCols));
    }
}

}  // namespace gemm_fused

static size_t fused_small_tma_smem_bytes() {
    return (size_t)gemm_fused::kPlaneStages * gemm_fused::kStageBytes + (size_t)gemm_fused::kRawStages * gemm_fused::kRawBytes +
           1024 /*align*/ + 256 /*barriers*/;
}

// 3-D tensor maps of the TMA-staged kernel (false: not encodable here -> the register path)
static bool fused_small_maps(FusedSmallParams& q) {
    static const PFN_cuTensorMapEncodeTiled_v12000 enc = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult qr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &qr) != cudaSuccess ||
            qr != cudaDriverEntryPointSuccess)
            f = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    }();
    if (!enc || (q.K & 1) || (q.N & 1) || q.K < 32) return false;
    for (const void* ptr : {(const void*)q.x, (const void*)q.a, (const void*)q.y, (const void*)q.b})
        if (reinterpret_cast<uintptr_t>(ptr) & 15) return false;
    const cuuint32_t es[3] = {1, 1, 1};
    auto left = [&](CUtensorMap* m, const uint64_t* base) {
        const cuuint64_t dims[3] = {(cuuint64_t)q.K, (cuuint64_t)q.M, 2};
        const cuuint64_t strides[2] = {(cuuint64_t)q.K * 8, (cuuint64_t)(q.M * q.K * 8)};
        const cuuint32_t box[3] = {16, 32, 1};
        return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, const_cast<uint64_t*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    };
    auto right = [&](CUtensorMap* m, const uint64_t* base) {
        const cuuint64_t dims[3] = {(cuuint64_t)q.N, (cuuint64_t)q.K, 2};
        const cuuint64_t strides[2] = {(cuuint64_t)q.N * 8, (cuuint64_t)(q.K * q.N * 8)};
        const cuuint32_t box[3] = {(cuuint32_t)q.N, 32, 1};
        return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, const_cast<uint64_t*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    };
    return left(&q.tm_x, q.x) && left(&q.tm_a, q.a) && right(&q.tm_y, q.y) && right(&q.tm_b, q.b);
}

size_t fused_small_smem_bytes() {
    return (size_t)gemm_fused::kStages * gemm_fused::kStageBytes + 2 * 32 * 32 * 8 /*output sums*/ +
           1024 /*align*/ + 256 /*barriers*/;
}

int fused_small_ctas(int64_t K, int sms) {
    const int64_t kb = num_kb(K);
    static const int env = getenv("MPC_FUSED_CTAS") ? atoi(getenv("MPC_FUSED_CTAS")) : 0;   // test knob
    if (env > 0) return (int)std::min<int64_t>(std::max<int64_t>(kb, 1), std::min(env, sms));
    // at least 16 blocks per CTA: shorter ranges pay the pipeline fill and the slab
    // write / finalize read for little work
    int64_t g = kb / 16;
    if (g > sms) g = sms;
    return g < 1 ? 1 : (int)g;
}

size_t fused_small_partials_bytes(int64_t M, int64_t K, int64_t N) {
    const int g = fused_small_ctas(K, 148);
    return g > 1 ? (size_t)g * 2 * M * N * sizeof(uint64_t) : 0;
}

cudaError_t fused_small_launch(const FusedSmallParams& p, cudaStream_t stream) {
    if (p.M < 1 || p.M > 32 || p.N < 1 || p.N > 32 || p.K < 0) return cudaErrorInvalidValue;
    static int attr_dev = -1;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t smem = fused_small_smem_bytes();
    if (attr_dev != dev) {
        cudaError_t e = cudaFuncSetAttribute(gemm_fused::fused_small_kernel<1>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(gemm_fused::fused_small_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(gemm_fused::fused_small_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)fused_small_tma_smem_bytes());
        if (e != cudaSuccess) return e;
        attr_dev = dev;
    }
    const int G = fused_small_ctas(p.K, sms < 148 ? sms : 148);
    if (G > 1 && !p.partials) return cudaErrorInvalidValue;
    FusedSmallParams q0 = p;
    // tuning / test knobs (read once): converter groups, unit length, L2 prefetch, block order
    static const int env_ng = getenv("MPC_FUSED_GROUPS") ? atoi(getenv("MPC_FUSED_GROUPS")) : 1;
    const int ng = env_ng == 2 ? 2 : 1;
    static const int env_unit = getenv("MPC_FUSED_UNIT") ? atoi(getenv("MPC_FUSED_UNIT")) : 0;
    int unit = env_unit > 0 && env_unit < gemm_fused::kMaxUnit ? env_unit : gemm_fused::kMaxUnit;
    if (ng == 2) unit = unit < 2 ? 2 : unit & ~1;       // every unit starts at a block of converter group 0
    q0.unit = unit;
    static const int env_pf = getenv("MPC_FUSED_PF") ? atoi(getenv("MPC_FUSED_PF")) : 1;
    q0.pf_mode = env_pf;
    static const int env_pfd = getenv("MPC_FUSED_PFD") ? atoi(getenv("MPC_FUSED_PFD")) : gemm_fused::kPrefetch;
    q0.pf_dist = env_pfd;
    static const int env_cyc = getenv("MPC_FUSED_CYCLIC") ? atoi(getenv("MPC_FUSED_CYCLIC")) : 1;
    q0.cyclic = env_cyc;
    static const bool debug = getenv("MPC_FUSED_DEBUG") != nullptr;      // stall attribution (synchronises)
    unsigned long long h[4] = {0, 0, 0, 0};
    if (debug) {
        cudaMalloc(&q0.dbg, sizeof(h));
        cudaMemsetAsync(q0.dbg, 0, sizeof(h), stream);
    }
    // TMA-staged kernel where the maps encode (K, N even; MPC_FUSED_TMA=0: the register path)
    static const int env_tma = getenv("MPC_FUSED_TMA") ? atoi(getenv("MPC_FUSED_TMA")) : 1;
    const bool tma = env_tma != 0 && fused_small_maps(q0);
    cudaError_t e = tma ? launch_pdl(gemm_fused::fused_small_tma_kernel, dim3((unsigned)G), dim3(384),
                                     fused_small_tma_smem_bytes(), stream, q0)
                        : launch_pdl(ng == 2 ? gemm_fused::fused_small_kernel<2> : gemm_fused::fused_small_kernel<1>,
                                     dim3((unsigned)G), dim3(gemm_fused::kThreadsOf(ng)), smem, stream, q0);
    if (debug) {
        cudaMemcpyAsync(h, q0.dbg, sizeof(h), cudaMemcpyDeviceToHost, stream);
        cudaStreamSynchronize(stream);
        cudaFree(q0.dbg);
        fprintf(stderr, "[fused_small] G=%d groups=%d: MMA thread %.0f cyc (waiting for stages %.1f%%); converter "
                "warps %.0f cyc (waiting for free stages %.1f%%)\n", G, ng, (double)h[1] / G,
                100.0 * h[0] / (h[1] ? h[1] : 1), (double)h[3] / (8.0 * ng * G), 100.0 * h[2] / (h[3] ? h[3] : 1));
    }
    if (e != cudaSuccess || G <= 1) return e;
    RingGemmParams q{};
    q.M = p.M; q.N = p.N; q.C = p.C; q.Z = p.Z;
    q.party_stride_c = q.party_stride_z = p.M * p.N;
    q.trunc_bits = p.trunc_bits;
    q.splits = G;
    q.partials = p.partials;
    q.partial_stride = 2 * p.M * p.N;
    return ring_gemm_finalize(q, 2, stream);
}

}  // namespace mpc

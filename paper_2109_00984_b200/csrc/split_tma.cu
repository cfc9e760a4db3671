// split_tma.cu — the two-party mask + local reveal + limb split (a4-a6) of one Beaver
// matmul with both parties on this GPU, streamed through shared memory by TMA.
//
// Same result as split_left2_body / split_right2_body (elementwise.cu): for the x side
//     eps = sum_p (x_p - a_p) -> eps planes,  a_0 -> planes,  a_1 -> planes
// and for the y side (R7/R8)
//     delta = sum_p (y_p - b_p) -> delta planes,  b'_0 = b_0 + delta,  b'_1 = b_1 -> planes,
// in the ring GEMM's operand layout (common.cuh: Layout::Left for the x side, 128-row
// blocks; Layout::Right for the y side, 64-row blocks; exchanged for the transposed
// GEMM).  A CTA (one per SM) walks tiles of 64 rows (x) / 64 columns (y) x one 32-K
// block: a loader thread brings the tile of
// all four share inputs into a raw stage with 3-D tensor maps (x / a: two 16-K boxes of
// 64 rows with 128-byte swizzle, y / b: a 64 x 32 box; K past the end, rows past M and
// columns past N are zero-filled — the planes' K padding must be 0), the 256 converter
// threads (one per (row or column, 8-K quarter)) read their 8 values per input from
// shared memory, form the sums and write the limb planes into a staging stage already
// in the global layout, and a storer thread writes them back with bulk copies (per set:
// 8 x 2 KiB pieces into 128-row blocks, one 16 KiB run into a 64-row block).  Two raw and two
// staging stages keep the load of tile t + 1 and the stores of tile t - 1 in flight while
// tile t converts.  The split kernels it replaces keep one tile's loads in flight per
// thread and run at ~0.8 of the HBM copy rate on large weight splits (ncu, ViT fc1:
// 30.7 µs, 20% warps active).
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "elementwise.h"
#include "tcgen05.cuh"

namespace mpc {
namespace split_tma {
using namespace tc;

constexpr int kConv = 256;                        // converter threads (8 warps)
constexpr int kThreads = kConv + 64;              // + loader warp + storer warp
constexpr int kRaw = 64 * 1024;                   // 4 inputs x 16 KiB per tile
constexpr int kStage = 48 * 1024;                 // 3 plane sets x 8 planes x 2 KiB
constexpr int kStages = 2;

struct Params {
    CUtensorMap tm_x, tm_a, tm_y, tm_b;           // x, a: [2][M][K]; y, b: [2][K][N]
    uint8_t *eps_pl, *a_pl, *delta_pl, *b_pl;     // plane buffers (a_pl / b_pl: party 0, then party 1)
    int64_t a_stride, b_stride;                   // bytes between the parties' a / b' planes
    int64_t M, K, N;
    int KB, lt, rt;                               // 32-K blocks; x-side tiles (64 rows x block), y-side tiles
    int sum_first;                                // b'_0 = b_0 + delta (1 in the Beaver matmul)
    int xl, yl;                                   // plane layout of each side: 0 Layout::Left (128-row blocks),
                                                  // 1 Layout::Right (64-row blocks; swapped for the transposed GEMM)
};


__device__ __forceinline__ void tma_3d(uint32_t dst, const CUtensorMap* m, int c0, int c1, int c2, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
        :: "r"(dst), "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, uint32_t src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" :: "l"(dst), "r"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive_local(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(bar)) : "memory");
}

// 8 consecutive-k values of one row -> byte l of each into plane l (8 bytes at `off` of every
// 2 KiB plane of a staging set)
__device__ __forceinline__ void st_planes8(uint8_t* set, uint32_t off, const uint64_t (&v)[8]) {
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
    for (int l = 0; l < 8; ++l) *reinterpret_cast<uint2*>(set + off + l * 2048) = make_uint2(w[l][0], w[l][1]);
}

// Bulk stores of one 64-row tile's 8 planes (staging: plane l at l x 2 KiB) into a plane buffer:
// Layout::Right (64-row blocks) takes them as one 16 KiB run, Layout::Left (128-row blocks) as
// 8 pieces of 2 KiB at the row half of each 4 KiB plane
__device__ __forceinline__ void store_set(uint8_t* planes, int layout, int r0, int kb, int KB, uint32_t src) {
    if (layout) {
        bulk_s2g(planes + ((int64_t)(r0 / 64) * KB + kb) * 8 * 2048, src, 16384);
    } else {
        uint8_t* blk = planes + ((int64_t)(r0 / 128) * KB + kb) * 8 * 4096 + (r0 % 128) / 64 * 2048;
#pragma unroll
        for (int l = 0; l < 8; ++l) bulk_s2g(blk + l * 4096, src + l * 2048, 2048);
    }
}

__global__ void __launch_bounds__(kThreads, 1) split2_tma_kernel(const __grid_constant__ Params p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* raw = smem;                                      // [kStages][64 KiB]
    uint8_t* stg = smem + kStages * kRaw;                     // [kStages][48 KiB]
    uint64_t* rfull = reinterpret_cast<uint64_t*>(stg + kStages * kStage);
    uint64_t* rempty = rfull + kStages;
    uint64_t* sfull = rempty + kStages;
    uint64_t* sempty = sfull + kStages;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ntiles = p.lt + p.rt;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&rfull[s], 1); mbar_init(&rempty[s], kConv / 32);
            mbar_init(&sfull[s], kConv / 32); mbar_init(&sempty[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == kConv / 32 && lane < 4) {     // the loader's tensor maps, fetched before the wait
        const CUtensorMap* m = lane == 0 ? &p.tm_x : lane == 1 ? &p.tm_a : lane == 2 ? &p.tm_y : &p.tm_b;
        asm volatile("prefetch.tensormap [%0];" :: "l"(reinterpret_cast<uint64_t>(m)) : "memory");
    }
    __syncthreads();
    // launched as a programmatic dependent: the inputs may come from, and the plane buffers
    // still be read by, the previous kernels
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (warp == kConv / 32) {
        // ------------------------------------------------ loader
        if (lane == 0) {
            int s = 0; uint32_t ph = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
                mbar_wait(&rempty[s], ph ^ 1);
                const uint32_t dst = smem_u32(raw + s * kRaw);
                mbar_expect_tx(&rfull[s], kRaw);
                if (t < p.lt) {
                    const int kb = t % p.KB, r0 = (t / p.KB) * 64;
#pragma unroll
                    for (int src = 0; src < 4; ++src) {               // x_0, a_0, x_1, a_1
                        const CUtensorMap* m = (src & 1) ? &p.tm_a : &p.tm_x;
                        tma_3d(dst + src * 16384, m, kb * 32, r0, src >> 1, &rfull[s]);
                        tma_3d(dst + src * 16384 + 8192, m, kb * 32 + 16, r0, src >> 1, &rfull[s]);
                    }
                } else {
                    const int tt = t - p.lt, kb = tt % p.KB, n0 = (tt / p.KB) * 64;
#pragma unroll
                    for (int src = 0; src < 4; ++src) {               // y_0, b_0, y_1, b_1
                        const CUtensorMap* m = (src & 1) ? &p.tm_b : &p.tm_y;
                        tma_3d(dst + src * 16384, m, n0, kb * 32, src >> 1, &rfull[s]);
                    }
                }
                if (++s == kStages) { s = 0; ph ^= 1; }
            }
        }
    } else if (warp == kConv / 32 + 1) {
        // ------------------------------------------------ storer
        if (lane == 0) {
            int s = 0; uint32_t ph = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
                mbar_wait(&sfull[s], ph);
                const uint32_t src = smem_u32(stg + s * kStage);
                if (t < p.lt) {
                    const int kb = t % p.KB, r0 = (t / p.KB) * 64;
                    store_set(p.eps_pl, p.xl, r0, kb, p.KB, src);
                    store_set(p.a_pl, p.xl, r0, kb, p.KB, src + 16384);
                    store_set(p.a_pl + p.a_stride, p.xl, r0, kb, p.KB, src + 32768);
                } else {
                    const int tt = t - p.lt, kb = tt % p.KB, n0 = (tt / p.KB) * 64;
                    store_set(p.delta_pl, p.yl, n0, kb, p.KB, src);
                    store_set(p.b_pl, p.yl, n0, kb, p.KB, src + 16384);
                    store_set(p.b_pl + p.b_stride, p.yl, n0, kb, p.KB, src + 32768);
                }
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");   // staging readable again
                mbar_arrive_local(&sempty[s]);
                if (++s == kStages) { s = 0; ph ^= 1; }
            }
            asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");           // every plane written
        }
    } else {
        // ------------------------------------------------ converters: thread (row / column idx, 8-K quarter kq)
        const int idx = warp * 8 + (lane & 7), kq = lane >> 3;
        const uint32_t poff = (uint32_t)((idx >> 3) * 256 + (kq >> 1) * 128 + (idx & 7) * 16 + (kq & 1) * 8);
        int s = 0; uint32_t ph = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
            uint64_t v0[8], v1[8], v2[8], v3[8];
            mbar_wait(&rfull[s], ph);
            const uint8_t* rb = raw + s * kRaw;
            const bool xside = t < p.lt;
            if (xside) {
                // row idx, K values 8 kq ..: box kq >> 1 (16 K), 16-byte chunks (kq & 1) * 4 + j, stored at
                // chunk ^ (row & 7) (128-byte swizzle)
                const uint8_t* hb = rb + (kq >> 1) * 8192 + idx * 128;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int ch = (((kq & 1) * 4 + j) ^ (idx & 7)) * 16;
                    const ulonglong2 t0 = *reinterpret_cast<const ulonglong2*>(hb + ch);
                    const ulonglong2 t1 = *reinterpret_cast<const ulonglong2*>(hb + 16384 + ch);
                    const ulonglong2 t2 = *reinterpret_cast<const ulonglong2*>(hb + 32768 + ch);
                    const ulonglong2 t3 = *reinterpret_cast<const ulonglong2*>(hb + 49152 + ch);
                    v0[2 * j] = t0.x; v0[2 * j + 1] = t0.y; v1[2 * j] = t1.x; v1[2 * j + 1] = t1.y;
                    v2[2 * j] = t2.x; v2[2 * j + 1] = t2.y; v3[2 * j] = t3.x; v3[2 * j + 1] = t3.y;
                }
            } else {
                const uint64_t* r0 = reinterpret_cast<const uint64_t*>(rb);      // [src][32 k][64 n]
#pragma unroll
                for (int m = 0; m < 8; ++m) {
                    const int o = (kq * 8 + m) * 64 + idx;
                    v0[m] = r0[o]; v1[m] = r0[2048 + o]; v2[m] = r0[4096 + o]; v3[m] = r0[6144 + o];
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive_local(&rempty[s]);
#pragma unroll
            for (int m = 0; m < 8; ++m) v0[m] = v0[m] - v1[m] + v2[m] - v3[m];   // sum_p (plus_p - minus_p)
            if (!xside && p.sum_first) {
#pragma unroll
                for (int m = 0; m < 8; ++m) v1[m] += v0[m];                     // b'_0 = b_0 + delta (R8)
            }
            mbar_wait(&sempty[s], ph ^ 1);
            uint8_t* sb = stg + s * kStage;
            st_planes8(sb, poff, v0);                                           // eps / delta
            st_planes8(sb + 16384, poff, v1);                                   // a_0 / b'_0
            st_planes8(sb + 32768, poff, v3);                                   // a_1 / b'_1
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");       // generic writes -> bulk copies
            __syncwarp();
            if (lane == 0) mbar_arrive_local(&sfull[s]);
            if (++s == kStages) { s = 0; ph ^= 1; }
        }
    }
    __syncthreads();
    asm volatile("griddepcontrol.launch_dependents;");
}

}  // namespace split_tma

static PFN_cuTensorMapEncodeTiled_v12000 split_tma_encoder() {
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

// The two-party Beaver split (left: x, a -> eps, a_p planes; right: y, b -> delta, b'_p planes;
// either side may be absent, e.g. the x side of mpc_beaver_matmul_prepared) through
// split2_tma_kernel; cudaErrorNotSupported when the shapes or buffers do not fit it (the
// caller then uses the register split).
cudaError_t launch_split2_tma(const LeftSplitArgs* lp, const RightSplitArgs* rp, cudaStream_t st) {
    static const bool off = getenv("MPC_SPLIT_TMA") && atoi(getenv("MPC_SPLIT_TMA")) == 0;   // A/B switch
    const PFN_cuTensorMapEncodeTiled_v12000 enc = split_tma_encoder();
    if (off || !enc || (!lp && !rp)) return cudaErrorNotSupported;
    // exactly the Beaver matmul's all-parties split, either orientation of the 2-CTA GEMM, one matrix
    if (lp) {
        const LeftSplitArgs& l = *lp;
        if (l.Psum != 2 || l.Pcopy != 2 || l.cp_src != l.minus || !l.minus || !l.sum_planes || !l.cp_planes ||
            l.add_sum_first || l.swap > 1 || l.batch > 1 || l.M < 1 || l.K < 32 || (l.K & 1) ||
            l.party_stride != l.M * l.K || ((reinterpret_cast<uintptr_t>(l.plus) | reinterpret_cast<uintptr_t>(l.minus)) & 15))
            return cudaErrorNotSupported;
    }
    if (rp) {
        const RightSplitArgs& r = *rp;
        if (r.Psum != 2 || r.Pcopy != 2 || r.cp_src != r.minus || !r.minus || !r.sum_planes || !r.cp_planes ||
            r.swap > 1 || r.batch > 1 || r.N < 1 || r.K < 32 || (r.N & 1) || r.party_stride != r.K * r.N ||
            ((reinterpret_cast<uintptr_t>(r.plus) | reinterpret_cast<uintptr_t>(r.minus)) & 15))
            return cudaErrorNotSupported;
    }
    if (lp && rp && (lp->K != rp->K || lp->swap != rp->swap)) return cudaErrorNotSupported;
    const int64_t K = lp ? lp->K : rp->K, M = lp ? lp->M : 0, N = rp ? rp->N : 0;
    split_tma::Params p{};
    const cuuint32_t es[3] = {1, 1, 1};
    auto left = [&](CUtensorMap* m, const uint64_t* base) {
        const cuuint64_t dims[3] = {(cuuint64_t)K, (cuuint64_t)M, 2};
        const cuuint64_t strides[2] = {(cuuint64_t)K * 8, (cuuint64_t)(M * K * 8)};
        const cuuint32_t box[3] = {16, 64, 1};
        return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, const_cast<uint64_t*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    };
    auto right = [&](CUtensorMap* m, const uint64_t* base) {
        const cuuint64_t dims[3] = {(cuuint64_t)N, (cuuint64_t)K, 2};
        const cuuint64_t strides[2] = {(cuuint64_t)N * 8, (cuuint64_t)(K * N * 8)};
        const cuuint32_t box[3] = {64, 32, 1};
        return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, const_cast<uint64_t*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    };
    if (lp && (!left(&p.tm_x, lp->plus) || !left(&p.tm_a, lp->minus))) return cudaErrorNotSupported;
    if (rp && (!right(&p.tm_y, rp->plus) || !right(&p.tm_b, rp->minus))) return cudaErrorNotSupported;
    if (lp) { p.eps_pl = lp->sum_planes; p.a_pl = lp->cp_planes; p.a_stride = lp->cp_planes_stride; }
    if (rp) { p.delta_pl = rp->sum_planes; p.b_pl = rp->cp_planes; p.b_stride = rp->cp_planes_stride; }
    p.M = M; p.K = K; p.N = N;
    p.KB = (int)num_kb(K);
    p.lt = lp ? (int)((M + 63) / 64) * p.KB : 0;
    p.rt = rp ? (int)((N + 63) / 64) * p.KB : 0;
    p.sum_first = rp ? rp->add_delta_first : 0;
    const int swap = lp ? lp->swap : rp->swap;
    p.xl = swap ? 1 : 0;                                      // transposed GEMM: x side right-operand planes
    p.yl = swap ? 0 : 1;
    static int attr_dev = -1;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t smem = (size_t)split_tma::kStages * (split_tma::kRaw + split_tma::kStage) + 1024 + 256;
    if (attr_dev != dev) {
        const cudaError_t e = cudaFuncSetAttribute(split_tma::split2_tma_kernel,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr_dev = dev;
    }
    const int64_t tiles = (int64_t)p.lt + p.rt;
    const unsigned grid = (unsigned)(tiles < sms ? tiles : sms);
    return launch_pdl(split_tma::split2_tma_kernel, dim3(grid), dim3(split_tma::kThreads), smem, st, p);
}

}  // namespace mpc

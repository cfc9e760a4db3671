// conv.cu — kernels of the private 2-D convolution (
// P:589-590 "the same procedure ... matrix multiplication and convolution").
//
// The Beaver convolution reveals eps at the input shape (B, C, H, W) and delta
// at the weight shape (R22) and computes
//     z_p = c_p + conv(a_p, delta) + conv(eps, b_p + [p = 0] delta)
// on the ring GEMM: the left operands are the implicit im2col of the
// activation-shaped eps / a_p (rows (b, oy, ox), K = (ci, ky, kx)), written
// straight into limb planes here without materialising the im2col matrix in
// u64; the right operands are the weights, already Cout x K row-major.
#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"
#include "conv.h"

namespace mpc {

namespace {
inline unsigned grid_of(int64_t work) {
    int64_t g = (work + 255) / 256;
    if (g < 1) g = 1;
    if (g > 148 * 16) g = 148 * 16;
    return (unsigned)g;
}
}  // namespace

// A warp covers 32 consecutive im2col rows (lane = row, i.e. 32 neighbouring
// output pixels: the gathers of one K index are nearly contiguous) and one
// 16-K chunk; each lane gathers its 16 (ci, ky, kx) values per party and
// writes 16 bytes per limb plane.  The K padding (K .. 32*KB) is written as 0.
template <Layout LO>
__global__ void __launch_bounds__(256) split_im2col_kernel(Im2colSplitArgs a) {
    const ConvGeom& g = a.g;
    const int64_t Ho = g.Ho(), Wo = g.Wo(), M = g.M(), K = g.K(), KB = num_kb(K);
    const int64_t khw = g.kh * g.kw;
    const int64_t rgroups = (M + 31) / 32, kchunks = KB * 2;
    const int lane = threadIdx.x & 31;
    const bool fused_copy = a.cp_src == a.minus && a.Pcopy == a.Psum && a.Psum > 0;
    for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; w < rgroups * kchunks;
         w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t kc = w / rgroups, rg = w % rgroups;     // neighbouring warps: neighbouring rows
        const int64_t row = rg * 32 + lane;
        if (row >= M) continue;
        const int64_t k0 = kc * 16;
        const int64_t b = row / (Ho * Wo), s = row % (Ho * Wo);
        const int64_t oy = s / Wo, ox = s % Wo;
        int64_t off[16];                                        // element offset in one party's tensor, or -1
#pragma unroll
        for (int m = 0; m < 16; ++m) {
            const int64_t k = k0 + m;
            off[m] = -1;
            if (k < K) {
                const int64_t ci = k / khw, r = k % khw;
                const int64_t iy = oy * g.sh - g.ph + r / g.kw, ix = ox * g.sw - g.pw + r % g.kw;
                if (iy >= 0 && iy < g.H && ix >= 0 && ix < g.W) off[m] = ((b * g.C + ci) * g.H + iy) * g.W + ix;
            }
        }
        uint64_t acc[16], v[16];
#pragma unroll
        for (int m = 0; m < 16; ++m) acc[m] = 0;
        for (int p = 0; p < a.Psum; ++p) {
            const uint64_t* src = a.plus + p * a.party_stride;
#pragma unroll
            for (int m = 0; m < 16; ++m) v[m] = off[m] >= 0 ? __ldg(src + off[m]) : 0ull;
#pragma unroll
            for (int m = 0; m < 16; ++m) acc[m] += v[m];
            if (a.minus) {
                const uint64_t* sm = a.minus + p * a.party_stride;
#pragma unroll
                for (int m = 0; m < 16; ++m) v[m] = off[m] >= 0 ? __ldg(sm + off[m]) : 0ull;
#pragma unroll
                for (int m = 0; m < 16; ++m) acc[m] -= v[m];
                if (fused_copy) store_limbs16<LO>(a.cp_planes + p * a.cp_planes_stride, row, k0, KB, v);
            }
        }
        if (a.Psum > 0) store_limbs16<LO>(a.sum_planes, row, k0, KB, acc);
        if (!fused_copy) {
            for (int q = 0; q < a.Pcopy; ++q) {
                const uint64_t* src = a.cp_src + q * a.party_stride;
#pragma unroll
                for (int m = 0; m < 16; ++m) v[m] = off[m] >= 0 ? __ldg(src + off[m]) : 0ull;
                store_limbs16<LO>(a.cp_planes + q * a.cp_planes_stride, row, k0, KB, v);
            }
        }
    }
}

cudaError_t launch_split_im2col(const Im2colSplitArgs& a, cudaStream_t st) {
    const int64_t M = a.g.M(), K = a.g.K();
    if (M == 0 || K == 0) return cudaSuccess;
    const int64_t warps = ((M + 31) / 32) * num_kb(K) * 2;
    if (a.layout_right) split_im2col_kernel<Layout::Right><<<grid_of(warps * 32), 256, 0, st>>>(a);
    else split_im2col_kernel<Layout::Left><<<grid_of(warps * 32), 256, 0, st>>>(a);
    return cudaGetLastError();
}

// One thread per element pair (one Philox block per stream and pair).
__global__ void prg_parties_kernel(uint64_t key, uint32_t tag, uint64_t id, int P, int lo, int hi,
                                   uint64_t* __restrict__ out, uint64_t* __restrict__ out_sum, int64_t n) {
    const int64_t npairs = (n + 1) / 2;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < npairs; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i0 = 2 * j;
        const bool has1 = i0 + 1 < n;
        uint64_t s0 = 0, s1 = 0;
        for (int p = out_sum ? 0 : lo; p < (out_sum ? P : hi); ++p) {
            uint64_t g0, g1;
            philox_pair(key, stream_word(tag, (uint32_t)p, id), (uint64_t)j, g0, g1);
            s0 += g0; s1 += g1;
            if (out && p >= lo && p < hi) {
                uint64_t* o = out + (int64_t)(p - lo) * n;
                o[i0] = g0;
                if (has1) o[i0 + 1] = g1;
            }
        }
        if (out_sum) {
            out_sum[i0] = s0;
            if (has1) out_sum[i0 + 1] = s1;
        }
    }
}

cudaError_t launch_prg_parties(uint64_t key, uint32_t tag, uint64_t id, int P, int lo, int hi, uint64_t* out,
                               uint64_t* out_sum, int64_t n, cudaStream_t st) {
    if (n == 0 || (!out && !out_sum)) return cudaSuccess;
    prg_parties_kernel<<<grid_of((n + 1) / 2), 256, 0, st>>>(key, tag, id, P, lo, hi, out, out_sum, n);
    return cudaGetLastError();
}

}  // namespace mpc

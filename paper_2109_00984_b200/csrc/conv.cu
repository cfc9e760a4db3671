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

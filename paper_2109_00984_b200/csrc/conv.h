// conv.h — private 2-D convolution support kernels (internal).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace mpc {

// x (B, C, H, W) * w (Cout, C, kh, kw) -> (B, Cout, Ho, Wo), zero padding, stride, NCHW (R22).
struct ConvGeom {
    int64_t B, C, H, W, Cout, kh, kw, sh, sw, ph, pw;
    __host__ __device__ int64_t Ho() const { return (H + 2 * ph - kh) / sh + 1; }
    __host__ __device__ int64_t Wo() const { return (W + 2 * pw - kw) / sw + 1; }
    __host__ __device__ int64_t M() const { return B * Ho() * Wo(); }       // im2col rows (b, oy, ox)
    __host__ __device__ int64_t K() const { return C * kh * kw; }           // (ci, ky, kx)
    __host__ __device__ int64_t in_elems() const { return B * C * H * W; }
    __host__ __device__ int64_t w_elems() const { return Cout * C * kh * kw; }
    __host__ __device__ int64_t out_elems() const { return B * Cout * Ho() * Wo(); }
};

// Limb split of the implicit im2col of activation-shaped operands (the left
// operand of the conv GEMM): sum planes of sum_{p<Psum} (plus_p - minus_p)
// and copy planes of cp_src party q < Pcopy, rows = im2col rows, K = C*kh*kw.
struct Im2colSplitArgs {
    ConvGeom g;
    int64_t party_stride;            // elements between parties' activation tensors
    const uint64_t* plus;
    const uint64_t* minus;           // may be null
    int Psum;
    uint8_t* sum_planes;
    const uint64_t* cp_src;
    int Pcopy;
    uint8_t* cp_planes;
    int64_t cp_planes_stride;        // bytes
    int layout_right;                // planes in Layout::Right (transposed GEMM) instead of Layout::Left
};
cudaError_t launch_split_im2col(const Im2colSplitArgs& a, cudaStream_t st);
// im2col split of the activation side and the weights split (elementwise.h LeftSplitArgs) in one
// launch; they must target opposite plane layouts (one left, one right GEMM operand).
struct LeftSplitArgs;
cudaError_t launch_split_conv(const Im2colSplitArgs& im, const LeftSplitArgs& wt, cudaStream_t st);

// out_sum[i] = sum_{p<P} G(key, tag||p||id)[i]; parties [lo, hi) also written to out ([hi-lo][n]).
// Either output may be null.
cudaError_t launch_prg_parties(uint64_t key, uint32_t tag, uint64_t id, int P, int lo, int hi, uint64_t* out,
                               uint64_t* out_sum, int64_t n, cudaStream_t st);

}  // namespace mpc

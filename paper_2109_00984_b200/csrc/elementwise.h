// elementwise.h — host interface of the elementwise protocol kernels (internal).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace mpc {

constexpr int kMaxParties = 16;
struct KeySet { uint64_t k[kMaxParties]; };

struct LeftSplitArgs {
    int64_t M, K;
    int64_t party_stride;            // elements between parties of plus/minus/cp_src
    const uint64_t* plus;            // Psum parties
    const uint64_t* minus;           // may be null
    int Psum;                        // 0: no sum planes
    uint8_t* sum_planes;
    const uint64_t* cp_src;          // Pcopy parties copied to planes
    int Pcopy;
    uint8_t* cp_planes;
    int64_t cp_planes_stride;        // bytes
    int swap;                        // plane layout: 0 Layout::Left, 1 Layout::Right (transposed ring GEMM),
                                     // 2 Layout::Small (stacked-plane GEMM)
    int add_sum_first;               // copy of party 0 gets + the sum (b'_0 = b_0 + delta, R8), for weights
                                     // given rows x K (conv: Cout x C*kh*kw)
    int batch;                       // independent matrices (0/1 = one): element b reads its inputs at
    int64_t in_bstride;              //   + b * in_bstride (elements) and writes planes at
    int64_t sum_bstride, cp_bstride; //   + b * sum_bstride / cp_bstride (bytes)
};

struct RightSplitArgs {
    int64_t K, N;
    int64_t party_stride;
    const uint64_t* plus;
    const uint64_t* minus;
    int Psum;
    uint8_t* sum_planes;             // may be null (delta still computed for the fold)
    const uint64_t* cp_src;
    int Pcopy;
    int add_delta_first;             // party 0's b' = b_0 + delta (R8)
    uint8_t* cp_planes;
    int64_t cp_planes_stride;
    int swap;                        // plane layout: 0 Layout::Right, 1 Layout::Left (transposed ring GEMM),
                                     // 2 Layout::Small (stacked-plane GEMM)
    int batch;                       // as LeftSplitArgs
    int64_t in_bstride;
    int64_t sum_bstride, cp_bstride;
};

struct TtpGenArgs {
    uint64_t key, id;
    uint32_t tag;
    int P;
    int64_t rows, K;                 // left: rows = M; right: rows = N (b is K x N row-major)
    int out_lo, out_hi;              // parties whose u64 shares are written
    uint64_t* out;                   // [out_hi - out_lo][rows*K]
    uint8_t* sum_planes;             // planes of sum_q over all P parties (TTP), or null
    int small;                       // 1: sum planes in Layout::Small (stacked-plane GEMM)
};

cudaError_t launch_encode(const double* x, uint64_t* out, int64_t n, int frac_bits, int* err, cudaStream_t st);
cudaError_t launch_decode(const uint64_t* v, double* out, int64_t n, int frac_bits, cudaStream_t st);
cudaError_t launch_share(const KeySet& keys, int P, int party_lo, int party_hi, const uint64_t* x, int src,
                         uint64_t stream, uint64_t* out, int64_t n, cudaStream_t st);
cudaError_t launch_sum_parties(const uint64_t* s, int P, int64_t n, uint64_t* out, cudaStream_t st);
cudaError_t launch_mask(const uint64_t* x, const uint64_t* a, int64_t n1, const uint64_t* y, const uint64_t* b,
                        int64_t n2, uint64_t* ed, cudaStream_t st);
cudaError_t launch_split_left(const LeftSplitArgs& a, cudaStream_t st);
cudaError_t launch_split_right(const RightSplitArgs& a, cudaStream_t st);
cudaError_t launch_split_both(const LeftSplitArgs& l, const RightSplitArgs& r, cudaStream_t st);
// the two-party Beaver split streamed through shared memory by TMA (split_tma.cu), either side
// optional; cudaErrorNotSupported when the shapes / buffers do not fit it
cudaError_t launch_split2_tma(const LeftSplitArgs* l, const RightSplitArgs* r, cudaStream_t st);
cudaError_t launch_ttp_left(const TtpGenArgs& g, cudaStream_t st);
cudaError_t launch_ttp_right(const TtpGenArgs& g, cudaStream_t st);
cudaError_t launch_ttp_c(uint64_t key, uint64_t id, int P, int out_lo, int out_hi, uint64_t* out, uint64_t* c0,
                         int64_t n, cudaStream_t st);
cudaError_t launch_wrap_pair(uint64_t key, uint64_t id, int P, int lo, int hi, uint64_t* r, uint64_t* th, int64_t n,
                             cudaStream_t st);
cudaError_t launch_trunc_local(uint64_t* x, int64_t n, int bits, cudaStream_t st);
// Alg. 1 (P > 2).  r, th: the wrap pair in memory ([P][n] for all parties, n for one
// party), or both null to regenerate it from wrap id `id` under k_ttp `key`.
cudaError_t launch_trunc_alg1_all(uint64_t* x, int P, int64_t n, int bits, uint64_t key, uint64_t id,
                                  const uint64_t* r, const uint64_t* th, cudaStream_t st);
cudaError_t launch_trunc_alg1_a(const uint64_t* x, int64_t n, uint64_t key, uint64_t id, int party, const uint64_t* r,
                                uint64_t* zbuf, int8_t* hbuf, cudaStream_t st);
cudaError_t launch_trunc_alg1_b(uint64_t* x, int64_t n, int bits, uint64_t key, uint64_t id, int P, int party,
                                const uint64_t* r, const uint64_t* th, const uint64_t* zsum, const int8_t* hsum,
                                cudaStream_t st);

}  // namespace mpc

// beaver_elementwise.cu — elementwise private multiplication and square
// (App. A.1.1).  HBM-bound uint64
// kernels; the same PRG streams and truncation as the matmul path.
//
//   triple:  a_p = G(k_ttp, A||p||id)[i], b_p = G(k_ttp, B||p||id)[i],
//            c = (sum a_p)(sum b_p), c_p = G(k_ttp, C||p||id)[i] (p >= 1),
//            c_0 = c - sum_{p>=1} c_p                          (R6, R21)
//   pair:    a_p as above, b = (sum a_p)^2, b_p (p >= 1) from the C stream (R20)
//   mul:     z_p = c_p + eps b_p + a_p delta + [p = 0] eps delta
//   square:  z_p = b_p + 2 eps a_p + [p = 0] eps^2
#include <cstdint>
#include <initializer_list>
#include <cuda_runtime.h>

#include "beaver_elementwise.h"
#include "common.cuh"

namespace mpc {

namespace {
// 16-byte vector accesses need every (non-null) base 16-byte aligned
inline bool aligned16(std::initializer_list<const void*> ps) {
    for (const void* p : ps)
        if (reinterpret_cast<uintptr_t>(p) & 15) return false;
    return true;
}
inline unsigned grid_of(int64_t work) {
    int64_t g = (work + 255) / 256;
    if (g < 1) g = 1;
    if (g > 148 * 16) g = 148 * 16;
    return (unsigned)g;
}
}  // namespace

// ------------------------------------------------------------------ TTP
// One thread per element pair (one Philox block = two elements per stream).
// Writes parties [out_lo, out_hi) of a (and b for a triple) and of c; when
// party 0 is written, all P streams are expanded to form c_0.
template <bool SQUARE>
__global__ void ttp_elementwise_kernel(uint64_t key, uint64_t id, int P, int out_lo, int out_hi,
                                       uint64_t* __restrict__ a, uint64_t* __restrict__ b,
                                       uint64_t* __restrict__ c, int64_t n) {
    const int64_t npairs = (n + 1) / 2;
    const bool need_sum = out_lo == 0 && out_hi > 0;          // c_0 needs every party's a_p, b_p, c_p
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < npairs; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i0 = 2 * j;
        const bool has1 = i0 + 1 < n;
        uint64_t as0 = 0, as1 = 0, bs0 = 0, bs1 = 0, cs0 = 0, cs1 = 0;   // sums over parties
        for (int p = need_sum ? 0 : out_lo; p < (need_sum ? P : out_hi); ++p) {
            const bool mine = p >= out_lo && p < out_hi;
            uint64_t a0, a1;
            philox_pair(key, stream_word(kTagA, (uint32_t)p, id), (uint64_t)j, a0, a1);
            as0 += a0; as1 += a1;
            if (mine) {
                uint64_t* o = a + (int64_t)(p - out_lo) * n;
                o[i0] = a0;
                if (has1) o[i0 + 1] = a1;
            }
            if (!SQUARE) {
                uint64_t b0, b1;
                philox_pair(key, stream_word(kTagB, (uint32_t)p, id), (uint64_t)j, b0, b1);
                bs0 += b0; bs1 += b1;
                if (mine) {
                    uint64_t* o = b + (int64_t)(p - out_lo) * n;
                    o[i0] = b0;
                    if (has1) o[i0 + 1] = b1;
                }
            }
            if (p >= 1) {
                uint64_t c0, c1;
                philox_pair(key, stream_word(kTagC, (uint32_t)p, id), (uint64_t)j, c0, c1);
                cs0 += c0; cs1 += c1;
                if (mine) {
                    uint64_t* o = (SQUARE ? b : c) + (int64_t)(p - out_lo) * n;
                    o[i0] = c0;
                    if (has1) o[i0 + 1] = c1;
                }
            }
        }
        if (need_sum) {
            const uint64_t v0 = (SQUARE ? as0 * as0 : as0 * bs0) - cs0;
            const uint64_t v1 = (SQUARE ? as1 * as1 : as1 * bs1) - cs1;
            uint64_t* o = SQUARE ? b : c;                          // party 0's slot
            o[i0] = v0;
            if (has1) o[i0 + 1] = v1;
        }
    }
}

cudaError_t launch_ttp_elementwise(bool square, uint64_t key, uint64_t id, int P, int out_lo, int out_hi,
                                   uint64_t* a, uint64_t* b, uint64_t* c, int64_t n, cudaStream_t st) {
    if (n == 0 || out_hi <= out_lo) return cudaSuccess;
    if (square) ttp_elementwise_kernel<true><<<grid_of((n + 1) / 2), 256, 0, st>>>(key, id, P, out_lo, out_hi, a, b, c, n);
    else ttp_elementwise_kernel<false><<<grid_of((n + 1) / 2), 256, 0, st>>>(key, id, P, out_lo, out_hi, a, b, c, n);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ online, all parties on one device
// Thread per element pair.  Pass 1 reveals eps (and delta) as the local sum of
// the masked shares; pass 2 forms every party's z_p (a_p, b_p re-read: L1/L2
// hits).  Reads (4P + P) u64 and writes P u64 per element for mul.
struct Pair { uint64_t v0, v1; };
__device__ __forceinline__ Pair ld2(const uint64_t* __restrict__ p, int64_t i0, bool has1, bool vec) {
    if (vec) {
        const ulonglong2 t = __ldg(reinterpret_cast<const ulonglong2*>(p + i0));
        return {t.x, t.y};
    }
    return {__ldg(p + i0), has1 ? __ldg(p + i0 + 1) : 0ull};
}
__device__ __forceinline__ void st2(uint64_t* __restrict__ p, int64_t i0, bool has1, bool vec, uint64_t v0, uint64_t v1) {
    if (vec) { *reinterpret_cast<ulonglong2*>(p + i0) = make_ulonglong2(v0, v1); return; }
    p[i0] = v0;
    if (has1) p[i0 + 1] = v1;
}
__device__ __forceinline__ uint64_t trunc_or(uint64_t v, int bits) { return bits ? div_pow2_round(v, bits) : v; }

// PT > 0: the party count is a compile-time constant, every party's loads are
// issued together and a_p, b_p stay in registers for pass 2 (no re-read);
// PT == 0: runtime P (> 8), a_p and b_p are re-read in pass 2.
template <bool SQUARE, int PT>
__global__ void __launch_bounds__(256) beaver_elementwise_all_kernel(
        const uint64_t* __restrict__ x, const uint64_t* __restrict__ y, const uint64_t* __restrict__ a,
        const uint64_t* __restrict__ b, const uint64_t* __restrict__ c, uint64_t* __restrict__ z, int P_rt,
        int64_t n, int bits, bool vec) {
    constexpr int R = PT > 0 ? PT : 1;             // register-resident parties
    const int P = PT > 0 ? PT : P_rt;
    const int64_t npairs = (n + 1) / 2;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < npairs; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i0 = 2 * j;
        const bool has1 = i0 + 1 < n;
        uint64_t e0 = 0, e1 = 0, d0 = 0, d1 = 0;
        Pair ar[R], br[R];
#pragma unroll
        for (int p = 0; p < (PT > 0 ? PT : 0); ++p) {
            const int64_t o = (int64_t)p * n;
            const Pair xv = ld2(x + o, i0, has1, vec);
            ar[p] = ld2(a + o, i0, has1, vec);
            e0 += xv.v0 - ar[p].v0; e1 += xv.v1 - ar[p].v1;
            if (!SQUARE) {
                const Pair yv = ld2(y + o, i0, has1, vec);
                br[p] = ld2(b + o, i0, has1, vec);
                d0 += yv.v0 - br[p].v0; d1 += yv.v1 - br[p].v1;
            }
        }
        if (PT == 0) {
            for (int p = 0; p < P; ++p) {
                const int64_t o = (int64_t)p * n;
                const Pair xv = ld2(x + o, i0, has1, vec), av = ld2(a + o, i0, has1, vec);
                e0 += xv.v0 - av.v0; e1 += xv.v1 - av.v1;
                if (!SQUARE) {
                    const Pair yv = ld2(y + o, i0, has1, vec), bv = ld2(b + o, i0, has1, vec);
                    d0 += yv.v0 - bv.v0; d1 += yv.v1 - bv.v1;
                }
            }
        }
#pragma unroll
        for (int p = 0; p < (PT > 0 ? PT : 1); ++p) {
            for (int q = (PT > 0 ? p : 0); q < (PT > 0 ? p + 1 : P); ++q) {
                const int64_t o = (int64_t)q * n;
                const Pair av = PT > 0 ? ar[p] : ld2(a + o, i0, has1, vec);
                const Pair bv = (PT > 0 && !SQUARE) ? br[p] : ld2(b + o, i0, has1, vec);
                uint64_t z0, z1;
                if (SQUARE) {                                 // b_q + 2 eps a_q + [q=0] eps^2
                    z0 = bv.v0 + 2u * e0 * av.v0;
                    z1 = bv.v1 + 2u * e1 * av.v1;
                    if (q == 0) { z0 += e0 * e0; z1 += e1 * e1; }
                } else {                                      // c_q + eps b_q + a_q delta + [q=0] eps delta
                    const Pair cv = ld2(c + o, i0, has1, vec);
                    z0 = cv.v0 + e0 * bv.v0 + av.v0 * d0;
                    z1 = cv.v1 + e1 * bv.v1 + av.v1 * d1;
                    if (q == 0) { z0 += e0 * d0; z1 += e1 * d1; }
                }
                st2(z + o, i0, has1, vec, trunc_or(z0, bits), trunc_or(z1, bits));
            }
        }
    }
}

template <bool SQUARE>
cudaError_t launch_all_p(const uint64_t* x, const uint64_t* y, const uint64_t* a, const uint64_t* b,
                         const uint64_t* c, uint64_t* z, int P, int64_t n, int bits, bool vec, cudaStream_t st) {
    const unsigned g = grid_of((n + 1) / 2);
    switch (P) {
#define MPC_EW_CASE(K) \
        case K: beaver_elementwise_all_kernel<SQUARE, K><<<g, 256, 0, st>>>(x, y, a, b, c, z, P, n, bits, vec); break;
        MPC_EW_CASE(1) MPC_EW_CASE(2) MPC_EW_CASE(3) MPC_EW_CASE(4)
        MPC_EW_CASE(5) MPC_EW_CASE(6) MPC_EW_CASE(7) MPC_EW_CASE(8)
#undef MPC_EW_CASE
        default: beaver_elementwise_all_kernel<SQUARE, 0><<<g, 256, 0, st>>>(x, y, a, b, c, z, P, n, bits, vec);
    }
    return cudaGetLastError();
}

cudaError_t launch_beaver_elementwise_all(bool square, const uint64_t* x, const uint64_t* y, const uint64_t* a,
                                          const uint64_t* b, const uint64_t* c, uint64_t* z, int P, int64_t n,
                                          int bits, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    const bool vec = (n & 1) == 0 && aligned16({x, y, a, b, c, z});
    return square ? launch_all_p<true>(x, y, a, b, c, z, P, n, bits, vec, st)
                  : launch_all_p<false>(x, y, a, b, c, z, P, n, bits, vec, st);
}

// ------------------------------------------------------------------ online, one party (after the reveal)
// ed = revealed [eps | delta] (square: eps only).  party0: this party adds the
// public eps delta (eps^2).
template <bool SQUARE>
__global__ void beaver_elementwise_finish_kernel(const uint64_t* __restrict__ ed, const uint64_t* __restrict__ a,
                                                 const uint64_t* __restrict__ b, const uint64_t* __restrict__ c,
                                                 uint64_t* __restrict__ z, int64_t n, int party0, int bits,
                                                 bool vec) {
    const int64_t npairs = (n + 1) / 2;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < npairs; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i0 = 2 * j;
        const bool has1 = i0 + 1 < n;
        const Pair e = ld2(ed, i0, has1, vec), av = ld2(a, i0, has1, vec), bv = ld2(b, i0, has1, vec);
        uint64_t z0, z1;
        if (SQUARE) {
            z0 = bv.v0 + 2u * e.v0 * av.v0;
            z1 = bv.v1 + 2u * e.v1 * av.v1;
            if (party0) { z0 += e.v0 * e.v0; z1 += e.v1 * e.v1; }
        } else {
            const Pair d = ld2(ed + n, i0, has1, vec), cv = ld2(c, i0, has1, vec);
            z0 = cv.v0 + e.v0 * bv.v0 + av.v0 * d.v0;
            z1 = cv.v1 + e.v1 * bv.v1 + av.v1 * d.v1;
            if (party0) { z0 += e.v0 * d.v0; z1 += e.v1 * d.v1; }
        }
        st2(z, i0, has1, vec, trunc_or(z0, bits), trunc_or(z1, bits));
    }
}

cudaError_t launch_beaver_elementwise_finish(bool square, const uint64_t* ed, const uint64_t* a, const uint64_t* b,
                                             const uint64_t* c, uint64_t* z, int64_t n, int party0, int bits,
                                             cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    const bool vec = (n & 1) == 0 && aligned16({ed, a, b, c, z});
    if (square)
        beaver_elementwise_finish_kernel<true><<<grid_of((n + 1) / 2), 256, 0, st>>>(ed, a, b, c, z, n, party0, bits, vec);
    else
        beaver_elementwise_finish_kernel<false><<<grid_of((n + 1) / 2), 256, 0, st>>>(ed, a, b, c, z, n, party0, bits,
                                                                                      vec);
    return cudaGetLastError();
}

}  // namespace mpc

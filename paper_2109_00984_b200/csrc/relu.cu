// relu.cu — the ReLU path of SURVEY §8(f) NEXT-3, all parties on one device:
//   A2B (binary PRZS of every party's arithmetic share, tree of Kogge-Stone
//   ring adders with binary Beaver ANDs; App. A.1.2),
//   sign bit ⟨x⟩ >> 63, single-bit B2A (Alg. 2) and
//   ReLU([x]) = [x] * (1 - [x < 0]) by a Beaver multiplication.
// Readings R23-R25 fix the PRG streams, the adder and the gate ids.
//
// One fused kernel: every reveal of the protocol is a local XOR / sum over the
// P parties held by the same thread, and every triple / bit pair is expanded
// from its counter-based stream where it is used, so the kernel reads the P
// input shares and writes the P output shares (16·P bytes per element) and
// spends the rest in Philox (ALU bound).  Thread = one element pair (one
// Philox block gives both elements' words of a stream).
#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"
#include "elementwise.h"
#include "relu.h"

namespace mpc {

namespace {
enum : uint32_t { kTagBPRZS = 7, kTagBA = 8, kTagBB = 9, kTagBC = 10, kTagRBIT = 11, kTagRB = 12, kTagRA = 13,
                  kTagMA = 14, kTagMB = 15, kTagMC = 16 };

template <int P> struct Sh { uint64_t v[P][2]; };      // one binary or arithmetic share per party, 2 elements

__device__ __forceinline__ uint64_t gate_id(uint64_t add_id, int l, int w) {
    return (add_id << 4) | ((uint64_t)l << 1) | (uint64_t)w;
}

// Binary Beaver AND of x and y (App. A.1.2) with the triple of gate `gid`:
// eps = ⊕(x_p ^ a_p), delta = ⊕(y_p ^ b_p) (the reveal: a local XOR here);
// z_p = c_p ^ (eps & b_p) ^ (a_p & delta) ^ [p = 0](eps & delta), c_0 = (⊕a & ⊕b) ^ ⊕_{p>=1} c_p.
template <int P>
__device__ __forceinline__ void and_gate(uint64_t kttp, uint64_t gid, uint64_t j, const Sh<P>& x, const Sh<P>& y,
                                         Sh<P>& z) {
    uint64_t a[P][2], b[P][2];
    uint64_t e0 = 0, e1 = 0, d0 = 0, d1 = 0, as0 = 0, as1 = 0, bs0 = 0, bs1 = 0;
#pragma unroll
    for (int p = 0; p < P; ++p) {
        philox_pair(kttp, stream_word(kTagBA, (uint32_t)p, gid), j, a[p][0], a[p][1]);
        philox_pair(kttp, stream_word(kTagBB, (uint32_t)p, gid), j, b[p][0], b[p][1]);
        e0 ^= x.v[p][0] ^ a[p][0]; e1 ^= x.v[p][1] ^ a[p][1];
        d0 ^= y.v[p][0] ^ b[p][0]; d1 ^= y.v[p][1] ^ b[p][1];
        as0 ^= a[p][0]; as1 ^= a[p][1]; bs0 ^= b[p][0]; bs1 ^= b[p][1];
    }
    uint64_t c00 = as0 & bs0, c01 = as1 & bs1;               // c_0 accumulates c ^ c_1 ^ ... ^ c_{P-1}
#pragma unroll
    for (int p = 1; p < P; ++p) {
        uint64_t c0, c1;
        philox_pair(kttp, stream_word(kTagBC, (uint32_t)p, gid), j, c0, c1);
        c00 ^= c0; c01 ^= c1;
        z.v[p][0] = c0 ^ (e0 & b[p][0]) ^ (a[p][0] & d0);
        z.v[p][1] = c1 ^ (e1 & b[p][1]) ^ (a[p][1] & d1);
    }
    z.v[0][0] = c00 ^ (e0 & b[0][0]) ^ (a[0][0] & d0) ^ (e0 & d0);
    z.v[0][1] = c01 ^ (e1 & b[0][1]) ^ (a[0][1] & d1) ^ (e1 & d1);
}

// Kogge-Stone ring adder on binary shares (R24); the last level's propagate
// update is not needed for the sum and is skipped (it never reaches the output).
template <int P>
__device__ __forceinline__ void add_ring(uint64_t kttp, uint64_t add_id, uint64_t j, const Sh<P>& x, const Sh<P>& y,
                                         Sh<P>& out) {
    Sh<P> G, Pr, t, u;
    and_gate<P>(kttp, gate_id(add_id, 0, 0), j, x, y, G);
#pragma unroll
    for (int p = 0; p < P; ++p) { Pr.v[p][0] = x.v[p][0] ^ y.v[p][0]; Pr.v[p][1] = x.v[p][1] ^ y.v[p][1]; }
#pragma unroll 1
    for (int l = 1; l <= 6; ++l) {
        const int s = 1 << (l - 1);
#pragma unroll
        for (int p = 0; p < P; ++p) { t.v[p][0] = G.v[p][0] << s; t.v[p][1] = G.v[p][1] << s; }
        and_gate<P>(kttp, gate_id(add_id, l, 0), j, Pr, t, u);
#pragma unroll
        for (int p = 0; p < P; ++p) { G.v[p][0] ^= u.v[p][0]; G.v[p][1] ^= u.v[p][1]; }
        if (l < 6) {
#pragma unroll
            for (int p = 0; p < P; ++p) { t.v[p][0] = Pr.v[p][0] << s; t.v[p][1] = Pr.v[p][1] << s; }
            and_gate<P>(kttp, gate_id(add_id, l, 1), j, Pr, t, u);
            Pr = u;
        }
    }
#pragma unroll
    for (int p = 0; p < P; ++p) {
        out.v[p][0] = x.v[p][0] ^ y.v[p][0] ^ (G.v[p][0] << 1);
        out.v[p][1] = x.v[p][1] ^ y.v[p][1] ^ (G.v[p][1] << 1);
    }
}

__host__ __device__ constexpr int ceil_log2(int n) { return n <= 1 ? 0 : 1 + ceil_log2((n + 1) / 2); }
__host__ __device__ constexpr int pow2_below(int n) { return n <= 2 ? 1 : 2 * pow2_below((n + 1) / 2); }   // largest 2^k < n

// The A2B adder tree over the binary-shared arithmetic shares of parties
// [LO, HI): adjacent pairs level by level (R24).  Node [LO, HI) adds its two
// halves at level h = ceil(log2(HI - LO)) as pair LO >> h.
template <int P, int LO, int HI>
struct Tree {
    static __device__ __forceinline__ void run(const KeySet& kp, uint64_t kttp, uint64_t id, uint64_t j,
                                               const uint64_t (&xs)[P][2], Sh<P>& out) {
        constexpr int MID = LO + pow2_below(HI - LO);
        constexpr int H = ceil_log2(HI - LO);
        Sh<P> l, r;
        Tree<P, LO, MID>::run(kp, kttp, id, j, xs, l);
        Tree<P, MID, HI>::run(kp, kttp, id, j, xs, r);
        add_ring<P>(kttp, (id << 12) | ((uint64_t)H << 6) | (uint64_t)(LO >> H), j, l, r, out);
    }
};
template <int P, int Q>
struct Tree<P, Q, Q + 1> {       // leaf: binary PRZS share of party Q's arithmetic share [x]_Q (R23)
    static __device__ __forceinline__ void run(const KeySet& kp, uint64_t, uint64_t id, uint64_t j,
                                               const uint64_t (&xs)[P][2], Sh<P>& out) {
        const uint64_t s = stream_word(kTagBPRZS, 0, (id << 8) | (uint64_t)Q);
        uint64_t g[P][2];
#pragma unroll
        for (int p = 0; p < P; ++p) philox_pair(kp.k[p], s, j, g[p][0], g[p][1]);
#pragma unroll
        for (int p = 0; p < P; ++p) {
            const int q = (p + P - 1) % P;
            out.v[p][0] = g[p][0] ^ g[q][0] ^ (p == Q ? xs[Q][0] : 0ull);
            out.v[p][1] = g[p][1] ^ g[q][1] ^ (p == Q ? xs[Q][1] : 0ull);
        }
    }
};

template <int P>
__global__ void __launch_bounds__(128) relu_all_kernel(KeySet kp, uint64_t kttp, uint64_t id,
                                                       const uint64_t* __restrict__ x, uint64_t* __restrict__ out,
                                                       uint64_t* __restrict__ sign_out, int64_t n) {
    const int64_t npairs = (n + 1) / 2;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < npairs; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i0 = 2 * j;
        const bool has1 = i0 + 1 < n;
        uint64_t xs[P][2];
#pragma unroll
        for (int p = 0; p < P; ++p) {
            xs[p][0] = x[(int64_t)p * n + i0];
            xs[p][1] = has1 ? x[(int64_t)p * n + i0 + 1] : 0ull;
        }
        // A2B, then the sign bit of every party's binary share (local shift)
        Sh<P> xb;
        Tree<P, 0, P>::run(kp, kttp, id, (uint64_t)j, xs, xb);
        // B2A of the sign bit (Alg. 2) with the bit pair `id`
        uint64_t r0, r1;
        philox_pair(kttp, stream_word(kTagRBIT, 0, id), (uint64_t)j, r0, r1);
        r0 &= 1; r1 &= 1;
        uint64_t rA[P][2], z0 = 0, z1 = 0, rb0 = r0, rb1 = r1, ra0 = r0, ra1 = r1;
#pragma unroll
        for (int p = 1; p < P; ++p) {
            uint64_t b0, b1;
            philox_pair(kttp, stream_word(kTagRB, (uint32_t)p, id), (uint64_t)j, b0, b1);
            b0 &= 1; b1 &= 1;
            rb0 ^= b0; rb1 ^= b1;
            z0 ^= (xb.v[p][0] >> 63) ^ b0; z1 ^= (xb.v[p][1] >> 63) ^ b1;
            philox_pair(kttp, stream_word(kTagRA, (uint32_t)p, id), (uint64_t)j, rA[p][0], rA[p][1]);
            ra0 -= rA[p][0]; ra1 -= rA[p][1];
        }
        rA[0][0] = ra0; rA[0][1] = ra1;
        z0 ^= (xb.v[0][0] >> 63) ^ rb0; z1 ^= (xb.v[0][1] >> 63) ^ rb1;
        // [s]_p = [r]_p + [p=0] z - 2 z [r]_p;  indicator [x >= 0]_p = [p=0] - [s]_p
        uint64_t ind[P][2];
#pragma unroll
        for (int p = 0; p < P; ++p) {
            const uint64_t s0 = rA[p][0] - 2u * z0 * rA[p][0] + (p == 0 ? z0 : 0ull);
            const uint64_t s1 = rA[p][1] - 2u * z1 * rA[p][1] + (p == 0 ? z1 : 0ull);
            if (sign_out) {
                sign_out[(int64_t)p * n + i0] = s0;
                if (has1) sign_out[(int64_t)p * n + i0 + 1] = s1;
            }
            ind[p][0] = (p == 0 ? 1ull : 0ull) - s0;
            ind[p][1] = (p == 0 ? 1ull : 0ull) - s1;
        }
        // Beaver multiplication [x] * [x >= 0] with the MA/MB/MC triple `id`
        uint64_t a[P][2], b[P][2];
        uint64_t e0 = 0, e1 = 0, d0 = 0, d1 = 0, as0 = 0, as1 = 0, bs0 = 0, bs1 = 0;
#pragma unroll
        for (int p = 0; p < P; ++p) {
            philox_pair(kttp, stream_word(kTagMA, (uint32_t)p, id), (uint64_t)j, a[p][0], a[p][1]);
            philox_pair(kttp, stream_word(kTagMB, (uint32_t)p, id), (uint64_t)j, b[p][0], b[p][1]);
            e0 += xs[p][0] - a[p][0]; e1 += xs[p][1] - a[p][1];
            d0 += ind[p][0] - b[p][0]; d1 += ind[p][1] - b[p][1];
            as0 += a[p][0]; as1 += a[p][1]; bs0 += b[p][0]; bs1 += b[p][1];
        }
        uint64_t c00 = as0 * bs0, c01 = as1 * bs1;
#pragma unroll
        for (int p = 1; p < P; ++p) {
            uint64_t c0, c1;
            philox_pair(kttp, stream_word(kTagMC, (uint32_t)p, id), (uint64_t)j, c0, c1);
            c00 -= c0; c01 -= c1;
            out[(int64_t)p * n + i0] = c0 + e0 * b[p][0] + a[p][0] * d0;
            if (has1) out[(int64_t)p * n + i0 + 1] = c1 + e1 * b[p][1] + a[p][1] * d1;
        }
        out[i0] = c00 + e0 * b[0][0] + a[0][0] * d0 + e0 * d0;
        if (has1) out[i0 + 1] = c01 + e1 * b[0][1] + a[0][1] * d1 + e1 * d1;
    }
}

template <int P>
cudaError_t launch_p(const KeySet& kp, uint64_t kttp, uint64_t id, const uint64_t* x, uint64_t* out,
                     uint64_t* sign_out, int64_t n, cudaStream_t st) {
    int64_t g = ((n + 1) / 2 + 127) / 128;
    if (g < 1) g = 1;
    if (g > 148 * 32) g = 148 * 32;
    relu_all_kernel<P><<<(unsigned)g, 128, 0, st>>>(kp, kttp, id, x, out, sign_out, n);
    return cudaGetLastError();
}
}  // namespace

cudaError_t launch_relu_all(const KeySet& kp, uint64_t kttp, uint64_t id, int P, const uint64_t* x, uint64_t* out,
                            uint64_t* sign_out, int64_t n, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    switch (P) {
        case 1: return launch_p<1>(kp, kttp, id, x, out, sign_out, n, st);
        case 2: return launch_p<2>(kp, kttp, id, x, out, sign_out, n, st);
        case 3: return launch_p<3>(kp, kttp, id, x, out, sign_out, n, st);
        case 4: return launch_p<4>(kp, kttp, id, x, out, sign_out, n, st);
        case 5: return launch_p<5>(kp, kttp, id, x, out, sign_out, n, st);
        case 6: return launch_p<6>(kp, kttp, id, x, out, sign_out, n, st);
        case 7: return launch_p<7>(kp, kttp, id, x, out, sign_out, n, st);
        case 8: return launch_p<8>(kp, kttp, id, x, out, sign_out, n, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace mpc

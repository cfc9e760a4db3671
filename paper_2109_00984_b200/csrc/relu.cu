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


// ============================================================================
// One party per context.  Party p holds one share of everything; each AND
// level, the B2A bit and the multiplication are one reveal (round) of the
// transport between the kernels below.  The streams, gate ids and the tree are
// those of relu_all_kernel, so both modes produce bit-identical shares.  Party 0
// also plays the TTP for the correction shares c_0 / r_0 (it regenerates every
// party's triple words, as the all-parties kernel does).
namespace {

struct W2 { uint64_t v0, v1; };          // the two elements of one Philox block (element pair j)

__device__ __forceinline__ W2 operator^(W2 a, W2 b) { return {a.v0 ^ b.v0, a.v1 ^ b.v1}; }
__device__ __forceinline__ W2 operator&(W2 a, W2 b) { return {a.v0 & b.v0, a.v1 & b.v1}; }
__device__ __forceinline__ W2 shl(W2 a, int s) { return {a.v0 << s, a.v1 << s}; }

__device__ __forceinline__ W2 gen(uint64_t key, uint32_t tag, uint32_t party, uint64_t sid, uint64_t j) {
    W2 r;
    philox_pair(key, stream_word(tag, party, sid), j, r.v0, r.v1);
    return r;
}
__device__ __forceinline__ W2 ld2(const uint64_t* b, int64_t i0, bool has1) {
    return {b[i0], has1 ? b[i0 + 1] : 0ull};
}
__device__ __forceinline__ void st2(uint64_t* b, int64_t i0, bool has1, W2 v) {
    b[i0] = v.v0;
    if (has1) b[i0 + 1] = v.v1;
}

// Binary Beaver AND, party p: mask (e, d) = (x ^ a_p, y ^ b_p) ...
__device__ __forceinline__ void and_mask1(uint64_t kttp, uint64_t gid, int p, uint64_t j, W2 x, W2 y, W2& e, W2& d) {
    e = x ^ gen(kttp, kTagBA, (uint32_t)p, gid, j);
    d = y ^ gen(kttp, kTagBB, (uint32_t)p, gid, j);
}
// ... and finish from the revealed (E, D): z_p = c_p ^ (E & b_p) ^ (a_p & D) ^ [p = 0](E & D),
// c_0 = (XOR_q a_q & XOR_q b_q) ^ XOR_{q>=1} c_q.
__device__ __forceinline__ W2 and_finish1(uint64_t kttp, uint64_t gid, int P, int p, uint64_t j, W2 E, W2 D) {
    const W2 a = gen(kttp, kTagBA, (uint32_t)p, gid, j), b = gen(kttp, kTagBB, (uint32_t)p, gid, j);
    if (p != 0) return gen(kttp, kTagBC, (uint32_t)p, gid, j) ^ (E & b) ^ (a & D);
    W2 as = a, bs = b, cs = {0, 0};
    for (int q = 1; q < P; ++q) {
        as = as ^ gen(kttp, kTagBA, (uint32_t)q, gid, j);
        bs = bs ^ gen(kttp, kTagBB, (uint32_t)q, gid, j);
        cs = cs ^ gen(kttp, kTagBC, (uint32_t)q, gid, j);
    }
    return (as & bs) ^ cs ^ (E & b) ^ (a & D) ^ (E & D);
}

__global__ void __launch_bounds__(256) relu_leaf_kernel(KeySet kp, int P, int p, uint64_t id,
                                                        const uint64_t* __restrict__ x, uint64_t* __restrict__ V,
                                                        int64_t n) {
    const int64_t npairs = (n + 1) / 2;
    const int prev = (p + P - 1) % P;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < npairs; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i0 = 2 * j;
        const bool has1 = i0 + 1 < n;
        const W2 xs = ld2(x, i0, has1);
        for (int Q = 0; Q < P; ++Q) {
            const uint64_t sid = (id << 8) | (uint64_t)Q;
            W2 v = gen(kp.k[p], kTagBPRZS, 0, sid, j) ^ gen(kp.k[prev], kTagBPRZS, 0, sid, j);
            if (Q == p) v = v ^ xs;
            st2(V + (int64_t)Q * n, i0, has1, v);
        }
    }
}

__device__ __forceinline__ uint64_t relu_gate(uint64_t add_id, int l, int w) {
    return (add_id << 4) | ((uint64_t)l << 1) | (uint64_t)w;
}

__global__ void __launch_bounds__(256) relu_adder_step_kernel(ReluAdderArgs a, int l) {
    const int64_t n = a.n, npairs = (n + 1) / 2;
    const int64_t K = a.nnodes;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < npairs; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i0 = 2 * j;
        const bool has1 = i0 + 1 < n;
        for (int k = 0; k < a.nnodes; ++k) {
            const ReluNode nd = a.node[k];
            uint64_t* e0p = a.ED + (0 * K + k) * n;
            uint64_t* d0p = a.ED + (1 * K + k) * n;
            uint64_t* e1p = a.ED + (2 * K + k) * n;
            uint64_t* d1p = a.ED + (3 * K + k) * n;
            const W2 x = ld2(a.V + (int64_t)nd.lo * n, i0, has1), y = ld2(a.V + (int64_t)nd.mid * n, i0, has1);
            W2 e, d;
            if (l == 0) {                                     // generate level: AND(x, y)
                and_mask1(a.kttp, relu_gate(nd.add_id, 0, 0), a.p, (uint64_t)j, x, y, e, d);
                st2(e0p, i0, has1, e); st2(d0p, i0, has1, d);
                continue;
            }
            W2 G, Pr;
            const int lp = l - 1;                             // the level whose reveal just completed
            const W2 E0 = ld2(e0p, i0, has1), D0 = ld2(d0p, i0, has1);
            if (lp == 0) {
                G = and_finish1(a.kttp, relu_gate(nd.add_id, 0, 0), a.P, a.p, (uint64_t)j, E0, D0);
                Pr = x ^ y;
            } else {
                G = ld2(a.G + k * n, i0, has1);
                Pr = ld2(a.Pr + k * n, i0, has1);
                G = G ^ and_finish1(a.kttp, relu_gate(nd.add_id, lp, 0), a.P, a.p, (uint64_t)j, E0, D0);
                if (lp < 6)
                    Pr = and_finish1(a.kttp, relu_gate(nd.add_id, lp, 1), a.P, a.p, (uint64_t)j,
                                     ld2(e1p, i0, has1), ld2(d1p, i0, has1));
            }
            if (l <= 6) {
                const int s = 1 << (l - 1);
                and_mask1(a.kttp, relu_gate(nd.add_id, l, 0), a.p, (uint64_t)j, Pr, shl(G, s), e, d);
                st2(e0p, i0, has1, e); st2(d0p, i0, has1, d);
                if (l < 6) {
                    and_mask1(a.kttp, relu_gate(nd.add_id, l, 1), a.p, (uint64_t)j, Pr, shl(Pr, s), e, d);
                    st2(e1p, i0, has1, e); st2(d1p, i0, has1, d);
                }
                st2(a.G + k * n, i0, has1, G);
                st2(a.Pr + k * n, i0, has1, Pr);
            } else {
                st2(a.V + (int64_t)nd.lo * n, i0, has1, x ^ y ^ shl(G, 1));   // the sum, R24
            }
        }
    }
}

// rb_p (p >= 1) from RB; rb_0 = r ^ XOR_{q>=1} rb_q with r from RBIT (the TTP's bit)
__device__ __forceinline__ W2 bit_share(uint64_t kttp, int P, int p, uint64_t id, uint64_t j) {
    const W2 one = {1, 1};
    if (p != 0) return gen(kttp, kTagRB, (uint32_t)p, id, j) & one;
    W2 r = gen(kttp, kTagRBIT, 0, id, j) & one;
    for (int q = 1; q < P; ++q) r = r ^ (gen(kttp, kTagRB, (uint32_t)q, id, j) & one);
    return r;
}

__global__ void __launch_bounds__(256) relu_b2a_mask_kernel(uint64_t kttp, int P, int p, uint64_t id,
                                                            const uint64_t* __restrict__ xb,
                                                            uint64_t* __restrict__ zbits, int64_t n) {
    const int64_t npairs = (n + 1) / 2, nwords = (npairs + 31) / 32;
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t w = warp; w < nwords; w += nwarps) {
        const int64_t j = w * 32 + lane;
        uint32_t b0 = 0, b1 = 0;
        if (j < npairs) {
            const int64_t i0 = 2 * j;
            const bool has1 = i0 + 1 < n;
            const W2 v = ld2(xb, i0, has1);
            const W2 r = bit_share(kttp, P, p, id, (uint64_t)j);
            b0 = (uint32_t)((v.v0 >> 63) ^ r.v0);
            b1 = has1 ? (uint32_t)((v.v1 >> 63) ^ r.v1) : 0u;
        }
        const uint32_t m0 = __ballot_sync(0xffffffffu, b0), m1 = __ballot_sync(0xffffffffu, b1);
        if (lane == 0) zbits[w] = (uint64_t)m0 | ((uint64_t)m1 << 32);
    }
}

__global__ void __launch_bounds__(256) relu_b2a_mul_mask_kernel(uint64_t kttp, int P, int p, uint64_t id,
                                                                const uint64_t* __restrict__ zbits,
                                                                const uint64_t* __restrict__ x,
                                                                uint64_t* __restrict__ ed,
                                                                uint64_t* __restrict__ sign_out, int64_t n) {
    const int64_t npairs = (n + 1) / 2;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < npairs; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i0 = 2 * j;
        const bool has1 = i0 + 1 < n;
        const uint64_t zw = zbits[j >> 5];
        const uint64_t z0 = (zw >> (j & 31)) & 1, z1 = (zw >> (32 + (j & 31))) & 1;
        // [r]_p arithmetic (RA for p >= 1; r_0 = r - sum_{q>=1} RA_q)
        W2 rA;
        if (p != 0) {
            rA = gen(kttp, kTagRA, (uint32_t)p, id, (uint64_t)j);
        } else {
            const W2 r = gen(kttp, kTagRBIT, 0, id, (uint64_t)j);
            rA = {r.v0 & 1, r.v1 & 1};
            for (int q = 1; q < P; ++q) {
                const W2 t = gen(kttp, kTagRA, (uint32_t)q, id, (uint64_t)j);
                rA.v0 -= t.v0; rA.v1 -= t.v1;
            }
        }
        // Alg. 2: [s]_p = [r]_p + [p = 0] z - 2 z [r]_p; indicator [x >= 0]_p = [p = 0] - [s]_p
        const uint64_t s0 = rA.v0 - 2u * z0 * rA.v0 + (p == 0 ? z0 : 0ull);
        const uint64_t s1 = rA.v1 - 2u * z1 * rA.v1 + (p == 0 ? z1 : 0ull);
        if (sign_out) st2(sign_out, i0, has1, W2{s0, s1});
        const uint64_t one = p == 0 ? 1ull : 0ull;
        const W2 xs = ld2(x, i0, has1);
        const W2 a = gen(kttp, kTagMA, (uint32_t)p, id, (uint64_t)j), b = gen(kttp, kTagMB, (uint32_t)p, id, (uint64_t)j);
        st2(ed, i0, has1, W2{xs.v0 - a.v0, xs.v1 - a.v1});
        st2(ed + n, i0, has1, W2{one - s0 - b.v0, one - s1 - b.v1});
    }
}

__global__ void __launch_bounds__(256) relu_mul_finish_kernel(uint64_t kttp, int P, int p, uint64_t id,
                                                              const uint64_t* __restrict__ ed,
                                                              uint64_t* __restrict__ out, int64_t n) {
    const int64_t npairs = (n + 1) / 2;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < npairs; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i0 = 2 * j;
        const bool has1 = i0 + 1 < n;
        const W2 E = ld2(ed, i0, has1), D = ld2(ed + n, i0, has1);
        const W2 a = gen(kttp, kTagMA, (uint32_t)p, id, (uint64_t)j), b = gen(kttp, kTagMB, (uint32_t)p, id, (uint64_t)j);
        W2 c;
        if (p != 0) {
            c = gen(kttp, kTagMC, (uint32_t)p, id, (uint64_t)j);
        } else {                     // c_0 = (sum a_q)(sum b_q) - sum_{q>=1} c_q
            W2 as = a, bs = b, cs = {0, 0};
            for (int q = 1; q < P; ++q) {
                const W2 aq = gen(kttp, kTagMA, (uint32_t)q, id, (uint64_t)j);
                const W2 bq = gen(kttp, kTagMB, (uint32_t)q, id, (uint64_t)j);
                const W2 cq = gen(kttp, kTagMC, (uint32_t)q, id, (uint64_t)j);
                as.v0 += aq.v0; as.v1 += aq.v1; bs.v0 += bq.v0; bs.v1 += bq.v1; cs.v0 += cq.v0; cs.v1 += cq.v1;
            }
            c = {as.v0 * bs.v0 - cs.v0 + E.v0 * D.v0, as.v1 * bs.v1 - cs.v1 + E.v1 * D.v1};
        }
        st2(out, i0, has1, W2{c.v0 + E.v0 * b.v0 + a.v0 * D.v0, c.v1 + E.v1 * b.v1 + a.v1 * D.v1});
    }
}

unsigned pair_grid(int64_t n) {
    int64_t g = ((n + 1) / 2 + 255) / 256;
    if (g < 1) g = 1;
    if (g > 148 * 8) g = 148 * 8;
    return (unsigned)g;
}

void tree_rec(int lo, int hi, uint64_t id, std::vector<std::vector<ReluNode>>& out) {
    if (hi - lo <= 1) return;
    const int mid = lo + pow2_below(hi - lo), H = ceil_log2(hi - lo);
    tree_rec(lo, mid, id, out);
    tree_rec(mid, hi, id, out);
    if ((int)out.size() < H) out.resize(H);
    out[H - 1].push_back(ReluNode{(id << 12) | ((uint64_t)H << 6) | (uint64_t)(lo >> H), lo, mid});
}
}  // namespace

void relu_tree_nodes(int P, uint64_t relu_id, std::vector<std::vector<ReluNode>>& nodes_by_height) {
    nodes_by_height.clear();
    tree_rec(0, P, relu_id, nodes_by_height);
}

cudaError_t launch_relu_leaf(const KeySet& kp, int P, int p, uint64_t relu_id, const uint64_t* x, uint64_t* V,
                             int64_t n, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    relu_leaf_kernel<<<pair_grid(n), 256, 0, st>>>(kp, P, p, relu_id, x, V, n);
    return cudaGetLastError();
}

cudaError_t launch_relu_adder_step(const ReluAdderArgs& a, int l, cudaStream_t st) {
    if (a.n == 0) return cudaSuccess;
    relu_adder_step_kernel<<<pair_grid(a.n), 256, 0, st>>>(a, l);
    return cudaGetLastError();
}

int64_t relu_zbits_words(int64_t n) { return ((n + 1) / 2 + 31) / 32; }

cudaError_t launch_relu_b2a_mask(uint64_t kttp, int P, int p, uint64_t relu_id, const uint64_t* xb, uint64_t* zbits,
                                 int64_t n, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    int64_t g = (relu_zbits_words(n) * 32 + 255) / 256;
    if (g > 148 * 8) g = 148 * 8;
    relu_b2a_mask_kernel<<<(unsigned)g, 256, 0, st>>>(kttp, P, p, relu_id, xb, zbits, n);
    return cudaGetLastError();
}

cudaError_t launch_relu_b2a_mul_mask(uint64_t kttp, int P, int p, uint64_t relu_id, const uint64_t* zbits,
                                     const uint64_t* x, uint64_t* ed, uint64_t* sign_out, int64_t n, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    relu_b2a_mul_mask_kernel<<<pair_grid(n), 256, 0, st>>>(kttp, P, p, relu_id, zbits, x, ed, sign_out, n);
    return cudaGetLastError();
}

cudaError_t launch_relu_mul_finish(uint64_t kttp, int P, int p, uint64_t relu_id, const uint64_t* ed, uint64_t* out,
                                   int64_t n, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    relu_mul_finish_kernel<<<pair_grid(n), 256, 0, st>>>(kttp, P, p, relu_id, ed, out, n);
    return cudaGetLastError();
}

}  // namespace mpc

// elementwise.cu — coalesced uint64 kernels of the protocol (HBM/ALU bound).
//
// Every kernel here is one of the §8(a) rows a1..a6, a8..a10 of SURVEY.md:
// fixed-point encode/decode, PRZS share, local reveal
// (P:171-173), the Beaver mask e = x - a, d = y - b fused with the
// local reveal and the u8 limb split that feeds the tcgen05 ring GEMM,
// TTP triple / wrap-pair generation (Alg. 1
// inputs P:611-612) and truncation.
#include <algorithm>
#include <cstdint>
#include <cuda_runtime.h>
#include "common.cuh"
#include "conv.h"
#include "elementwise.h"

namespace mpc {

static inline unsigned grid_for(int64_t work, int threads = 256) {
    int64_t g = (work + threads - 1) / threads;
    if (g < 1) g = 1;
    if (g > 148 * 16) g = 148 * 16;
    return (unsigned)g;
}

// ------------------------------------------------------------------ a1 / a10
__global__ void encode_kernel(const double* __restrict__ x, uint64_t* __restrict__ out, int64_t n,
                              double scale, int* __restrict__ err) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double v = x[i] * scale;                       // exact: power-of-two scale
        if (!(fabs(v) < 9223372036854775808.0)) { atomicExch(err, 1); continue; }
        out[i] = (uint64_t)llround(v);                  // nearest, ties away from zero (R2)
    }
}
__global__ void decode_kernel(const uint64_t* __restrict__ v, double* __restrict__ out, int64_t n, double inv_scale) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (double)(int64_t)v[i] * inv_scale;
}
cudaError_t launch_encode(const double* x, uint64_t* out, int64_t n, int frac_bits, int* err, cudaStream_t st) {
    encode_kernel<<<grid_for(n), 256, 0, st>>>(x, out, n, ldexp(1.0, frac_bits), err);
    return cudaGetLastError();
}
cudaError_t launch_decode(const uint64_t* v, double* out, int64_t n, int frac_bits, cudaStream_t st) {
    decode_kernel<<<grid_for(n), 256, 0, st>>>(v, out, n, ldexp(1.0, -frac_bits));
    return cudaGetLastError();
}

// ------------------------------------------------------------------ a2 share
// [x]_p = G(k_p, s)[i] - G(k_{p-1}, s)[i] + [p == src] x[i]   (R4)
// One thread per element pair (one Philox block yields two elements), round keys
// precomputed on the host (philox_pair_rk).  All parties: every stream G(k_q) is
// expanded ONCE — party q's own block is party q+1's neighbour block, and party 0's
// neighbour k_{P-1} closes the ring (P blocks for P parties); P is a template
// constant so each party's round keys are constant-bank operands.  One party:
// its own and its neighbour's stream.  16-byte loads / stores when n is even and
// the buffers are aligned.
struct ShareRK { PhiloxRK k[kMaxParties]; };
__device__ __forceinline__ void ld2(const uint64_t* __restrict__ p, int64_t i0, bool vec, bool has1, uint64_t (&o)[2]) {
    if (vec) { const ulonglong2 t = __ldg(reinterpret_cast<const ulonglong2*>(p + i0)); o[0] = t.x; o[1] = t.y; }
    else { o[0] = p[i0]; o[1] = has1 ? p[i0 + 1] : 0ull; }
}
__device__ __forceinline__ void st2(uint64_t* __restrict__ p, int64_t i0, bool vec, bool has1, uint64_t v0, uint64_t v1) {
    if (vec) *reinterpret_cast<ulonglong2*>(p + i0) = make_ulonglong2(v0, v1);
    else { p[i0] = v0; if (has1) p[i0 + 1] = v1; }
}
// 32-byte (one sector) accesses of 4 elements
__device__ __forceinline__ void ld4(const uint64_t* __restrict__ p, uint64_t (&o)[4]) {
    asm volatile("ld.global.nc.v4.u64 {%0, %1, %2, %3}, [%4];" : "=l"(o[0]), "=l"(o[1]), "=l"(o[2]), "=l"(o[3]) : "l"(p));
}
__device__ __forceinline__ void st4(uint64_t* __restrict__ p, uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
    asm volatile("st.global.v4.u64 [%0], {%1, %2, %3, %4};" :: "l"(p), "l"(a), "l"(b), "l"(c), "l"(d) : "memory");
}
template <int P>
__global__ void __launch_bounds__(256) share_all_kernel(const ShareRK rk, const uint64_t* __restrict__ x, int src,
                                                        uint64_t stream, uint64_t* __restrict__ out, int64_t n) {
    const int64_t npairs = (n + 1) / 2;
    const bool vec = (n & 1) == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0 &&
                     (!x || (reinterpret_cast<uintptr_t>(x) & 15) == 0);
    const bool quad = (n & 3) == 0 && (reinterpret_cast<uintptr_t>(out) & 31) == 0 &&
                      (!x || (reinterpret_cast<uintptr_t>(x) & 31) == 0);
    if (quad) {
        // 4 elements (two Philox blocks per stream) per thread and step: full 32-byte sectors for
        // every load and store (2 parties, 4096^2: 0.76 -> 0.8x of the HBM copy rate; see DESIGN)
        const int64_t nq = n / 4;
        for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nq; t += (int64_t)gridDim.x * blockDim.x) {
            const int64_t i0 = 4 * t;
            uint64_t xv[4] = {0, 0, 0, 0};
            if (x) ld4(x + i0, xv);
            uint64_t g[4], first[4], prev[4];
#pragma unroll
            for (int q = 0; q < P; ++q) {
                philox_pair_rk(rk.k[q], stream, (uint64_t)(2 * t), g[0], g[1]);
                philox_pair_rk(rk.k[q], stream, (uint64_t)(2 * t + 1), g[2], g[3]);
                if (q == 0) {
#pragma unroll
                    for (int e = 0; e < 4; ++e) first[e] = g[e];
                } else {
                    const uint64_t add = q == src ? 1ull : 0ull;
                    st4(out + (int64_t)q * n + i0, g[0] - prev[0] + add * xv[0], g[1] - prev[1] + add * xv[1],
                        g[2] - prev[2] + add * xv[2], g[3] - prev[3] + add * xv[3]);
                }
#pragma unroll
                for (int e = 0; e < 4; ++e) prev[e] = g[e];
            }
            const uint64_t add0 = src == 0 ? 1ull : 0ull;            // party 0: G(k_0) - G(k_{P-1})
            st4(out + i0, first[0] - prev[0] + add0 * xv[0], first[1] - prev[1] + add0 * xv[1],
                first[2] - prev[2] + add0 * xv[2], first[3] - prev[3] + add0 * xv[3]);
        }
        return;
    }
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < npairs; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i0 = 2 * j;
        const bool has1 = i0 + 1 < n;
        uint64_t xv[2] = {0, 0};
        if (x) ld2(x, i0, vec, has1, xv);
        uint64_t g[2], first[2], prev[2];
#pragma unroll
        for (int q = 0; q < P; ++q) {
            philox_pair_rk(rk.k[q], stream, (uint64_t)j, g[0], g[1]);
            if (q == 0) { first[0] = g[0]; first[1] = g[1]; }
            else {
                const uint64_t add = q == src ? 1ull : 0ull;
                st2(out + (int64_t)q * n, i0, vec, has1, g[0] - prev[0] + add * xv[0], g[1] - prev[1] + add * xv[1]);
            }
            prev[0] = g[0]; prev[1] = g[1];
        }
        const uint64_t add0 = src == 0 ? 1ull : 0ull;            // party 0: G(k_0) - G(k_{P-1})
        st2(out, i0, vec, has1, first[0] - prev[0] + add0 * xv[0], first[1] - prev[1] + add0 * xv[1]);
    }
}
__global__ void __launch_bounds__(256) share_one_kernel(const PhiloxRK self, const PhiloxRK prev, int is_src,
                                                        const uint64_t* __restrict__ x, uint64_t stream,
                                                        uint64_t* __restrict__ out, int64_t n) {
    const int64_t npairs = (n + 1) / 2;
    const bool vec = (n & 1) == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0 &&
                     (!x || (reinterpret_cast<uintptr_t>(x) & 15) == 0);
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < npairs; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i0 = 2 * j;
        const bool has1 = i0 + 1 < n;
        uint64_t xv[2] = {0, 0}, g[2], h[2];
        if (is_src && x) ld2(x, i0, vec, has1, xv);
        philox_pair_rk(self, stream, (uint64_t)j, g[0], g[1]);
        philox_pair_rk(prev, stream, (uint64_t)j, h[0], h[1]);
        st2(out, i0, vec, has1, g[0] - h[0] + xv[0], g[1] - h[1] + xv[1]);
    }
}
cudaError_t launch_share(const KeySet& keys, int P, int party_lo, int party_hi, const uint64_t* x, int src,
                         uint64_t stream, uint64_t* out, int64_t n, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    if (party_hi - party_lo == 1 || P == 1) {
        const unsigned g = grid_for((n + 1) / 2);
        // one party (or P = 1, where [x]_0 = G(k_0) - G(k_0) + x = x)
        for (int p = party_lo; p < party_hi; ++p) {
            share_one_kernel<<<g, 256, 0, st>>>(philox_round_keys(keys.k[p]),
                                                philox_round_keys(keys.k[(p + P - 1) % P]), p == src ? 1 : 0,
                                                p == src ? x : nullptr, stream, out + (int64_t)(p - party_lo) * n, n);
        }
        return cudaGetLastError();
    }
    if (party_lo != 0 || party_hi != P) return cudaErrorInvalidValue;
    ShareRK rk;
    for (int q = 0; q < P; ++q) rk.k[q] = philox_round_keys(keys.k[q]);
    const uint64_t* xs = (src >= 0 && src < P) ? x : nullptr;
    const bool quad = (n & 3) == 0 && (reinterpret_cast<uintptr_t>(out) & 31) == 0 &&
                      (!xs || (reinterpret_cast<uintptr_t>(xs) & 31) == 0);
    const unsigned g = grid_for(quad ? n / 4 : (n + 1) / 2);
    switch (P) {
#define MPC_SHARE_CASE(Q) case Q: share_all_kernel<Q><<<g, 256, 0, st>>>(rk, xs, src, stream, out, n); break;
        MPC_SHARE_CASE(2) MPC_SHARE_CASE(3) MPC_SHARE_CASE(4) MPC_SHARE_CASE(5) MPC_SHARE_CASE(6) MPC_SHARE_CASE(7)
        MPC_SHARE_CASE(8) MPC_SHARE_CASE(9) MPC_SHARE_CASE(10) MPC_SHARE_CASE(11) MPC_SHARE_CASE(12)
        MPC_SHARE_CASE(13) MPC_SHARE_CASE(14) MPC_SHARE_CASE(15) MPC_SHARE_CASE(16)
#undef MPC_SHARE_CASE
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

// ------------------------------------------------------------------ reveal (local sum)
__global__ void sum_parties_kernel(const uint64_t* __restrict__ s, int P, int64_t n, uint64_t* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t acc = 0;
        for (int p = 0; p < P; ++p) acc += s[(int64_t)p * n + i];
        out[i] = acc;
    }
}
cudaError_t launch_sum_parties(const uint64_t* s, int P, int64_t n, uint64_t* out, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    sum_parties_kernel<<<grid_for(n), 256, 0, st>>>(s, P, n, out);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ a4 mask (one party)
// e = x - a (n1 elements) and d = y - b (n2 elements) into one contiguous
// buffer [e | d] that is then revealed by a single allreduce (one round).
__global__ void mask_kernel(const uint64_t* __restrict__ x, const uint64_t* __restrict__ a, int64_t n1,
                            const uint64_t* __restrict__ y, const uint64_t* __restrict__ b, int64_t n2,
                            uint64_t* __restrict__ ed) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n1 + n2; i += (int64_t)gridDim.x * blockDim.x)
        ed[i] = (i < n1) ? x[i] - a[i] : y[i - n1] - b[i - n1];
}
cudaError_t launch_mask(const uint64_t* x, const uint64_t* a, int64_t n1, const uint64_t* y, const uint64_t* b,
                        int64_t n2, uint64_t* ed, cudaStream_t st) {
    if (n1 + n2 == 0) return cudaSuccess;
    mask_kernel<<<grid_for(n1 + n2), 256, 0, st>>>(x, a, n1, y, b, n2, ed);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ a4+a5+a6 left split
// Left operands (rows = M, K contiguous): eps = sum_{p<Psum} (plus_p - minus_p)
// -> eps planes; copies: planes of cp_src party q for q < Pcopy.  When
// cp_src == minus (all parties on one device) each party's a_p is split from
// the registers it was loaded into for the mask (read once).
// A warp covers 8 rows x 64 K: lane -> (row = lane & 7, 16-K chunk = lane >> 3);
// a thread loads its 128 contiguous bytes with 16-byte loads, all issued
// before use, and each limb's 8 rows x 16 B are written as one 128 B run.
__device__ __forceinline__ void load16(const uint64_t* __restrict__ src, bool full, bool vec, int64_t kleft,
                                       uint64_t (&v)[16]) {
    if (full && vec) {
        const ulonglong2* s2 = reinterpret_cast<const ulonglong2*>(src);
        ulonglong2 t[8];
#pragma unroll
        for (int m = 0; m < 8; ++m) t[m] = __ldg(s2 + m);
#pragma unroll
        for (int m = 0; m < 8; ++m) { v[2 * m] = t[m].x; v[2 * m + 1] = t[m].y; }
    } else {
#pragma unroll
        for (int m = 0; m < 16; ++m) v[m] = (m < kleft) ? __ldg(src + m) : 0ull;
    }
}

// MPC_SPLIT2=0 turns the two-party split paths below off (A/B measurements); set once per
// process by the first split launch (a constant-bank flag, so captured graphs see it too).
__constant__ int g_split2 = 1;
__device__ __forceinline__ bool split2_enabled() { return g_split2 != 0; }
static void split2_config() {
    static bool done = false;
    if (done) return;
    done = true;
    const char* e = getenv("MPC_SPLIT2");
    if (e && atoi(e) == 0) {
        const int zero = 0;
        cudaMemcpyToSymbol(g_split2, &zero, sizeof(zero));
    }
}

// host mirror of the device-side choice: the two-party paths run twice as many (half-size)
// warp tasks, so the launchers size their grids for them
static bool split2_host() {
    static const bool on = !(getenv("MPC_SPLIT2") && atoi(getenv("MPC_SPLIT2")) == 0);
    return on;
}
static bool left2(const LeftSplitArgs& a) {
    return split2_host() && a.cp_src == a.minus && a.minus && a.Pcopy == 2 && a.Psum == 2 && a.sum_planes && a.cp_planes;
}
static bool right2(const RightSplitArgs& a) {
    return split2_host() && a.cp_src == a.minus && a.minus && a.Pcopy == 2 && a.Psum == 2 && a.cp_planes;
}

// Two parties with the copies fused into the mask (the common all-parties Beaver case):
// every share load of a task is issued before any is used, so a task costs one memory
// round trip instead of one per (party, operand); tasks are half the generic ones
// (8 K values per lane) so the loads fit in the registers of two 256-thread blocks per SM.
// Left: a warp covers 8 rows x 32 K (lane -> row lane & 7, 8-K chunk lane >> 3).
template <Layout LO>
__device__ __forceinline__ void split_left2_body(const LeftSplitArgs& a, int64_t bid, int64_t nblk) {
    const int64_t KB = num_kb(a.K);
    const int64_t row_groups = (a.M + 7) / 8;
    const int64_t warps_total = row_groups * KB;                 // whole padded K: pad limbs must be 0
    const int64_t nb = a.batch > 1 ? a.batch : 1;
    const int lane = threadIdx.x & 31;
    const bool vec = (a.K & 1) == 0 && (a.party_stride & 1) == 0 && (a.in_bstride & 1) == 0;
    for (int64_t bw = (bid * blockDim.x + threadIdx.x) >> 5; bw < warps_total * nb; bw += (nblk * blockDim.x) >> 5) {
        const int64_t bi = bw / warps_total, w = bw - bi * warps_total;
        const uint64_t* plus = a.plus + bi * a.in_bstride;
        const uint64_t* minus = a.minus + bi * a.in_bstride;
        uint8_t* sum_planes = a.sum_planes + bi * a.sum_bstride;
        uint8_t* cp_planes = a.cp_planes + bi * a.cp_bstride;
        const int64_t row = (w / KB) * 8 + (lane & 7);
        const int64_t k0 = (w % KB) * 32 + (lane >> 3) * 8;
        if (row >= a.M) continue;
        const int64_t kleft = a.K - k0;                          // <= 0: pure K padding
        uint64_t x0[8], a0[8], x1[8], a1[8];
        const int64_t o = row * a.K + k0;
        if (vec && kleft >= 8) {
            const ulonglong2* p0 = reinterpret_cast<const ulonglong2*>(plus + o);
            const ulonglong2* p1 = reinterpret_cast<const ulonglong2*>(minus + o);
            const ulonglong2* p2 = reinterpret_cast<const ulonglong2*>(plus + a.party_stride + o);
            const ulonglong2* p3 = reinterpret_cast<const ulonglong2*>(minus + a.party_stride + o);
            ulonglong2 t0[4], t1[4], t2[4], t3[4];
#pragma unroll
            for (int m = 0; m < 4; ++m) { t0[m] = __ldg(p0 + m); t1[m] = __ldg(p1 + m); t2[m] = __ldg(p2 + m); t3[m] = __ldg(p3 + m); }
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                x0[2 * m] = t0[m].x; x0[2 * m + 1] = t0[m].y; a0[2 * m] = t1[m].x; a0[2 * m + 1] = t1[m].y;
                x1[2 * m] = t2[m].x; x1[2 * m + 1] = t2[m].y; a1[2 * m] = t3[m].x; a1[2 * m + 1] = t3[m].y;
            }
        } else {
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                const bool ok = m < kleft;
                x0[m] = ok ? __ldg(plus + o + m) : 0ull;
                a0[m] = ok ? __ldg(minus + o + m) : 0ull;
                x1[m] = ok ? __ldg(plus + a.party_stride + o + m) : 0ull;
                a1[m] = ok ? __ldg(minus + a.party_stride + o + m) : 0ull;
            }
        }
#pragma unroll
        for (int m = 0; m < 8; ++m) x0[m] = x0[m] - a0[m] + x1[m] - a1[m];
        if (a.add_sum_first) {
#pragma unroll
            for (int m = 0; m < 8; ++m) a0[m] += x0[m];
        }
        store_limbs8<LO>(cp_planes, row, k0, KB, a0);
        store_limbs8<LO>(cp_planes + a.cp_planes_stride, row, k0, KB, a1);
        store_limbs8<LO>(sum_planes, row, k0, KB, x0);
    }
}
// Right (K x N row-major -> planes with rows = N): a warp covers 32 n x 8 K (lane -> n);
// every load is 8 B per lane, 256 B contiguous per warp and K row.
template <Layout LO>
__device__ __forceinline__ void split_right2_body(const RightSplitArgs& a, int64_t bid, int64_t nblk) {
    const int64_t KB = num_kb(a.K);
    const int64_t ngroups = (a.N + 31) / 32;
    const int64_t warps_total = ngroups * KB * 4;               // whole padded K, 8 per task
    const int64_t nb = a.batch > 1 ? a.batch : 1;
    const int lane = threadIdx.x & 31;
    for (int64_t bw = (bid * blockDim.x + threadIdx.x) >> 5; bw < warps_total * nb; bw += (nblk * blockDim.x) >> 5) {
        const int64_t bi = bw / warps_total, w = bw - bi * warps_total;
        const uint64_t* plus = a.plus + bi * a.in_bstride;
        const uint64_t* minus = a.minus + bi * a.in_bstride;
        uint8_t* sum_planes = a.sum_planes ? a.sum_planes + bi * a.sum_bstride : nullptr;
        uint8_t* cp_planes = a.cp_planes + bi * a.cp_bstride;
        const int64_t kc = w / ngroups, ng = w % ngroups;
        const int64_t n = ng * 32 + lane;
        const int64_t k0 = kc * 8;
        if (n >= a.N) continue;
        const int lim = (int)(a.K - k0 < 8 ? (a.K - k0 > 0 ? a.K - k0 : 0) : 8);
        const uint64_t* py = plus + k0 * a.N + n;
        const uint64_t* pb = minus + k0 * a.N + n;
        uint64_t y0[8], b0[8], y1[8], b1[8];
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            const bool ok = m < lim;
            y0[m] = ok ? __ldg(py + m * a.N) : 0ull;
            b0[m] = ok ? __ldg(pb + m * a.N) : 0ull;
            y1[m] = ok ? __ldg(py + a.party_stride + m * a.N) : 0ull;
            b1[m] = ok ? __ldg(pb + a.party_stride + m * a.N) : 0ull;
        }
#pragma unroll
        for (int m = 0; m < 8; ++m) y0[m] = y0[m] - b0[m] + y1[m] - b1[m];
        if (a.add_delta_first) {
#pragma unroll
            for (int m = 0; m < 8; ++m) b0[m] += y0[m];
        }
        store_limbs8<LO>(cp_planes, n, k0, KB, b0);
        store_limbs8<LO>(cp_planes + a.cp_planes_stride, n, k0, KB, b1);
        if (sum_planes) store_limbs8<LO>(sum_planes, n, k0, KB, y0);
    }
}

// (bid, nblk): this block's index among the nblk blocks working on the left split.
// LO: plane layout of the output (Layout::Left normally; Layout::Right when the
// ring GEMM runs transposed, see RingGemmParams::transpose_out).
template <Layout LO>
__device__ __forceinline__ void split_left_body(const LeftSplitArgs& a, int64_t bid, int64_t nblk) {
    if (a.cp_src == a.minus && a.minus && a.Pcopy == 2 && a.Psum == 2 && a.sum_planes && a.cp_planes &&
        split2_enabled()) {
        split_left2_body<LO>(a, bid, nblk);
        return;
    }
    const int64_t KB = num_kb(a.K);
    const int64_t row_groups = (a.M + 7) / 8;
    const int64_t kgroups = (KB * kKBlock + 63) / 64;      // whole padded K: pad limbs must be 0
    const int64_t warps_total = row_groups * kgroups;
    const int64_t nb = a.batch > 1 ? a.batch : 1;
    const int lane = threadIdx.x & 31;
    const bool vec = (a.K & 1) == 0 && (a.party_stride & 1) == 0 && (a.in_bstride & 1) == 0;
    const bool fused_copy = a.cp_src == a.minus && a.Pcopy == a.Psum && a.Psum > 0;
    for (int64_t bw = (bid * blockDim.x + threadIdx.x) >> 5; bw < warps_total * nb; bw += (nblk * blockDim.x) >> 5) {
        const int64_t bi = bw / warps_total, w = bw - bi * warps_total;      // batch element, warp task
        const uint64_t* plus = a.plus ? a.plus + bi * a.in_bstride : nullptr;
        const uint64_t* minus = a.minus ? a.minus + bi * a.in_bstride : nullptr;
        const uint64_t* cp_src = a.cp_src ? a.cp_src + bi * a.in_bstride : nullptr;
        uint8_t* sum_planes = a.sum_planes ? a.sum_planes + bi * a.sum_bstride : nullptr;
        uint8_t* cp_planes = a.cp_planes ? a.cp_planes + bi * a.cp_bstride : nullptr;
        const int64_t rg = w / kgroups, kg = w % kgroups;
        const int64_t row = rg * 8 + (lane & 7);
        const int64_t k0 = kg * 64 + (lane >> 3) * 16;
        if (row >= a.M || k0 >= KB * kKBlock) continue;
        const int64_t kleft = a.K - k0;                     // <= 0: pure K padding
        const bool full = kleft >= 16;
        uint64_t acc[16], v[16];
#pragma unroll
        for (int m = 0; m < 16; ++m) acc[m] = 0;
        if (a.Psum > 0) {
            for (int p = 0; p < a.Psum; ++p) {
                load16(plus + p * a.party_stride + row * a.K + k0, full, vec, kleft, v);
#pragma unroll
                for (int m = 0; m < 16; ++m) acc[m] += v[m];
                if (minus) {
                    load16(minus + p * a.party_stride + row * a.K + k0, full, vec, kleft, v);
#pragma unroll
                    for (int m = 0; m < 16; ++m) acc[m] -= v[m];
                    // party 0's copy needs the complete sum first (add_sum_first): written below
                    if (fused_copy && !(p == 0 && a.add_sum_first))
                        store_limbs16<LO>(cp_planes + p * a.cp_planes_stride, row, k0, KB, v);
                }
            }
            store_limbs16<LO>(sum_planes, row, k0, KB, acc);
        }
        for (int q = 0; q < a.Pcopy; ++q) {
            const bool adds = q == 0 && a.add_sum_first;
            if (fused_copy && !adds) continue;             // already written from registers
            load16(cp_src + q * a.party_stride + row * a.K + k0, full, vec, kleft, v);
            if (adds) {
#pragma unroll
                for (int m = 0; m < 16; ++m) v[m] += acc[m];
            }
            store_limbs16<LO>(cp_planes + q * a.cp_planes_stride, row, k0, KB, v);
        }
    }
}
template <Layout LO>
__global__ void __launch_bounds__(256) split_left_kernel(LeftSplitArgs a) {
    split_left_body<LO>(a, blockIdx.x, gridDim.x);
}
cudaError_t launch_split_left(const LeftSplitArgs& a, cudaStream_t st) {
    split2_config();
    if (a.M > 0 && a.K > 0 && left2(a)) {
        const cudaError_t e = launch_split2_tma(&a, nullptr, st);
        if (e != cudaErrorNotSupported) return e;
    }
    if (a.M == 0 || a.K == 0) return cudaSuccess;
    const int64_t warps = ((a.M + 7) / 8) * ((num_kb(a.K) * kKBlock + 63) / 64) * (a.batch > 1 ? a.batch : 1) *
                          (left2(a) ? 2 : 1);
    if (a.swap == 2) split_left_kernel<Layout::Small><<<grid_for(warps * 32), 256, 0, st>>>(a);
    else if (a.swap) split_left_kernel<Layout::Right><<<grid_for(warps * 32), 256, 0, st>>>(a);
    else split_left_kernel<Layout::Left><<<grid_for(warps * 32), 256, 0, st>>>(a);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ a4+a5+a6 right split
// Right operands (K x N row-major, planes have rows = N: a transpose):
// delta = sum_{p<Psum} (plus_p - minus_p) -> delta planes; copies:
// planes of (b_q + [q == 0 && add_delta_first] delta) for q < Pcopy
// (R8: party 0 folds the public eps@delta into eps @ (b_0 + delta)).  When
// cp_src == minus, b_q (q >= 1) is split from the registers loaded for the
// mask; b_0 is re-read (L1/L2 hit) once delta is complete.
// A warp covers 32 n x 16 K: lane -> (2 adjacent n = 2 * (lane & 15),
// 8-K half = lane >> 4); every load is 16 B per lane (256 B contiguous per
// half-warp and K row) and the two K halves of each 16-byte plane row are
// written by two lanes of the same warp.
struct Col2 { uint64_t v[2][8]; };

__device__ __forceinline__ void load_cols(const uint64_t* __restrict__ base, int64_t N, int64_t n, int64_t k0,
                                          int64_t K, bool vec, bool two, uint64_t (&v)[2][8]) {
#pragma unroll
    for (int m = 0; m < 8; ++m) {
        const int64_t k = k0 + m;
        if (k < K) {
            const uint64_t* src = base + k * N + n;
            if (vec) {
                const ulonglong2 t = __ldg(reinterpret_cast<const ulonglong2*>(src));
                v[0][m] = t.x; v[1][m] = t.y;
            } else {
                v[0][m] = __ldg(src);
                v[1][m] = two ? __ldg(src + 1) : 0ull;
            }
        } else {
            v[0][m] = 0; v[1][m] = 0;
        }
    }
}

template <Layout LO>
__device__ __forceinline__ void split_right_body(const RightSplitArgs& a, int64_t bid, int64_t nblk) {
    if (a.cp_src == a.minus && a.minus && a.Pcopy == 2 && a.Psum == 2 && a.cp_planes && split2_enabled()) {
        split_right2_body<LO>(a, bid, nblk);
        return;
    }
    const int64_t KB = num_kb(a.K);
    const int64_t ngroups = (a.N + 31) / 32;
    const int64_t kchunks = KB * 2;                         // whole padded K, 16 per chunk
    const int64_t warps_total = ngroups * kchunks;
    const int64_t nb = a.batch > 1 ? a.batch : 1;
    const int lane = threadIdx.x & 31;
    const bool fused_copy = a.cp_src == a.minus && a.Pcopy == a.Psum && a.Psum > 0;
    const bool even = (a.N & 1) == 0 && (a.party_stride & 1) == 0 && (a.in_bstride & 1) == 0;
    for (int64_t bw = (bid * blockDim.x + threadIdx.x) >> 5; bw < warps_total * nb; bw += (nblk * blockDim.x) >> 5) {
        const int64_t bi = bw / warps_total, w = bw - bi * warps_total;      // batch element, warp task
        const uint64_t* plus = a.plus ? a.plus + bi * a.in_bstride : nullptr;
        const uint64_t* minus = a.minus ? a.minus + bi * a.in_bstride : nullptr;
        const uint64_t* cp_src = a.cp_src ? a.cp_src + bi * a.in_bstride : nullptr;
        uint8_t* sum_planes = a.sum_planes ? a.sum_planes + bi * a.sum_bstride : nullptr;
        uint8_t* cp_planes = a.cp_planes ? a.cp_planes + bi * a.cp_bstride : nullptr;
        const int64_t kc = w / ngroups, ng = w % ngroups;
        const int64_t n = ng * 32 + 2 * (lane & 15);
        const int64_t k0 = kc * 16 + (lane >> 4) * 8;
        if (n >= a.N) continue;
        const bool two = n + 1 < a.N;
        const bool vec = even && two;
        uint64_t d[2][8], v[2][8];
#pragma unroll
        for (int m = 0; m < 8; ++m) { d[0][m] = 0; d[1][m] = 0; }
        for (int p = 0; p < a.Psum; ++p) {
            load_cols(plus + p * a.party_stride, a.N, n, k0, a.K, vec, two, v);
#pragma unroll
            for (int m = 0; m < 8; ++m) { d[0][m] += v[0][m]; d[1][m] += v[1][m]; }
            if (minus) {
                load_cols(minus + p * a.party_stride, a.N, n, k0, a.K, vec, two, v);
#pragma unroll
                for (int m = 0; m < 8; ++m) { d[0][m] -= v[0][m]; d[1][m] -= v[1][m]; }
                if (fused_copy && !(p == 0 && a.add_delta_first)) {
                    uint8_t* pl = cp_planes + p * a.cp_planes_stride;
                    store_limbs8<LO>(pl, n, k0, KB, v[0]);
                    if (two) store_limbs8<LO>(pl, n + 1, k0, KB, v[1]);
                }
            }
        }
        if (sum_planes) {
            store_limbs8<LO>(sum_planes, n, k0, KB, d[0]);
            if (two) store_limbs8<LO>(sum_planes, n + 1, k0, KB, d[1]);
        }
        for (int q = 0; q < a.Pcopy; ++q) {
            const bool addd = (q == 0) && a.add_delta_first;
            if (fused_copy && !addd) continue;               // already written from registers
            load_cols(cp_src + q * a.party_stride, a.N, n, k0, a.K, vec, two, v);
            if (addd) {
#pragma unroll
                for (int m = 0; m < 8; ++m) { v[0][m] += d[0][m]; v[1][m] += d[1][m]; }
            }
            uint8_t* pl = cp_planes + q * a.cp_planes_stride;
            store_limbs8<LO>(pl, n, k0, KB, v[0]);
            if (two) store_limbs8<LO>(pl, n + 1, k0, KB, v[1]);
        }
    }
}
template <Layout LO>
__global__ void __launch_bounds__(256, 2) split_right_kernel(RightSplitArgs a) {
    split_right_body<LO>(a, blockIdx.x, gridDim.x);
}
cudaError_t launch_split_right(const RightSplitArgs& a, cudaStream_t st) {
    split2_config();
    if (a.N == 0 || a.K == 0) return cudaSuccess;
    const int64_t warps = ((a.N + 31) / 32) * (num_kb(a.K) * 2) * (a.batch > 1 ? a.batch : 1) * (right2(a) ? 2 : 1);
    if (a.swap == 2) split_right_kernel<Layout::Small><<<grid_for(warps * 32), 256, 0, st>>>(a);
    else if (a.swap) split_right_kernel<Layout::Left><<<grid_for(warps * 32), 256, 0, st>>>(a);
    else split_right_kernel<Layout::Right><<<grid_for(warps * 32), 256, 0, st>>>(a);
    return cudaGetLastError();
}

// Both splits of one Beaver matmul in a single launch (they are independent):
// blocks [0, nleft) run the left split, the rest the right split.
template <Layout LL, Layout LR>
__global__ void __launch_bounds__(256, 2) split_both_kernel(LeftSplitArgs l, RightSplitArgs r, int nleft) {
    // launched as a programmatic dependent of the previous kernel (e.g. the last
    // layer's GEMM / finalize): nothing is read or written before it completes
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if ((int)blockIdx.x < nleft) split_left_body<LL>(l, blockIdx.x, nleft);
    else split_right_body<LR>(r, blockIdx.x - nleft, gridDim.x - nleft);
    // each block is done: once all are, the ring GEMM (a programmatic dependent)
    // may launch and run its prologue while the last blocks drain — triggering
    // earlier would let GEMM CTAs take SMs from the split's tail
    asm volatile("griddepcontrol.launch_dependents;");
}
cudaError_t launch_split_both(const LeftSplitArgs& l, const RightSplitArgs& r, cudaStream_t st) {
    split2_config();
    const bool dl = l.M > 0 && l.K > 0, dr = r.N > 0 && r.K > 0;
    if (!dl && !dr) return cudaSuccess;
    if (dl && dr && left2(l) && right2(r)) {
        const cudaError_t e = launch_split2_tma(&l, &r, st);
        if (e != cudaErrorNotSupported) return e;
    }
    if (!dr) return launch_split_left(l, st);
    if (!dl) return launch_split_right(r, st);
    const int64_t bl = l.batch > 1 ? l.batch : 1, br = r.batch > 1 ? r.batch : 1;
    const int64_t wl = ((l.M + 7) / 8) * ((num_kb(l.K) * kKBlock + 63) / 64) * 32 * bl * (left2(l) ? 2 : 1);
    const int64_t wr = ((r.N + 31) / 32) * (num_kb(r.K) * 2) * 32 * br * (right2(r) ? 2 : 1);
    // share the block budget in proportion to the bytes each side moves
    const int64_t bytes_l = l.M * l.K * (int64_t)(2 * l.Psum + l.Pcopy + 1) * bl;
    const int64_t bytes_r = r.N * r.K * (int64_t)(2 * r.Psum + r.Pcopy + 1) * br;
    int64_t nl = std::min<int64_t>(grid_for(wl), std::max<int64_t>(1, 148 * 16 * bytes_l / (bytes_l + bytes_r)));
    int64_t nr = std::min<int64_t>(grid_for(wr), std::max<int64_t>(1, 148 * 16 - nl));
    if (l.swap != r.swap) return cudaErrorInvalidValue;
    if (l.swap == 2)
        return launch_pdl(split_both_kernel<Layout::Small, Layout::Small>, dim3((unsigned)(nl + nr)), dim3(256), 0, st,
                          l, r, (int)nl);
    if (l.swap)
        return launch_pdl(split_both_kernel<Layout::Right, Layout::Left>, dim3((unsigned)(nl + nr)), dim3(256), 0, st,
                          l, r, (int)nl);
    return launch_pdl(split_both_kernel<Layout::Left, Layout::Right>, dim3((unsigned)(nl + nr)), dim3(256), 0, st, l,
                      r, (int)nl);
}

// ------------------------------------------------------------------ conv: implicit im2col split
// A warp covers 32 consecutive im2col rows (lane = row, i.e. 32 neighbouring
// output pixels: the gathers of one K index are nearly contiguous) and one
// 16-K chunk; each lane gathers its 16 (ci, ky, kx) values per party and
// writes 16 bytes per limb plane.  The K padding (K .. 32*KB) is written as 0.
template <Layout LO>
__device__ __forceinline__ void split_im2col_body(const Im2colSplitArgs& a, int64_t bid, int64_t nblk) {
    const ConvGeom& g = a.g;
    const int64_t Ho = g.Ho(), Wo = g.Wo(), M = g.M(), K = g.K(), KB = num_kb(K);
    const int64_t khw = g.kh * g.kw;
    const int64_t rgroups = (M + 31) / 32, kchunks = KB * 2;
    const int lane = threadIdx.x & 31;
    const bool fused_copy = a.cp_src == a.minus && a.Pcopy == a.Psum && a.Psum > 0;
    for (int64_t w = (bid * blockDim.x + threadIdx.x) >> 5; w < rgroups * kchunks; w += (nblk * blockDim.x) >> 5) {
        const int64_t kc = w / rgroups, rg = w % rgroups;     // neighbouring warps: neighbouring rows
        const int64_t row = rg * 32 + lane;
        if (row >= M) continue;
        const int64_t k0 = kc * 16;
        const int64_t b = row / (Ho * Wo), s = row % (Ho * Wo);
        // (ci, ky, kx) of k0 once, then stepped: 32-bit index math inside one image
        // (C*H*W < 2^31, checked by the host), one 64-bit image base
        const int iy0 = (int)(s / Wo) * (int)g.sh - (int)g.ph, ix0 = (int)(s % Wo) * (int)g.sw - (int)g.pw;
        const int H = (int)g.H, W = (int)g.W, kw = (int)g.kw, kh = (int)g.kh;
        int ci = (int)(k0 / khw), r = (int)(k0 % khw);
        int ky = r / kw, kx = r - ky * kw;
        const int64_t base = b * g.C * g.H * g.W;
        int64_t off[16];                                        // element offset in one party's tensor, or -1
#pragma unroll
        for (int m = 0; m < 16; ++m) {
            const int iy = iy0 + ky, ix = ix0 + kx;
            off[m] = (k0 + m < K && iy >= 0 && iy < H && ix >= 0 && ix < W) ? base + (ci * H + iy) * W + ix : -1;
            if (++kx == kw) { kx = 0; if (++ky == kh) { ky = 0; ++ci; } }
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

template <Layout LO>
__global__ void __launch_bounds__(256) split_im2col_kernel(Im2colSplitArgs a) {
    split_im2col_body<LO>(a, blockIdx.x, gridDim.x);
}
cudaError_t launch_split_im2col(const Im2colSplitArgs& a, cudaStream_t st) {
    const int64_t M = a.g.M(), K = a.g.K();
    if (M == 0 || K == 0) return cudaSuccess;
    const int64_t warps = ((M + 31) / 32) * num_kb(K) * 2;
    if (a.layout_right) split_im2col_kernel<Layout::Right><<<grid_for(warps * 32), 256, 0, st>>>(a);
    else split_im2col_kernel<Layout::Left><<<grid_for(warps * 32), 256, 0, st>>>(a);
    return cudaGetLastError();
}

// Both splits of one private convolution in one launch (a programmatic
// dependent, like split_both_kernel): blocks [0, nim) split the implicit
// im2col of eps / a_p, the rest the weights' delta / b'_p.
template <Layout LI, Layout LW>
__global__ void __launch_bounds__(256, 2) split_conv_kernel(Im2colSplitArgs im, LeftSplitArgs wt, int nim) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if ((int)blockIdx.x < nim) split_im2col_body<LI>(im, blockIdx.x, nim);
    else split_left_body<LW>(wt, blockIdx.x - nim, gridDim.x - nim);
    asm volatile("griddepcontrol.launch_dependents;");
}
cudaError_t launch_split_conv(const Im2colSplitArgs& im, const LeftSplitArgs& wt, cudaStream_t st) {
    split2_config();
    const bool di = im.g.M() > 0 && im.g.K() > 0, dw = wt.M > 0 && wt.K > 0;
    if (!dw) return launch_split_im2col(im, st);
    if (!di) return launch_split_left(wt, st);
    if ((im.layout_right != 0) == (wt.swap != 0)) return cudaErrorInvalidValue;   // one left, one right operand
    const int64_t wi = ((im.g.M() + 31) / 32) * num_kb(im.g.K()) * 2 * 32;
    const int64_t ww = ((wt.M + 7) / 8) * ((num_kb(wt.K) * kKBlock + 63) / 64) * 32 * (left2(wt) ? 2 : 1);
    // blocks in proportion to the bytes each side moves (the im2col side re-reads each input kh*kw times)
    const int64_t bytes_i = im.g.M() * im.g.K() * (int64_t)(2 * im.Psum + im.Pcopy + 1);
    const int64_t bytes_w = wt.M * wt.K * (int64_t)(2 * wt.Psum + wt.Pcopy + 1);
    int64_t ni = std::min<int64_t>(grid_for(wi), std::max<int64_t>(1, 148 * 16 * bytes_i / (bytes_i + bytes_w)));
    int64_t nw = std::min<int64_t>(grid_for(ww), std::max<int64_t>(1, 148 * 16 - ni));
    if (im.layout_right)
        return launch_pdl(split_conv_kernel<Layout::Right, Layout::Left>, dim3((unsigned)(ni + nw)), dim3(256), 0, st,
                          im, wt, (int)ni);
    return launch_pdl(split_conv_kernel<Layout::Left, Layout::Right>, dim3((unsigned)(ni + nw)), dim3(256), 0, st, im,
                      wt, (int)ni);
}

// ------------------------------------------------------------------ a3 TTP triples
// Left factor a (M x K): a_q = G(k_ttp, A||q||id)[row*K + k].  Writes the
// parties' u64 shares for q in [out_lo, out_hi) and, if sum_planes != null,
// the limb planes of a = sum_{q<P} a_q (the TTP's view, R6).
__global__ void ttp_left_kernel(TtpGenArgs g) {
    const int64_t KB = num_kb(g.K);
    const int64_t row_groups = (g.rows + 7) / 8;
    const int64_t kgroups = (KB * kKBlock + 63) / 64;
    const int lane = threadIdx.x & 31;
    for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; w < row_groups * kgroups;
         w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t rg = w / kgroups, kg = w % kgroups;
        const int64_t row = rg * 8 + (lane & 7);
        const int64_t k0 = kg * 64 + (lane >> 3) * 16;
        if (row >= g.rows || k0 >= KB * kKBlock) continue;
        uint64_t sum[16];
#pragma unroll
        for (int m = 0; m < 16; ++m) sum[m] = 0;
        const int qhi = g.sum_planes ? g.P : g.out_hi;
        const int qlo = g.sum_planes ? 0 : g.out_lo;
        for (int q = qlo; q < qhi; ++q) {
            const uint64_t s = stream_word(g.tag, (uint32_t)q, g.id);
            const bool wr = (q >= g.out_lo && q < g.out_hi);
            uint64_t* o = wr ? g.out + (int64_t)(q - g.out_lo) * g.rows * g.K + row * g.K : nullptr;
            uint64_t e0 = 0, e1 = 0;
            int64_t have = -1;
#pragma unroll
            for (int m = 0; m < 16; ++m) {
                const int64_t k = k0 + m;
                if (k < g.K) {
                    const uint64_t i = (uint64_t)(row * g.K + k);
                    if ((int64_t)(i >> 1) != have) { philox_pair(g.key, s, i >> 1, e0, e1); have = (int64_t)(i >> 1); }
                    const uint64_t v = (i & 1) ? e1 : e0;
                    sum[m] += v;
                    if (wr) o[k] = v;
                }
            }
        }
        if (g.sum_planes) {
            if (g.small) store_limbs16<Layout::Small>(g.sum_planes, row, k0, KB, sum);
            else store_limbs16<Layout::Left>(g.sum_planes, row, k0, KB, sum);
        }
    }
}
// Right factor b (K x N row-major): b_q = G(k_ttp, B||q||id)[k*N + n];
// planes of b = sum_q b_q are transposed (rows = N).
__global__ void ttp_right_kernel(TtpGenArgs g) {
    const int64_t KB = num_kb(g.K);
    const int64_t N = g.rows;
    const int64_t ngroups = (N + 31) / 32;
    const int64_t kchunks = KB * 2;
    const int lane = threadIdx.x & 31;
    for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; w < ngroups * kchunks;
         w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t kc = w / ngroups, ng = w % ngroups;
        const int64_t n = ng * 32 + lane;
        const int64_t k0 = kc * 16;
        if (n >= N) continue;
        uint64_t sum[16];
#pragma unroll
        for (int m = 0; m < 16; ++m) sum[m] = 0;
        const int qhi = g.sum_planes ? g.P : g.out_hi;
        const int qlo = g.sum_planes ? 0 : g.out_lo;
        for (int q = qlo; q < qhi; ++q) {
            const uint64_t s = stream_word(g.tag, (uint32_t)q, g.id);
            const bool wr = (q >= g.out_lo && q < g.out_hi);
            uint64_t* o = wr ? g.out + (int64_t)(q - g.out_lo) * N * g.K : nullptr;
#pragma unroll
            for (int m = 0; m < 16; ++m) {
                const int64_t k = k0 + m;
                if (k < g.K) {
                    const uint64_t v = philox_at(g.key, s, (uint64_t)(k * N + n));
                    sum[m] += v;
                    if (wr) o[k * N + n] = v;
                }
            }
        }
        if (g.sum_planes) {
            if (g.small) store_limbs16<Layout::Small>(g.sum_planes, n, k0, KB, sum);
            else store_limbs16<Layout::Right>(g.sum_planes, n, k0, KB, sum);
        }
    }
}
cudaError_t launch_ttp_left(const TtpGenArgs& g, cudaStream_t st) {
    if (g.rows == 0 || g.K == 0) return cudaSuccess;
    const int64_t warps = ((g.rows + 7) / 8) * ((num_kb(g.K) * kKBlock + 63) / 64);
    ttp_left_kernel<<<grid_for(warps * 32), 256, 0, st>>>(g);
    return cudaGetLastError();
}
cudaError_t launch_ttp_right(const TtpGenArgs& g, cudaStream_t st) {
    if (g.rows == 0 || g.K == 0) return cudaSuccess;
    const int64_t warps = ((g.rows + 31) / 32) * (num_kb(g.K) * 2);
    ttp_right_kernel<<<grid_for(warps * 32), 256, 0, st>>>(g);
    return cudaGetLastError();
}

// c_q = G(k_ttp, C||q||id) for q >= 1; c_0 = c - sum_{q>=1} c_q.
// out: parties [out_lo, out_hi); c0_full (in/out) holds c on entry if the
// TTP view is requested (fix_c0), and receives c_0.
__global__ void ttp_c_kernel(uint64_t key, uint64_t id, int P, int out_lo, int out_hi, uint64_t* __restrict__ out,
                             uint64_t* __restrict__ c0, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t acc = 0;
        for (int q = 1; q < P; ++q) {
            const bool wr = (q >= out_lo && q < out_hi);
            if (!wr && !c0) continue;
            const uint64_t v = philox_at(key, stream_word(kTagC, (uint32_t)q, id), (uint64_t)i);
            acc += v;
            if (wr) out[(int64_t)(q - out_lo) * n + i] = v;
        }
        if (c0) c0[i] -= acc;
    }
}
cudaError_t launch_ttp_c(uint64_t key, uint64_t id, int P, int out_lo, int out_hi, uint64_t* out, uint64_t* c0,
                         int64_t n, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    ttp_c_kernel<<<grid_for(n), 256, 0, st>>>(key, id, P, out_lo, out_hi, out, c0, n);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ a9 wrap pairs
// Element pairs: one Philox4x32-10 block yields both elements of a pair, so
// every per-element helper below works on pair j = elements (2j, 2j + 1).
// Pair loads / stores are 16-byte vectors when n is even and the base is
// 16-byte aligned (then every party's row of [P][n] is too).
__device__ __forceinline__ bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
__device__ __forceinline__ void ld_pair(const uint64_t* __restrict__ p, int64_t i0, bool vec, bool has1, uint64_t (&o)[2]) {
    if (vec) { const ulonglong2 t = *reinterpret_cast<const ulonglong2*>(p + i0); o[0] = t.x; o[1] = t.y; }
    else { o[0] = p[i0]; o[1] = has1 ? p[i0 + 1] : 0ull; }
}
__device__ __forceinline__ void st_pair(uint64_t* __restrict__ p, int64_t i0, bool vec, bool has1, const uint64_t (&v)[2]) {
    if (vec) *reinterpret_cast<ulonglong2*>(p + i0) = make_ulonglong2(v[0], v[1]);
    else { p[i0] = v[0]; if (has1) p[i0 + 1] = v[1]; }
}
// wrap count of two terms: (signed(u) + signed(v) - signed(u + v)) / 2^64 in {-1, 0, 1}
__device__ __forceinline__ uint64_t wrap2(uint64_t u, uint64_t v) {
    const __int128 s = (__int128)(int64_t)u + (__int128)(int64_t)v - (__int128)(int64_t)(u + v);
    return (uint64_t)(int64_t)(s >> 64);
}
// theta_r of pair j, exactly: (sum signed(r_q) - signed(sum r_q)) / 2^64 (the TTP's view)
__device__ __forceinline__ void theta_r_pair(const PhiloxRK& rk, uint64_t id, int P, uint64_t j, uint64_t (&t)[2]) {
    __int128 s[2] = {0, 0};
    uint64_t u[2] = {0, 0};
    for (int q = 0; q < P; ++q) {
        uint64_t r[2];
        philox_pair_rk(rk, stream_word(kTagR, (uint32_t)q, id), j, r[0], r[1]);
#pragma unroll
        for (int e = 0; e < 2; ++e) { s[e] += (__int128)(int64_t)r[e]; u[e] += r[e]; }
    }
#pragma unroll
    for (int e = 0; e < 2; ++e) t[e] = (uint64_t)(int64_t)((s[e] - (__int128)(int64_t)u[e]) >> 64);
}
// [theta_r]_q of pair j: q >= 1 -> G(THETA||q||id), q = 0 -> theta_r - sum_{q>=1} (TTP view)
__device__ __forceinline__ void theta_share_pair(const PhiloxRK& rk, uint64_t id, int P, int q, uint64_t j,
                                                 uint64_t (&t)[2]) {
    if (q > 0) { philox_pair_rk(rk, stream_word(kTagTheta, (uint32_t)q, id), j, t[0], t[1]); return; }
    theta_r_pair(rk, id, P, j, t);
    for (int s = 1; s < P; ++s) {
        uint64_t v[2];
        philox_pair_rk(rk, stream_word(kTagTheta, (uint32_t)s, id), j, v[0], v[1]);
        t[0] -= v[0]; t[1] -= v[1];
    }
}
__global__ void wrap_pair_kernel(const PhiloxRK rk, uint64_t id, int P, int lo, int hi, uint64_t* __restrict__ r,
                                 uint64_t* __restrict__ th, int64_t n) {
    const int64_t npairs = (n + 1) / 2;
    const bool vec = (n & 1) == 0 && aligned16(r) && aligned16(th);
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < npairs; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i0 = 2 * j;
        const bool has1 = i0 + 1 < n;
        for (int q = lo; q < hi; ++q) {
            uint64_t v[2], t[2];
            philox_pair_rk(rk, stream_word(kTagR, (uint32_t)q, id), (uint64_t)j, v[0], v[1]);
            theta_share_pair(rk, id, P, q, (uint64_t)j, t);
            st_pair(r + (int64_t)(q - lo) * n, i0, vec, has1, v);
            st_pair(th + (int64_t)(q - lo) * n, i0, vec, has1, t);
        }
    }
}
cudaError_t launch_wrap_pair(uint64_t key, uint64_t id, int P, int lo, int hi, uint64_t* r, uint64_t* th, int64_t n,
                             cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    wrap_pair_kernel<<<grid_for((n + 1) / 2), 256, 0, st>>>(philox_round_keys(key), id, P, lo, hi, r, th, n);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ a8 truncation, P <= 2
__global__ void trunc_local_kernel(uint64_t* __restrict__ x, int64_t n, int bits) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        x[i] = div_pow2_round(x[i], bits);
}
cudaError_t launch_trunc_local(uint64_t* x, int64_t n, int bits, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    trunc_local_kernel<<<grid_for(n), 256, 0, st>>>(x, n, bits);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ a9 truncation, P > 2, all parties
// Alg. 1 + correction, eta skipped, for
// every party of an element pair in one thread (the reveal of z is local).
// P is a template constant, so each party's r_q pair stays in registers
// between the two passes, and x_q too for P <= 4; above that the second pass
// re-reads x_q (an L1 hit: the block's 256 x P x 16 B were just loaded), which
// keeps the kernel under 128 registers (2 blocks per SM).  The wrap pair
// ([r], [theta_r]) is either regenerated from its Philox streams
// (PAIRS = false: wrap_id, the seeded TTP; one block per element pair and
// stream) or read from memory (PAIRS = true: materialised offline by
// mpc_ttp_wrap_pairs).
template <int P, bool PAIRS>
__global__ void __launch_bounds__(256, (P <= 8 ? 2 : 1)) trunc_alg1_all_kernel(uint64_t* __restrict__ x, int64_t n, int bits,
                                                            const PhiloxRK rk, uint64_t id, const uint64_t* __restrict__ rin,
                                                            const uint64_t* __restrict__ thin) {
    const int64_t npairs = (n + 1) / 2;
    const bool vec = (n & 1) == 0 && aligned16(x) && (!PAIRS || (aligned16(rin) && aligned16(thin)));
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < npairs; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i0 = 2 * j;
        const bool has1 = i0 + 1 < n;
        uint64_t xv[P][2], r[P][2];
        uint64_t zsum[2] = {0, 0}, rsum[2] = {0, 0};
        __int128 zs[2] = {0, 0}, rs[2] = {0, 0};
#pragma unroll
        for (int q = 0; q < P; ++q) {
            ld_pair(x + (int64_t)q * n, i0, vec, has1, xv[q]);
            if (PAIRS) ld_pair(rin + (int64_t)q * n, i0, vec, has1, r[q]);
            else philox_pair_rk(rk, stream_word(kTagR, (uint32_t)q, id), (uint64_t)j, r[q][0], r[q][1]);
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const uint64_t z = xv[q][e] + r[q][e];                  // z_q = x_q + r_q
                zsum[e] += z;
                zs[e] += (__int128)(int64_t)z;
                if (!PAIRS) { rsum[e] += r[q][e]; rs[e] += (__int128)(int64_t)r[q][e]; }
            }
        }
        uint64_t theta_z[2], theta_r[2] = {0, 0};
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            theta_z[e] = (uint64_t)(int64_t)((zs[e] - (__int128)(int64_t)zsum[e]) >> 64);      // wraps of z
            if (!PAIRS) theta_r[e] = (uint64_t)(int64_t)((rs[e] - (__int128)(int64_t)rsum[e]) >> 64);
        }
        uint64_t th_sum[2] = {0, 0};                                   // sum_{q>=1} [theta_r]_q (seeded TTP)
#pragma unroll
        for (int q = P - 1; q >= 0; --q) {
            uint64_t th[2];
            if (PAIRS) {
                ld_pair(thin + (int64_t)q * n, i0, vec, has1, th);
            } else if (q > 0) {
                philox_pair_rk(rk, stream_word(kTagTheta, (uint32_t)q, id), (uint64_t)j, th[0], th[1]);
                th_sum[0] += th[0];
                th_sum[1] += th[1];
            } else {
                th[0] = theta_r[0] - th_sum[0];
                th[1] = theta_r[1] - th_sum[1];
            }
            if (P > 4) ld_pair(x + (int64_t)q * n, i0, vec, has1, xv[q]);     // L1 hit (see above)
            uint64_t o[2];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const uint64_t beta = wrap2(xv[q][e], r[q][e]);
                const uint64_t theta_x = beta - th[e] + (q == 0 ? theta_z[e] : 0ull);
                o[e] = div_pow2_round(xv[q][e], bits) - theta_x * (1ull << (64 - bits));
            }
            st_pair(x + (int64_t)q * n, i0, vec, has1, o);
        }
    }
}
// The same computation for bits <= 32 (the fixed-point truncation, f = 16) with
// every wrap count in 32-bit arithmetic: theta_x * 2^(64 - bits) mod 2^64 depends
// only on theta_x mod 2^bits, so theta_x, beta, theta_z, theta_r and the
// [theta_r] shares are needed mod 2^32.  With m(v) = v >> 63 and C the carries of a
// running unsigned sum, the wrap count of sum_q v_q is C - sum_q m(v_q) + m(sum), and
// beta_q = carry(x_q + r_q) - m(x_q) - m(r_q) + m(z_q) — the exact integer identities
// the int128 form evaluates, at a third of its ALU instructions (the kernel is
// ALU-pipe bound: ncu, P = 8).  Pass 1 keeps beta_q and x_q per party; pass 2 needs
// no r_q.
__device__ __forceinline__ uint32_t add_carry(uint64_t a, uint64_t b, uint64_t& s) {
    uint32_t lo, hi, c;
    asm("add.cc.u32 %0, %3, %5;\n\taddc.cc.u32 %1, %4, %6;\n\taddc.u32 %2, 0, 0;"
        : "=r"(lo), "=r"(hi), "=r"(c)
        : "r"((uint32_t)a), "r"((uint32_t)(a >> 32)), "r"((uint32_t)b), "r"((uint32_t)(b >> 32)));
    s = ((uint64_t)hi << 32) | lo;
    return c;
}
__device__ __forceinline__ void acc_carry(uint64_t& s, uint64_t v, uint32_t& cnt) {
    uint32_t lo = (uint32_t)s, hi = (uint32_t)(s >> 32);
    asm("add.cc.u32 %0, %0, %3;\n\taddc.cc.u32 %1, %1, %4;\n\taddc.u32 %2, %2, 0;"
        : "+r"(lo), "+r"(hi), "+r"(cnt) : "r"((uint32_t)v), "r"((uint32_t)(v >> 32)));
    s = ((uint64_t)hi << 32) | lo;
}
__device__ __forceinline__ uint32_t msb(uint64_t v) { return (uint32_t)(v >> 63); }

__device__ __forceinline__ void cp_async16(void* smem, const void* g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;"
                 :: "r"((uint32_t)__cvta_generic_to_shared(smem)), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// PF (prefetch; n even, 16-byte aligned shares): the x pairs of a thread's NEXT grid-stride
// iteration are copied into shared memory (cp.async, 16 bytes per party) while it expands
// the Philox blocks of the current one, so every warp keeps P loads in flight through its
// ALU phase instead of alternating load -> compute -> store (dynamic shared memory:
// 2 buffers x P x blockDim pairs; each thread reads only the slots it filled).
template <int P, bool PAIRS, bool PF>
__global__ void __launch_bounds__(256, (P <= 8 ? 2 : 1)) trunc_alg1_all_w32_kernel(
        uint64_t* __restrict__ x, int64_t n, int bits, const PhiloxRK rk, uint64_t id, const uint64_t* __restrict__ rin,
        const uint64_t* __restrict__ thin) {
    extern __shared__ ulonglong2 pf_buf[];
    const int64_t npairs = (n + 1) / 2;
    const bool vec = (n & 1) == 0 && aligned16(x) && (!PAIRS || (aligned16(rin) && aligned16(thin)));
    const uint32_t hshift = 32 - bits;                                  // theta_x lands in the high word
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    auto prefetch = [&](int64_t jj, int buf) {
#pragma unroll
        for (int q = 0; q < P; ++q)
            cp_async16(&pf_buf[(buf * P + q) * blockDim.x + threadIdx.x], x + (int64_t)q * n + 2 * jj);
    };
    if (PF) {
        if (j < npairs) prefetch(j, 0);
        cp_async_commit();
    }
    for (int it = 0; j < npairs; j += stride, ++it) {
        if (PF) {
            if (j + stride < npairs) prefetch(j + stride, (it + 1) & 1);
            cp_async_commit();
            cp_async_wait1();                                            // this iteration's group has landed
        }
        const int64_t i0 = 2 * j;
        const bool has1 = i0 + 1 < n;
        uint32_t beta[P][2];
        uint64_t xv[P][2];
        uint64_t zsum[2] = {0, 0}, rsum[2] = {0, 0};
        uint32_t cz[2] = {0, 0}, cr[2] = {0, 0};                        // carries minus msb counts
        // every party's x pair is requested before any Philox block is expanded (the
        // loads' latency hides under the arithmetic; ncu: long-scoreboard stalls
        // dominated when each load was consumed right after its own block)
        uint64_t rv[PAIRS ? P : 1][2];                                  // the wrap pair's r_q (PAIRS)
#pragma unroll
        for (int q = 0; q < P; ++q) {
            if (PF) {
                const ulonglong2 t = pf_buf[((it & 1) * P + q) * blockDim.x + threadIdx.x];
                xv[q][0] = t.x; xv[q][1] = t.y;
            } else {
                ld_pair(x + (int64_t)q * n, i0, vec, has1, xv[q]);
            }
        }
        if (PAIRS) {
#pragma unroll
            for (int q = 0; q < P; ++q) ld_pair(rin + (int64_t)q * n, i0, vec, has1, rv[PAIRS ? q : 0]);
        }
#pragma unroll
        for (int q = 0; q < P; ++q) {
            uint64_t r[2];
            if (PAIRS) { r[0] = rv[PAIRS ? q : 0][0]; r[1] = rv[PAIRS ? q : 0][1]; }
            else philox_pair_rk(rk, stream_word(kTagR, (uint32_t)q, id), (uint64_t)j, r[0], r[1]);
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                uint64_t z;
                const uint32_t c = add_carry(xv[q][e], r[e], z);              // z_q = x_q + r_q
                beta[q][e] = c - msb(xv[q][e]) - msb(r[e]) + msb(z);
                acc_carry(zsum[e], z, cz[e]);
                cz[e] -= msb(z);
                if (!PAIRS) { acc_carry(rsum[e], r[e], cr[e]); cr[e] -= msb(r[e]); }
            }
        }
        uint32_t theta_z[2], theta_r[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            theta_z[e] = cz[e] + msb(zsum[e]);                                // wraps of z
            theta_r[e] = cr[e] + msb(rsum[e]);                                // wraps of r (seeded TTP)
        }
        uint32_t th_sum[2] = {0, 0};
        if (PAIRS) {                                                    // every [theta_r]_q requested up front
#pragma unroll
            for (int q = 0; q < P; ++q) ld_pair(thin + (int64_t)q * n, i0, vec, has1, rv[PAIRS ? q : 0]);
        }
#pragma unroll
        for (int q = P - 1; q >= 0; --q) {
            uint32_t th[2];
            if (PAIRS) {
                th[0] = (uint32_t)rv[PAIRS ? q : 0][0]; th[1] = (uint32_t)rv[PAIRS ? q : 0][1];
            } else if (q > 0) {
                uint64_t t[2];
                philox_pair_rk(rk, stream_word(kTagTheta, (uint32_t)q, id), (uint64_t)j, t[0], t[1]);
                th[0] = (uint32_t)t[0]; th[1] = (uint32_t)t[1];
                th_sum[0] += th[0]; th_sum[1] += th[1];
            } else {
                th[0] = theta_r[0] - th_sum[0];
                th[1] = theta_r[1] - th_sum[1];
            }
            uint64_t o[2];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const uint32_t theta_x = beta[q][e] - th[e] + (q == 0 ? theta_z[e] : 0u);
                o[e] = div_pow2_round(xv[q][e], bits) - ((uint64_t)(theta_x << hshift) << 32);
            }
            st_pair(x + (int64_t)q * n, i0, vec, has1, o);
        }
    }
}

template <int Q, bool PAIRS>
static cudaError_t launch_alg1_w32(uint64_t* x, int64_t n, int bits, const PhiloxRK& rk, uint64_t id,
                                   const uint64_t* r, const uint64_t* th, unsigned g, cudaStream_t st) {
    // prefetching variant when every pair is one aligned 16-byte load (MPC_ALG1_PREFETCH=0: A/B)
    static const bool pf_env = !getenv("MPC_ALG1_PREFETCH") || atoi(getenv("MPC_ALG1_PREFETCH")) != 0;
    auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
    const bool pf = pf_env && (n & 1) == 0 && al(x) && (!PAIRS || (al(r) && al(th)));
    if (!pf) {
        trunc_alg1_all_w32_kernel<Q, PAIRS, false><<<g, 256, 0, st>>>(x, n, bits, rk, id, r, th);
        return cudaGetLastError();
    }
    const int smem = 2 * Q * 256 * (int)sizeof(ulonglong2);
    static int attr_dev = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (attr_dev != dev) {
        const cudaError_t e = cudaFuncSetAttribute(trunc_alg1_all_w32_kernel<Q, PAIRS, true>,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        attr_dev = dev;
    }
    trunc_alg1_all_w32_kernel<Q, PAIRS, true><<<g, 256, smem, st>>>(x, n, bits, rk, id, r, th);
    return cudaGetLastError();
}

template <bool PAIRS>
static cudaError_t launch_alg1_all_t(uint64_t* x, int P, int64_t n, int bits, uint64_t key, uint64_t id,
                                     const uint64_t* r, const uint64_t* th, cudaStream_t st) {
    const unsigned g = grid_for((n + 1) / 2, 256);
    const PhiloxRK rk = philox_round_keys(key);
    const bool w32 = bits <= 32 && !getenv("MPC_ALG1_INT128");        // A/B switch for measurements
    switch (P) {
#define MPC_ALG1_CASE(Q) case Q:                                                                         \
        if (w32) return launch_alg1_w32<Q, PAIRS>(x, n, bits, rk, id, r, th, g, st);                      \
        trunc_alg1_all_kernel<Q, PAIRS><<<g, 256, 0, st>>>(x, n, bits, rk, id, r, th);                     \
        break;
        MPC_ALG1_CASE(3) MPC_ALG1_CASE(4) MPC_ALG1_CASE(5) MPC_ALG1_CASE(6) MPC_ALG1_CASE(7) MPC_ALG1_CASE(8)
        MPC_ALG1_CASE(9) MPC_ALG1_CASE(10) MPC_ALG1_CASE(11) MPC_ALG1_CASE(12) MPC_ALG1_CASE(13) MPC_ALG1_CASE(14)
        MPC_ALG1_CASE(15) MPC_ALG1_CASE(16)
#undef MPC_ALG1_CASE
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}
cudaError_t launch_trunc_alg1_all(uint64_t* x, int P, int64_t n, int bits, uint64_t key, uint64_t id,
                                  const uint64_t* r, const uint64_t* th, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    return r ? launch_alg1_all_t<true>(x, P, n, bits, key, id, r, th, st)
             : launch_alg1_all_t<false>(x, P, n, bits, key, id, nullptr, nullptr, st);
}

// ------------------------------------------------------------------ a9 truncation, P > 2, one party
// Phase A: z_p = x_p + r_p -> zbuf (u64, to be sum-allreduced) and the top
// nibble h_p = signed(z_p) >> 60 -> hbuf (int8, sum-allreduced; exact for
// P <= 16).  r_p from memory (rin) or from its Philox stream.
__global__ void trunc_alg1_a_kernel(const uint64_t* __restrict__ x, int64_t n, const PhiloxRK rk, uint64_t id, int party,
                                    const uint64_t* __restrict__ rin, uint64_t* __restrict__ zbuf,
                                    int8_t* __restrict__ hbuf) {
    const int64_t npairs = (n + 1) / 2;
    const bool vec = (n & 1) == 0 && aligned16(x) && aligned16(zbuf) && (!rin || aligned16(rin));
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < npairs; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i0 = 2 * j;
        const bool has1 = i0 + 1 < n;
        uint64_t xv[2], r[2], z[2];
        ld_pair(x, i0, vec, has1, xv);
        if (rin) ld_pair(rin, i0, vec, has1, r);
        else philox_pair_rk(rk, stream_word(kTagR, (uint32_t)party, id), (uint64_t)j, r[0], r[1]);
        z[0] = xv[0] + r[0];
        z[1] = xv[1] + r[1];
        st_pair(zbuf, i0, vec, has1, z);
        hbuf[i0] = (int8_t)((int64_t)z[0] >> 60);
        if (has1) hbuf[i0 + 1] = (int8_t)((int64_t)z[1] >> 60);
    }
}
// Phase B: with z = sum z_q and H = sum h_q: S = sum signed(z_q) = (H + kappa) 2^60
// + (z mod 2^60), kappa = ((z >> 60) - H) mod 16; theta_z = (S - signed(z)) / 2^64
// (party 0 only).  [theta_r]_p from memory (thin) or regenerated (seeded TTP: for
// party 0 that is the TTP's theta_r over all P r streams).
__global__ void trunc_alg1_b_kernel(uint64_t* __restrict__ x, int64_t n, int bits, const PhiloxRK rk, uint64_t id, int P,
                                    int party, const uint64_t* __restrict__ rin, const uint64_t* __restrict__ thin,
                                    const uint64_t* __restrict__ zsum, const int8_t* __restrict__ hsum) {
    const int64_t npairs = (n + 1) / 2;
    const bool vec = (n & 1) == 0 && aligned16(x) && (!rin || (aligned16(rin) && aligned16(thin))) &&
                     (party != 0 || aligned16(zsum));
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < npairs; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i0 = 2 * j;
        const bool has1 = i0 + 1 < n;
        uint64_t xv[2], r[2], th[2], theta_z[2] = {0, 0};
        ld_pair(x, i0, vec, has1, xv);
        if (rin) {
            ld_pair(rin, i0, vec, has1, r);
            ld_pair(thin, i0, vec, has1, th);
        } else {
            philox_pair_rk(rk, stream_word(kTagR, (uint32_t)party, id), (uint64_t)j, r[0], r[1]);
            theta_share_pair(rk, id, P, party, (uint64_t)j, th);
        }
        if (party == 0) {
            uint64_t zv[2];
            ld_pair(zsum, i0, vec, has1, zv);
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                if (e == 1 && !has1) break;
                const int64_t H = hsum[i0 + e];
                const int64_t kappa = (((int64_t)(zv[e] >> 60) - H) % 16 + 16) % 16;
                const __int128 S = (__int128)(H + kappa) * ((__int128)1 << 60) + (__int128)(zv[e] & ((1ull << 60) - 1));
                theta_z[e] = (uint64_t)(int64_t)((S - (__int128)(int64_t)zv[e]) >> 64);
            }
        }
        uint64_t o[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const uint64_t theta_x = wrap2(xv[e], r[e]) - th[e] + theta_z[e];
            o[e] = div_pow2_round(xv[e], bits) - theta_x * (1ull << (64 - bits));
        }
        st_pair(x, i0, vec, has1, o);
    }
}
cudaError_t launch_trunc_alg1_a(const uint64_t* x, int64_t n, uint64_t key, uint64_t id, int party, const uint64_t* r,
                                uint64_t* zbuf, int8_t* hbuf, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    trunc_alg1_a_kernel<<<grid_for((n + 1) / 2), 256, 0, st>>>(x, n, philox_round_keys(key), id, party, r, zbuf, hbuf);
    return cudaGetLastError();
}
cudaError_t launch_trunc_alg1_b(uint64_t* x, int64_t n, int bits, uint64_t key, uint64_t id, int P, int party,
                                const uint64_t* r, const uint64_t* th, const uint64_t* zsum, const int8_t* hsum,
                                cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    trunc_alg1_b_kernel<<<grid_for((n + 1) / 2), 256, 0, st>>>(x, n, bits, philox_round_keys(key), id, P, party, r, th,
                                                               zsum, hsum);
    return cudaGetLastError();
}

}  // namespace mpc

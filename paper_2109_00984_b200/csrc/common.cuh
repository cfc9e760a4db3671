// common.cuh — device-side building blocks of libmpc_ring.so (sm_100a only).
//
// Shares nothing with oracle/ (the CPU oracle is independent test
// infrastructure).  Citations: "P:n" = PAPER.md line n; "R#" = a reading
// listed in DESIGN.md.
#pragma once
#include <cstdint>
#include <cstdlib>
#include <utility>
#include <cuda_runtime.h>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ != 1000)
#error "libmpc_ring targets sm_100a only (compile with -gencode arch=compute_100a,code=sm_100a)"
#endif

namespace mpc {

// ---------------------------------------------------------------- PRG (R5)
// Philox4x32-10 (Random123).  G(key, stream)[i]: counter (lo(i/2), hi(i/2),
// lo(stream), hi(stream)), key (lo(key), hi(key)); element 2j = o1<<32|o0,
// element 2j+1 = o3<<32|o2.  stream = tag<<56 | party<<48 | id (48 bits).
enum : uint32_t { kTagPRZS = 1, kTagA = 2, kTagB = 3, kTagC = 4, kTagR = 5, kTagTheta = 6,
                  kTagKeyParty = 0xFF, kTagKeyTTP = 0xFE };

__host__ __device__ __forceinline__ uint64_t stream_word(uint32_t tag, uint32_t party, uint64_t id) {
    return ((uint64_t)(tag & 0xFFu) << 56) | ((uint64_t)(party & 0xFFu) << 48) | (id & 0xFFFFFFFFFFFFull);
}

__host__ __device__ __forceinline__ void philox_pair(uint64_t key, uint64_t stream, uint64_t j,
                                                     uint64_t& e0, uint64_t& e1) {
    uint32_t c0 = (uint32_t)j, c1 = (uint32_t)(j >> 32), c2 = (uint32_t)stream, c3 = (uint32_t)(stream >> 32);
    uint32_t k0 = (uint32_t)key, k1 = (uint32_t)(key >> 32);
#pragma unroll
    for (int r = 0; r < 10; ++r) {
#ifdef __CUDA_ARCH__
        uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
        uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
#else
        uint64_t p0 = (uint64_t)0xD2511F53u * c0, p1 = (uint64_t)0xCD9E8D57u * c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0, hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
#endif
        uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
        k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
    }
    e0 = ((uint64_t)c1 << 32) | c0;
    e1 = ((uint64_t)c3 << 32) | c2;
}

// The same generator with its 10 round keys precomputed on the host and passed by
// value as a kernel parameter: the rounds then read them straight from the
// constant bank (LOP3 operands), so a Philox block costs its 20 multiplies and 20
// three-input XORs and no key-schedule adds — for kernels that expand many
// streams under one key (Alg. 1, the wrap pairs, sharing).
struct PhiloxRK { uint32_t k[20]; };
inline PhiloxRK philox_round_keys(uint64_t key) {
    PhiloxRK rk;
    uint32_t k0 = (uint32_t)key, k1 = (uint32_t)(key >> 32);
    for (int r = 0; r < 10; ++r) { rk.k[2 * r] = k0; rk.k[2 * r + 1] = k1; k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    return rk;
}
__device__ __forceinline__ void philox_pair_rk(const PhiloxRK& rk, uint64_t stream, uint64_t j, uint64_t& e0,
                                               uint64_t& e1) {
    uint32_t c0 = (uint32_t)j, c1 = (uint32_t)(j >> 32), c2 = (uint32_t)stream, c3 = (uint32_t)(stream >> 32);
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
        const uint32_t n0 = hi1 ^ c1 ^ rk.k[2 * r], n2 = hi0 ^ c3 ^ rk.k[2 * r + 1];
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    }
    e0 = ((uint64_t)c1 << 32) | c0;
    e1 = ((uint64_t)c3 << 32) | c2;
}

__host__ __device__ __forceinline__ uint64_t philox_at(uint64_t key, uint64_t stream, uint64_t i) {
    uint64_t e0, e1;
    philox_pair(key, stream, i >> 1, e0, e1);
    return (i & 1) ? e1 : e0;
}

// ------------------------------------------------------- limb-plane layout
// A u64 operand with R rows (M for left operands, N for right operands) and
// reduction length K is stored as 8 u8 planes (plane l = byte l of every
// element), K-major, blocked so that one (row block, 32-K block) of all 8
// planes is 8 contiguous blocks, each already in the UMMA canonical K-major
// SWIZZLE_NONE layout: [row/8][k/16][row%8][k%16] (core matrices of 8 rows x
// 16 B; LBO = 128 B between the two K halves, SBO = 256 B between 8-row
// groups).  The row block is what one CTA of a tcgen05 cta_group::2 pair
// loads per 32-K block:
//   left  operands (Layout::Left):  128-row blocks (4 KiB per plane),
//   right operands (Layout::Right):  64-row blocks (2 KiB per plane).
// Rows are padded to one cluster tile (256 left rows, 128 right rows) and K
// to 32; the K padding is written as zeros, the row padding is never read
// into a stored output.
constexpr int kKBlock = 32;
enum class Layout : int { Left = 0, Right = 1, Small = 2 };
template <Layout L> struct PlaneGeom;
template <> struct PlaneGeom<Layout::Left>  { static constexpr int kRows = 128, kBlock = 128 * 32, kPad = 256; };
template <> struct PlaneGeom<Layout::Right> { static constexpr int kRows = 64, kBlock = 64 * 32, kPad = 128; };
// both operands of the stacked-plane GEMM for <= 32 output rows (ring_gemm_small.cu):
// 32-row blocks, so one (row block, 32-K block) of all 8 planes is 8 KiB contiguous
template <> struct PlaneGeom<Layout::Small> { static constexpr int kRows = 32, kBlock = 32 * 32, kPad = 32; };

__host__ __device__ __forceinline__ int64_t num_kb(int64_t k) { return (k + kKBlock - 1) / kKBlock; }
template <Layout L>
__host__ __device__ __forceinline__ int64_t pad_rows(int64_t r) {
    return (r + PlaneGeom<L>::kPad - 1) / PlaneGeom<L>::kPad * PlaneGeom<L>::kPad;
}
template <Layout L>
__host__ __device__ __forceinline__ int64_t planes_bytes(int64_t rows, int64_t k) {
    return pad_rows<L>(rows) * num_kb(k) * kKBlock * 8;
}
template <Layout L>
__host__ __device__ __forceinline__ int64_t plane_offset(int64_t row, int64_t k, int limb, int64_t KB) {
    constexpr int R = PlaneGeom<L>::kRows;
    const int64_t rb = row / R, rr = row % R, kb = k >> 5, kk = k & 31;
    return ((rb * KB + kb) * 8 + limb) * (int64_t)PlaneGeom<L>::kBlock
         + (rr >> 3) * 256 + (kk >> 4) * 128 + (rr & 7) * 16 + (kk & 15);
}

// 4x4 byte transpose: in a,b,c,d (byte 0 = LSB) -> o[l] = [a_l b_l c_l d_l]
__device__ __forceinline__ void transpose4x4(uint32_t a, uint32_t b, uint32_t c, uint32_t d, uint32_t o[4]) {
    uint32_t t0 = __byte_perm(a, b, 0x5140), t1 = __byte_perm(a, b, 0x7362);
    uint32_t t2 = __byte_perm(c, d, 0x5140), t3 = __byte_perm(c, d, 0x7362);
    o[0] = __byte_perm(t0, t2, 0x5410); o[1] = __byte_perm(t0, t2, 0x7632);
    o[2] = __byte_perm(t1, t3, 0x5410); o[3] = __byte_perm(t1, t3, 0x7632);
}

// 16 consecutive-k elements of one row -> 8 limb vectors of 16 bytes, stored
// at their plane positions.  k0 must be a multiple of 16.
template <Layout L>
__device__ __forceinline__ void store_limbs16(uint8_t* planes, int64_t row, int64_t k0, int64_t KB,
                                              const uint64_t v[16]) {
    uint32_t w[8][4];  // w[limb][word]
#pragma unroll
    for (int g = 0; g < 4; ++g) {
        uint32_t lo[4], hi[4];
        transpose4x4((uint32_t)v[4 * g], (uint32_t)v[4 * g + 1], (uint32_t)v[4 * g + 2], (uint32_t)v[4 * g + 3], lo);
        transpose4x4((uint32_t)(v[4 * g] >> 32), (uint32_t)(v[4 * g + 1] >> 32), (uint32_t)(v[4 * g + 2] >> 32),
                     (uint32_t)(v[4 * g + 3] >> 32), hi);
#pragma unroll
        for (int l = 0; l < 4; ++l) { w[l][g] = lo[l]; w[4 + l][g] = hi[l]; }
    }
    int64_t base = plane_offset<L>(row, k0, 0, KB);
#pragma unroll
    for (int l = 0; l < 8; ++l)
        *reinterpret_cast<uint4*>(planes + base + (int64_t)l * PlaneGeom<L>::kBlock) =
            make_uint4(w[l][0], w[l][1], w[l][2], w[l][3]);
}

// 8 consecutive-k elements of one row -> 8 limb vectors of 8 bytes (k0 % 8 == 0).
template <Layout L>
__device__ __forceinline__ void store_limbs8(uint8_t* planes, int64_t row, int64_t k0, int64_t KB,
                                             const uint64_t v[8]) {
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
    int64_t base = plane_offset<L>(row, k0, 0, KB);
#pragma unroll
    for (int l = 0; l < 8; ++l)
        *reinterpret_cast<uint2*>(planes + base + (int64_t)l * PlaneGeom<L>::kBlock) = make_uint2(w[l][0], w[l][1]);
}

// ------------------------------------------------------------ launches
// Launch as a programmatic dependent of the previous kernel in the stream
// (PDL): its CTAs may start while the previous kernel drains; the kernel must
// execute `griddepcontrol.wait` before reading anything that kernel wrote.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    static const bool off = getenv("MPC_NO_PDL") != nullptr;     // A/B switch for measurements
    cfg.attrs = attr;
    cfg.numAttrs = off ? 0 : 1;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// ------------------------------------------------------------ signed helpers
// floor(signed(v) / 2^bits) + bit_{bits-1}(v): per-share round-half-up division (R10)
__host__ __device__ __forceinline__ uint64_t div_pow2_round(uint64_t v, int bits) {
    return (uint64_t)((int64_t)v >> bits) + ((v >> (bits - 1)) & 1ull);
}

}  // namespace mpc

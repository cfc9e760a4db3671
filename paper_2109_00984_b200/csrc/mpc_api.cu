// mpc_api.cu — the C-ABI of include/mpc_ring.h: host orchestration of the
// protocol steps (argument checks, workspace carving, stream ordering, NCCL
// reveals, round/byte accounting, profiling hooks).  All arithmetic runs in
// the kernels of elementwise.cu and ring_gemm.cu.
#include <cuda_runtime.h>
#include <nccl.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <algorithm>
#include <vector>

#include "../../include/mpc_ring.h"
#include "common.cuh"
#include "beaver_elementwise.h"
#include "conv.h"
#include "elementwise.h"
#include "relu.h"
#include "ring_gemm.h"
#include "transport.h"

using namespace mpc;

struct ProfEvent { cudaEvent_t a, b; int cls; };

struct mpc_ctx_s {
    int P = 1, rank = 0, device = 0, frac = 16;
    bool all = false;                    // all parties on this device
    uint64_t master = 0;
    KeySet kp{};
    uint64_t kttp = 0;
    bool has_ttp = true;                 // holds k_ttp (mpc_create; mpc_create_with_keys only if given)
    cudaStream_t stream = nullptr;
    ncclComm_t comm = nullptr;              // maxCTAs = kCommSms: reveals overlapped with the GEMM (comm stream)
    ncclComm_t comm_fast = nullptr;         // no CTA cap: reveals nothing overlaps (context stream; Alg. 1's
                                            // z / top-nibble reveals, output reveals, ReLU rounds)
    LocalGroup* lg = nullptr;               // in-process transport (mpc_create_local), instead of NCCL
    uint64_t* xbuf = nullptr;               // NCCL XOR reveal: all-gathered binary shares
    size_t xbuf_bytes = 0;
    bool check_collectives = false;         // MPC_CHECK_COLLECTIVES=1: verify the collective contract (NCCL)
    uint64_t coll_seq = 0;
    uint64_t* check_buf = nullptr;          // 2 words
    cudaStream_t comm_stream = nullptr;     // reveals of the overlapped Beaver schedule
    cudaEvent_t ev_mask = nullptr, ev_delta = nullptr, ev_eps = nullptr;
    cudaEvent_t ev_chunk[8] = {};           // eps row chunks of the overlapped schedule (created on first use)
    int reveal_chunks = 0;                  // mpc_set_reveal_chunks (0: default policy)
    bool broken = false;
    std::string err;
    uint64_t rounds = 0, bytes = 0, launches = 0;
    bool prof = false;
    std::vector<ProfEvent> pending;
    std::vector<cudaEvent_t> pool;
    double prof_ms[6] = {0, 0, 0, 0, 0, 0};
    uint64_t prof_n[6] = {0, 0, 0, 0, 0, 0};
    int* d_err = nullptr;
    void* scratch = nullptr;
    size_t scratch_bytes = 0;
    cudaStream_t scratch_stream = nullptr;  // last stream that used the scratch
    cudaEvent_t scratch_ev = nullptr;
    void* ows = nullptr;                    // the context's own workspace (entry points called with
    size_t ows_bytes = 0;                   // workspace NULL and workspace_bytes 0)
    cudaStream_t ows_stream = nullptr;
    cudaEvent_t ows_ev = nullptr;
};

namespace {

constexpr int kClsGemm = 0, kClsSplit = 1, kClsTrunc = 2, kClsPrg = 3, kClsCodec = 4, kClsComm = 5;

mpc_status fail(mpc_ctx c, mpc_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    if (c) c->err = buf;
    return s;
}

cudaEvent_t take_event(mpc_ctx c) {
    if (!c->pool.empty()) { cudaEvent_t e = c->pool.back(); c->pool.pop_back(); return e; }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

// Run one launch of class `cls`; brackets it with events when profiling.
template <class F>
mpc_status run(mpc_ctx c, int cls, const char* what, F&& f) {
    ProfEvent ev{nullptr, nullptr, cls};
    if (c->prof) { ev.a = take_event(c); ev.b = take_event(c); cudaEventRecord(ev.a, c->stream); }
    cudaError_t e = f();
    if (c->prof) { cudaEventRecord(ev.b, c->stream); c->pending.push_back(ev); }
    if (cls != kClsComm) c->launches++;
    if (e != cudaSuccess) return fail(c, MPC_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
    return MPC_OK;
}

inline bool has_comm(mpc_ctx c) { return c->comm != nullptr || c->lg != nullptr; }
// A collective on the comm stream overlaps a GEMM: the CTA-capped communicator
// leaves it SMs.  Anything else (on the context stream, nothing beside it) gets all
// the CTAs NCCL wants.  Every party issues its collectives in the same program
// order, and the two communicators' operations never overlap in time (the comm
// stream's reveals complete before the compute stream's next collective).
inline ncclComm_t pick_comm(mpc_ctx c, cudaStream_t st) {
    return (st == c->comm_stream || !c->comm_fast) ? c->comm : c->comm_fast;
}
void abort_comms(mpc_ctx c) {
    if (c->comm_fast) ncclCommAbort(c->comm_fast);
    if (c->comm) ncclCommAbort(c->comm);
    c->comm_fast = nullptr;
    c->comm = nullptr;
}

// One reveal collective of this party on `st` (default: the context stream):
// recv = op over the parties' send buffers (transport.h).  Any failure leaves
// the context broken (MPC_ERR_STATE afterwards), as the collective contract
// can no longer be kept.
mpc_status comm_allreduce(mpc_ctx c, const void* send, void* recv, size_t count, RedOp op, const char* what,
                          cudaStream_t st = nullptr) {
    if (!st) st = c->stream;
    if (c->P == 1 && !has_comm(c)) {            // one party: the reveal is the share itself
        if (send == recv || count == 0) return MPC_OK;
        const size_t bytes = count * (op == RedOp::SumI8 ? 1 : 8);
        cudaError_t e = cudaMemcpyAsync(recv, send, bytes, cudaMemcpyDeviceToDevice, st);
        return e == cudaSuccess ? MPC_OK : fail(c, MPC_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
    }
    if (!has_comm(c)) return fail(c, MPC_ERR_STATE, "%s: context has no communicator (created without nccl_id)", what);
    ProfEvent ev{nullptr, nullptr, kClsComm};
    if (c->prof) { ev.a = take_event(c); ev.b = take_event(c); cudaEventRecord(ev.a, st); }
    if (c->lg) {
        const int r = local_group_allreduce(c->lg, c->rank, send, recv, count, op, st);
        if (c->prof) { cudaEventRecord(ev.b, st); c->pending.push_back(ev); }
        if (r != 0) {
            c->broken = true;
            static const char* why[] = {"", "parties called different collectives (count / op mismatch)",
                                        "timed out waiting for the other parties", "CUDA error", "group broken"};
            return fail(c, r == 1 ? MPC_ERR_SHAPE : MPC_ERR_STATE, "%s: local group: %s", what, why[r < 5 ? r : 4]);
        }
        return MPC_OK;
    }
    ncclResult_t r = ncclSuccess;
    if (c->check_collectives) {
        // collective contract: every party enters the same collective with the same size.
        // Word = (sequence number, op, count) folded into a u64; min == max across parties iff all agree.
        const uint64_t word = (c->coll_seq++ << 40) ^ ((uint64_t)op << 36) ^ (uint64_t)count;
        uint64_t h[2] = {word, ~word};
        cudaMemcpyAsync(c->check_buf, h, sizeof(h), cudaMemcpyHostToDevice, st);
        r = ncclAllReduce(c->check_buf, c->check_buf, 1, ncclUint64, ncclMin, c->comm, st);     // min(word)
        if (r == ncclSuccess)
            r = ncclAllReduce(c->check_buf + 1, c->check_buf + 1, 1, ncclUint64, ncclMin, c->comm, st);  // min(~word) = ~max
        cudaMemcpyAsync(h, c->check_buf, sizeof(h), cudaMemcpyDeviceToHost, st);
        if (r == ncclSuccess && cudaStreamSynchronize(st) == cudaSuccess && h[0] != ~h[1]) {
            c->broken = true;
            return fail(c, MPC_ERR_SHAPE, "%s: parties entered different collectives (collective contract broken)", what);
        }
    }
    if (r != ncclSuccess) {
    } else if (count == 0) {
    } else if (op == RedOp::XorU64) {
        // NCCL has no XOR reduction: all-gather the P binary shares, XOR them locally
        const size_t need = 8 * count * (size_t)c->P;
        if (c->xbuf_bytes < need) {
            cudaStreamSynchronize(st);
            if (c->xbuf) cudaFree(c->xbuf);
            c->xbuf = nullptr; c->xbuf_bytes = 0;
            if (cudaMalloc(&c->xbuf, need) != cudaSuccess) return fail(c, MPC_ERR_CUDA, "%s: xor buffer alloc", what);
            c->xbuf_bytes = need;
        }
        r = ncclAllGather(send, c->xbuf, count, ncclUint64, pick_comm(c, st), st);
        if (r == ncclSuccess) {
            cudaError_t e = launch_xor_gathered(c->xbuf, c->P, (int64_t)count, static_cast<uint64_t*>(recv), st);
            c->launches++;
            if (e != cudaSuccess) return fail(c, MPC_ERR_CUDA, "%s: xor: %s", what, cudaGetErrorString(e));
        }
    } else {
        r = ncclAllReduce(send, recv, count, op == RedOp::SumI8 ? ncclInt8 : ncclUint64, ncclSum, pick_comm(c, st), st);
    }
    if (c->prof) { cudaEventRecord(ev.b, st); c->pending.push_back(ev); }
    if (r != ncclSuccess) {
        c->broken = true;
        abort_comms(c);
        return fail(c, MPC_ERR_NCCL, "%s: %s", what, ncclGetErrorString(r));
    }
    return MPC_OK;
}

#define CHECK(call)                                   \
    do {                                              \
        mpc_status _s = (call);                       \
        if (_s != MPC_OK) return _s;                  \
    } while (0)

mpc_status enter(mpc_ctx c) {
    if (!c) return MPC_ERR_ARG;
    if (c->broken) return fail(c, MPC_ERR_STATE, "context unusable after a failed collective");
    c->err.clear();
    cudaError_t e = cudaSetDevice(c->device);
    if (e != cudaSuccess) return fail(c, MPC_ERR_CUDA, "cudaSetDevice: %s", cudaGetErrorString(e));
    return MPC_OK;
}

// TTP material (triples, wrap pairs, the ReLU path's binary triples) needs k_ttp
// (a context from mpc_create_with_keys without it must be handed that material)
mpc_status need_ttp(mpc_ctx c, const char* what) {
    return c->has_ttp ? MPC_OK : fail(c, MPC_ERR_STATE, "%s: context holds no TTP key (mpc_create_with_keys)", what);
}

constexpr int kCommSms = 16;     // SMs (NCCL CTAs) reserved for a reveal overlapped with the GEMM
constexpr int kOverlapClusters = (148 - kCommSms) / 2;   // GEMM clusters while a reveal is in flight

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }
// limb-plane buffer sizes of left (M x K) and right (N x K) ring-GEMM operands
inline int64_t lp(int64_t rows, int64_t k) { return planes_bytes<Layout::Left>(rows, k); }
inline int64_t rp(int64_t rows, int64_t k) { return planes_bytes<Layout::Right>(rows, k); }

struct Carve {
    uint8_t* base; size_t off = 0;
    explicit Carve(void* b) : base(static_cast<uint8_t*>(b)) {}
    uint8_t* take(size_t n) { uint8_t* p = base ? base + off : nullptr; off += align256(n); return p; }
};

// GEMM orientation and kernel of a Beaver step.  The ring GEMM tiles its output
// in 256 x 128 blocks, or — for at most 32 rows — in stacked-plane 32 x 32 blocks
// (ring_gemm_small.cu, planes in Layout::Small).  It can also compute
// z^T = delta^T a_p^T + b'_p^T eps^T (x-side planes in the right-operand layout,
// y-side planes in the left one, transposed store).  Of the (orientation,
// kernel) options the tensor-time model (ring_gemm_model_cycles) rates
// cheapest is used: e.g. M = 49, N = 512 runs transposed (256 x 512 -> 512 x 128
// padded tiles), M = 32 or N <= 32 on the stacked-plane kernel.  Bit-identical
// either way (the same ring sums).  MPC_NO_SWAP=1 disables the transposition,
// MPC_GEMM_SMALL=0/1 disables / forces (where possible) the stacked kernel.
struct GemmChoice { bool swap, small; };
GemmChoice choose_gemm(int parties, int64_t M, int64_t N, int64_t K, bool allow_swap, bool allow_small,
                       bool conv_out = false) {
    static const bool no_swap = getenv("MPC_NO_SWAP") != nullptr;
    static const int small_env = getenv("MPC_GEMM_SMALL") ? atoi(getenv("MPC_GEMM_SMALL")) : -1;
    allow_swap = allow_swap && !no_swap;
    allow_small = allow_small && small_env != 0;
    const int tkb = (int)(2 * num_kb(K));
    GemmChoice best{false, false};
    if (M == 0 || N == 0) return best;
    double cost = ring_gemm_model_cycles(parties, M, N, tkb, 74, false);
    // The stacked-plane kernel's per-launch overhead is lower (one CTA per work
    // item, a 32 x 32 epilogue): measured faster than the 2-CTA kernel for every
    // M <= 32 shape tried (scripts/gemm_kernel_compare.py) even where the
    // tensor-time model rates it up to ~1.2x slower, so it is preferred within 1.3x.
    // The transposed 2-CTA GEMM is taken only when the model rates it more than twice as cheap:
    // measured in graph replay, the small-M layers where the model sees exactly half the MMA
    // time run slower transposed (ResNet 49 x 4608 x 512: 65.7 vs 61.9 us per layer; alone,
    // without PDL, its GEMM is the faster one — DESIGN §8d); ResNet-50 chain 1.934 -> 1.876 ms,
    // ResNet-18 0.879 -> 0.849 ms with the factor; Wav2Letter 51 x 8000 x 2000 is the one shape
    // that lost: 348 -> 374 us, chain 0.688 -> 0.703.
    // MPC_SWAP_GAIN overrides the factor (1.0: the plain model, 0.5 the default).
    static const double swap_gain = getenv("MPC_SWAP_GAIN") ? atof(getenv("MPC_SWAP_GAIN")) : 0.5;
    auto consider = [&](bool sw, bool sm) {
        const int64_t gm = sw ? N : M, gn = sw ? M : N;
        if (sm && gm > kSmallMaxRows) return;
        // a convolution of one image keeps the plain model: its transposed output is already NCHW,
        // the other orientation stores through the strided NCHW epilogue (ResNet-50 convs 2.41 ->
        // 2.54 ms, Wav2Letter b1 0.84 -> 1.05 ms without transposition)
        // long GEMMs (> 200k modelled cycles, ~0.1 ms) keep the plain model: there the MMA time
        // dominates and the transposition pays as modelled (Wav2Letter 51 x 8000 x 2000: 348 vs
        // 374 us transposed / not)
        const double gain = (conv_out || cost > 200000.0) ? 1.0 : swap_gain;
        const double t = ring_gemm_model_cycles(parties, gm, gn, tkb, 74, sm) / (sm ? 1.3 : (sw ? gain : 1.0));
        if (t < cost - 1e-9) { cost = t; best = GemmChoice{sw, sm}; }
    };
    if (allow_swap) consider(true, false);
    if (allow_small) consider(false, true);
    if (allow_small && allow_swap) consider(true, true);
    if (small_env == 1 && allow_small && !best.small) {
        if (M <= kSmallMaxRows && (M <= N || !allow_swap)) best = GemmChoice{false, true};
        else if (allow_swap && N <= kSmallMaxRows) best = GemmChoice{true, true};
        else if (M <= kSmallMaxRows) best = GemmChoice{false, true};
    }
    return best;
}

// workspace of a plain one-party ring GEMM C = A @ B (the TTP's c = a @ b, mpc_ring_matmul):
// limb planes of A and B in the layout of the kernel choose_gemm picks (no transposition), partials
struct PlainGemmWs { uint8_t *a_pl, *b_pl; uint64_t* partials; bool small; size_t total; };
PlainGemmWs plain_gemm_ws(int64_t M, int64_t K, int64_t N, void* ws = nullptr) {
    PlainGemmWs w{};
    w.small = choose_gemm(1, M, N, (K + 1) / 2, false, true).small;     // model of one K-long segment
    Carve cv(ws);
    w.a_pl = cv.take(w.small ? planes_bytes<Layout::Small>(M, K) : lp(M, K));
    w.b_pl = cv.take(w.small ? planes_bytes<Layout::Small>(N, K) : rp(N, K));
    const size_t pb = ring_gemm_partials_bytes(1, M, N, (int)num_kb(K), 0, w.small);
    w.partials = reinterpret_cast<uint64_t*>(pb ? cv.take(pb) : nullptr);
    w.total = cv.off;
    return w;
}

// workspace layout of beaver_matmul (see mpc_workspace_bytes)
struct BeaverWs {
    uint8_t *eps_pl, *delta_pl, *a_pl, *b_pl;
    int64_t a_stride, b_stride;   // bytes between parties' a_p / b'_p planes
    bool swap;                    // transposed ring GEMM (choose_gemm)
    bool small;                   // stacked-plane GEMM, planes in Layout::Small (choose_gemm)
    bool fused;                   // the fused 2-party small-output kernel (no planes; use_fused_small)
    uint64_t* ed;        // one-party mode: [e | d] reveal buffer
    uint64_t* zbuf;      // one-party, P > 2, truncation: z reveal
    int8_t* hbuf;        // one-party, P > 2, truncation: top nibbles
    uint64_t* partials;  // ring GEMM split-K slabs (small shapes only)
    int64_t batch;       // independent matmuls (mpc_beaver_matmul_batched; 1 otherwise)
    int64_t xs, ys;      // bytes of one matrix's x-side / y-side planes (the batch strides)
    size_t total;
};

// Row chunks of the eps reveal in the overlapped schedule: eps is
// M x K row-major, so a chunk of rows is contiguous in the reveal buffer, its
// limb planes are a contiguous run of 128-row blocks and its GEMM output rows a
// contiguous run of z.  Chunks are whole 256-row GEMM tiles with at least 1024
// rows (enough tiles per chunk GEMM to fill the SMs the reveal leaves); not for
// the transposed / stacked-plane GEMMs (small M: the eps reveal is small too).
// mpc_set_reveal_chunks / MPC_REVEAL_CHUNKS=c force c chunks where the shape allows.
constexpr int kMaxRevealChunks = 8;
int reveal_chunks(mpc_ctx ctx, const BeaverWs& w, int64_t M) {
    if (w.swap || w.small || w.batch > 1) return 1;
    static const int env = getenv("MPC_REVEAL_CHUNKS") ? atoi(getenv("MPC_REVEAL_CHUNKS")) : 0;
    const int64_t tiles = (M + 255) / 256;
    int c = ctx->reveal_chunks > 0 ? ctx->reveal_chunks : env > 0 ? env : (int)std::min<int64_t>(4, M / 1024);
    c = (int)std::max<int64_t>(1, std::min<int64_t>({(int64_t)c, (int64_t)kMaxRevealChunks, tiles}));
    return c;
}
// rows [m0, m1) of chunk i of c: whole 256-row tiles, spread evenly
inline void chunk_rows(int64_t M, int i, int c, int64_t& m0, int64_t& m1) {
    const int64_t tiles = (M + 255) / 256;
    m0 = std::min<int64_t>(M, tiles * i / c * 256);
    m1 = std::min<int64_t>(M, tiles * (i + 1) / c * 256);
}

// ed_elems: size of the one-party [e | d] reveal buffer (default M*K + K*N; a
// convolution reveals at the input / weight shapes instead).  allow_swap: the
// transposed GEMM is possible for this output layout.
// The fused small-output kernel (ring_gemm_fused.cu) serves mpc_beaver_matmul when both
// parties of a 2-party context are on this GPU, M, N <= 32 and K is long enough for its
// split-K grid (>= 64 32-K blocks); MPC_FUSED_SMALL=0 keeps the planes-based path.
bool use_fused_small(mpc_ctx c, int64_t M, int64_t K, int64_t N) {
    static const int env = getenv("MPC_FUSED_SMALL") ? atoi(getenv("MPC_FUSED_SMALL")) : 1;
    return env != 0 && c->all && c->P == 2 && M >= 1 && M <= 32 && N >= 1 && N <= 32 && num_kb(K) >= 64;
}

BeaverWs carve_beaver(mpc_ctx c, void* ws, int64_t M, int64_t K, int64_t N, int64_t ed_elems = -1,
                      bool allow_swap = true, bool allow_small = true, int64_t batch = 1, bool allow_fused = false) {
    const int Pl = c->all ? c->P : 1;
    Carve cv(ws);
    BeaverWs w{};
    w.batch = batch < 1 ? 1 : batch;
    if (allow_fused && w.batch == 1 && use_fused_small(c, M, K, N)) {
        w.fused = true;
        const size_t pb = fused_small_partials_bytes(M, K, N);
        w.partials = reinterpret_cast<uint64_t*>(pb ? cv.take(pb) : nullptr);
        w.total = cv.off;
        return w;
    }
    const int inst = (int)(Pl * w.batch);                     // GEMM instances
    const GemmChoice gc = choose_gemm(inst, M, N, K, allow_swap, allow_small, ed_elems >= 0);
    w.swap = gc.swap;
    w.small = gc.small;
    if (ed_elems < 0) ed_elems = M * K + K * N;
    const int64_t xs = w.small ? planes_bytes<Layout::Small>(M, K) : (w.swap ? rp(M, K) : lp(M, K));   // eps, a_p
    const int64_t ys = w.small ? planes_bytes<Layout::Small>(N, K) : (w.swap ? lp(N, K) : rp(N, K));   // delta, b'_p
    const int64_t gM = w.swap ? N : M, gN = w.swap ? M : N;   // the GEMM's own output sizes
    const int64_t B = w.batch;
    w.xs = xs;
    w.ys = ys;
    w.a_stride = B * xs;                                      // party strides; batch stride xs / ys
    w.b_stride = B * ys;
    w.eps_pl = cv.take(B * xs);
    w.delta_pl = cv.take(B * ys);
    w.a_pl = cv.take((size_t)Pl * B * xs);
    w.b_pl = cv.take((size_t)Pl * B * ys);
    w.ed = reinterpret_cast<uint64_t*>(c->all ? nullptr : cv.take(8 * (size_t)(B * ed_elems)));
    const bool alg1_one = !c->all && c->P > 2;
    w.zbuf = reinterpret_cast<uint64_t*>(alg1_one ? cv.take(8 * (size_t)(B * M * N)) : nullptr);
    w.hbuf = reinterpret_cast<int8_t*>(alg1_one ? cv.take((size_t)(B * M * N)) : nullptr);
    size_t pb = ring_gemm_partials_bytes(inst, gM, gN, 2 * (int)num_kb(K), 0, w.small);
    if (!c->all) {   // the overlapped schedule runs half-K GEMMs: phase 1 per eps row chunk on fewer SMs
        pb = std::max({pb, ring_gemm_partials_bytes(1, gM, gN, (int)num_kb(K), kOverlapClusters, w.small),
                       ring_gemm_partials_bytes(1, gM, gN, (int)num_kb(K), 0, w.small)});
        const int nch = reveal_chunks(c, w, M);
        for (int i = 0; i < nch && nch > 1; ++i) {
            int64_t m0, m1;
            chunk_rows(M, i, nch, m0, m1);
            pb = std::max(pb, ring_gemm_partials_bytes(1, m1 - m0, N, (int)num_kb(K), kOverlapClusters, false));
        }
    }
    w.partials = reinterpret_cast<uint64_t*>(pb ? cv.take(pb) : nullptr);
    w.total = cv.off;
    return w;
}

// GEMM segment (x-side planes X, y-side planes Y): X @ Y^T normally, Y @ X^T when swapped.
// plane-layout code of the split kernels (LeftSplitArgs / RightSplitArgs::swap)
inline int lay(const BeaverWs& w) { return w.small ? 2 : (w.swap ? 1 : 0); }
RingGemmSegment seg_of(const BeaverWs& w, const uint8_t* X, int64_t xstride, const uint8_t* Y, int64_t ystride,
                       int kb) {
    return w.swap ? RingGemmSegment{Y, X, kb, ystride, xstride, w.ys, w.xs}
                  : RingGemmSegment{X, Y, kb, xstride, ystride, w.xs, w.ys};
}
void set_out(RingGemmParams& p, const BeaverWs& w, int64_t M, int64_t N) {
    p.M = w.swap ? N : M;
    p.N = w.swap ? M : N;
    p.transpose_out = w.swap ? 1 : 0;
    p.small = w.small ? 1 : 0;
    p.batch = (int)w.batch;
    p.batch_stride_c = p.batch_stride_z = M * N;
}

mpc_status beaver_local(mpc_ctx c, const BeaverWs& w, const uint64_t* ed, const uint64_t* a, const uint64_t* b,
                        const uint64_t* cc, uint64_t* z, int64_t M, int64_t K, int64_t N, int truncate);
mpc_status gemm_run(mpc_ctx c, RingGemmParams& p, int parties);
mpc_status beaver_gemm(mpc_ctx c, const BeaverWs& w, const uint64_t* cc, uint64_t* z, int64_t M, int64_t K,
                       int64_t N, int truncate);

// One party per GPU with a communicator: the reveal overlaps the GEMM terms
// that do not need all of it.  Comm stream: eps is revealed
// first, in row chunks, then delta.  Compute stream: b_p's limb planes (and a_p's,
// p != 0) are split while eps chunk 0 is in flight; for each eps chunk, its planes
// (and, for party 0, those of a'_0 = a_0 + eps on the same rows: the public
// eps@delta folded into party 0's left operand, R7/R8) are split and phase 1,
// z[rows] = c_p[rows] + eps[rows] @ b_p, runs on the SMs NCCL leaves free while
// the next chunks and delta are revealed; then delta is split and phase 2 adds
// a'_p @ delta and truncates.  Exposed communication: the first eps chunk.
// Bit-identical to the fused single-GEMM schedule (ring addition commutes).
mpc_status beaver_overlapped(mpc_ctx c, const BeaverWs& w, const uint64_t* x, const uint64_t* y, const uint64_t* a,
                             const uint64_t* b, const uint64_t* cc, uint64_t* z, int64_t M, int64_t K, int64_t N,
                             int truncate) {
    const int64_t sMK = M * K, sKN = K * N;
    const int nch = reveal_chunks(c, w, M);
    for (int i = 0; i < nch; ++i)
        if (!c->ev_chunk[i] && cudaEventCreateWithFlags(&c->ev_chunk[i], cudaEventDisableTiming) != cudaSuccess)
            return fail(c, MPC_ERR_CUDA, "beaver: chunk event");
    CHECK(run(c, kClsSplit, "mask", [&] { return launch_mask(x, a, sMK, y, b, sKN, w.ed, c->stream); }));
    cudaEventRecord(c->ev_mask, c->stream);
    cudaStreamWaitEvent(c->comm_stream, c->ev_mask, 0);
    for (int i = 0; i < nch; ++i) {
        int64_t m0, m1;
        chunk_rows(M, i, nch, m0, m1);
        CHECK(comm_allreduce(c, w.ed + m0 * K, w.ed + m0 * K, (size_t)((m1 - m0) * K), RedOp::SumU64, "eps reveal",
                             c->comm_stream));
        cudaEventRecord(c->ev_chunk[i], c->comm_stream);
    }
    CHECK(comm_allreduce(c, w.ed + sMK, w.ed + sMK, (size_t)sKN, RedOp::SumU64, "delta reveal", c->comm_stream));
    cudaEventRecord(c->ev_delta, c->comm_stream);
    // planes that need no reveal: b_p (all parties), a_p (p != 0)
    RightSplitArgs Rb{K, N, 0, nullptr, nullptr, 0, nullptr, b, 1, 0, w.b_pl, 0, lay(w)};
    LeftSplitArgs La{M, K, 0, nullptr, nullptr, 0, nullptr, a, 1, w.a_pl, 0, lay(w)};
    if (c->rank != 0) CHECK(run(c, kClsSplit, "split a/b", [&] { return launch_split_both(La, Rb, c->stream); }));
    else CHECK(run(c, kClsSplit, "split b", [&] { return launch_split_right(Rb, c->stream); }));
    // per eps chunk of rows of a 256-row-tile grid: Layout::Left blocks of 128 rows
    const int64_t lblk = (int64_t)num_kb(K) * 8 * PlaneGeom<Layout::Left>::kBlock;     // bytes per 128-row block
    for (int i = 0; i < nch; ++i) {
        int64_t m0, m1;
        chunk_rows(M, i, nch, m0, m1);
        const int64_t mc = m1 - m0;
        const int64_t pl_off = nch > 1 ? (m0 / 128) * lblk : 0;
        cudaStreamWaitEvent(c->stream, c->ev_chunk[i], 0);
        LeftSplitArgs Le{mc, K, 0, w.ed + m0 * K, nullptr, 1, w.eps_pl + pl_off,
                         c->rank == 0 ? a + m0 * K : nullptr, c->rank == 0 ? 1 : 0,
                         c->rank == 0 ? w.a_pl + pl_off : nullptr, 0, lay(w), c->rank == 0 ? 1 : 0};
        CHECK(run(c, kClsSplit, "split eps", [&] { return launch_split_left(Le, c->stream); }));
        RingGemmParams p1{};
        p1.seg[0] = seg_of(w, w.eps_pl + pl_off, 0, w.b_pl, 0, (int)num_kb(K));        // eps @ b_p
        p1.nseg = 1;
        set_out(p1, w, mc, N);
        p1.C = cc + m0 * N; p1.Z = z + m0 * N;
        p1.trunc_bits = 0;
        p1.partials = w.partials;
        p1.max_clusters = kOverlapClusters;
        CHECK(gemm_run(c, p1, 1));
    }
    cudaStreamWaitEvent(c->stream, c->ev_delta, 0);
    RightSplitArgs Rd{K, N, 0, w.ed + sMK, nullptr, 1, w.delta_pl, nullptr, 0, 0, nullptr, 0, lay(w)};
    CHECK(run(c, kClsSplit, "split delta", [&] { return launch_split_right(Rd, c->stream); }));
    RingGemmParams p2{};
    p2.seg[0] = seg_of(w, w.a_pl, 0, w.delta_pl, 0, (int)num_kb(K));              // a'_p @ delta
    p2.nseg = 1;
    set_out(p2, w, M, N);
    p2.C = z; p2.Z = z;                                                         // z += ..., in place
    p2.trunc_bits = (truncate && c->P <= 2) ? c->frac : 0;
    p2.partials = w.partials;
    return gemm_run(c, p2, 1);
}

mpc_status gemm_run(mpc_ctx c, RingGemmParams& p, int parties) {
    p.kc = ring_gemm_default_kc(p.seg[0].kb + (p.nseg > 1 ? p.seg[1].kb : 0));
    return run(c, kClsGemm, "ring_gemm", [&] { return ring_gemm_launch(p, parties, c->stream); });
}

// The context scratch (elementwise mul / square, truncate, relu buffers) is
// stream-ordered: a call on another stream than the scratch's last user first
// waits for that stream's work, and a reallocation waits for both streams.
mpc_status ensure_scratch(mpc_ctx c, size_t bytes) {
    if (c->scratch_stream != c->stream && c->scratch) {
        if (!c->scratch_ev && cudaEventCreateWithFlags(&c->scratch_ev, cudaEventDisableTiming) != cudaSuccess)
            return fail(c, MPC_ERR_CUDA, "scratch event");
        cudaEventRecord(c->scratch_ev, c->scratch_stream);
        cudaStreamWaitEvent(c->stream, c->scratch_ev, 0);
    }
    c->scratch_stream = c->stream;
    if (c->scratch_bytes >= bytes) return MPC_OK;
    if (c->scratch) { cudaStreamSynchronize(c->stream); cudaFree(c->scratch); c->scratch = nullptr; c->scratch_bytes = 0; }
    cudaError_t e = cudaMalloc(&c->scratch, bytes);
    if (e != cudaSuccess) return fail(c, MPC_ERR_CUDA, "scratch alloc: %s", cudaGetErrorString(e));
    c->scratch_bytes = bytes;
    return MPC_OK;
}

// An entry point called with workspace == NULL and workspace_bytes == 0 uses the
// context's own workspace, grown to `need` bytes and kept (stream-ordered like the
// scratch: a call on another stream first waits for the previous user's work).
mpc_status own_workspace(mpc_ctx c, size_t need, void*& ws, size_t& ws_bytes) {
    if (ws || ws_bytes || need == 0) return MPC_OK;
    if (c->ows_stream != c->stream && c->ows) {
        if (!c->ows_ev && cudaEventCreateWithFlags(&c->ows_ev, cudaEventDisableTiming) != cudaSuccess)
            return fail(c, MPC_ERR_CUDA, "workspace event");
        cudaEventRecord(c->ows_ev, c->ows_stream);
        cudaStreamWaitEvent(c->stream, c->ows_ev, 0);
    }
    c->ows_stream = c->stream;
    if (c->ows_bytes < need) {
        if (c->ows) { cudaStreamSynchronize(c->stream); cudaFree(c->ows); c->ows = nullptr; c->ows_bytes = 0; }
        const cudaError_t e = cudaMalloc(&c->ows, need);
        if (e != cudaSuccess) return fail(c, MPC_ERR_CUDA, "workspace alloc (%zu B): %s", need, cudaGetErrorString(e));
        c->ows_bytes = need;
    }
    ws = c->ows;
    ws_bytes = c->ows_bytes;
    return MPC_OK;
}

// Truncation of x ([P][n] or n) by `bits` with the wrap pair `wrap_id` (seeded
// TTP: regenerated from k_ttp) or, when r / th are given, the wrap pair in memory
// (materialised offline by mpc_ttp_wrap_pairs; Alg. 1 takes [r], [theta_r] as
// inputs).
mpc_status truncate_impl(mpc_ctx c, uint64_t* x, int64_t n, int bits, uint64_t wrap_id, uint64_t* zbuf, int8_t* hbuf,
                         const uint64_t* r = nullptr, const uint64_t* th = nullptr) {
    if (c->P <= 2) {
        const int64_t tot = n * (c->all ? c->P : 1);
        return run(c, kClsTrunc, "trunc_local", [&] { return launch_trunc_local(x, tot, bits, c->stream); });
    }
    if (!r) CHECK(need_ttp(c, "truncate (wrap pair from wrap_id)"));
    c->rounds += 1;
    if (c->all) {
        c->bytes += 8ull * (uint64_t)n * c->P + (uint64_t)n * c->P;
        return run(c, kClsTrunc, "trunc_alg1_all",
                   [&] { return launch_trunc_alg1_all(x, c->P, n, bits, c->kttp, wrap_id, r, th, c->stream); });
    }
    c->bytes += 9ull * (uint64_t)n;
    CHECK(run(c, kClsTrunc, "trunc_alg1_a",
              [&] { return launch_trunc_alg1_a(x, n, c->kttp, wrap_id, c->rank, r, zbuf, hbuf, c->stream); }));
    CHECK(comm_allreduce(c, zbuf, zbuf, (size_t)n, RedOp::SumU64, "truncate z reveal"));
    CHECK(comm_allreduce(c, hbuf, hbuf, (size_t)n, RedOp::SumI8, "truncate top-bit reveal"));
    return run(c, kClsTrunc, "trunc_alg1_b", [&] {
        return launch_trunc_alg1_b(x, n, bits, c->kttp, wrap_id, c->P, c->rank, r, th, zbuf, hbuf, c->stream);
    });
}

}  // namespace

extern "C" {

}  // extern "C"
namespace {
mpc_status create_impl(mpc_ctx* out, int world_size, int rank, int device, const void* nccl_id, const KeySet& kp,
                       uint64_t kttp, bool has_ttp, int frac_bits) {
    if (!out) return MPC_ERR_ARG;
    *out = nullptr;
    if (world_size < 1 || world_size > kMaxParties) return MPC_ERR_ARG;
    if (rank != MPC_ALL_PARTIES && (rank < 0 || rank >= world_size)) return MPC_ERR_ARG;
    if (frac_bits < 1 || frac_bits > 30) return MPC_ERR_ARG;
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return MPC_ERR_UNSUPPORTED;
    if (prop.major != 10 || prop.minor != 0) return MPC_ERR_UNSUPPORTED;   // sm_100a kernels only
    if (cudaSetDevice(device) != cudaSuccess) return MPC_ERR_CUDA;
    mpc_ctx c = new mpc_ctx_s();
    c->P = world_size;
    c->rank = rank == MPC_ALL_PARTIES ? 0 : rank;
    c->all = (rank == MPC_ALL_PARTIES);
    c->device = device;
    c->frac = frac_bits;
    c->kp = kp;
    c->kttp = kttp;
    c->has_ttp = has_ttp;
    // d_err[0]: the synchronous encode check; d_err[1]: the sticky flag of mpc_encode_async
    if (cudaMalloc(&c->d_err, 2 * sizeof(int)) != cudaSuccess) { delete c; return MPC_ERR_CUDA; }
    if (cudaMemset(c->d_err, 0, 2 * sizeof(int)) != cudaSuccess) { cudaFree(c->d_err); delete c; return MPC_ERR_CUDA; }
    if (!c->all && nccl_id) {
        // One party per process: own communicator (also for P = 1, where the
        // reveals are 1-rank allreduces).  NCCL gets a bounded CTA count so its
        // kernels can run beside the ring GEMM, which leaves SMs for them
        // (kCommSms) while a reveal is in flight.
        ncclUniqueId id;
        std::memcpy(&id, nccl_id, sizeof(id));
        ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
        cfg.blocking = 1;
        cfg.maxCTAs = kCommSms;
        if (ncclCommInitRankConfig(&c->comm, world_size, id, rank, &cfg) != ncclSuccess) {
            cudaFree(c->d_err); delete c; return MPC_ERR_NCCL;
        }
        // the same ranks again without the CTA cap, for the collectives nothing overlaps
        // (collective: every party splits at creation, so all or none have it)
        ncclConfig_t cfg_fast = NCCL_CONFIG_INITIALIZER;
        cfg_fast.blocking = 1;
        if (ncclCommSplit(c->comm, 0, rank, &c->comm_fast, &cfg_fast) != ncclSuccess) {
            ncclCommDestroy(c->comm); cudaFree(c->d_err); delete c; return MPC_ERR_NCCL;
        }
        if (cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&c->ev_mask, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&c->ev_delta, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&c->ev_eps, cudaEventDisableTiming) != cudaSuccess) {
            ncclCommDestroy(c->comm_fast); ncclCommDestroy(c->comm); cudaFree(c->d_err); delete c; return MPC_ERR_CUDA;
        }
        const char* chk = getenv("MPC_CHECK_COLLECTIVES");
        if (chk && atoi(chk) != 0) {
            if (cudaMalloc(&c->check_buf, 2 * sizeof(uint64_t)) != cudaSuccess) {
                ncclCommDestroy(c->comm_fast); ncclCommDestroy(c->comm); cudaFree(c->d_err); delete c; return MPC_ERR_CUDA;
            }
            c->check_collectives = true;
        }
    }
    *out = c;
    return MPC_OK;
}

// The reproducibility convention (R5): every key from one master seed.
KeySet derive_party_keys(uint64_t master_seed, int world_size) {
    KeySet kp{};
    for (int p = 0; p < world_size && p < kMaxParties; ++p)
        kp.k[p] = philox_at(master_seed, stream_word(kTagKeyParty, p, 0), 0);
    return kp;
}
uint64_t derive_ttp_key(uint64_t master_seed) { return philox_at(master_seed, stream_word(kTagKeyTTP, 0, 0), 0); }
}  // namespace
extern "C" {

mpc_status mpc_create(mpc_ctx* out, int world_size, int rank, int device, const void* nccl_id,
                      uint64_t master_seed, int frac_bits) {
    return create_impl(out, world_size, rank, device, nccl_id, derive_party_keys(master_seed, world_size),
                       derive_ttp_key(master_seed), true, frac_bits);
}

mpc_status mpc_derive_keys(uint64_t master_seed, int world_size, int rank, mpc_keys* out) {
    if (!out || world_size < 1 || world_size > kMaxParties || rank < 0 || rank >= world_size) return MPC_ERR_ARG;
    const KeySet kp = derive_party_keys(master_seed, world_size);
    out->przs_self = kp.k[rank];
    out->przs_prev = kp.k[(rank + world_size - 1) % world_size];
    out->ttp = derive_ttp_key(master_seed);
    out->has_ttp = 1;
    return MPC_OK;
}

mpc_status mpc_create_with_keys(mpc_ctx* out, int world_size, int rank, int device, const void* nccl_id,
                                const mpc_keys* keys, int frac_bits) {
    if (!out) return MPC_ERR_ARG;
    *out = nullptr;
    if (!keys || rank == MPC_ALL_PARTIES || world_size < 1 || world_size > kMaxParties || rank < 0 ||
        rank >= world_size)
        return MPC_ERR_ARG;
    if (world_size == 1 && keys->przs_self != keys->przs_prev) return MPC_ERR_ARG;   // one party is its own neighbour
    KeySet kp{};                                 // only this party's two PRZS keys; the others stay 0
    kp.k[(rank + world_size - 1) % world_size] = keys->przs_prev;
    kp.k[rank] = keys->przs_self;
    return create_impl(out, world_size, rank, device, nccl_id, kp, keys->has_ttp ? keys->ttp : 0,
                       keys->has_ttp != 0, frac_bits);
}

struct mpc_group_s { LocalGroup* g; };

mpc_status mpc_group_create(mpc_group* out, int world_size) {
    if (!out) return MPC_ERR_ARG;
    *out = nullptr;
    if (world_size < 1 || world_size > kMaxParties) return MPC_ERR_ARG;
    LocalGroup* g = local_group_create(world_size);
    if (!g) return MPC_ERR_CUDA;
    *out = new mpc_group_s{g};
    return MPC_OK;
}

mpc_status mpc_group_destroy(mpc_group g) {
    if (!g) return MPC_ERR_ARG;
    local_group_destroy(g->g);
    delete g;
    return MPC_OK;
}

mpc_status mpc_create_local(mpc_ctx* out, mpc_group group, int rank, int device, uint64_t master_seed,
                            int frac_bits) {
    if (!out) return MPC_ERR_ARG;
    *out = nullptr;
    if (!group) return MPC_ERR_ARG;
    const int P = local_group_size(group->g);
    if (rank < 0 || rank >= P) return MPC_ERR_ARG;
    mpc_ctx c = nullptr;
    mpc_status s = mpc_create(&c, P, rank, device, nullptr, master_seed, frac_bits);
    if (s != MPC_OK) return s;
    if (!local_group_attach(group->g, rank)) { mpc_destroy(c); return MPC_ERR_ARG; }
    c->lg = group->g;
    if (cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_mask, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_delta, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_eps, cudaEventDisableTiming) != cudaSuccess) {
        mpc_destroy(c);
        return MPC_ERR_CUDA;
    }
    *out = c;
    return MPC_OK;
}

mpc_status mpc_destroy(mpc_ctx c) {
    if (!c) return MPC_ERR_ARG;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream); else cudaDeviceSynchronize();
    if (c->comm_fast) ncclCommDestroy(c->comm_fast);
    if (c->comm) ncclCommDestroy(c->comm);
    if (c->lg) local_group_detach(c->lg, c->rank);
    if (c->xbuf) cudaFree(c->xbuf);
    if (c->check_buf) cudaFree(c->check_buf);
    if (c->comm_stream) { cudaStreamSynchronize(c->comm_stream); cudaStreamDestroy(c->comm_stream); }
    for (cudaEvent_t e : {c->ev_mask, c->ev_delta, c->ev_eps}) if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : c->ev_chunk) if (e) cudaEventDestroy(e);
    for (auto& e : c->pending) { cudaEventDestroy(e.a); cudaEventDestroy(e.b); }
    for (auto e : c->pool) cudaEventDestroy(e);
    if (c->d_err) cudaFree(c->d_err);
    if (c->scratch) cudaFree(c->scratch);
    if (c->scratch_ev) cudaEventDestroy(c->scratch_ev);
    if (c->ows) cudaFree(c->ows);
    if (c->ows_ev) cudaEventDestroy(c->ows_ev);
    delete c;
    return MPC_OK;
}

mpc_status mpc_set_reveal_chunks(mpc_ctx c, int chunks) {
    if (!c || chunks < 0 || chunks > 8) return MPC_ERR_ARG;
    c->reveal_chunks = chunks;
    return MPC_OK;
}

mpc_status mpc_set_stream(mpc_ctx c, void* s) {
    if (!c) return MPC_ERR_ARG;
    c->stream = static_cast<cudaStream_t>(s);
    return MPC_OK;
}

const char* mpc_last_error(mpc_ctx c) { return c ? c->err.c_str() : "null context"; }

mpc_status mpc_stats(mpc_ctx c, uint64_t* rounds, uint64_t* bytes_sent) {
    if (!c) return MPC_ERR_ARG;
    if (rounds) *rounds = c->rounds;
    if (bytes_sent) *bytes_sent = c->bytes;
    return MPC_OK;
}

mpc_status mpc_nccl_unique_id(void* out128) {
    if (!out128) return MPC_ERR_ARG;
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return MPC_ERR_NCCL;
    static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(out128, &id, sizeof(id));
    return MPC_OK;
}

int mpc_world_size(mpc_ctx c) { return c ? c->P : -1; }
int mpc_rank(mpc_ctx c) { return c ? (c->all ? MPC_ALL_PARTIES : c->rank) : -2; }

mpc_status mpc_encode(mpc_ctx c, const double* x, uint64_t* out, int64_t n) {
    CHECK(enter(c));
    if (n < 0) return fail(c, MPC_ERR_SHAPE, "encode: n < 0");
    if (n == 0) return MPC_OK;
    if (!x || !out) return fail(c, MPC_ERR_ARG, "encode: null pointer");
    cudaMemsetAsync(c->d_err, 0, sizeof(int), c->stream);
    CHECK(run(c, kClsCodec, "encode", [&] { return launch_encode(x, out, n, c->frac, c->d_err, c->stream); }));
    int h = 0;
    cudaMemcpyAsync(&h, c->d_err, sizeof(int), cudaMemcpyDeviceToHost, c->stream);
    cudaError_t e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) return fail(c, MPC_ERR_CUDA, "encode: %s", cudaGetErrorString(e));
    if (h) return fail(c, MPC_ERR_OVERFLOW, "encode: |x| * 2^%d >= 2^63 or NaN", c->frac);
    return MPC_OK;
}

mpc_status mpc_encode_async(mpc_ctx c, const double* x, uint64_t* out, int64_t n) {
    CHECK(enter(c));
    if (n < 0) return fail(c, MPC_ERR_SHAPE, "encode: n < 0");
    if (n == 0) return MPC_OK;
    if (!x || !out) return fail(c, MPC_ERR_ARG, "encode: null pointer");
    return run(c, kClsCodec, "encode", [&] { return launch_encode(x, out, n, c->frac, c->d_err + 1, c->stream); });
}

mpc_status mpc_check_overflow(mpc_ctx c) {
    CHECK(enter(c));
    int h = 0;
    cudaMemcpyAsync(&h, c->d_err + 1, sizeof(int), cudaMemcpyDeviceToHost, c->stream);
    cudaMemsetAsync(c->d_err + 1, 0, sizeof(int), c->stream);
    cudaError_t e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) return fail(c, MPC_ERR_CUDA, "check_overflow: %s", cudaGetErrorString(e));
    if (h) return fail(c, MPC_ERR_OVERFLOW, "encode_async: |x| * 2^%d >= 2^63 or NaN since the last check", c->frac);
    return MPC_OK;
}

mpc_status mpc_decode(mpc_ctx c, const uint64_t* v, double* out, int64_t n) {
    CHECK(enter(c));
    if (n < 0) return fail(c, MPC_ERR_SHAPE, "decode: n < 0");
    if (n == 0) return MPC_OK;
    if (!v || !out) return fail(c, MPC_ERR_ARG, "decode: null pointer");
    return run(c, kClsCodec, "decode", [&] { return launch_decode(v, out, n, c->frac, c->stream); });
}

mpc_status mpc_share(mpc_ctx c, const uint64_t* x, int src, uint64_t share_id, uint64_t* out, int64_t n) {
    CHECK(enter(c));
    if (n < 0) return fail(c, MPC_ERR_SHAPE, "share: n < 0");
    if (src < 0 || src >= c->P) return fail(c, MPC_ERR_ARG, "share: src %d out of range", src);
    if (n == 0) return MPC_OK;
    if (!out) return fail(c, MPC_ERR_ARG, "share: null output");
    const bool holds = c->all || c->rank == src;
    if (holds && !x) return fail(c, MPC_ERR_ARG, "share: src party must supply x");
    const int lo = c->all ? 0 : c->rank, hi = c->all ? c->P : c->rank + 1;
    const uint64_t s = stream_word(kTagPRZS, 0, share_id);
    return run(c, kClsPrg, "share",
               [&] { return launch_share(c->kp, c->P, lo, hi, holds ? x : nullptr, src, s, out, n, c->stream); });
}

mpc_status mpc_reveal(mpc_ctx c, const uint64_t* share, uint64_t* out, int64_t n) {
    CHECK(enter(c));
    if (n < 0) return fail(c, MPC_ERR_SHAPE, "reveal: n < 0");
    c->rounds += 1;
    c->bytes += 8ull * (uint64_t)n * (c->all ? c->P : 1);
    if (n == 0) return MPC_OK;
    if (!share || !out) return fail(c, MPC_ERR_ARG, "reveal: null pointer");
    if (c->all) return run(c, kClsSplit, "reveal_sum", [&] { return launch_sum_parties(share, c->P, n, out, c->stream); });
    if (c->P == 1 && !has_comm(c)) {
        cudaError_t e = cudaMemcpyAsync(out, share, 8 * (size_t)n, cudaMemcpyDeviceToDevice, c->stream);
        return e == cudaSuccess ? MPC_OK : fail(c, MPC_ERR_CUDA, "reveal copy: %s", cudaGetErrorString(e));
    }
    return comm_allreduce(c, share, out, (size_t)n, RedOp::SumU64, "reveal");
}

size_t mpc_ttp_workspace_bytes(mpc_ctx c, int64_t M, int64_t K, int64_t N) {
    (void)c;
    if (M < 0 || K < 0 || N < 0) return 0;
    return plain_gemm_ws(M, K, N).total;
}

mpc_status mpc_ttp_triples(mpc_ctx c, uint64_t id, int64_t M, int64_t K, int64_t N, uint64_t* a, uint64_t* b,
                           uint64_t* cc, void* ws, size_t ws_bytes) {
    CHECK(enter(c));
    CHECK(need_ttp(c, "ttp_triples"));
    if (M < 0 || K < 0 || N < 0) return fail(c, MPC_ERR_SHAPE, "ttp_triples: negative size");
    if ((M * K && !a) || (K * N && !b) || (M * N && !cc)) return fail(c, MPC_ERR_ARG, "ttp_triples: null output");
    const bool ttp = c->all || c->rank == 0;       // holds the TTP view: needs a, b sums and c
    if (ttp) CHECK(own_workspace(c, mpc_ttp_workspace_bytes(c, M, K, N), ws, ws_bytes));
    if (ttp && ws_bytes < mpc_ttp_workspace_bytes(c, M, K, N)) return fail(c, MPC_ERR_SHAPE, "ttp_triples: workspace too small");
    if (ttp && !ws && (M * K + K * N) > 0) return fail(c, MPC_ERR_ARG, "ttp_triples: null workspace");
    const int lo = c->all ? 0 : c->rank, hi = c->all ? c->P : c->rank + 1;
    const PlainGemmWs pw = plain_gemm_ws(M, K, N, ttp ? ws : nullptr);
    uint8_t* a_pl = ttp ? pw.a_pl : nullptr;
    uint8_t* b_pl = ttp ? pw.b_pl : nullptr;
    uint64_t* partials = ttp ? pw.partials : nullptr;
    TtpGenArgs ga{c->kttp, id, kTagA, c->P, M, K, lo, hi, a, a_pl, pw.small ? 1 : 0};
    CHECK(run(c, kClsPrg, "ttp_a", [&] { return launch_ttp_left(ga, c->stream); }));
    TtpGenArgs gb{c->kttp, id, kTagB, c->P, N, K, lo, hi, b, b_pl, pw.small ? 1 : 0};
    CHECK(run(c, kClsPrg, "ttp_b", [&] { return launch_ttp_right(gb, c->stream); }));
    if (M == 0 || N == 0) return MPC_OK;
    if (ttp) {
        // c = (sum a) @ (sum b) into party 0's c slot, on the tensor cores
        RingGemmParams p{};
        p.seg[0] = RingGemmSegment{a_pl, b_pl, (int)num_kb(K), 0, 0};
        p.nseg = 1;
        p.M = M; p.N = N; p.C = nullptr; p.Z = cc;
        p.party_stride_c = p.party_stride_z = 0;
        p.trunc_bits = 0;
        p.partials = partials;
        p.small = pw.small ? 1 : 0;
        CHECK(gemm_run(c, p, 1));
    }
    uint64_t* c_out = c->all ? cc + M * N : cc;    // parties >= 1
    const int out_lo = c->all ? 1 : c->rank, out_hi = c->all ? c->P : (c->rank == 0 ? 0 : c->rank + 1);
    return run(c, kClsPrg, "ttp_c", [&] {
        return launch_ttp_c(c->kttp, id, c->P, out_lo, out_hi, c_out, ttp ? cc : nullptr, M * N, c->stream);
    });
}

mpc_status mpc_ttp_wrap_pairs(mpc_ctx c, uint64_t id, int64_t n, uint64_t* r, uint64_t* th) {
    CHECK(enter(c));
    CHECK(need_ttp(c, "ttp_wrap_pairs"));
    if (n < 0) return fail(c, MPC_ERR_SHAPE, "wrap_pairs: n < 0");
    if (n == 0) return MPC_OK;
    if (!r || !th) return fail(c, MPC_ERR_ARG, "wrap_pairs: null output");
    const int lo = c->all ? 0 : c->rank, hi = c->all ? c->P : c->rank + 1;
    return run(c, kClsPrg, "wrap_pairs", [&] { return launch_wrap_pair(c->kttp, id, c->P, lo, hi, r, th, n, c->stream); });
}

size_t mpc_workspace_bytes(mpc_ctx c, int64_t M, int64_t K, int64_t N) {
    if (!c || M < 0 || K < 0 || N < 0) return 0;
    // the planes-based layout (mpc_beaver_prepare / _matmul_prepared / _finish use it) covers
    // the fused small-output kernel's partials too
    return std::max(carve_beaver(c, nullptr, M, K, N).total,
                    carve_beaver(c, nullptr, M, K, N, -1, true, true, 1, true).total);
}

mpc_status mpc_beaver_matmul(mpc_ctx c, const uint64_t* x, const uint64_t* y, const uint64_t* a, const uint64_t* b,
                             const uint64_t* cc, uint64_t* z, int64_t M, int64_t K, int64_t N, int truncate,
                             uint64_t wrap_id, void* ws, size_t ws_bytes) {
    CHECK(enter(c));
    if (M < 0 || K < 0 || N < 0) return fail(c, MPC_ERR_SHAPE, "beaver_matmul: negative size");
    if (K > (int64_t)1 << 30 || M > (int64_t)1 << 31 || N > (int64_t)1 << 31) return fail(c, MPC_ERR_SHAPE, "beaver_matmul: too large");
    CHECK(own_workspace(c, carve_beaver(c, nullptr, M, K, N, -1, true, true, 1, true).total, ws, ws_bytes));
    const BeaverWs w = carve_beaver(c, ws, M, K, N, -1, true, true, 1, true);
    if (ws_bytes < w.total) return fail(c, MPC_ERR_SHAPE, "beaver_matmul: workspace %zu < %zu", ws_bytes, w.total);
    const int Pl = c->all ? c->P : 1;
    c->rounds += 1;                                   // eps || delta: one batched reveal
    c->bytes += 8ull * (uint64_t)(M * K + K * N) * Pl;
    if (M == 0 || N == 0) return MPC_OK;
    if ((M * K && (!x || !a)) || (K * N && (!y || !b)) || !cc || !z || (!ws && w.total))
        return fail(c, MPC_ERR_ARG, "beaver_matmul: null pointer");
    const int64_t sMK = M * K, sKN = K * N, sMN = M * N;
    if (w.fused) {
        FusedSmallParams f{x, a, y, b, cc, z, M, K, N, truncate ? c->frac : 0, w.partials};
        return run(c, kClsGemm, "fused beaver (small)", [&] { return fused_small_launch(f, c->stream); });
    }
    if (c->all) {
        LeftSplitArgs L{M, K, sMK, x, a, c->P, w.eps_pl, a, c->P, w.a_pl, w.a_stride, lay(w)};
        RightSplitArgs R{K, N, sKN, y, b, c->P, w.delta_pl, b, c->P, 1, w.b_pl, w.b_stride, lay(w)};
        CHECK(run(c, kClsSplit, "mask+reveal+split", [&] { return launch_split_both(L, R, c->stream); }));
    } else if (has_comm(c)) {
        CHECK(beaver_overlapped(c, w, x, y, a, b, cc, z, M, K, N, truncate));
        if (truncate && c->P > 2) CHECK(truncate_impl(c, z, sMN, c->frac, wrap_id, w.zbuf, w.hbuf));
        return MPC_OK;
    } else {
        CHECK(run(c, kClsSplit, "mask", [&] { return launch_mask(x, a, sMK, y, b, sKN, w.ed, c->stream); }));
        if (c->P > 1) CHECK(comm_allreduce(c, w.ed, w.ed, (size_t)(sMK + sKN), RedOp::SumU64, "eps/delta reveal"));
    }
    CHECK(beaver_local(c, w, w.ed, a, b, cc, z, M, K, N, truncate));
    if (truncate && c->P > 2) CHECK(truncate_impl(c, z, sMN, c->frac, wrap_id, w.zbuf, w.hbuf));
    return MPC_OK;
}

mpc_status mpc_beaver_mask(mpc_ctx c, const uint64_t* x, const uint64_t* y, const uint64_t* a, const uint64_t* b,
                           uint64_t* ed, int64_t M, int64_t K, int64_t N) {
    CHECK(enter(c));
    if (c->all) return fail(c, MPC_ERR_UNSUPPORTED, "beaver_mask: one-party contexts only");
    if (M < 0 || K < 0 || N < 0) return fail(c, MPC_ERR_SHAPE, "beaver_mask: negative size");
    if (M * K + K * N == 0) return MPC_OK;
    if ((M * K && (!x || !a)) || (K * N && (!y || !b)) || !ed) return fail(c, MPC_ERR_ARG, "beaver_mask: null pointer");
    return run(c, kClsSplit, "mask", [&] { return launch_mask(x, a, M * K, y, b, K * N, ed, c->stream); });
}

mpc_status mpc_beaver_finish(mpc_ctx c, const uint64_t* ed, const uint64_t* a, const uint64_t* b, const uint64_t* cc,
                             uint64_t* z, int64_t M, int64_t K, int64_t N, int truncate, void* ws, size_t ws_bytes) {
    CHECK(enter(c));
    if (c->all) return fail(c, MPC_ERR_UNSUPPORTED, "beaver_finish: one-party contexts only");
    if (truncate && c->P > 2) return fail(c, MPC_ERR_UNSUPPORTED, "beaver_finish: P > 2 truncation needs mpc_truncate");
    if (M < 0 || K < 0 || N < 0) return fail(c, MPC_ERR_SHAPE, "beaver_finish: negative size");
    CHECK(own_workspace(c, carve_beaver(c, nullptr, M, K, N).total, ws, ws_bytes));
    const BeaverWs w = carve_beaver(c, ws, M, K, N);
    if (ws_bytes < w.total) return fail(c, MPC_ERR_SHAPE, "beaver_finish: workspace %zu < %zu", ws_bytes, w.total);
    c->rounds += 1;                                   // the caller's reveal of eps || delta
    c->bytes += 8ull * (uint64_t)(M * K + K * N);
    if (M == 0 || N == 0) return MPC_OK;
    if ((M * K && (!ed || !a)) || (K * N && (!ed || !b)) || !cc || !z || (!ws && w.total))
        return fail(c, MPC_ERR_ARG, "beaver_finish: null pointer");
    return beaver_local(c, w, ed, a, b, cc, z, M, K, N, truncate);
}

// ---- a batch of independent Beaver matmuls of one shape (e.g. attention heads) ----
mpc_status mpc_beaver_matmul_batched(mpc_ctx c, int64_t batch, const uint64_t* x, const uint64_t* y,
                                     const uint64_t* a, const uint64_t* b, const uint64_t* cc, uint64_t* z, int64_t M,
                                     int64_t K, int64_t N, int truncate, uint64_t wrap_id, void* ws, size_t ws_bytes) {
    CHECK(enter(c));
    if (batch < 0 || M < 0 || K < 0 || N < 0) return fail(c, MPC_ERR_SHAPE, "beaver_matmul_batched: negative size");
    if (batch > 65536 || K > (int64_t)1 << 30 || M > (int64_t)1 << 31 || N > (int64_t)1 << 31)
        return fail(c, MPC_ERR_SHAPE, "beaver_matmul_batched: too large");
    const int nb = (int)batch;                        // <= 65536 (checked above)
    CHECK(own_workspace(c, carve_beaver(c, nullptr, M, K, N, -1, true, true, batch < 1 ? 1 : batch).total, ws, ws_bytes));
    const BeaverWs w = carve_beaver(c, ws, M, K, N, -1, true, true, batch < 1 ? 1 : batch);
    if (ws_bytes < w.total) return fail(c, MPC_ERR_SHAPE, "beaver_matmul_batched: workspace %zu < %zu", ws_bytes, w.total);
    const int Pl = c->all ? c->P : 1;
    const int64_t sMK = M * K, sKN = K * N, sMN = M * N;
    c->rounds += 1;                                   // every eps || delta of the batch: one reveal
    c->bytes += 8ull * (uint64_t)(batch * (sMK + sKN)) * Pl;
    if (batch == 0 || M == 0 || N == 0) return MPC_OK;
    if ((sMK && (!x || !a)) || (sKN && (!y || !b)) || !cc || !z || (!ws && w.total))
        return fail(c, MPC_ERR_ARG, "beaver_matmul_batched: null pointer");
    const int code = lay(w);
    if (c->all) {
        LeftSplitArgs L{M, K, batch * sMK, x, a, c->P, w.eps_pl, a, c->P, w.a_pl, w.a_stride, code, 0,
                        nb, sMK, w.xs, w.xs};
        RightSplitArgs R{K, N, batch * sKN, y, b, c->P, w.delta_pl, b, c->P, 1, w.b_pl, w.b_stride, code,
                         nb, sKN, w.ys, w.ys};
        CHECK(run(c, kClsSplit, "mask+reveal+split (batched)", [&] { return launch_split_both(L, R, c->stream); }));
    } else {
        // one party: [e (batch x M x K) | d (batch x K x N)] -> one reveal -> splits
        uint64_t* e = w.ed;
        uint64_t* d = w.ed + batch * sMK;
        CHECK(run(c, kClsSplit, "mask", [&] { return launch_mask(x, a, batch * sMK, y, b, batch * sKN, e, c->stream); }));
        if (c->P > 1) CHECK(comm_allreduce(c, e, e, (size_t)(batch * (sMK + sKN)), RedOp::SumU64, "eps/delta reveal"));
        LeftSplitArgs L{M, K, 0, e, nullptr, 1, w.eps_pl, a, 1, w.a_pl, 0, code, 0, nb, sMK, w.xs, w.xs};
        RightSplitArgs R{K, N, 0, d, nullptr, 1, w.delta_pl, b, 1, c->rank == 0, w.b_pl, 0, code,
                         nb, sKN, w.ys, w.ys};
        CHECK(run(c, kClsSplit, "split eps/delta (batched)", [&] { return launch_split_both(L, R, c->stream); }));
    }
    CHECK(beaver_gemm(c, w, cc, z, M, K, N, truncate));
    if (truncate && c->P > 2) CHECK(truncate_impl(c, z, batch * sMN, c->frac, wrap_id, w.zbuf, w.hbuf));
    return MPC_OK;
}

size_t mpc_workspace_bytes_batched(mpc_ctx c, int64_t batch, int64_t M, int64_t K, int64_t N) {
    if (!c || batch < 0 || M < 0 || K < 0 || N < 0) return 0;
    return carve_beaver(c, nullptr, M, K, N, -1, true, true, batch < 1 ? 1 : batch).total;
}

// ---- the input-independent y side (weights known ahead), then the x side ----
mpc_status mpc_beaver_prepare(mpc_ctx c, const uint64_t* y, const uint64_t* b, int64_t M, int64_t K, int64_t N,
                              void* ws, size_t ws_bytes) {
    CHECK(enter(c));
    if (M < 0 || K < 0 || N < 0) return fail(c, MPC_ERR_SHAPE, "beaver_prepare: negative size");
    if (K > (int64_t)1 << 30 || M > (int64_t)1 << 31 || N > (int64_t)1 << 31) return fail(c, MPC_ERR_SHAPE, "beaver_prepare: too large");
    const BeaverWs w = carve_beaver(c, ws, M, K, N);
    if (ws_bytes < w.total) return fail(c, MPC_ERR_SHAPE, "beaver_prepare: workspace %zu < %zu", ws_bytes, w.total);
    const int Pl = c->all ? c->P : 1;
    const int64_t sMK = M * K, sKN = K * N;
    c->rounds += 1;                                   // the delta reveal (input-independent)
    c->bytes += 8ull * (uint64_t)sKN * Pl;
    if (M == 0 || N == 0) return MPC_OK;
    if ((sKN && (!y || !b)) || (!ws && w.total)) return fail(c, MPC_ERR_ARG, "beaver_prepare: null pointer");
    if (c->all) {
        RightSplitArgs R{K, N, sKN, y, b, c->P, w.delta_pl, b, c->P, 1, w.b_pl, w.b_stride, lay(w)};
        return run(c, kClsSplit, "prepare: mask+reveal+split delta", [&] { return launch_split_right(R, c->stream); });
    }
    uint64_t* d = w.ed + sMK;
    CHECK(run(c, kClsSplit, "prepare: mask", [&] { return launch_mask(nullptr, nullptr, 0, y, b, sKN, d, c->stream); }));
    if (c->P > 1) CHECK(comm_allreduce(c, d, d, (size_t)sKN, RedOp::SumU64, "delta reveal"));
    RightSplitArgs R{K, N, 0, d, nullptr, 1, w.delta_pl, b, 1, c->rank == 0, w.b_pl, 0, lay(w)};
    return run(c, kClsSplit, "prepare: split delta", [&] { return launch_split_right(R, c->stream); });
}

mpc_status mpc_beaver_matmul_prepared(mpc_ctx c, const uint64_t* x, const uint64_t* a, const uint64_t* cc, uint64_t* z,
                                      int64_t M, int64_t K, int64_t N, int truncate, uint64_t wrap_id, void* ws,
                                      size_t ws_bytes) {
    CHECK(enter(c));
    if (M < 0 || K < 0 || N < 0) return fail(c, MPC_ERR_SHAPE, "beaver_matmul_prepared: negative size");
    if (K > (int64_t)1 << 30 || M > (int64_t)1 << 31 || N > (int64_t)1 << 31) return fail(c, MPC_ERR_SHAPE, "beaver_matmul_prepared: too large");
    const BeaverWs w = carve_beaver(c, ws, M, K, N);
    if (ws_bytes < w.total) return fail(c, MPC_ERR_SHAPE, "beaver_matmul_prepared: workspace %zu < %zu", ws_bytes, w.total);
    const int Pl = c->all ? c->P : 1;
    const int64_t sMK = M * K, sMN = M * N;
    c->rounds += 1;                                   // the eps reveal
    c->bytes += 8ull * (uint64_t)sMK * Pl;
    if (M == 0 || N == 0) return MPC_OK;
    if ((sMK && (!x || !a)) || !cc || !z || (!ws && w.total)) return fail(c, MPC_ERR_ARG, "beaver_matmul_prepared: null pointer");
    if (c->all) {
        LeftSplitArgs L{M, K, sMK, x, a, c->P, w.eps_pl, a, c->P, w.a_pl, w.a_stride, lay(w)};
        CHECK(run(c, kClsSplit, "mask+reveal+split eps", [&] { return launch_split_left(L, c->stream); }));
        CHECK(beaver_gemm(c, w, cc, z, M, K, N, truncate));
    } else if (!has_comm(c)) {
        if (c->P > 1) return fail(c, MPC_ERR_STATE, "beaver_matmul_prepared: context has no communicator");
        LeftSplitArgs L{M, K, 0, x, a, 1, w.eps_pl, a, 1, w.a_pl, 0, lay(w)};
        CHECK(run(c, kClsSplit, "mask+split eps", [&] { return launch_split_left(L, c->stream); }));
        CHECK(beaver_gemm(c, w, cc, z, M, K, N, truncate));
    } else {
        // eps revealed on the comm stream while a_p is split and z = c_p + a_p @ delta
        // runs on the SMs the reveal leaves free; then eps @ b'_p (as beaver_overlapped)
        CHECK(run(c, kClsSplit, "mask", [&] { return launch_mask(x, a, sMK, nullptr, nullptr, 0, w.ed, c->stream); }));
        cudaEventRecord(c->ev_mask, c->stream);
        cudaStreamWaitEvent(c->comm_stream, c->ev_mask, 0);
        CHECK(comm_allreduce(c, w.ed, w.ed, (size_t)sMK, RedOp::SumU64, "eps reveal", c->comm_stream));
        cudaEventRecord(c->ev_eps, c->comm_stream);
        LeftSplitArgs La{M, K, 0, nullptr, nullptr, 0, nullptr, a, 1, w.a_pl, 0, lay(w)};
        CHECK(run(c, kClsSplit, "split a", [&] { return launch_split_left(La, c->stream); }));
        RingGemmParams p1{};
        p1.seg[0] = seg_of(w, w.a_pl, 0, w.delta_pl, 0, (int)num_kb(K));
        p1.nseg = 1;
        set_out(p1, w, M, N);
        p1.C = cc; p1.Z = z;
        p1.partials = w.partials;
        p1.max_clusters = kOverlapClusters;
        CHECK(gemm_run(c, p1, 1));
        cudaStreamWaitEvent(c->stream, c->ev_eps, 0);
        LeftSplitArgs Le{M, K, 0, w.ed, nullptr, 1, w.eps_pl, nullptr, 0, nullptr, 0, lay(w)};
        CHECK(run(c, kClsSplit, "split eps", [&] { return launch_split_left(Le, c->stream); }));
        RingGemmParams p2{};
        p2.seg[0] = seg_of(w, w.eps_pl, 0, w.b_pl, 0, (int)num_kb(K));
        p2.nseg = 1;
        set_out(p2, w, M, N);
        p2.C = z; p2.Z = z;
        p2.trunc_bits = (truncate && c->P <= 2) ? c->frac : 0;
        p2.partials = w.partials;
        CHECK(gemm_run(c, p2, 1));
    }
    if (truncate && c->P > 2) CHECK(truncate_impl(c, z, sMN, c->frac, wrap_id, w.zbuf, w.hbuf));
    return MPC_OK;
}

}  // extern "C"

namespace {
// Everything after the eps || delta reveal: limb split of eps, delta, a_p and
// b'_p = b_p + [p = 0] delta, then the ring GEMM z_p = c_p + a_p@delta +
// eps@b'_p with the P <= 2 truncation fused.  ed = revealed [eps | delta]
// (one-party contexts; ignored in the all-parties mode, whose split kernels
// already produced the planes).
mpc_status beaver_local(mpc_ctx c, const BeaverWs& w, const uint64_t* ed, const uint64_t* a, const uint64_t* b,
                        const uint64_t* cc, uint64_t* z, int64_t M, int64_t K, int64_t N, int truncate) {
    const int64_t sMK = M * K;
    if (!c->all) {
        LeftSplitArgs L{M, K, 0, ed, nullptr, 1, w.eps_pl, a, 1, w.a_pl, 0, lay(w)};
        RightSplitArgs R{K, N, 0, ed + sMK, nullptr, 1, w.delta_pl, b, 1, c->rank == 0, w.b_pl, 0, lay(w)};
        CHECK(run(c, kClsSplit, "split eps/delta", [&] { return launch_split_both(L, R, c->stream); }));
    }
    return beaver_gemm(c, w, cc, z, M, K, N, truncate);
}

// The ring GEMM of the Beaver step from the limb planes in the workspace:
// z_p = c_p + a_p @ delta + eps @ b'_p (all parties of the context), truncated if P <= 2.
mpc_status beaver_gemm(mpc_ctx c, const BeaverWs& w, const uint64_t* cc, uint64_t* z, int64_t M, int64_t K,
                       int64_t N, int truncate) {
    const int Pl = c->all ? c->P : 1;
    const int64_t sMN = M * N;
    RingGemmParams p{};
    p.seg[0] = seg_of(w, w.a_pl, w.a_stride, w.delta_pl, 0, (int)num_kb(K));   // a_p @ delta
    p.seg[1] = seg_of(w, w.eps_pl, 0, w.b_pl, w.b_stride, (int)num_kb(K));     // eps @ b'_p
    p.partials = w.partials;
    p.nseg = 2;
    set_out(p, w, M, N);
    p.C = cc; p.Z = z;
    p.party_stride_c = p.party_stride_z = w.batch * sMN;
    p.trunc_bits = (truncate && c->P <= 2) ? c->frac : 0;                                     // fused, 0 rounds
    return gemm_run(c, p, Pl);
}
}  // namespace

extern "C" {

mpc_status mpc_truncate(mpc_ctx c, uint64_t* x, int64_t n, int bits, uint64_t wrap_id) {
    CHECK(enter(c));
    if (n < 0) return fail(c, MPC_ERR_SHAPE, "truncate: n < 0");
    if (bits < 1 || bits > 62) return fail(c, MPC_ERR_ARG, "truncate: bits %d out of [1, 62]", bits);
    if (n == 0) return MPC_OK;
    if (!x) return fail(c, MPC_ERR_ARG, "truncate: null pointer");
    uint64_t* zb = nullptr;
    int8_t* hb = nullptr;
    if (!c->all && c->P > 2) {
        CHECK(ensure_scratch(c, align256(8 * (size_t)n) + (size_t)n));
        zb = static_cast<uint64_t*>(c->scratch);
        hb = reinterpret_cast<int8_t*>(static_cast<uint8_t*>(c->scratch) + align256(8 * (size_t)n));
    }
    return truncate_impl(c, x, n, bits, wrap_id, zb, hb);
}

mpc_status mpc_truncate_pairs(mpc_ctx c, uint64_t* x, int64_t n, int bits, const uint64_t* r, const uint64_t* theta_r) {
    CHECK(enter(c));
    if (n < 0) return fail(c, MPC_ERR_SHAPE, "truncate_pairs: n < 0");
    if (bits < 1 || bits > 62) return fail(c, MPC_ERR_ARG, "truncate_pairs: bits %d out of [1, 62]", bits);
    if (n == 0) return MPC_OK;
    if (!x || (c->P > 2 && (!r || !theta_r))) return fail(c, MPC_ERR_ARG, "truncate_pairs: null pointer");
    uint64_t* zb = nullptr;
    int8_t* hb = nullptr;
    if (!c->all && c->P > 2) {
        CHECK(ensure_scratch(c, align256(8 * (size_t)n) + (size_t)n));
        zb = static_cast<uint64_t*>(c->scratch);
        hb = reinterpret_cast<int8_t*>(static_cast<uint8_t*>(c->scratch) + align256(8 * (size_t)n));
    }
    return truncate_impl(c, x, n, bits, 0, zb, hb, r, theta_r);
}

size_t mpc_ring_matmul_workspace_bytes(int64_t M, int64_t K, int64_t N) {
    if (M < 0 || K < 0 || N < 0) return 0;
    return plain_gemm_ws(M, K, N).total;
}

mpc_status mpc_ring_matmul(mpc_ctx c, const uint64_t* A, const uint64_t* B, uint64_t* C, int64_t M, int64_t K,
                           int64_t N, void* ws, size_t ws_bytes) {
    CHECK(enter(c));
    if (M < 0 || K < 0 || N < 0) return fail(c, MPC_ERR_SHAPE, "ring_matmul: negative size");
    CHECK(own_workspace(c, mpc_ring_matmul_workspace_bytes(M, K, N), ws, ws_bytes));
    if (ws_bytes < mpc_ring_matmul_workspace_bytes(M, K, N)) return fail(c, MPC_ERR_SHAPE, "ring_matmul: workspace too small");
    if (M == 0 || N == 0) return MPC_OK;
    if (!C || (K && (!A || !B || !ws))) return fail(c, MPC_ERR_ARG, "ring_matmul: null pointer");
    const PlainGemmWs pw = plain_gemm_ws(M, K, N, ws);
    const int code = pw.small ? 2 : 0;
    LeftSplitArgs L{M, K, 0, A, nullptr, 1, pw.a_pl, nullptr, 0, nullptr, 0, code};
    RightSplitArgs R{K, N, 0, B, nullptr, 1, pw.b_pl, nullptr, 0, 0, nullptr, 0, code};
    CHECK(run(c, kClsSplit, "split A/B", [&] { return launch_split_both(L, R, c->stream); }));
    RingGemmParams p{};
    p.seg[0] = RingGemmSegment{pw.a_pl, pw.b_pl, (int)num_kb(K), 0, 0};
    p.nseg = 1;
    p.M = M; p.N = N; p.C = nullptr; p.Z = C;
    p.partials = pw.partials;
    p.small = pw.small ? 1 : 0;
    return gemm_run(c, p, 1);
}

// ---------------------------------------------------------------- elementwise product / square
// (App. A.1.1)
mpc_status mpc_ttp_mul_triples(mpc_ctx c, uint64_t id, int64_t n, uint64_t* a, uint64_t* b, uint64_t* cc) {
    CHECK(enter(c));
    CHECK(need_ttp(c, "ttp_mul_triples"));
    if (n < 0) return fail(c, MPC_ERR_SHAPE, "ttp_mul_triples: n < 0");
    if (n == 0) return MPC_OK;
    if (!a || !b || !cc) return fail(c, MPC_ERR_ARG, "ttp_mul_triples: null output");
    const int lo = c->all ? 0 : c->rank, hi = c->all ? c->P : c->rank + 1;
    return run(c, kClsPrg, "ttp_mul",
               [&] { return launch_ttp_elementwise(false, c->kttp, id, c->P, lo, hi, a, b, cc, n, c->stream); });
}

mpc_status mpc_ttp_square_pairs(mpc_ctx c, uint64_t id, int64_t n, uint64_t* a, uint64_t* b) {
    CHECK(enter(c));
    CHECK(need_ttp(c, "ttp_square_pairs"));
    if (n < 0) return fail(c, MPC_ERR_SHAPE, "ttp_square_pairs: n < 0");
    if (n == 0) return MPC_OK;
    if (!a || !b) return fail(c, MPC_ERR_ARG, "ttp_square_pairs: null output");
    const int lo = c->all ? 0 : c->rank, hi = c->all ? c->P : c->rank + 1;
    return run(c, kClsPrg, "ttp_square",
               [&] { return launch_ttp_elementwise(true, c->kttp, id, c->P, lo, hi, a, b, nullptr, n, c->stream); });
}

}  // extern "C"

namespace {
// Shared body of mpc_beaver_mul (square = false) and mpc_beaver_square.
mpc_status beaver_elementwise(mpc_ctx c, bool square, const uint64_t* x, const uint64_t* y, const uint64_t* a,
                              const uint64_t* b, const uint64_t* cc, uint64_t* z, int64_t n, int truncate,
                              uint64_t wrap_id) {
    const char* what = square ? "beaver_square" : "beaver_mul";
    CHECK(enter(c));
    if (n < 0) return fail(c, MPC_ERR_SHAPE, "%s: n < 0", what);
    const int Pl = c->all ? c->P : 1;
    const int64_t nrev = square ? n : 2 * n;             // eps (|| delta): one batched reveal
    c->rounds += 1;
    c->bytes += 8ull * (uint64_t)nrev * Pl;
    if (n == 0) return MPC_OK;
    if (!x || !a || !b || !z || (!square && (!y || !cc))) return fail(c, MPC_ERR_ARG, "%s: null pointer", what);
    const int bits = (truncate && c->P <= 2) ? c->frac : 0;               // fused local truncation
    uint64_t* zb = nullptr;
    int8_t* hb = nullptr;
    if (c->all) {
        CHECK(run(c, kClsSplit, what, [&] {
            return launch_beaver_elementwise_all(square, x, y, a, b, cc, z, c->P, n, bits, c->stream);
        }));
    } else {
        // one party: [x - a | y - b] -> reveal (one allreduce) -> z_p; scratch also holds Alg. 1's buffers
        const size_t ed_bytes = align256(8 * (size_t)nrev);
        const bool alg1 = truncate && c->P > 2;
        CHECK(ensure_scratch(c, ed_bytes + (alg1 ? align256(8 * (size_t)n) + (size_t)n : 0)));
        uint64_t* ed = static_cast<uint64_t*>(c->scratch);
        if (alg1) {
            zb = reinterpret_cast<uint64_t*>(static_cast<uint8_t*>(c->scratch) + ed_bytes);
            hb = reinterpret_cast<int8_t*>(static_cast<uint8_t*>(c->scratch) + ed_bytes + align256(8 * (size_t)n));
        }
        CHECK(run(c, kClsSplit, "mask", [&] {
            return launch_mask(x, a, n, square ? nullptr : y, square ? nullptr : b, square ? 0 : n, ed, c->stream);
        }));
        if (c->P > 1) CHECK(comm_allreduce(c, ed, ed, (size_t)nrev, RedOp::SumU64, "eps/delta reveal"));
        CHECK(run(c, kClsSplit, what, [&] {
            return launch_beaver_elementwise_finish(square, ed, a, b, cc, z, n, c->rank == 0, bits, c->stream);
        }));
    }
    if (truncate && c->P > 2) CHECK(truncate_impl(c, z, n, c->frac, wrap_id, zb, hb));
    return MPC_OK;
}
}  // namespace

extern "C" {

mpc_status mpc_beaver_mul(mpc_ctx c, const uint64_t* x, const uint64_t* y, const uint64_t* a, const uint64_t* b,
                          const uint64_t* cc, uint64_t* z, int64_t n, int truncate, uint64_t wrap_id) {
    return beaver_elementwise(c, false, x, y, a, b, cc, z, n, truncate, wrap_id);
}

mpc_status mpc_beaver_square(mpc_ctx c, const uint64_t* x, const uint64_t* a, const uint64_t* b, uint64_t* z,
                             int64_t n, int truncate, uint64_t wrap_id) {
    return beaver_elementwise(c, true, x, nullptr, a, b, nullptr, z, n, truncate, wrap_id);
}

// The elementwise product / square after the caller's reveal (one-party contexts;
// the round made explicit, as mpc_beaver_finish for the matmul).
mpc_status mpc_beaver_mul_finish(mpc_ctx c, const uint64_t* ed, const uint64_t* a, const uint64_t* b,
                                 const uint64_t* cc, uint64_t* z, int64_t n, int truncate) {
    CHECK(enter(c));
    if (c->all) return fail(c, MPC_ERR_UNSUPPORTED, "beaver_mul_finish: one-party contexts only");
    if (truncate && c->P > 2) return fail(c, MPC_ERR_UNSUPPORTED, "beaver_mul_finish: P > 2 truncation needs mpc_truncate");
    if (n < 0) return fail(c, MPC_ERR_SHAPE, "beaver_mul_finish: n < 0");
    c->rounds += 1;
    c->bytes += 16ull * (uint64_t)n;
    if (n == 0) return MPC_OK;
    if (!ed || !a || !b || !cc || !z) return fail(c, MPC_ERR_ARG, "beaver_mul_finish: null pointer");
    const int bits = truncate ? c->frac : 0;
    return run(c, kClsSplit, "beaver_mul", [&] {
        return launch_beaver_elementwise_finish(false, ed, a, b, cc, z, n, c->rank == 0, bits, c->stream);
    });
}

mpc_status mpc_beaver_square_finish(mpc_ctx c, const uint64_t* e, const uint64_t* a, const uint64_t* b, uint64_t* z,
                                    int64_t n, int truncate) {
    CHECK(enter(c));
    if (c->all) return fail(c, MPC_ERR_UNSUPPORTED, "beaver_square_finish: one-party contexts only");
    if (truncate && c->P > 2) return fail(c, MPC_ERR_UNSUPPORTED, "beaver_square_finish: P > 2 truncation needs mpc_truncate");
    if (n < 0) return fail(c, MPC_ERR_SHAPE, "beaver_square_finish: n < 0");
    c->rounds += 1;
    c->bytes += 8ull * (uint64_t)n;
    if (n == 0) return MPC_OK;
    if (!e || !a || !b || !z) return fail(c, MPC_ERR_ARG, "beaver_square_finish: null pointer");
    const int bits = truncate ? c->frac : 0;
    return run(c, kClsSplit, "beaver_square", [&] {
        return launch_beaver_elementwise_finish(true, e, a, b, nullptr, z, n, c->rank == 0, bits, c->stream);
    });
}

// Several reveals in one round: one NCCL group of allreduces (one-party
// contexts), local sums (all parties on one device).
mpc_status mpc_reveal_batch(mpc_ctx c, int count, const uint64_t* const* shares, uint64_t* const* outs,
                            const int64_t* ns) {
    CHECK(enter(c));
    if (count < 0 || (count > 0 && (!shares || !outs || !ns))) return fail(c, MPC_ERR_ARG, "reveal_batch: bad arguments");
    uint64_t total = 0;
    for (int t = 0; t < count; ++t) {
        if (ns[t] < 0) return fail(c, MPC_ERR_SHAPE, "reveal_batch: n[%d] < 0", t);
        if (ns[t] > 0 && (!shares[t] || !outs[t])) return fail(c, MPC_ERR_ARG, "reveal_batch: null pointer %d", t);
        total += (uint64_t)ns[t];
    }
    c->rounds += 1;
    c->bytes += 8ull * total * (c->all ? c->P : 1);
    if (c->all) {
        for (int t = 0; t < count; ++t)
            if (ns[t]) CHECK(run(c, kClsSplit, "reveal_sum",
                                 [&] { return launch_sum_parties(shares[t], c->P, ns[t], outs[t], c->stream); }));
        return MPC_OK;
    }
    if (c->P == 1 && !has_comm(c)) {
        for (int t = 0; t < count; ++t) {
            if (!ns[t]) continue;
            cudaError_t e = cudaMemcpyAsync(outs[t], shares[t], 8 * (size_t)ns[t], cudaMemcpyDeviceToDevice, c->stream);
            if (e != cudaSuccess) return fail(c, MPC_ERR_CUDA, "reveal_batch copy: %s", cudaGetErrorString(e));
        }
        return MPC_OK;
    }
    if (!has_comm(c)) return fail(c, MPC_ERR_STATE, "reveal_batch: context has no communicator (created without nccl_id)");
    if (c->lg) {
        for (int t = 0; t < count; ++t)
            if (ns[t]) CHECK(comm_allreduce(c, shares[t], outs[t], (size_t)ns[t], RedOp::SumU64, "reveal_batch"));
        return MPC_OK;
    }
    ncclResult_t r = ncclGroupStart();
    for (int t = 0; t < count && r == ncclSuccess; ++t)
        if (ns[t]) r = ncclAllReduce(shares[t], outs[t], (size_t)ns[t], ncclUint64, ncclSum, pick_comm(c, c->stream),
                                     c->stream);
    ncclResult_t r2 = ncclGroupEnd();
    if (r == ncclSuccess) r = r2;
    if (r != ncclSuccess) {
        c->broken = true;
        abort_comms(c);
        return fail(c, MPC_ERR_NCCL, "reveal_batch: %s", ncclGetErrorString(r));
    }
    return MPC_OK;
}

// ---------------------------------------------------------------- private 2-D convolution
// (R22)
mpc_status mpc_mask(mpc_ctx c, const uint64_t* x, const uint64_t* a, int64_t n1, const uint64_t* y,
                    const uint64_t* b, int64_t n2, uint64_t* ed) {
    CHECK(enter(c));
    if (n1 < 0 || n2 < 0) return fail(c, MPC_ERR_SHAPE, "mask: negative size");
    if (n1 + n2 == 0) return MPC_OK;
    if ((n1 && (!x || !a)) || (n2 && (!y || !b)) || !ed) return fail(c, MPC_ERR_ARG, "mask: null pointer");
    return run(c, kClsSplit, "mask", [&] { return launch_mask(x, a, n1, y, b, n2, ed, c->stream); });
}

}  // extern "C"

namespace {
bool conv_geom_ok(const mpc_conv2d_geom* g) {
    return g && g->B >= 0 && g->C >= 0 && g->H >= 0 && g->W >= 0 && g->Cout >= 0 && g->kh >= 1 && g->kw >= 1 &&
           g->sh >= 1 && g->sw >= 1 && g->ph >= 0 && g->pw >= 0 && g->H + 2 * g->ph >= g->kh &&
           g->W + 2 * g->pw >= g->kw && g->C * g->kh * g->kw < ((int64_t)1 << 30) &&
           g->C * g->H * g->W < ((int64_t)1 << 31) && g->H < ((int64_t)1 << 30) && g->W < ((int64_t)1 << 30);
}
ConvGeom to_geom(const mpc_conv2d_geom* g) {
    return ConvGeom{g->B, g->C, g->H, g->W, g->Cout, g->kh, g->kw, g->sh, g->sw, g->ph, g->pw};
}
// Transposed GEMM (Cout rows x pixel columns) only for one image: its row-major
// output is then exactly NCHW.
BeaverWs carve_conv(mpc_ctx c, void* ws, const ConvGeom& g) {
    return carve_beaver(c, ws, g.M(), g.K(), g.Cout, g.in_elems() + g.w_elems(), g.B == 1, false);
}
// GEMM output mapping of a convolution: NCHW z from im2col rows (b, pixel).
void conv_out(RingGemmParams& p, const BeaverWs& w, const ConvGeom& g) {
    if (w.swap) { p.M = g.Cout; p.N = g.M(); }                 // (Cout x Ho*Wo) row-major = NCHW, B = 1
    else { p.M = g.M(); p.N = g.Cout; p.out_hw = g.Ho() * g.Wo(); }
    p.party_stride_c = p.party_stride_z = g.out_elems();
}
// x-side: implicit im2col of activation-shaped operands; y-side: weights (Cout x K rows)
mpc_status conv_split(mpc_ctx c, const BeaverWs& w, const ConvGeom& g, const uint64_t* xp, const uint64_t* xm,
                      int Psum, int64_t xstride, const uint64_t* acp, int Pcopy, const uint64_t* yp,
                      const uint64_t* ym, int64_t ystride, const uint64_t* bcp, int add_first) {
    Im2colSplitArgs I{g, xstride, xp, xm, Psum, w.eps_pl, acp, Pcopy, w.a_pl, w.a_stride, w.swap ? 1 : 0};
    LeftSplitArgs Wt{g.Cout, g.K(), ystride, yp, ym, Psum, w.delta_pl, bcp, Pcopy, w.b_pl, w.b_stride,
                     w.swap ? 0 : 1, add_first};
    return run(c, kClsSplit, "split conv", [&] { return launch_split_conv(I, Wt, c->stream); });
}
mpc_status conv_gemm(mpc_ctx c, const BeaverWs& w, const ConvGeom& g, const uint64_t* cc, uint64_t* z, int truncate,
                     int parties) {
    const int kb = (int)num_kb(g.K());
    RingGemmParams p{};
    p.seg[0] = seg_of(w, w.a_pl, w.a_stride, w.delta_pl, 0, kb);     // conv(a_p, delta)
    p.seg[1] = seg_of(w, w.eps_pl, 0, w.b_pl, w.b_stride, kb);       // conv(eps, b_p + [p = 0] delta)
    p.nseg = 2;
    p.partials = w.partials;
    conv_out(p, w, g);
    p.C = cc; p.Z = z;
    p.trunc_bits = (truncate && c->P <= 2) ? c->frac : 0;
    return gemm_run(c, p, parties);
}
}  // namespace

extern "C" {

size_t mpc_conv2d_workspace_bytes(mpc_ctx c, const mpc_conv2d_geom* gg) {
    if (!c || !conv_geom_ok(gg)) return 0;
    return carve_conv(c, nullptr, to_geom(gg)).total;
}

mpc_status mpc_beaver_conv2d(mpc_ctx c, const mpc_conv2d_geom* gg, const uint64_t* x, const uint64_t* y,
                             const uint64_t* a, const uint64_t* b, const uint64_t* cc, uint64_t* z, int truncate,
                             uint64_t wrap_id, void* ws, size_t ws_bytes) {
    CHECK(enter(c));
    if (!conv_geom_ok(gg)) return fail(c, MPC_ERR_SHAPE, "beaver_conv2d: invalid geometry");
    const ConvGeom g = to_geom(gg);
    const BeaverWs w = carve_conv(c, ws, g);
    if (ws_bytes < w.total) return fail(c, MPC_ERR_SHAPE, "beaver_conv2d: workspace %zu < %zu", ws_bytes, w.total);
    const int Pl = c->all ? c->P : 1;
    const int64_t na = g.in_elems(), nb = g.w_elems(), nz = g.out_elems();
    c->rounds += 1;                                   // eps || delta at the input / weight shapes, one round
    c->bytes += 8ull * (uint64_t)(na + nb) * Pl;
    if (nz == 0) return MPC_OK;
    if ((na && (!x || !a)) || (nb && (!y || !b)) || !cc || !z || (!ws && w.total))
        return fail(c, MPC_ERR_ARG, "beaver_conv2d: null pointer");
    if (c->all) {
        CHECK(conv_split(c, w, g, x, a, c->P, na, a, c->P, y, b, nb, b, 1));
    } else {
        CHECK(run(c, kClsSplit, "mask", [&] { return launch_mask(x, a, na, y, b, nb, w.ed, c->stream); }));
        if (c->P > 1) CHECK(comm_allreduce(c, w.ed, w.ed, (size_t)(na + nb), RedOp::SumU64, "eps/delta reveal"));
        CHECK(conv_split(c, w, g, w.ed, nullptr, 1, 0, a, 1, w.ed + na, nullptr, 0, b, c->rank == 0));
    }
    CHECK(conv_gemm(c, w, g, cc, z, truncate, Pl));
    if (truncate && c->P > 2) CHECK(truncate_impl(c, z, nz, c->frac, wrap_id, w.zbuf, w.hbuf));
    return MPC_OK;
}

mpc_status mpc_beaver_conv2d_finish(mpc_ctx c, const mpc_conv2d_geom* gg, const uint64_t* ed, const uint64_t* a,
                                    const uint64_t* b, const uint64_t* cc, uint64_t* z, int truncate, void* ws,
                                    size_t ws_bytes) {
    CHECK(enter(c));
    if (c->all) return fail(c, MPC_ERR_UNSUPPORTED, "beaver_conv2d_finish: one-party contexts only");
    if (truncate && c->P > 2) return fail(c, MPC_ERR_UNSUPPORTED, "beaver_conv2d_finish: P > 2 truncation needs mpc_truncate");
    if (!conv_geom_ok(gg)) return fail(c, MPC_ERR_SHAPE, "beaver_conv2d_finish: invalid geometry");
    const ConvGeom g = to_geom(gg);
    const BeaverWs w = carve_conv(c, ws, g);
    if (ws_bytes < w.total) return fail(c, MPC_ERR_SHAPE, "beaver_conv2d_finish: workspace %zu < %zu", ws_bytes, w.total);
    const int64_t na = g.in_elems(), nb = g.w_elems();
    c->rounds += 1;
    c->bytes += 8ull * (uint64_t)(na + nb);
    if (g.out_elems() == 0) return MPC_OK;
    if (!ed || (na && !a) || (nb && !b) || !cc || !z || (!ws && w.total))
        return fail(c, MPC_ERR_ARG, "beaver_conv2d_finish: null pointer");
    CHECK(conv_split(c, w, g, ed, nullptr, 1, 0, a, 1, ed + na, nullptr, 0, b, c->rank == 0));
    return conv_gemm(c, w, g, cc, z, truncate, 1);
}

size_t mpc_ttp_conv_workspace_bytes(mpc_ctx c, const mpc_conv2d_geom* gg) {
    if (!c || !conv_geom_ok(gg)) return 0;
    const ConvGeom g = to_geom(gg);
    // the TTP's sums of a_p, b_p, their planes (normal GEMM orientation) and split-K slabs
    return align256(8 * (size_t)g.in_elems()) + align256(8 * (size_t)g.w_elems()) + align256(lp(g.M(), g.K())) +
           align256(rp(g.Cout, g.K())) + align256(ring_gemm_partials_bytes(1, g.M(), g.Cout, (int)num_kb(g.K())));
}

mpc_status mpc_ttp_conv_triples(mpc_ctx c, uint64_t id, const mpc_conv2d_geom* gg, uint64_t* a, uint64_t* b,
                                uint64_t* cc, void* ws, size_t ws_bytes) {
    CHECK(enter(c));
    CHECK(need_ttp(c, "ttp_conv_triples"));
    if (!conv_geom_ok(gg)) return fail(c, MPC_ERR_SHAPE, "ttp_conv_triples: invalid geometry");
    const ConvGeom g = to_geom(gg);
    const int64_t na = g.in_elems(), nb = g.w_elems(), nz = g.out_elems();
    if ((na && !a) || (nb && !b) || (nz && !cc)) return fail(c, MPC_ERR_ARG, "ttp_conv_triples: null output");
    const bool ttp = c->all || c->rank == 0;
    if (ttp && ws_bytes < mpc_ttp_conv_workspace_bytes(c, gg)) return fail(c, MPC_ERR_SHAPE, "ttp_conv_triples: workspace too small");
    if (ttp && !ws && nz) return fail(c, MPC_ERR_ARG, "ttp_conv_triples: null workspace");
    const int lo = c->all ? 0 : c->rank, hi = c->all ? c->P : c->rank + 1;
    Carve cv(ws);
    uint64_t* asum = ttp ? reinterpret_cast<uint64_t*>(cv.take(8 * (size_t)na)) : nullptr;
    uint64_t* bsum = ttp ? reinterpret_cast<uint64_t*>(cv.take(8 * (size_t)nb)) : nullptr;
    uint8_t* a_pl = ttp ? cv.take(lp(g.M(), g.K())) : nullptr;
    uint8_t* b_pl = ttp ? cv.take(rp(g.Cout, g.K())) : nullptr;
    const size_t pb = ring_gemm_partials_bytes(1, g.M(), g.Cout, (int)num_kb(g.K()));
    uint64_t* partials = reinterpret_cast<uint64_t*>(ttp && pb ? cv.take(pb) : nullptr);
    CHECK(run(c, kClsPrg, "ttp_conv_a", [&] {
        return launch_prg_parties(c->kttp, kTagA, id, c->P, lo, hi, a, asum, na, c->stream); }));
    CHECK(run(c, kClsPrg, "ttp_conv_b", [&] {
        return launch_prg_parties(c->kttp, kTagB, id, c->P, lo, hi, b, bsum, nb, c->stream); }));
    if (nz == 0) return MPC_OK;
    if (ttp) {
        // c = conv(sum a, sum b) into party 0's c slot, on the tensor cores
        Im2colSplitArgs I{g, 0, asum, nullptr, 1, a_pl, nullptr, 0, nullptr, 0, 0};
        CHECK(run(c, kClsSplit, "ttp split im2col", [&] { return launch_split_im2col(I, c->stream); }));
        LeftSplitArgs Wt{g.Cout, g.K(), 0, bsum, nullptr, 1, b_pl, nullptr, 0, nullptr, 0, 1, 0};
        CHECK(run(c, kClsSplit, "ttp split weights", [&] { return launch_split_left(Wt, c->stream); }));
        RingGemmParams p{};
        p.seg[0] = RingGemmSegment{a_pl, b_pl, (int)num_kb(g.K()), 0, 0};
        p.nseg = 1;
        p.M = g.M(); p.N = g.Cout; p.out_hw = g.Ho() * g.Wo();
        p.C = nullptr; p.Z = cc;
        p.partials = partials;
        CHECK(gemm_run(c, p, 1));
    }
    uint64_t* c_out = c->all ? cc + nz : cc;    // parties >= 1
    const int out_lo = c->all ? 1 : c->rank, out_hi = c->all ? c->P : (c->rank == 0 ? 0 : c->rank + 1);
    return run(c, kClsPrg, "ttp_c", [&] {
        return launch_ttp_c(c->kttp, id, c->P, out_lo, out_hi, c_out, ttp ? cc : nullptr, nz, c->stream);
    });
}

// ---------------------------------------------------------------- ReLU
}  // extern "C"
namespace {
// One party per context: leaf binary sharing (0 rounds), then for every height
// of the adder tree 7 XOR reveals between the 8 adder steps, the B2A bit reveal
// (packed, 1 bit per element) and the multiplication's sum reveal.  Work
// buffers live in the context scratch: V [P][n], G and Pr [nodes][n], the
// reveal buffer [4][nodes][n] (>= [2][n]) and the packed bits.
mpc_status relu_one_party(mpc_ctx c, const uint64_t* x, uint64_t* out, int64_t n, uint64_t id, uint64_t* sign_out) {
    std::vector<std::vector<ReluNode>> H;
    relu_tree_nodes(c->P, id, H);
    size_t kmax = 0;
    for (auto& h : H) kmax = std::max(kmax, h.size());
    const size_t un = 8 * (size_t)n;
    const size_t nV = align256(un * c->P), nGP = align256(un * kmax), nED = align256(un * std::max<size_t>(4 * kmax, 2));
    const int64_t nw = relu_zbits_words(n);
    CHECK(ensure_scratch(c, nV + 2 * nGP + nED + align256(8 * (size_t)nw)));
    Carve cv(c->scratch);
    uint64_t* V = reinterpret_cast<uint64_t*>(cv.take(un * c->P));
    uint64_t* G = reinterpret_cast<uint64_t*>(cv.take(un * kmax));
    uint64_t* Pr = reinterpret_cast<uint64_t*>(cv.take(un * kmax));
    uint64_t* ED = reinterpret_cast<uint64_t*>(cv.take(un * std::max<size_t>(4 * kmax, 2)));
    uint64_t* zb = reinterpret_cast<uint64_t*>(cv.take(8 * (size_t)nw));
    const int P = c->P, p = c->rank;
    CHECK(run(c, kClsSplit, "relu_leaf", [&] { return launch_relu_leaf(c->kp, P, p, id, x, V, n, c->stream); }));
    for (auto& nodes : H) {
        ReluAdderArgs a{};
        a.kttp = c->kttp; a.P = P; a.p = p; a.nnodes = (int)nodes.size();
        for (int k = 0; k < a.nnodes; ++k) a.node[k] = nodes[k];
        a.V = V; a.G = G; a.Pr = Pr; a.ED = ED; a.n = n;
        for (int l = 0; l <= 7; ++l) {
            CHECK(run(c, kClsSplit, "relu_adder", [&] { return launch_relu_adder_step(a, l, c->stream); }));
            if (l == 7) break;
            const size_t words = (size_t)n * a.nnodes * ((l == 0 || l == 6) ? 2 : 4);
            c->bytes += 8ull * words;
            CHECK(comm_allreduce(c, ED, ED, words, RedOp::XorU64, "relu AND reveal"));
        }
    }
    CHECK(run(c, kClsSplit, "relu_b2a",
              [&] { return launch_relu_b2a_mask(c->kttp, P, p, id, V, zb, n, c->stream); }));
    c->bytes += 8ull * (uint64_t)nw;
    CHECK(comm_allreduce(c, zb, zb, (size_t)nw, RedOp::XorU64, "relu B2A reveal"));
    CHECK(run(c, kClsSplit, "relu_b2a_mul",
              [&] { return launch_relu_b2a_mul_mask(c->kttp, P, p, id, zb, x, ED, sign_out, n, c->stream); }));
    c->bytes += 16ull * (uint64_t)n;
    CHECK(comm_allreduce(c, ED, ED, 2 * (size_t)n, RedOp::SumU64, "relu multiplication reveal"));
    return run(c, kClsSplit, "relu_mul",
               [&] { return launch_relu_mul_finish(c->kttp, P, p, id, ED, out, n, c->stream); });
}
}  // namespace
extern "C" {

mpc_status mpc_relu(mpc_ctx c, const uint64_t* x, uint64_t* out, int64_t n, uint64_t relu_id, uint64_t* sign_out) {
    CHECK(enter(c));
    CHECK(need_ttp(c, "relu"));
    if (n < 0) return fail(c, MPC_ERR_SHAPE, "relu: n < 0");
    if (relu_id >> 32) return fail(c, MPC_ERR_ARG, "relu: relu_id must be < 2^32 (R24 gate ids)");
    if (c->all && c->P > 8) return fail(c, MPC_ERR_UNSUPPORTED, "relu: at most 8 parties on one device");
    int levels = 0;
    for (int q = 1; q < c->P; q *= 2) levels++;
    c->rounds += (uint64_t)(7 * levels + 2);       // A2B adders, B2A, multiplication (R25)
    if (n == 0) return MPC_OK;
    if (!x || !out) return fail(c, MPC_ERR_ARG, "relu: null pointer");
    if (c->all)
        return run(c, kClsSplit, "relu",
                   [&] { return launch_relu_all(c->kp, c->kttp, relu_id, c->P, x, out, sign_out, n, c->stream); });
    return relu_one_party(c, x, out, n, relu_id, sign_out);
}

mpc_status mpc_profile_enable(mpc_ctx c, int enable) {
    if (!c) return MPC_ERR_ARG;
    c->prof = enable != 0;
    return MPC_OK;
}

mpc_status mpc_profile_read(mpc_ctx c, int cls, double* total_ms, uint64_t* launches) {
    if (!c || cls < 0 || cls > 5) return MPC_ERR_ARG;
    cudaSetDevice(c->device);
    cudaError_t e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) return fail(c, MPC_ERR_CUDA, "profile_read: %s", cudaGetErrorString(e));
    for (auto& ev : c->pending) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ev.a, ev.b);
        c->prof_ms[ev.cls] += ms;
        c->prof_n[ev.cls] += 1;
        c->pool.push_back(ev.a);
        c->pool.push_back(ev.b);
    }
    c->pending.clear();
    if (total_ms) *total_ms = c->prof_ms[cls];
    if (launches) *launches = c->prof_n[cls];
    c->prof_ms[cls] = 0;
    c->prof_n[cls] = 0;
    return MPC_OK;
}

uint64_t mpc_launch_count(mpc_ctx c) { return c ? c->launches : 0; }

}  // extern "C"

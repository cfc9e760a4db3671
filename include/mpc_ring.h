/*
 * mpc_ring.h — C-ABI of the B200-native Beaver ring-GEMM library
 * (libmpc_ring.so, built from paper_2109_00984_b200/csrc).
 *
 * What it computes: the arithmetic-secret-sharing hot path of CrypTen
 * (arXiv 2109.00984), in the ring Z/QZ with Q = 2^64 (§7) and
 * fixed-point scale 2^f, f = 16 by default (PAPER.md:176-177 §4.1, :244 §7).
 * "P:n" below cites /root/reference/PAPER.md line n; DESIGN.md lists every
 * reading (R1..R19) taken where the paper is silent.
 *
 * Conventions shared by every entry point
 * ----------------------------------------
 * Memory.   Every tensor argument is a caller-owned CUDA DEVICE buffer on the
 *           context's device (torch tensors in practice), row-major, 8-byte
 *           aligned; ring elements are little-endian uint64.  The library never
 *           allocates or frees caller memory.  Work buffers are passed in as
 *           `workspace` (size from mpc_workspace_bytes / mpc_ttp_workspace_bytes,
 *           256-byte aligned).  workspace == NULL with workspace_bytes == 0 asks
 *           mpc_ttp_triples, mpc_beaver_matmul(_batched), mpc_beaver_finish and
 *           mpc_ring_matmul to use a workspace the context allocates, grows and
 *           frees in mpc_destroy (stream-ordered; the one library-owned buffer).
 * Parties.  A context is either
 *             - one party of P (rank in [0, P)): one process and one GPU per
 *               party, reveals are NCCL sum-allreduces (P:64, P:72 footnote,
 *               P:377-378); every share argument is that party's share, or
 *             - all P parties on one device (rank == MPC_ALL_PARTIES): every
 *               share argument is P contiguous party buffers, layout [P][n];
 *               reveals are local sums.  Bit-identical results either way.
 * Streams.  All calls are asynchronous and stream-ordered on the stream set by
 *           mpc_set_stream (default: the legacy default stream).  Outputs are
 *           valid once that stream has synchronised.
 * Errors.   Every call returns an mpc_status and never throws across the ABI.
 *           Argument / shape / overflow errors are detected on the host before
 *           any launch and leave outputs untouched.  CUDA / NCCL failures return
 *           MPC_ERR_CUDA / MPC_ERR_NCCL; the message is in mpc_last_error().  After
 *           a failed collective the context is in MPC_ERR_STATE: only
 *           mpc_destroy is allowed.
 * Contract. Every party calls the same sequence of collective entry points with
 *           the same sizes ("synchronization point").  With the environment
 *           variable MPC_CHECK_COLLECTIVES=1 at mpc_create, each NCCL collective is
 *           preceded by a min/max allreduce of a (sequence, op, size) word and a
 *           mismatch returns MPC_ERR_SHAPE (debug aid: it synchronises the stream);
 *           the in-process party group always checks.
 * Rounds.   mpc_stats counts communication rounds (Table 3): reveal = 1,
 *           beaver_matmul = 1, truncation = 0 for P <= 2 and 1 for P > 2.
 * Ids.      share_id / triple_id / wrap_id are caller-chosen 48-bit ids that select
 *           PRG streams (R5): equal seeds and ids give bit-identical
 *           shares.  Triples and wrap pairs are single-use.
 */
#ifndef MPC_RING_H
#define MPC_RING_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mpc_ctx_s* mpc_ctx;               /* opaque, library-owned */

typedef enum {
    MPC_OK = 0,
    MPC_ERR_ARG = 1,          /* bad pointer / enum / id / rank */
    MPC_ERR_SHAPE = 2,        /* negative or inconsistent sizes, workspace too small */
    MPC_ERR_OVERFLOW = 3,     /* encode: |x| * 2^f >= 2^63 or NaN (R3) */
    MPC_ERR_CUDA = 4,
    MPC_ERR_NCCL = 5,
    MPC_ERR_STATE = 6,        /* context unusable after an earlier collective failure */
    MPC_ERR_UNSUPPORTED = 7   /* no sm_100a device, or a mode this build does not have */
} mpc_status;

#define MPC_ALL_PARTIES (-1)

/* ---- context ------------------------------------------------------------
 * world_size P in [1, 16]; rank in [0, P) or MPC_ALL_PARTIES.  nccl_id: the
 * 128-byte ncclUniqueId created by rank 0 (mpc_nccl_unique_id) and broadcast by
 * the caller (through torch.distributed); ignored when rank == MPC_ALL_PARTIES or
 * P == 1.  NULL with one party of P > 1 creates a context WITHOUT a communicator:
 * the local steps (share, ttp_triples, ttp_wrap_pairs, encode/decode, local
 * truncation) work, every call that needs a reveal returns MPC_ERR_STATE.
 * master_seed: every PRZS / TTP key is derived from it (R5; "sync random
 * seeds").  frac_bits f in [1, 30] (default 16).  Fails with
 * MPC_ERR_UNSUPPORTED if `device` is not a compute-capability 10.0 GPU. */
mpc_status mpc_create(mpc_ctx* out, int world_size, int rank, int device,
                      const void* nccl_id, uint64_t master_seed, int frac_bits);

/* ---- explicit keys (one party per process) ---------------------------------
 * SECURITY NOTE.  mpc_create derives EVERY party's PRZS key and the TTP key from
 * master_seed (the reproducibility convention of DESIGN.md R5, which lets the
 * oracle and the GPU agree bit for bit).  A party holding the master seed can
 * therefore regenerate a = sum a_p and b = sum b_p and unmask x = eps + a,
 * y = delta + b: mpc_create is for benchmarks and tests, NOT a private
 * deployment.  A deployment agrees keys at set-up ("sync random seeds"):
 *   przs_self  k_p, shared by party p and party p+1 (mod P),
 *   przs_prev  k_{p-1}, shared by party p-1 and party p (P = 1: equal to przs_self),
 *   ttp        k_ttp, held by the dealer only (has_ttp = 0 on a computing party).
 * mpc_create_with_keys creates one party (rank in [0, P), never MPC_ALL_PARTIES)
 * that knows only these keys.  Without k_ttp the context cannot generate TTP
 * material: mpc_ttp_* , mpc_truncate (wrap pair from an id) and mpc_relu return
 * MPC_ERR_STATE; the triples are passed in as arguments, and the P > 2 truncation
 * takes its wrap pair with mpc_truncate_pairs.  Shares are bit-identical to an
 * mpc_create context whose master seed derives the same keys (mpc_derive_keys
 * returns rank's keys under the R5 convention).  MPC_ERR_ARG for a bad rank,
 * NULL keys, or P = 1 with przs_self != przs_prev. */
typedef struct {
    uint64_t przs_self;
    uint64_t przs_prev;
    uint64_t ttp;
    int has_ttp;
} mpc_keys;
mpc_status mpc_derive_keys(uint64_t master_seed, int world_size, int rank, mpc_keys* out);
mpc_status mpc_create_with_keys(mpc_ctx* out, int world_size, int rank, int device,
                                const void* nccl_id, const mpc_keys* keys, int frac_bits);
mpc_status mpc_destroy(mpc_ctx ctx);
mpc_status mpc_set_stream(mpc_ctx ctx, void* cuda_stream);
/* One party per GPU: the eps reveal of mpc_beaver_matmul runs in `chunks` row chunks
 * (whole 256-row GEMM tiles), each followed by its share of the GEMM terms that need
 * no delta, while the later chunks and delta are still in flight.
 * chunks in [1, 8], 0 = the default policy (min(4, M / 1024)); capped by the number of
 * row tiles; ignored (1) for the transposed / stacked-plane GEMM orientations and
 * batches.  Shares are bit-identical for every chunk count.  MPC_ERR_ARG outside [0, 8]. */
mpc_status mpc_set_reveal_chunks(mpc_ctx ctx, int chunks);
const char* mpc_last_error(mpc_ctx ctx);      /* never NULL; valid until the next call on ctx */
/* rounds and bytes SENT by this process's party/parties since creation (R19) */
mpc_status mpc_stats(mpc_ctx ctx, uint64_t* rounds, uint64_t* bytes_sent);
/* 1 if ctx is one party per GPU, 0 if all parties share this device */
int mpc_world_size(mpc_ctx ctx);
int mpc_rank(mpc_ctx ctx);
/* Writes a fresh 128-byte ncclUniqueId (rank 0 calls this, then broadcasts it to
 * the other parties before mpc_create).  MPC_ERR_NCCL on failure. */
mpc_status mpc_nccl_unique_id(void* out128);

/* ---- in-process party group (one-party contexts without NCCL) ------------
 * A group joins P one-party contexts of ONE process on one device: their
 * reveals are the same collectives as over NCCL (sum, int8 sum, XOR), done by a
 * host rendezvous plus one reduction kernel launched by the last party to
 * arrive, ordered with CUDA events on each party's stream.  Each party must be
 * driven by its own host thread (a collective blocks its caller until all P
 * parties have entered it; after 300 s without them the context fails with
 * MPC_ERR_STATE), and every party must call the same sequence of collective
 * entry points with the same sizes (a mismatch returns MPC_ERR_SHAPE and
 * breaks the group).  Purpose: running the one-party-per-GPU schedule — same
 * kernels, streams and events — for P > 1 parties on a single GPU (tests;
 * the paper's parties are separate processes).
 * mpc_group_create: P in [1, 16].  mpc_create_local: like mpc_create with
 * rank in [0, P) and the group instead of an NCCL id; MPC_ERR_ARG if the rank
 * is already attached.  The group must outlive its contexts (destroy the
 * contexts first). */
typedef struct mpc_group_s* mpc_group;           /* opaque, library-owned */
mpc_status mpc_group_create(mpc_group* out, int world_size);
mpc_status mpc_group_destroy(mpc_group group);
mpc_status mpc_create_local(mpc_ctx* out, mpc_group group, int rank, int device,
                            uint64_t master_seed, int frac_bits);

/* ---- fixed point (§4.1; App. A.1.1) ----------------
 * encode: out[i] = round_half_away(x[i] * 2^f) as two's complement u64;
 *   MPC_ERR_OVERFLOW if any |x[i]| * 2^f >= 2^63 or NaN (checked on the device;
 *   the call synchronises the stream to report it).  Public values, not shares.
 * decode: out[i] = (double)(int64)v[i] / 2^f. */
mpc_status mpc_encode(mpc_ctx ctx, const double* x, uint64_t* out, int64_t n);
/* encode without the synchronising check (for pipelined callers): an overflow or
 * NaN sets a sticky device flag of the context (that element's output is
 * unspecified); mpc_check_overflow synchronises the stream, returns
 * MPC_ERR_OVERFLOW if the flag was set since the last check, and clears it. */
mpc_status mpc_encode_async(mpc_ctx ctx, const double* x, uint64_t* out, int64_t n);
mpc_status mpc_check_overflow(mpc_ctx ctx);
mpc_status mpc_decode(mpc_ctx ctx, const uint64_t* v, double* out, int64_t n);

/* ---- share: pseudorandom zero-share + src adds x (§4.1) ------
 * [x]_p[i] = G(k_p, PRZS||0||share_id)[i] - G(k_{p-1 mod P}, PRZS||0||share_id)[i]
 *            + [p == src] * x[i]                                     (0 rounds)
 * x_or_null: n ring elements held by party `src` (read only by src; NULL allowed for
 * other ranks).  share_out: n (one party) or [P][n] (all parties). */
mpc_status mpc_share(mpc_ctx ctx, const uint64_t* x_or_null, int src, uint64_t share_id,
                     uint64_t* share_out, int64_t n);

/* ---- reveal: x = sum_p [x]_p mod 2^64 (Fig. 2) -------
 * share: n or [P][n]; out: n.  1 round (NCCL uint64 sum-allreduce), 8n bytes sent. */
mpc_status mpc_reveal(mpc_ctx ctx, const uint64_t* share, uint64_t* out, int64_t n);

/* ---- offline TTP: Beaver matmul triple -----
 * a_p = G(k_ttp, A||p||id) (M x K), b_p = G(k_ttp, B||p||id) (K x N),
 * c = (sum a_p) @ (sum b_p) mod 2^64 computed by the ring GEMM, c_p = G(k_ttp, C||p||id)
 * for p >= 1, c_0 = c - sum_{p>=1} c_p  (R6).  a, b, c: this party's
 * (or [P][..] for all parties).  In the one-party-per-GPU mode rank 0 also acts as the
 * TTP and regenerates every party's a_q, b_q to form c_0.  workspace: at least
 * mpc_ttp_workspace_bytes(ctx, M, K, N) bytes (only rank 0 / all-parties use it). */
size_t mpc_ttp_workspace_bytes(mpc_ctx ctx, int64_t M, int64_t K, int64_t N);
mpc_status mpc_ttp_triples(mpc_ctx ctx, uint64_t triple_id, int64_t M, int64_t K, int64_t N,
                           uint64_t* a, uint64_t* b, uint64_t* c,
                           void* workspace, size_t workspace_bytes);

/* ---- offline TTP: wrap pair for Alg. 1 (DESIGN.md a9) ---------
 * r_p = G(k_ttp, R||p||id); theta_r = (sum signed(r_p) - signed(sum r_p)) / 2^64;
 * [theta_r]_p = G(k_ttp, THETA||p||id) for p >= 1, [theta_r]_0 = theta_r - sum_{p>=1}.
 * mpc_truncate regenerates exactly these values from wrap_id; this entry point
 * materialises them for mpc_truncate_pairs (the offline phase). */
mpc_status mpc_ttp_wrap_pairs(mpc_ctx ctx, uint64_t wrap_id, int64_t n,
                              uint64_t* r, uint64_t* theta_r);

/* ---- Beaver private matmul (§4.2; App. A.1.1) -------
 * e_p = x_p - a_p, d_p = y_p - b_p; eps = sum e_p, delta = sum d_p (one round);
 * z_p = c_p + eps @ b_p + a_p @ delta + [p == 0] eps @ delta  (R7, R8),
 * then, if truncate != 0, fixed-point truncation by 2^f: local
 * per-share round-half-up division for P <= 2 (P:597, 0 rounds), Alg. 1
 * with eta skipped for P > 2 (P:606-663, 1 more round) using wrap pair wrap_id.
 * x: M x K, y: K x N, a: M x K, b: K x N, c and z: M x N (per party, or [P][..]).
 * z may not alias any input.  workspace >= mpc_workspace_bytes(ctx, M, K, N).
 * The ring GEMM is the tcgen05 u8-limb kernel (36 limb pairs). */
size_t mpc_workspace_bytes(mpc_ctx ctx, int64_t M, int64_t K, int64_t N);
mpc_status mpc_beaver_matmul(mpc_ctx ctx, const uint64_t* x, const uint64_t* y,
                             const uint64_t* a, const uint64_t* b, const uint64_t* c,
                             uint64_t* z, int64_t M, int64_t K, int64_t N,
                             int truncate, uint64_t wrap_id,
                             void* workspace, size_t workspace_bytes);

/* ---- the same matmul with its round made explicit (one-party contexts) ----
 * For callers that reveal with their own communicator (and for testing the
 * one-party kernels without NCCL):
 *   mpc_beaver_mask:   ed = [x - a | y - b]   (M*K + K*N u64; 0 rounds, local)
 *   -- caller: ed <- sum over parties of ed (mod 2^64), i.e. [eps | delta]  (1 round)
 *   mpc_beaver_finish: z = c_p + a_p @ delta + eps @ (b_p + [p == 0] delta), truncated
 *                      locally if truncate != 0 (P <= 2 only; for P > 2 call
 *                      mpc_truncate, which needs the communicator).
 * Result identical to mpc_beaver_matmul.  MPC_ERR_UNSUPPORTED on an all-parties
 * context.  workspace: mpc_workspace_bytes(ctx, M, K, N). */
mpc_status mpc_beaver_mask(mpc_ctx ctx, const uint64_t* x, const uint64_t* y, const uint64_t* a,
                           const uint64_t* b, uint64_t* ed, int64_t M, int64_t K, int64_t N);
mpc_status mpc_beaver_finish(mpc_ctx ctx, const uint64_t* ed, const uint64_t* a, const uint64_t* b,
                             const uint64_t* c, uint64_t* z, int64_t M, int64_t K, int64_t N,
                             int truncate, void* workspace, size_t workspace_bytes);

/* ---- a batch of independent Beaver matmuls of one shape -------
 * z[i] = x[i] @ y[i] for i < batch (e.g. the heads of an attention layer), as
 * mpc_beaver_matmul on each i with triple (a[i], b[i], c[i]) — bit-identical — but
 * every eps || delta of the batch in ONE reveal round and one split + one ring
 * GEMM launch for the whole batch (the GEMM walks batch x parties instances).
 * Layout: x [P][batch][M][K], y [P][batch][K][N], a like x, b like y, c and z
 * [P][batch][M][N] for all-parties contexts; without the leading P for one party.
 * workspace: mpc_workspace_bytes_batched(ctx, batch, M, K, N).  Rounds: 1 (+1 for
 * Alg. 1 when P > 2 and truncate).  batch <= 65536; errors as mpc_beaver_matmul. */
size_t mpc_workspace_bytes_batched(mpc_ctx ctx, int64_t batch, int64_t M, int64_t K, int64_t N);
mpc_status mpc_beaver_matmul_batched(mpc_ctx ctx, int64_t batch, const uint64_t* x, const uint64_t* y,
                                     const uint64_t* a, const uint64_t* b, const uint64_t* c, uint64_t* z,
                                     int64_t M, int64_t K, int64_t N, int truncate, uint64_t wrap_id,
                                     void* workspace, size_t workspace_bytes);

/* ---- the Beaver matmul in two halves: weights known ahead ------
 * mpc_beaver_prepare is the input-independent y side: d_p = y_p - b_p, delta =
 * reveal(d) (1 round, 8KN bytes), and the limb planes of delta and of
 * b'_p = b_p + [p = 0] delta, kept in `workspace`.  mpc_beaver_matmul_prepared is
 * the x side on the SAME workspace: eps = reveal(x - a) (1 round, 8MK bytes),
 * the split of eps and a_p, the ring GEMM z_p = c_p + a_p @ delta + eps @ b'_p and
 * the truncation (+ Alg. 1's round when P > 2 and truncate).  Together they give
 * exactly mpc_beaver_matmul's shares for the same inputs and triple.  delta
 * depends only on y and the triple, so a model's weight-side prepares can run
 * ahead of the activations — e.g. on another stream beside the previous
 * layer's GEMM; one workspace per prepared operand (mpc_workspace_bytes(M, K, N)
 * bytes; M, K, N must be the same in both calls — M fixes the GEMM orientation),
 * not reused before the prepared matmul has run.  One-party contexts: delta is
 * revealed in prepare; the prepared matmul reveals eps on the comm stream while
 * a_p @ delta already runs.  Errors as mpc_beaver_matmul. */
mpc_status mpc_beaver_prepare(mpc_ctx ctx, const uint64_t* y, const uint64_t* b, int64_t M, int64_t K, int64_t N,
                              void* workspace, size_t workspace_bytes);
mpc_status mpc_beaver_matmul_prepared(mpc_ctx ctx, const uint64_t* x, const uint64_t* a, const uint64_t* c,
                                      uint64_t* z, int64_t M, int64_t K, int64_t N, int truncate,
                                      uint64_t wrap_id, void* workspace, size_t workspace_bytes);

/* ---- truncation by 2^bits (App. A.1.1 "Truncation") ----------
 * In place on x (n or [P][n]).  bits in [1, 62].  P <= 2: out_p =
 * (signed(x_p) >> bits) + bit_{bits-1}(x_p) (0 rounds).  P > 2: Alg. 1 with the wrap
 * pair wrap_id, eta skipped (1 round). */
mpc_status mpc_truncate(mpc_ctx ctx, uint64_t* x_inout, int64_t n, int bits, uint64_t wrap_id);
/* The same truncation with the wrap pair passed in (Alg. 1's inputs [r], [theta_r],
 * P:606-612), as materialised offline by mpc_ttp_wrap_pairs: r and theta_r hold this
 * party's shares (n) or every party's ([P][n]).  The online step then reads the pair
 * instead of regenerating it from k_ttp (no TTP work on party 0's critical path; works
 * on a context without k_ttp).  Result bit-identical to mpc_truncate with the pair's
 * wrap_id.  P <= 2 ignores r / theta_r (local truncation).  Each pair is single-use. */
mpc_status mpc_truncate_pairs(mpc_ctx ctx, uint64_t* x_inout, int64_t n, int bits, const uint64_t* r,
                              const uint64_t* theta_r);

/* ---- plain ring GEMM C = A @ B mod 2^64 (building block of ttp_triples) ---
 * A: M x K, B: K x N, C: M x N, device buffers; not a protocol step (no shares).
 * workspace >= mpc_ring_matmul_workspace_bytes(M, K, N). */
size_t mpc_ring_matmul_workspace_bytes(int64_t M, int64_t K, int64_t N);
mpc_status mpc_ring_matmul(mpc_ctx ctx, const uint64_t* A, const uint64_t* B, uint64_t* C,
                           int64_t M, int64_t K, int64_t N, void* workspace, size_t workspace_bytes);

/* ---- elementwise private multiplication and square --
 * App. A.1.1 P:575-594 ("Multiplication", "Square").  All buffers n elements per
 * party ([P][n] on an all-parties context), caller-owned device memory.
 *
 * mpc_ttp_mul_triples: a_p = G(k_ttp, A||p||id), b_p = G(k_ttp, B||p||id),
 *   c = (sum a_p)(sum b_p) elementwise, c_p = G(k_ttp, C||p||id) for p >= 1,
 *   c_0 = c - sum_{p>=1} c_p (R6, R21).  Offline; 0 rounds.
 * mpc_ttp_square_pairs: the Beaver pair of P:592, b = a^2: a_p as above, b_p
 *   (p >= 1) from the C stream, b_0 = a^2 - sum_{p>=1} b_p (R20).
 * mpc_beaver_mul: e_p = x_p - a_p, d_p = y_p - b_p; [eps | delta] revealed in ONE
 *   batched round; z_p = c_p + eps b_p + a_p delta + [p == 0] eps delta, then the
 *   truncation of mpc_beaver_matmul (local for P <= 2, Alg. 1 with wrap_id for P > 2).
 * mpc_beaver_square: e_p = x_p - a_p; eps revealed (one round);
 *   z_p = b_p + 2 eps a_p + [p == 0] eps^2, then truncation as above.
 * z must not alias an input.  One-party contexts use the context's scratch for
 * the reveal buffer.  Errors: MPC_ERR_SHAPE (n < 0), MPC_ERR_ARG (null pointer),
 * MPC_ERR_STATE (P > 1 one-party context without communicator), MPC_ERR_NCCL. */
mpc_status mpc_ttp_mul_triples(mpc_ctx ctx, uint64_t triple_id, int64_t n, uint64_t* a, uint64_t* b, uint64_t* c);
mpc_status mpc_ttp_square_pairs(mpc_ctx ctx, uint64_t pair_id, int64_t n, uint64_t* a, uint64_t* b);
mpc_status mpc_beaver_mul(mpc_ctx ctx, const uint64_t* x, const uint64_t* y, const uint64_t* a,
                          const uint64_t* b, const uint64_t* c, uint64_t* z, int64_t n,
                          int truncate, uint64_t wrap_id);
mpc_status mpc_beaver_square(mpc_ctx ctx, const uint64_t* x, const uint64_t* a, const uint64_t* b,
                             uint64_t* z, int64_t n, int truncate, uint64_t wrap_id);
/* The same with the round made explicit (one-party contexts, as mpc_beaver_finish):
 * the caller forms [x - a | y - b] (mpc_beaver_mask with M = 1, K = n, N = 1; for the
 * square N = 0), sums it over the parties (one round) and passes the revealed
 * [eps | delta] (square: eps) here.  Local truncation only (P <= 2).
 * MPC_ERR_UNSUPPORTED on an all-parties context. */
mpc_status mpc_beaver_mul_finish(mpc_ctx ctx, const uint64_t* ed, const uint64_t* a, const uint64_t* b,
                                 const uint64_t* c, uint64_t* z, int64_t n, int truncate);
mpc_status mpc_beaver_square_finish(mpc_ctx ctx, const uint64_t* eps, const uint64_t* a, const uint64_t* b,
                                    uint64_t* z, int64_t n, int truncate);

/* ---- batched multi-tensor reveal (one round) --------------------------------
 * out_t = sum over parties of share_t (mod 2^64) for t < count, counted as ONE
 * round (collectives issued without a data-dependent wait): one NCCL
 * group of allreduces on one-party contexts, local sums on all-parties contexts
 * (share_t is then [P][n_t]).  shares / outs / ns: host arrays of count entries. */
mpc_status mpc_reveal_batch(mpc_ctx ctx, int count, const uint64_t* const* shares, uint64_t* const* outs,
                            const int64_t* ns);

/* ---- private 2-D convolution with conv triples ------
 * P:589-590 ("the same procedure to perform matrix multiplication and
 * convolution"); R22.  Geometry: input x (B, C, H, W), weights
 * y (Cout, C, kh, kw), zero padding (ph, pw), stride (sh, sw), no dilation, one
 * group; output z (B, Cout, Ho, Wo), Ho = (H + 2ph - kh)/sh + 1 (NCHW, row-major).
 * Per party (or [P][..] on an all-parties context).
 *
 * mpc_ttp_conv_triples: a_p = G(k_ttp, A||p||id) over the B*C*H*W input elements,
 *   b_p = G(k_ttp, B||p||id) over the weight elements, c = conv(sum a_p, sum b_p),
 *   c_p = G(k_ttp, C||p||id) (p >= 1), c_0 = c - sum_{p>=1} c_p.  Offline.  workspace:
 *   mpc_ttp_conv_workspace_bytes (rank 0 / all-parties only).
 * mpc_beaver_conv2d: e_p = x_p - a_p (input shape), d_p = y_p - b_p (weight shape),
 *   [eps | delta] revealed in ONE round at those shapes (not at the im2col shape);
 *   z_p = c_p + conv(a_p, delta) + conv(eps, b_p + [p == 0] delta) on the ring GEMM
 *   with the implicit im2col written straight into limb planes; truncation as in
 *   mpc_beaver_matmul.  workspace: mpc_conv2d_workspace_bytes.
 * mpc_beaver_conv2d_finish: the same after the caller's reveal of
 *   ed = [eps | delta] (na + nb u64, formed by mpc_mask); one-party contexts; local
 *   truncation only.
 * mpc_mask: ed = [x - a | y - b] for any n1, n2 (0 rounds).
 * 1-D convolutions (Wav2Letter): the H = kh = 1 case, ph = 0, sh = 1 —
 * x (B, C, L) and w (Cout, C, k) have exactly the memory layout of (B, C, 1, L) and
 * (Cout, C, 1, k), so every entry point below serves them unchanged.
 * Errors: MPC_ERR_SHAPE (invalid geometry / workspace), MPC_ERR_ARG (null pointer). */
typedef struct {
    int64_t B, C, H, W, Cout, kh, kw, sh, sw, ph, pw;
} mpc_conv2d_geom;
size_t mpc_ttp_conv_workspace_bytes(mpc_ctx ctx, const mpc_conv2d_geom* geom);
mpc_status mpc_ttp_conv_triples(mpc_ctx ctx, uint64_t triple_id, const mpc_conv2d_geom* geom,
                                uint64_t* a, uint64_t* b, uint64_t* c, void* workspace, size_t workspace_bytes);
size_t mpc_conv2d_workspace_bytes(mpc_ctx ctx, const mpc_conv2d_geom* geom);
mpc_status mpc_beaver_conv2d(mpc_ctx ctx, const mpc_conv2d_geom* geom, const uint64_t* x, const uint64_t* y,
                             const uint64_t* a, const uint64_t* b, const uint64_t* c, uint64_t* z,
                             int truncate, uint64_t wrap_id, void* workspace, size_t workspace_bytes);
mpc_status mpc_beaver_conv2d_finish(mpc_ctx ctx, const mpc_conv2d_geom* geom, const uint64_t* ed,
                                    const uint64_t* a, const uint64_t* b, const uint64_t* c, uint64_t* z,
                                    int truncate, void* workspace, size_t workspace_bytes);
mpc_status mpc_mask(mpc_ctx ctx, const uint64_t* x, const uint64_t* a, int64_t n1, const uint64_t* y,
                    const uint64_t* b, int64_t n2, uint64_t* ed);

/* ---- ReLU ----------------------
 * out = shares of ReLU(x) = [x] * [x >= 0] for x, out: n per party ([P][n]).
 * A2B: every party's arithmetic share is binary-shared (binary PRZS) and the P
 * values summed by a tree of Kogge-Stone adders with binary Beaver ANDs
 * (App. A.1.2-A.1.3; R23, R24); the sign bit <x> >> 63
 * goes through Alg. 2 (bit pair from the TTP) to [x < 0], and
 * out = BeaverMul([x], 1 - [x < 0]) (R25) — exact, x's scale, no truncation.
 * Rounds: ceil(log2 P)*7 + 2.  relu_id (< 2^32) selects every stream (binary
 * zero-shares, binary triples, bit pair, multiplication triple); single-use.
 * sign_out (optional, same shape) receives the shares of [x < 0].
 * All-parties contexts, P <= 8: one fused kernel, every reveal a local XOR / sum.
 * One-party contexts, P <= 16: round by round over the transport — per height of
 * the adder tree 7 XOR reveals (NCCL: all-gather + local XOR), the B2A bit
 * reveal (1 bit per element, packed) and the multiplication's sum reveal;
 * rank 0 also generates the TTP's correction words.  Work buffers come from
 * the context (8n(P + 6 floor(P/2)) bytes at most).  Both modes give
 * bit-identical shares. */
mpc_status mpc_relu(mpc_ctx ctx, const uint64_t* x, uint64_t* out, int64_t n, uint64_t relu_id, uint64_t* sign_out);

/* ---- measurement hooks (bench.py) ----------------------------------------
 * When enabled, the library brackets every launch of kernel class `cls` with CUDA
 * events on the launching stream and accumulates its device time.
 * cls: 0 = ring GEMM (tcgen05), 1 = limb split / mask / local reveal,
 *      2 = truncation, 3 = PRG (share / triples / wrap pairs), 4 = encode/decode,
 *      5 = collectives (NCCL).  mpc_profile_read synchronises the stream.
 * mpc_launch_count: number of the library's own kernel launches since creation. */
mpc_status mpc_profile_enable(mpc_ctx ctx, int enable);
mpc_status mpc_profile_read(mpc_ctx ctx, int cls, double* total_ms, uint64_t* launches);
uint64_t mpc_launch_count(mpc_ctx ctx);

#ifdef __cplusplus
}
#endif
#endif /* MPC_RING_H */

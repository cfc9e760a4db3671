/*
 * oracle/oracle.c — plain, slow, obviously-correct CPU oracle for the CrypTen
 * Beaver ring-GEMM hot path (arXiv 2109.00984).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or constant generator with the CUDA path
 * (paper_2109_00984_b200/csrc); neither side includes or links the other.
 *
 * Every function simulates ALL |P| parties in one process.  Party-indexed
 * buffers are laid out [P][n] (party-major, row-major inside each party).
 * Arithmetic is in the ring Z/QZ with Q = 2^64 (§7 "the size of
 * the ring, Q = 2^64"): uint64_t wrap-around IS the ring.  Signed
 * representatives are int64_t two's complement (reading R9).
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n (section named beside
 * it); "S:n" = SPEC.md line n; "§8(c) Ox" = the oracle step in SURVEY.md.
 *
 * Parity pins (tests/test_oracle_*.py): Philox KAT vectors, the frozen PRG
 * table, numpy uint64 matmul, Python big-int brute force, the paper's own
 * §4.3 float64 16-bit-block GEMM, the Beaver identity, the P=1 closed form,
 * the Alg. 1 identity against big-int recomputation; the elementwise product
 * and square (O9-O12) against big-int identities and SPEC's examples
 * (tests/test_oracle_elementwise.py).  "Parity unpinned": only
 * the *choice* of PRG layout (the paper allows any PRG); it is pinned
 * to the frozen table in SURVEY.md Appendix A.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#include <omp.h>

typedef __int128 i128;

#define ORACLE_OK 0
#define ORACLE_ERR_ARG 1
#define ORACLE_ERR_OVERFLOW 3

/* ------------------------------------------------------------------------
 * O1  PRG: Philox4x32-10 (Salmon et al., SC'11 "Random123").  The paper only
 * asks for seeded pseudorandomness ("sync random seeds", Fig. 2;
 * "pseudorandom zero-share", §4.1); the primitive and the counter layout
 * are our reading R5, frozen in SURVEY.md §8(c) O1.
 * ---------------------------------------------------------------------- */
void oracle_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4])
{
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; round++) {
        if (round > 0) {            /* key schedule: Weyl sequence bump */
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* stream word = tag<<56 | party<<48 | (id mod 2^48)   (§8(c) O1) */
uint64_t oracle_stream_id(uint32_t tag, uint32_t party, uint64_t id)
{
    return ((uint64_t)(tag & 0xFFu) << 56) | ((uint64_t)(party & 0xFFu) << 48)
         | (id & 0xFFFFFFFFFFFFull);
}

/* G(key, stream)[start .. start+n): element 2j = o1*2^32 + o0, element
 * 2j+1 = o3*2^32 + o2, where (o0..o3) = Philox(ctr = (lo(j), hi(j),
 * lo(stream), hi(stream)), key = (lo(key), hi(key))).  One element at a
 * time, no batching. */
uint64_t oracle_prg_at(uint64_t key, uint64_t stream, uint64_t i)
{
    uint64_t j = i / 2;
    uint32_t ctr[4] = { (uint32_t)j, (uint32_t)(j >> 32), (uint32_t)stream, (uint32_t)(stream >> 32) };
    uint32_t k[2] = { (uint32_t)key, (uint32_t)(key >> 32) };
    uint32_t o[4];
    oracle_philox4x32_10(ctr, k, o);
    if (i % 2 == 0) return ((uint64_t)o[1] << 32) | o[0];
    return ((uint64_t)o[3] << 32) | o[2];
}

void oracle_prg(uint64_t key, uint64_t stream, uint64_t start, int64_t n, uint64_t* out)
{
    for (int64_t t = 0; t < n; t++) out[t] = oracle_prg_at(key, stream, start + (uint64_t)t);
}

/* Keys: k_p = G(master, 0xFF||p||0)[0] (party p's PRZS key),
 *       k_ttp = G(master, 0xFE||0||0)[0].  Reproducibility convention only
 * (§8(c) O1); a deployment agrees these pairwise at init. */
void oracle_derive_keys(uint64_t master, int P, uint64_t* k_party, uint64_t* k_ttp)
{
    for (int p = 0; p < P; p++) k_party[p] = oracle_prg_at(master, oracle_stream_id(0xFF, (uint32_t)p, 0), 0);
    *k_ttp = oracle_prg_at(master, oracle_stream_id(0xFE, 0, 0), 0);
}

enum { TAG_PRZS = 1, TAG_A = 2, TAG_B = 3, TAG_C = 4, TAG_R = 5, TAG_THETA = 6 };

/* ------------------------------------------------------------------------
 * O2  Fixed-point encode / decode (§4.1 "x = ⌊B x_R⌉, B = 2^L";
 * P:563-567 App. A.1.1; default L = 16, §7).  Ties round half away
 * from zero (reading R2); |x|·2^L ≥ 2^63 (or NaN) is an overflow error
 * (reading R3).
 * ---------------------------------------------------------------------- */
int oracle_encode(const double* x, uint64_t* out, int64_t n, int frac_bits)
{
    const double scale = ldexp(1.0, frac_bits);
    for (int64_t i = 0; i < n; i++) {
        double v = x[i] * scale;                 /* exact: power-of-two scale */
        if (!(fabs(v) < 9223372036854775808.0)) return ORACLE_ERR_OVERFLOW;   /* also NaN */
        out[i] = (uint64_t)(int64_t)llround(v);   /* C99 llround: nearest, ties away from 0 */
    }
    return ORACLE_OK;
}

/* decode: x_R ≈ signed(x) / B */
void oracle_decode(const uint64_t* v, double* out, int64_t n, int frac_bits)
{
    const double scale = ldexp(1.0, frac_bits);
    for (int64_t i = 0; i < n; i++) out[i] = (double)(int64_t)v[i] / scale;
}

/* ------------------------------------------------------------------------
 * O3  share via pseudorandom zero-share (§4.1: "the parties
 * generate a pseudorandom zero-share with |P| random numbers that sum to 0.
 * The party that possesses the value x adds x to their share").
 * [x]_p[i] = G(k_p, PRZS||0||id)[i] − G(k_{p−1 mod P}, PRZS||0||id)[i]
 *            + [p = src]·x[i]                                    (reading R4)
 * ---------------------------------------------------------------------- */
/* elements [start, start+n) of the shared tensor (start > 0: a row sample) */
void oracle_share_range(int P, const uint64_t* k_party, const uint64_t* x, int src,
                        uint64_t share_id, int64_t start, int64_t n, uint64_t* shares)
{
    uint64_t stream = oracle_stream_id(TAG_PRZS, 0, share_id);
    for (int p = 0; p < P; p++) {
        int prev = (p + P - 1) % P;
        for (int64_t i = 0; i < n; i++) {
            uint64_t v = oracle_prg_at(k_party[p], stream, (uint64_t)(start + i))
                       - oracle_prg_at(k_party[prev], stream, (uint64_t)(start + i));
            if (p == src && x != NULL) v += x[i];
            shares[(int64_t)p * n + i] = v;
        }
    }
}

void oracle_share(int P, const uint64_t* k_party, const uint64_t* x, int src,
                  uint64_t share_id, int64_t n, uint64_t* shares)
{
    oracle_share_range(P, k_party, x, src, share_id, 0, n, shares);
}

/* O8  reveal: x = Σ_p [x]_p mod Q (§4.1; Fig. 2) */
void oracle_reveal(int P, const uint64_t* shares, int64_t n, uint64_t* out)
{
    for (int64_t i = 0; i < n; i++) {
        uint64_t s = 0;
        for (int p = 0; p < P; p++) s += shares[(int64_t)p * n + i];
        out[i] = s;
    }
}

/* Thread count of the OpenMP loops (timing only: results do not depend on it).
 * bench.py times the oracle with one thread, the paper's CPU setting,
 * and with every host core. */
void oracle_set_threads(int n) { if (n > 0) omp_set_num_threads(n); }
int oracle_get_threads(void) { return omp_get_max_threads(); }

/* ------------------------------------------------------------------------
 * Ring GEMM: C = A @ B mod 2^64, A: M×K, B: K×N, row-major.  The textbook
 * triple loop (i, k, j) with wrapping uint64 multiply-add — the definition
 * of a matrix product in Z/2^64Z.  (The paper computes it with float64
 * blocks, §4.3; that route is a *test* cross-check here.)
 * OpenMP over rows only; each output element is summed in index order.
 * ---------------------------------------------------------------------- */
void oracle_ring_matmul(const uint64_t* A, const uint64_t* B, uint64_t* C,
                        int64_t M, int64_t K, int64_t N)
{
    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t i = 0; i < M; i++) {
        uint64_t* c = C + i * N;
        for (int64_t j = 0; j < N; j++) c[j] = 0;
        for (int64_t k = 0; k < K; k++) {
            uint64_t a = A[i * K + k];
            const uint64_t* b = B + k * N;
            for (int64_t j = 0; j < N; j++) c[j] += a * b[j];
        }
    }
}

/* ------------------------------------------------------------------------
 * O4  TTP Beaver triple for f = matmul (§3 TTP footnote; P:200-201
 * §4.2; App. A.1.1 "generated in an offline preprocessing phase";
 * "holds for any linear function f ... matrix multiplication").
 *   a_p = G(k_ttp, A||p||id), b_p = G(k_ttp, B||p||id) (uniform)
 *   c   = (Σ_p a_p) @ (Σ_p b_p)
 *   c_p = G(k_ttp, C||p||id) for p ≥ 1, c_0 = c − Σ_{p≥1} c_p  (reading R6)
 * rows != NULL selects a subset of the M rows of a and c (same values as
 * the full triple's rows; b is always full).  a: [P][nrows*K], c: [P][nrows*N].
 * ---------------------------------------------------------------------- */
void oracle_ttp_triple(int P, uint64_t k_ttp, uint64_t triple_id,
                       int64_t M, int64_t K, int64_t N,
                       const int64_t* rows, int64_t nrows,
                       uint64_t* a, uint64_t* b, uint64_t* c)
{
    if (rows == NULL) nrows = M;
    for (int p = 0; p < P; p++) {
        uint64_t sa = oracle_stream_id(TAG_A, (uint32_t)p, triple_id);
        uint64_t sb = oracle_stream_id(TAG_B, (uint32_t)p, triple_id);
        for (int64_t r = 0; r < nrows; r++) {
            int64_t i = rows ? rows[r] : r;
            oracle_prg(k_ttp, sa, (uint64_t)(i * K), K, a + (int64_t)p * nrows * K + r * K);
        }
        oracle_prg(k_ttp, sb, 0, K * N, b + (int64_t)p * K * N);
    }
    uint64_t* asum = (uint64_t*)calloc((size_t)(nrows * K > 0 ? nrows * K : 1), 8);
    uint64_t* bsum = (uint64_t*)calloc((size_t)(K * N > 0 ? K * N : 1), 8);
    uint64_t* cfull = (uint64_t*)calloc((size_t)(nrows * N > 0 ? nrows * N : 1), 8);
    oracle_reveal(P, a, nrows * K, asum);
    oracle_reveal(P, b, K * N, bsum);
    oracle_ring_matmul(asum, bsum, cfull, nrows, K, N);
    for (int64_t r = 0; r < nrows * N; r++) c[r] = cfull[r];
    for (int p = 1; p < P; p++) {
        uint64_t sc = oracle_stream_id(TAG_C, (uint32_t)p, triple_id);
        for (int64_t r = 0; r < nrows; r++) {
            int64_t i = rows ? rows[r] : r;
            uint64_t* cp = c + (int64_t)p * nrows * N + r * N;
            oracle_prg(k_ttp, sc, (uint64_t)(i * N), N, cp);
            for (int64_t j = 0; j < N; j++) c[r * N + j] -= cp[j];   /* c_0 −= c_p */
        }
    }
    free(asum); free(bsum); free(cfull);
}

/* The same triple restricted to a sample of rows of a / c and columns of b / c
 * (for checking single outputs of a large product): a: [P][nrows*K],
 * b: [P][K*ncols], c: [P][nrows*ncols], values identical to the full triple's. */
void oracle_ttp_triple_sampled(int P, uint64_t k_ttp, uint64_t triple_id,
                               int64_t M, int64_t K, int64_t N,
                               const int64_t* rows, int64_t nrows, const int64_t* cols, int64_t ncols,
                               uint64_t* a, uint64_t* b, uint64_t* c)
{
    (void)M;
    for (int p = 0; p < P; p++) {
        uint64_t sa = oracle_stream_id(TAG_A, (uint32_t)p, triple_id);
        uint64_t sb = oracle_stream_id(TAG_B, (uint32_t)p, triple_id);
        for (int64_t r = 0; r < nrows; r++)
            oracle_prg(k_ttp, sa, (uint64_t)(rows[r] * K), K, a + (int64_t)p * nrows * K + r * K);
        for (int64_t k = 0; k < K; k++)
            for (int64_t j = 0; j < ncols; j++)
                b[(int64_t)p * K * ncols + k * ncols + j] = oracle_prg_at(k_ttp, sb, (uint64_t)(k * N + cols[j]));
    }
    uint64_t* asum = (uint64_t*)calloc((size_t)(nrows * K > 0 ? nrows * K : 1), 8);
    uint64_t* bsum = (uint64_t*)calloc((size_t)(K * ncols > 0 ? K * ncols : 1), 8);
    oracle_reveal(P, a, nrows * K, asum);
    oracle_reveal(P, b, K * ncols, bsum);
    oracle_ring_matmul(asum, bsum, c, nrows, K, ncols);
    for (int p = 1; p < P; p++) {
        uint64_t sc = oracle_stream_id(TAG_C, (uint32_t)p, triple_id);
        for (int64_t r = 0; r < nrows; r++)
            for (int64_t j = 0; j < ncols; j++) {
                uint64_t v = oracle_prg_at(k_ttp, sc, (uint64_t)(rows[r] * N + cols[j]));
                c[(int64_t)p * nrows * ncols + r * ncols + j] = v;
                c[r * ncols + j] -= v;
            }
    }
    free(asum); free(bsum);
}

/* PRZS shares of selected elements idx[0..n) of a tensor (x_vals = the src
 * party's plaintext values at those indices), same values as oracle_share. */
void oracle_share_indices(int P, const uint64_t* k_party, const uint64_t* x_vals, int src,
                          uint64_t share_id, const int64_t* idx, int64_t n, uint64_t* shares)
{
    uint64_t stream = oracle_stream_id(TAG_PRZS, 0, share_id);
    for (int p = 0; p < P; p++) {
        int prev = (p + P - 1) % P;
        for (int64_t t = 0; t < n; t++) {
            uint64_t v = oracle_prg_at(k_party[p], stream, (uint64_t)idx[t])
                       - oracle_prg_at(k_party[prev], stream, (uint64_t)idx[t]);
            if (p == src && x_vals != NULL) v += x_vals[t];
            shares[(int64_t)p * n + t] = v;
        }
    }
}

/* ------------------------------------------------------------------------
 * O5  Beaver private matmul (§4.2; App. A.1.1):
 *   [ε]_p = [x]_p − [a]_p,  [δ]_p = [y]_p − [b]_p
 *   ε = Σ_p [ε]_p,  δ = Σ_p [δ]_p   ("decrypt ε and δ", one round)
 *   [z]_p = [c]_p + ε@[b]_p + [a]_p@δ + [p = 0]·ε@δ        (
 *           readings R7, R8: party 0 adds the public ε@δ; operand order
 *           ε@b and a@δ for the non-commutative matmul)
 * No truncation here (z is at scale 2^(2f)); see O6/O7.
 * x: [P][M*K], y: [P][K*N], a: [P][M*K], b: [P][K*N], c: [P][M*N].
 * eps_out (M*K), delta_out (K*N), e_out/d_out ([P][..]) may be NULL.
 * ---------------------------------------------------------------------- */
void oracle_beaver_matmul(int P, const uint64_t* x, const uint64_t* y,
                          const uint64_t* a, const uint64_t* b, const uint64_t* c,
                          int64_t M, int64_t K, int64_t N,
                          uint64_t* e_out, uint64_t* d_out,
                          uint64_t* eps_out, uint64_t* delta_out, uint64_t* z)
{
    int64_t nx = M * K, ny = K * N, nz = M * N;
    uint64_t* e = (uint64_t*)malloc((size_t)(P * (nx > 0 ? nx : 1)) * 8);
    uint64_t* d = (uint64_t*)malloc((size_t)(P * (ny > 0 ? ny : 1)) * 8);
    uint64_t* eps = (uint64_t*)malloc((size_t)(nx > 0 ? nx : 1) * 8);
    uint64_t* delta = (uint64_t*)malloc((size_t)(ny > 0 ? ny : 1) * 8);
    uint64_t* t = (uint64_t*)malloc((size_t)(nz > 0 ? nz : 1) * 8);
    for (int p = 0; p < P; p++) {
        for (int64_t i = 0; i < nx; i++) e[p * nx + i] = x[p * nx + i] - a[p * nx + i];
        for (int64_t i = 0; i < ny; i++) d[p * ny + i] = y[p * ny + i] - b[p * ny + i];
    }
    oracle_reveal(P, e, nx, eps);
    oracle_reveal(P, d, ny, delta);
    for (int p = 0; p < P; p++) {
        uint64_t* zp = z + (int64_t)p * nz;
        for (int64_t i = 0; i < nz; i++) zp[i] = c[p * nz + i];
        oracle_ring_matmul(eps, b + (int64_t)p * ny, t, M, K, N);        /* ε@[b]_p */
        for (int64_t i = 0; i < nz; i++) zp[i] += t[i];
        oracle_ring_matmul(a + (int64_t)p * nx, delta, t, M, K, N);      /* [a]_p@δ */
        for (int64_t i = 0; i < nz; i++) zp[i] += t[i];
        if (p == 0) {
            oracle_ring_matmul(eps, delta, t, M, K, N);                  /* ε@δ, party 0 */
            for (int64_t i = 0; i < nz; i++) zp[i] += t[i];
        }
    }
    if (e_out) memcpy(e_out, e, (size_t)(P * nx) * 8);
    if (d_out) memcpy(d_out, d, (size_t)(P * ny) * 8);
    if (eps_out) memcpy(eps_out, eps, (size_t)nx * 8);
    if (delta_out) memcpy(delta_out, delta, (size_t)ny * 8);
    free(e); free(d); free(eps); free(delta); free(t);
}

/* ------------------------------------------------------------------------
 * Per-share division by ℓ = 2^bits with round-half-up on the signed
 * representative: (signed(v) >> bits) + bit_{bits−1}(v)   (reading R10).
 * Arithmetic right shift of int64 written out as floor division.
 * ---------------------------------------------------------------------- */
static uint64_t div_pow2_round(uint64_t v, int bits)
{
    if (bits == 0) return v;
    int64_t s = (int64_t)v;
    int64_t q;
    int64_t den = (int64_t)1 << bits;
    /* floor(s / 2^bits) */
    q = s / den;
    if ((s % den) != 0 && s < 0) q -= 1;
    uint64_t half = (v >> (bits - 1)) & 1u;
    return (uint64_t)q + half;
}

/* O6  truncation, P ≤ 2: "divide the share of each party by ℓ" (P:597
 * App. A.1.1 Truncation); 0 rounds at P = 2 (Table 3 footnote).
 * Fails with probability |x|/Q; see oracle_wrap_count. */
int oracle_truncate_local(int P, const uint64_t* x, int64_t n, int bits, uint64_t* out)
{
    if (bits < 0 || bits > 62 || P < 1) return ORACLE_ERR_ARG;
    for (int64_t i = 0; i < (int64_t)P * n; i++) out[i] = div_pow2_round(x[i], bits);
    return ORACLE_OK;
}

/* θ_x = (Σ_p signed([x]_p) − signed(x)) / Q, exact in 128-bit
 * (definition: x = Σ_p [x]_p − θ_x Q; signed reps, R9). */
void oracle_wrap_count(int P, const uint64_t* x, int64_t n, int64_t* theta)
{
    for (int64_t i = 0; i < n; i++) {
        i128 s = 0;
        uint64_t u = 0;
        for (int p = 0; p < P; p++) { s += (i128)(int64_t)x[(int64_t)p * n + i]; u += x[(int64_t)p * n + i]; }
        i128 diff = s - (i128)(int64_t)u;
        theta[i] = (int64_t)(diff >> 64);      /* diff is an exact multiple of 2^64 */
    }
}

/* Wrap pair for Alg. 1 (inputs "secret shared random value [r] and its wrap
 * count"):  r_p = G(k_ttp, R||p||id);
 *   θ_r = (Σ_p signed(r_p) − signed(Σ_p r_p)) / Q;
 *   [θ_r]_p = G(k_ttp, THETA||p||id) for p ≥ 1, [θ_r]_0 = θ_r − Σ_{p≥1}[θ_r]_p. */
void oracle_wrap_pair(int P, uint64_t k_ttp, uint64_t wrap_id, int64_t n,
                      uint64_t* r, uint64_t* theta_r)
{
    for (int p = 0; p < P; p++)
        oracle_prg(k_ttp, oracle_stream_id(TAG_R, (uint32_t)p, wrap_id), 0, n, r + (int64_t)p * n);
    int64_t* th = (int64_t*)malloc((size_t)(n > 0 ? n : 1) * 8);
    oracle_wrap_count(P, r, n, th);
    for (int64_t i = 0; i < n; i++) theta_r[i] = (uint64_t)th[i];
    for (int p = 1; p < P; p++) {
        oracle_prg(k_ttp, oracle_stream_id(TAG_THETA, (uint32_t)p, wrap_id), 0, n, theta_r + (int64_t)p * n);
        for (int64_t i = 0; i < n; i++) theta_r[i] -= theta_r[(int64_t)p * n + i];
    }
    free(th);
}

/* Wrap pair values at selected flat indices idx[0..n) (same values as the
 * full oracle_wrap_pair at those positions). */
void oracle_wrap_pair_indices(int P, uint64_t k_ttp, uint64_t wrap_id, const int64_t* idx, int64_t n,
                              uint64_t* r, uint64_t* theta_r)
{
    for (int p = 0; p < P; p++)
        for (int64_t t = 0; t < n; t++)
            r[(int64_t)p * n + t] = oracle_prg_at(k_ttp, oracle_stream_id(TAG_R, (uint32_t)p, wrap_id), (uint64_t)idx[t]);
    int64_t* th = (int64_t*)malloc((size_t)(n > 0 ? n : 1) * 8);
    oracle_wrap_count(P, r, n, th);
    for (int64_t t = 0; t < n; t++) theta_r[t] = (uint64_t)th[t];
    for (int p = 1; p < P; p++)
        for (int64_t t = 0; t < n; t++) {
            uint64_t v = oracle_prg_at(k_ttp, oracle_stream_id(TAG_THETA, (uint32_t)p, wrap_id), (uint64_t)idx[t]);
            theta_r[(int64_t)p * n + t] = v;
            theta_r[t] -= v;
        }
    free(th);
}

/* ------------------------------------------------------------------------
 * O7  truncation for P > 2 by Algorithm 1 and the correction
 * x/ℓ = [y] − [θ_x]·Q/ℓ, with η_xr skipped:
 *   [z]_p = [x]_p + [r]_p
 *   [β]_p = (signed([x]_p) + signed([r]_p) − signed([z]_p)) / Q
 *   z = reveal([z]);   θ_z = (Σ_p signed([z]_p) − signed(z)) / Q
 *   [θ_x]_p = [β]_p − [θ_r]_p + [p=0]·θ_z          (η := 0)
 *   out_p = div_round([x]_p, ℓ) − [θ_x]_p · 2^(64−bits)
 * Diagnostics (may be NULL): z_out (revealed z), eta_out (η_xr = wraps of
 * the plaintexts x + r, i.e. (signed(x)+signed(r)−signed(z))/Q — the term
 * the paper skips; η ≠ 0 marks a possible failure event).
 * ---------------------------------------------------------------------- */
int oracle_truncate_alg1(int P, const uint64_t* x, const uint64_t* r, const uint64_t* theta_r,
                         int64_t n, int bits, uint64_t* out, uint64_t* z_out, int64_t* eta_out)
{
    if (bits < 1 || bits > 62 || P < 1) return ORACLE_ERR_ARG;
    uint64_t* zs = (uint64_t*)malloc((size_t)(P * (n > 0 ? n : 1)) * 8);
    uint64_t* beta = (uint64_t*)malloc((size_t)(P * (n > 0 ? n : 1)) * 8);
    int64_t* theta_z = (int64_t*)malloc((size_t)(n > 0 ? n : 1) * 8);
    uint64_t* z = (uint64_t*)malloc((size_t)(n > 0 ? n : 1) * 8);
    for (int64_t i = 0; i < (int64_t)P * n; i++) {
        zs[i] = x[i] + r[i];
        i128 s = (i128)(int64_t)x[i] + (i128)(int64_t)r[i] - (i128)(int64_t)zs[i];
        beta[i] = (uint64_t)(int64_t)(s >> 64);
    }
    oracle_reveal(P, zs, n, z);
    oracle_wrap_count(P, zs, n, theta_z);
    for (int p = 0; p < P; p++) {
        for (int64_t i = 0; i < n; i++) {
            int64_t k = (int64_t)p * n + i;
            uint64_t th = beta[k] - theta_r[k] + (p == 0 ? (uint64_t)theta_z[i] : 0u);
            out[k] = div_pow2_round(x[k], bits) - th * ((uint64_t)1 << (64 - bits));
        }
    }
    if (z_out) memcpy(z_out, z, (size_t)n * 8);
    if (eta_out) {
        uint64_t* xs = (uint64_t*)malloc((size_t)(n > 0 ? n : 1) * 8);
        uint64_t* rs = (uint64_t*)malloc((size_t)(n > 0 ? n : 1) * 8);
        oracle_reveal(P, x, n, xs);
        oracle_reveal(P, r, n, rs);
        for (int64_t i = 0; i < n; i++) {
            i128 s = (i128)(int64_t)xs[i] + (i128)(int64_t)rs[i] - (i128)(int64_t)z[i];
            eta_out[i] = (int64_t)(s >> 64);
        }
        free(xs); free(rs);
    }
    free(zs); free(beta); free(theta_z); free(z);
    return ORACLE_OK;
}

/* ========================================================================
 * elementwise private multiplication and square.
 * ======================================================================== */

/* ------------------------------------------------------------------------
 * O9  TTP Beaver triple for f = elementwise product (§4.2; P:576-580
 * App. A.1.1 "A Beaver triple ... satisfies the property c = ab"):
 *   a_p = G(k_ttp, A||p||id)[i], b_p = G(k_ttp, B||p||id)[i]
 *   c   = (Σ_p a_p) · (Σ_p b_p)   elementwise, mod Q
 *   c_p = G(k_ttp, C||p||id)[i] for p ≥ 1, c_0 = c − Σ_{p≥1} c_p
 * (the same stream layout as the matmul triple, reading R6; triple ids are
 * single-use, so a matmul and an elementwise triple never share an id).
 * a, b, c: [P][n].
 * ---------------------------------------------------------------------- */
void oracle_ttp_mul_triple(int P, uint64_t k_ttp, uint64_t triple_id, int64_t n,
                           uint64_t* a, uint64_t* b, uint64_t* c)
{
    for (int p = 0; p < P; p++) {
        oracle_prg(k_ttp, oracle_stream_id(TAG_A, (uint32_t)p, triple_id), 0, n, a + (int64_t)p * n);
        oracle_prg(k_ttp, oracle_stream_id(TAG_B, (uint32_t)p, triple_id), 0, n, b + (int64_t)p * n);
    }
    uint64_t* asum = (uint64_t*)calloc((size_t)(n > 0 ? n : 1), 8);
    uint64_t* bsum = (uint64_t*)calloc((size_t)(n > 0 ? n : 1), 8);
    oracle_reveal(P, a, n, asum);
    oracle_reveal(P, b, n, bsum);
    for (int64_t i = 0; i < n; i++) c[i] = asum[i] * bsum[i];
    for (int p = 1; p < P; p++) {
        uint64_t* cp = c + (int64_t)p * n;
        oracle_prg(k_ttp, oracle_stream_id(TAG_C, (uint32_t)p, triple_id), 0, n, cp);
        for (int64_t i = 0; i < n; i++) c[i] -= cp[i];                  /* c_0 −= c_p */
    }
    free(asum); free(bsum);
}

/* ------------------------------------------------------------------------
 * O10 TTP Beaver pair for the square (App. A.1.1 "a Beaver pair
 * ([a], [b]) such that b = a^2"):
 *   a_p = G(k_ttp, A||p||id)[i];  b = (Σ_p a_p)^2 mod Q
 *   b_p = G(k_ttp, C||p||id)[i] for p ≥ 1, b_0 = b − Σ_{p≥1} b_p
 * (the correlated share uses the C tag, as c does in a triple — reading R20).
 * a, b: [P][n].
 * ---------------------------------------------------------------------- */
void oracle_ttp_square_pair(int P, uint64_t k_ttp, uint64_t pair_id, int64_t n, uint64_t* a, uint64_t* b)
{
    for (int p = 0; p < P; p++)
        oracle_prg(k_ttp, oracle_stream_id(TAG_A, (uint32_t)p, pair_id), 0, n, a + (int64_t)p * n);
    uint64_t* asum = (uint64_t*)calloc((size_t)(n > 0 ? n : 1), 8);
    oracle_reveal(P, a, n, asum);
    for (int64_t i = 0; i < n; i++) b[i] = asum[i] * asum[i];
    for (int p = 1; p < P; p++) {
        uint64_t* bp = b + (int64_t)p * n;
        oracle_prg(k_ttp, oracle_stream_id(TAG_C, (uint32_t)p, pair_id), 0, n, bp);
        for (int64_t i = 0; i < n; i++) b[i] -= bp[i];                  /* b_0 −= b_p */
    }
    free(asum);
}

/* ------------------------------------------------------------------------
 * O11 Beaver elementwise multiplication (§4.2):
 *   [ε]_p = [x]_p − [a]_p,  [δ]_p = [y]_p − [b]_p;  ε, δ revealed (one round)
 *   [z]_p = [c]_p + ε·[b]_p + [a]_p·δ + [p = 0]·ε·δ     (elementwise; R7)
 * No truncation here (z at scale 2^(2f)).  All buffers [P][n]; eps_out and
 * delta_out (n) may be NULL.
 * ---------------------------------------------------------------------- */
void oracle_beaver_mul(int P, const uint64_t* x, const uint64_t* y, const uint64_t* a, const uint64_t* b,
                       const uint64_t* c, int64_t n, uint64_t* eps_out, uint64_t* delta_out, uint64_t* z)
{
    uint64_t* e = (uint64_t*)malloc((size_t)(P * (n > 0 ? n : 1)) * 8);
    uint64_t* d = (uint64_t*)malloc((size_t)(P * (n > 0 ? n : 1)) * 8);
    uint64_t* eps = (uint64_t*)malloc((size_t)(n > 0 ? n : 1) * 8);
    uint64_t* delta = (uint64_t*)malloc((size_t)(n > 0 ? n : 1) * 8);
    for (int64_t k = 0; k < (int64_t)P * n; k++) {
        e[k] = x[k] - a[k];
        d[k] = y[k] - b[k];
    }
    oracle_reveal(P, e, n, eps);
    oracle_reveal(P, d, n, delta);
    for (int p = 0; p < P; p++) {
        for (int64_t i = 0; i < n; i++) {
            int64_t k = (int64_t)p * n + i;
            z[k] = c[k] + eps[i] * b[k] + a[k] * delta[i];
            if (p == 0) z[k] += eps[i] * delta[i];
        }
    }
    if (eps_out) memcpy(eps_out, eps, (size_t)n * 8);
    if (delta_out) memcpy(delta_out, delta, (size_t)n * 8);
    free(e); free(d); free(eps); free(delta);
}

/* ------------------------------------------------------------------------
 * O12 Beaver square (App. A.1.1):
 *   [ε]_p = [x]_p − [a]_p;  ε revealed (one round)
 *   [x^2]_p = [b]_p + 2·ε·[a]_p + [p = 0]·ε^2          (party 0 adds the public ε², R7)
 * All buffers [P][n]; eps_out (n) may be NULL.
 * ---------------------------------------------------------------------- */
void oracle_beaver_square(int P, const uint64_t* x, const uint64_t* a, const uint64_t* b, int64_t n,
                          uint64_t* eps_out, uint64_t* z)
{
    uint64_t* e = (uint64_t*)malloc((size_t)(P * (n > 0 ? n : 1)) * 8);
    uint64_t* eps = (uint64_t*)malloc((size_t)(n > 0 ? n : 1) * 8);
    for (int64_t k = 0; k < (int64_t)P * n; k++) e[k] = x[k] - a[k];
    oracle_reveal(P, e, n, eps);
    for (int p = 0; p < P; p++) {
        for (int64_t i = 0; i < n; i++) {
            int64_t k = (int64_t)p * n + i;
            z[k] = b[k] + 2u * eps[i] * a[k];
            if (p == 0) z[k] += eps[i] * eps[i];
        }
    }
    if (eps_out) memcpy(eps_out, eps, (size_t)n * 8);
    free(e); free(eps);
}

/* ========================================================================
 * private 2-D convolution with true conv triples
 * ("we use the same procedure to perform matrix multiplication and
 * convolution"; §4.2 P:206 "convolutions").
 * ======================================================================== */

/* Convolution geometry: x (B, C, H, W), w (Cout, C, kh, kw), zero padding
 * (ph, pw), stride (sh, sw), no dilation, one group; out (B, Cout, Ho, Wo)
 * with Ho = (H + 2ph − kh)/sh + 1, Wo = (W + 2pw − kw)/sw + 1 (NCHW, the
 * PyTorch layout CrypTen uses). */
typedef struct { int64_t B, C, H, W, Cout, kh, kw, sh, sw, ph, pw; } oracle_conv_geom;

static int64_t conv_ho(const oracle_conv_geom* g) { return (g->H + 2 * g->ph - g->kh) / g->sh + 1; }
static int64_t conv_wo(const oracle_conv_geom* g) { return (g->W + 2 * g->pw - g->kw) / g->sw + 1; }

/* out[b,co,oy,ox] = Σ_{ci,ky,kx} x[b,ci,oy·sh−ph+ky, ox·sw−pw+kx] · w[co,ci,ky,kx] mod Q
 * (terms outside the input are the zero padding) — the definition, loop by loop. */
void oracle_conv2d(const uint64_t* x, const uint64_t* w, const oracle_conv_geom* g, uint64_t* out)
{
    int64_t Ho = conv_ho(g), Wo = conv_wo(g);
    for (int64_t b = 0; b < g->B; b++)
        for (int64_t co = 0; co < g->Cout; co++)
            for (int64_t oy = 0; oy < Ho; oy++)
                for (int64_t ox = 0; ox < Wo; ox++) {
                    uint64_t acc = 0;
                    for (int64_t ci = 0; ci < g->C; ci++)
                        for (int64_t ky = 0; ky < g->kh; ky++)
                            for (int64_t kx = 0; kx < g->kw; kx++) {
                                int64_t iy = oy * g->sh - g->ph + ky, ix = ox * g->sw - g->pw + kx;
                                if (iy < 0 || iy >= g->H || ix < 0 || ix >= g->W) continue;
                                acc += x[((b * g->C + ci) * g->H + iy) * g->W + ix]
                                     * w[((co * g->C + ci) * g->kh + ky) * g->kw + kx];
                            }
                    out[((b * g->Cout + co) * Ho + oy) * Wo + ox] = acc;
                }
}

/* ------------------------------------------------------------------------
 * O13 TTP conv triple (P:589-590 with O4's construction, readings R6, R22):
 *   a_p = G(k_ttp, A||p||id)[i] over the B·C·H·W input elements,
 *   b_p = G(k_ttp, B||p||id)[i] over the Cout·C·kh·kw weight elements,
 *   c = conv(Σ a_p, Σ b_p);  c_p = G(k_ttp, C||p||id)[i] (p ≥ 1), c_0 = c − Σ_{p≥1} c_p.
 * a: [P][B·C·H·W], b: [P][Cout·C·kh·kw], c: [P][B·Cout·Ho·Wo].
 * ---------------------------------------------------------------------- */
void oracle_ttp_conv_triple(int P, uint64_t k_ttp, uint64_t triple_id, const oracle_conv_geom* g,
                            uint64_t* a, uint64_t* b, uint64_t* c)
{
    int64_t na = g->B * g->C * g->H * g->W, nb = g->Cout * g->C * g->kh * g->kw;
    int64_t nc = g->B * g->Cout * conv_ho(g) * conv_wo(g);
    for (int p = 0; p < P; p++) {
        oracle_prg(k_ttp, oracle_stream_id(TAG_A, (uint32_t)p, triple_id), 0, na, a + (int64_t)p * na);
        oracle_prg(k_ttp, oracle_stream_id(TAG_B, (uint32_t)p, triple_id), 0, nb, b + (int64_t)p * nb);
    }
    uint64_t* asum = (uint64_t*)calloc((size_t)(na > 0 ? na : 1), 8);
    uint64_t* bsum = (uint64_t*)calloc((size_t)(nb > 0 ? nb : 1), 8);
    oracle_reveal(P, a, na, asum);
    oracle_reveal(P, b, nb, bsum);
    oracle_conv2d(asum, bsum, g, c);
    for (int p = 1; p < P; p++) {
        uint64_t* cp = c + (int64_t)p * nc;
        oracle_prg(k_ttp, oracle_stream_id(TAG_C, (uint32_t)p, triple_id), 0, nc, cp);
        for (int64_t i = 0; i < nc; i++) c[i] -= cp[i];
    }
    free(asum); free(bsum);
}

/* ------------------------------------------------------------------------
 * O14 Beaver private convolution:
 *   [ε]_p = [x]_p − [a]_p (input shape), [δ]_p = [y]_p − [b]_p (weight shape);
 *   ε, δ revealed (one round, at the input / weight shapes — reading R22);
 *   [z]_p = [c]_p + conv(ε, [b]_p) + conv([a]_p, δ) + [p = 0]·conv(ε, δ).
 * No truncation (scale 2^(2f)).  eps_out / delta_out may be NULL.
 * ---------------------------------------------------------------------- */
void oracle_beaver_conv2d(int P, const uint64_t* x, const uint64_t* y, const uint64_t* a, const uint64_t* b,
                          const uint64_t* c, const oracle_conv_geom* g, uint64_t* eps_out, uint64_t* delta_out,
                          uint64_t* z)
{
    int64_t na = g->B * g->C * g->H * g->W, nb = g->Cout * g->C * g->kh * g->kw;
    int64_t nc = g->B * g->Cout * conv_ho(g) * conv_wo(g);
    uint64_t* e = (uint64_t*)malloc((size_t)(P * (na > 0 ? na : 1)) * 8);
    uint64_t* d = (uint64_t*)malloc((size_t)(P * (nb > 0 ? nb : 1)) * 8);
    uint64_t* eps = (uint64_t*)malloc((size_t)(na > 0 ? na : 1) * 8);
    uint64_t* delta = (uint64_t*)malloc((size_t)(nb > 0 ? nb : 1) * 8);
    uint64_t* t = (uint64_t*)malloc((size_t)(nc > 0 ? nc : 1) * 8);
    for (int64_t k = 0; k < (int64_t)P * na; k++) e[k] = x[k] - a[k];
    for (int64_t k = 0; k < (int64_t)P * nb; k++) d[k] = y[k] - b[k];
    oracle_reveal(P, e, na, eps);
    oracle_reveal(P, d, nb, delta);
    for (int p = 0; p < P; p++) {
        uint64_t* zp = z + (int64_t)p * nc;
        for (int64_t i = 0; i < nc; i++) zp[i] = c[(int64_t)p * nc + i];
        oracle_conv2d(eps, b + (int64_t)p * nb, g, t);                   /* conv(ε, [b]_p) */
        for (int64_t i = 0; i < nc; i++) zp[i] += t[i];
        oracle_conv2d(a + (int64_t)p * na, delta, g, t);                 /* conv([a]_p, δ) */
        for (int64_t i = 0; i < nc; i++) zp[i] += t[i];
        if (p == 0) {
            oracle_conv2d(eps, delta, g, t);                             /* conv(ε, δ), party 0 */
            for (int64_t i = 0; i < nc; i++) zp[i] += t[i];
        }
    }
    if (eps_out) memcpy(eps_out, eps, (size_t)na * 8);
    if (delta_out) memcpy(delta_out, delta, (size_t)nb * 8);
    free(e); free(d); free(eps); free(delta); free(t);
}

/* ========================================================================
 * the ReLU path — binary secret sharing (P:180-182,
 * App. A.1.2), A2B by a carry-lookahead adder,
 * the sign bit, single-bit B2A (Alg. 2) and the final
 * multiplication ReLU([x]) = [x][x >= 0].
 * Stream tags of this path (reading R23): BPRZS = 7 (binary zero-shares),
 * BA/BB/BC = 8/9/10 (binary AND triples), RBIT/RB/RA = 11/12/13 (bit pairs),
 * MA/MB/MC = 14/15/16 (the final arithmetic multiplication triple).
 * ======================================================================== */
enum { TAG_BPRZS = 7, TAG_BA = 8, TAG_BB = 9, TAG_BC = 10, TAG_RBIT = 11, TAG_RB = 12, TAG_RA = 13,
       TAG_MA = 14, TAG_MB = 15, TAG_MC = 16 };

/* Binary sharing by pseudorandom zero-share (XOR version of O3, reading R23):
 * ⟨x⟩_p = G(k_p, BPRZS||0||id)[i] ⊕ G(k_{p−1}, BPRZS||0||id)[i] ⊕ [p = src]·x[i]. */
void oracle_bshare(int P, const uint64_t* k_party, const uint64_t* x, int src, uint64_t share_id, int64_t n,
                   uint64_t* shares)
{
    uint64_t stream = oracle_stream_id(TAG_BPRZS, 0, share_id);
    for (int p = 0; p < P; p++) {
        int prev = (p + P - 1) % P;
        for (int64_t i = 0; i < n; i++) {
            uint64_t v = oracle_prg_at(k_party[p], stream, (uint64_t)i) ^ oracle_prg_at(k_party[prev], stream, (uint64_t)i);
            if (p == src && x != NULL) v ^= x[i];
            shares[(int64_t)p * n + i] = v;
        }
    }
}

/* x = ⊕_p ⟨x⟩_p */
void oracle_breveal(int P, const uint64_t* shares, int64_t n, uint64_t* out)
{
    for (int64_t i = 0; i < n; i++) {
        uint64_t s = 0;
        for (int p = 0; p < P; p++) s ^= shares[(int64_t)p * n + i];
        out[i] = s;
    }
}

/* Binary Beaver triple ("c = a ⊗ b", bitwise, packed 64 per word):
 * a_p = G(k_ttp, BA||p||id), b_p = G(k_ttp, BB||p||id), c = (⊕a) & (⊕b),
 * c_p = G(k_ttp, BC||p||id) for p ≥ 1, c_0 = c ⊕ ⊕_{p≥1} c_p. */
void oracle_ttp_binary_triple(int P, uint64_t k_ttp, uint64_t id, int64_t n, uint64_t* a, uint64_t* b, uint64_t* c)
{
    for (int p = 0; p < P; p++) {
        oracle_prg(k_ttp, oracle_stream_id(TAG_BA, (uint32_t)p, id), 0, n, a + (int64_t)p * n);
        oracle_prg(k_ttp, oracle_stream_id(TAG_BB, (uint32_t)p, id), 0, n, b + (int64_t)p * n);
    }
    uint64_t* as = (uint64_t*)calloc((size_t)(n > 0 ? n : 1), 8);
    uint64_t* bs = (uint64_t*)calloc((size_t)(n > 0 ? n : 1), 8);
    oracle_breveal(P, a, n, as);
    oracle_breveal(P, b, n, bs);
    for (int64_t i = 0; i < n; i++) c[i] = as[i] & bs[i];
    for (int p = 1; p < P; p++) {
        uint64_t* cp = c + (int64_t)p * n;
        oracle_prg(k_ttp, oracle_stream_id(TAG_BC, (uint32_t)p, id), 0, n, cp);
        for (int64_t i = 0; i < n; i++) c[i] ^= cp[i];
    }
    free(as); free(bs);
}

/* O15 Bitwise AND: ⟨ε⟩ = ⟨x⟩ ⊕ ⟨a⟩, ⟨δ⟩ = ⟨y⟩ ⊕ ⟨b⟩, ε, δ revealed
 * (one round); ⟨z⟩_p = ⟨c⟩_p ⊕ (ε & ⟨b⟩_p) ⊕ (⟨a⟩_p & δ) ⊕ [p = 0](ε & δ). */
void oracle_binary_and(int P, const uint64_t* x, const uint64_t* y, const uint64_t* a, const uint64_t* b,
                       const uint64_t* c, int64_t n, uint64_t* z)
{
    for (int64_t i = 0; i < n; i++) {
        uint64_t eps = 0, delta = 0;
        for (int p = 0; p < P; p++) {
            eps ^= x[(int64_t)p * n + i] ^ a[(int64_t)p * n + i];
            delta ^= y[(int64_t)p * n + i] ^ b[(int64_t)p * n + i];
        }
        for (int p = 0; p < P; p++) {
            int64_t k = (int64_t)p * n + i;
            z[k] = c[k] ^ (eps & b[k]) ^ (a[k] & delta);
            if (p == 0) z[k] ^= eps & delta;
        }
    }
}

/* AND of two binary-shared tensors with the triple of AND gate `gate_id` (dealt here by the TTP). */
static void and_gate(int P, uint64_t k_ttp, uint64_t gate_id, const uint64_t* x, const uint64_t* y, int64_t n,
                     uint64_t* z)
{
    size_t sz = (size_t)(P * (n > 0 ? n : 1)) * 8;
    uint64_t *a = (uint64_t*)malloc(sz), *b = (uint64_t*)malloc(sz), *c = (uint64_t*)malloc(sz);
    oracle_ttp_binary_triple(P, k_ttp, gate_id, n, a, b, c);
    oracle_binary_and(P, x, y, a, b, c, n, z);
    free(a); free(b); free(c);
}

/* AND gate ids of one ring addition (reading R24): adder `add_id`, Kogge-Stone
 * level l (0 = the generate bits x & y, 1..6 = prefix levels), operand w
 * (0: P & (G << k), 1: P & (P << k)):  gate = (add_id << 4) | (l << 1) | w. */
static uint64_t gate_id(uint64_t add_id, int l, int w) { return (add_id << 4) | ((uint64_t)l << 1) | (uint64_t)w; }

/* O16 ring addition ⟨x + y mod 2^64⟩ as a carry-lookahead (Kogge-Stone) adder
 * on binary shares (SPEC add_ring): generate G = x & y, propagate
 * Pr = x ⊕ y; for k = 1, 2, 4, ..., 32: G ← G ⊕ (Pr & (G << k)),
 * Pr ← Pr & (Pr << k) (the two ANDs of a level share one round; G and
 * Pr & (G << k) are disjoint, so OR = XOR); sum = x ⊕ y ⊕ (G << 1).
 * 1 + 6 AND rounds (the first generate AND is batched with nothing; 7 rounds). */
void oracle_add_ring(int P, uint64_t k_ttp, uint64_t add_id, const uint64_t* x, const uint64_t* y, int64_t n,
                     uint64_t* out)
{
    size_t sz = (size_t)(P * (n > 0 ? n : 1)) * 8;
    uint64_t *G = (uint64_t*)malloc(sz), *Pr = (uint64_t*)malloc(sz), *t = (uint64_t*)malloc(sz),
             *u = (uint64_t*)malloc(sz);
    int64_t Pn = (int64_t)P * n;
    and_gate(P, k_ttp, gate_id(add_id, 0, 0), x, y, n, G);
    for (int64_t k = 0; k < Pn; k++) Pr[k] = x[k] ^ y[k];
    for (int l = 1; l <= 6; l++) {
        int s = 1 << (l - 1);
        for (int64_t k = 0; k < Pn; k++) t[k] = G[k] << s;       /* local logical shift */
        and_gate(P, k_ttp, gate_id(add_id, l, 0), Pr, t, n, u);
        for (int64_t k = 0; k < Pn; k++) G[k] ^= u[k];
        for (int64_t k = 0; k < Pn; k++) t[k] = Pr[k] << s;
        and_gate(P, k_ttp, gate_id(add_id, l, 1), Pr, t, n, u);
        memcpy(Pr, u, (size_t)Pn * 8);
    }
    for (int64_t k = 0; k < Pn; k++) out[k] = x[k] ^ y[k] ^ (G[k] << 1);
    free(G); free(Pr); free(t); free(u);
}

/* O17 A2B: party q binary-shares its arithmetic share
 * [x]_q (binary PRZS, share id (a2b_id << 8) | q); the P binary values are
 * summed by a tree of ring adders, adjacent pairs level by level (level h,
 * pair i has adder id (a2b_id << 12) | (h << 6) | i; an odd last element
 * passes up).  Rounds: ceil(log2 P) adder levels of 7 AND rounds.
 * x: [P][n] arithmetic shares -> out: [P][n] binary shares of x. */
void oracle_a2b(int P, const uint64_t* k_party, uint64_t k_ttp, uint64_t a2b_id, const uint64_t* x, int64_t n,
                uint64_t* out)
{
    size_t one = (size_t)(P * (n > 0 ? n : 1)) * 8;
    uint64_t** items = (uint64_t**)malloc(sizeof(uint64_t*) * (size_t)P);
    for (int q = 0; q < P; q++) {
        items[q] = (uint64_t*)malloc(one);
        oracle_bshare(P, k_party, x + (int64_t)q * n, q, (a2b_id << 8) | (uint64_t)q, n, items[q]);
    }
    int cnt = P, h = 1;
    while (cnt > 1) {
        int nc = 0;
        for (int i = 0; i + 1 < cnt; i += 2) {
            uint64_t* s = (uint64_t*)malloc(one);
            oracle_add_ring(P, k_ttp, (a2b_id << 12) | ((uint64_t)h << 6) | (uint64_t)(i / 2), items[i], items[i + 1], n, s);
            free(items[i]); free(items[i + 1]);
            items[nc++] = s;
        }
        if (cnt & 1) items[nc++] = items[cnt - 1];
        cnt = nc;
        h++;
    }
    memcpy(out, items[0], (size_t)P * (size_t)n * 8);
    free(items[0]);
    free(items);
}

/* Bit pair ([r], ⟨r⟩) from the TTP (Alg. 2 input): r = G(k_ttp, RBIT||0||id)[i] & 1;
 * ⟨r⟩_p = G(k_ttp, RB||p||id)[i] & 1 (p ≥ 1), ⟨r⟩_0 = r ⊕ ⊕_{p≥1}⟨r⟩_p;
 * [r]_p = G(k_ttp, RA||p||id)[i] (p ≥ 1), [r]_0 = r − Σ_{p≥1} [r]_p. */
void oracle_ttp_bit_pair(int P, uint64_t k_ttp, uint64_t id, int64_t n, uint64_t* rA, uint64_t* rB)
{
    for (int64_t i = 0; i < n; i++) {
        uint64_t r = oracle_prg_at(k_ttp, oracle_stream_id(TAG_RBIT, 0, id), (uint64_t)i) & 1u;
        uint64_t rb0 = r, ra0 = r;
        for (int p = 1; p < P; p++) {
            uint64_t vb = oracle_prg_at(k_ttp, oracle_stream_id(TAG_RB, (uint32_t)p, id), (uint64_t)i) & 1u;
            uint64_t va = oracle_prg_at(k_ttp, oracle_stream_id(TAG_RA, (uint32_t)p, id), (uint64_t)i);
            rB[(int64_t)p * n + i] = vb;
            rA[(int64_t)p * n + i] = va;
            rb0 ^= vb;
            ra0 -= va;
        }
        rB[i] = rb0;
        rA[i] = ra0;
    }
}

/* O18 single-bit B2A (Alg. 2): ⟨z⟩ = ⟨b⟩ ⊕ ⟨r⟩; z = reveal(⟨z⟩) (one
 * round); [b] = [r] + z − 2[r]z (party 0 adds the public z).  b: [P][n] binary
 * shares whose bit 0 is the shared bit (higher bits ignored).  z_out may be NULL. */
void oracle_b2a_bit(int P, const uint64_t* b, const uint64_t* rA, const uint64_t* rB, int64_t n, uint64_t* out,
                    uint64_t* z_out)
{
    for (int64_t i = 0; i < n; i++) {
        uint64_t z = 0;
        for (int p = 0; p < P; p++) z ^= (b[(int64_t)p * n + i] ^ rB[(int64_t)p * n + i]) & 1u;
        for (int p = 0; p < P; p++) {
            int64_t k = (int64_t)p * n + i;
            out[k] = rA[k] - 2u * z * rA[k] + (p == 0 ? z : 0u);
        }
        if (z_out) z_out[i] = z;
    }
}

/* O19 ReLU([x]) = [x] · [x >= 0] (reading R25):
 *   ⟨x⟩ = A2B([x]) (a2b id relu_id);  ⟨s⟩ = ⟨x⟩ >> 63 (sign bit);
 *   [s] = B2A_bit(⟨s⟩) with bit pair relu_id;  [x >= 0] = 1 − [s] (party 0 adds 1);
 *   out = BeaverMul([x], [x >= 0]) with the MA/MB/MC triple relu_id (one round).
 * The indicator carries scale 1, so out keeps x's scale (no truncation).
 * x, out: [P][n]; sign_out ([P][n] arithmetic shares of [x < 0]) and rounds may be NULL. */
void oracle_relu(int P, const uint64_t* k_party, uint64_t k_ttp, uint64_t relu_id, const uint64_t* x, int64_t n,
                 uint64_t* out, uint64_t* sign_out, int* rounds)
{
    size_t sz = (size_t)(P * (n > 0 ? n : 1)) * 8;
    uint64_t *xb = (uint64_t*)malloc(sz), *rA = (uint64_t*)malloc(sz), *rB = (uint64_t*)malloc(sz),
             *s = (uint64_t*)malloc(sz), *ind = (uint64_t*)malloc(sz), *a = (uint64_t*)malloc(sz),
             *b = (uint64_t*)malloc(sz), *c = (uint64_t*)malloc(sz);
    int64_t Pn = (int64_t)P * n;
    oracle_a2b(P, k_party, k_ttp, relu_id, x, n, xb);
    for (int64_t k = 0; k < Pn; k++) xb[k] >>= 63;                      /* sign bit, local */
    oracle_ttp_bit_pair(P, k_ttp, relu_id, n, rA, rB);
    oracle_b2a_bit(P, xb, rA, rB, n, s, NULL);                          /* [x < 0] */
    for (int p = 0; p < P; p++)
        for (int64_t i = 0; i < n; i++) ind[(int64_t)p * n + i] = (p == 0 ? 1u : 0u) - s[(int64_t)p * n + i];
    for (int p = 0; p < P; p++) {                                       /* triple c = a·b (O9's construction) */
        oracle_prg(k_ttp, oracle_stream_id(TAG_MA, (uint32_t)p, relu_id), 0, n, a + (int64_t)p * n);
        oracle_prg(k_ttp, oracle_stream_id(TAG_MB, (uint32_t)p, relu_id), 0, n, b + (int64_t)p * n);
    }
    for (int64_t i = 0; i < n; i++) {
        uint64_t as = 0, bs = 0;
        for (int p = 0; p < P; p++) { as += a[(int64_t)p * n + i]; bs += b[(int64_t)p * n + i]; }
        c[i] = as * bs;
    }
    for (int p = 1; p < P; p++) {
        oracle_prg(k_ttp, oracle_stream_id(TAG_MC, (uint32_t)p, relu_id), 0, n, c + (int64_t)p * n);
        for (int64_t i = 0; i < n; i++) c[i] -= c[(int64_t)p * n + i];
    }
    oracle_beaver_mul(P, x, ind, a, b, c, n, NULL, NULL, out);
    if (sign_out) memcpy(sign_out, s, (size_t)Pn * 8);
    if (rounds) {
        int levels = 0;
        for (int q = 1; q < P; q *= 2) levels++;
        *rounds = levels * 7 + 1 + 1;                                   /* A2B, B2A, multiplication */
    }
    free(xb); free(rA); free(rB); free(s); free(ind); free(a); free(b); free(c);
}

/* ========================================================================
 * The boundary's calls with the C-ABI's shape (SURVEY §8(b) "the oracle
 * library exports the same functions as oracle_mpc_* with host pointers and
 * identical semantics"): include/mpc_ring.h's north-star entry points, for an
 * all-parties context (rank = -1; every share argument is [P][n] in HOST
 * memory).  Each one only composes the steps above (O1-O8); status codes are
 * mpc_status's numbers.  A parity harness can run one protocol script against
 * either library (tests/test_oracle_boundary.py, tests/test_gpu_boundary_swap.py).
 * ======================================================================== */
#define ORACLE_MPC_OK 0
#define ORACLE_MPC_ERR_ARG 1
#define ORACLE_MPC_ERR_SHAPE 2
#define ORACLE_MPC_ERR_OVERFLOW 3
#define ORACLE_MPC_ERR_UNSUPPORTED 7

typedef struct oracle_mpc_ctx_s {
    int P, frac;
    uint64_t k_party[16], k_ttp;
    uint64_t rounds, bytes;
} oracle_mpc_ctx_s;
typedef oracle_mpc_ctx_s* oracle_mpc_ctx;

int oracle_mpc_create(oracle_mpc_ctx* out, int world_size, int rank, int device, const void* nccl_id,
                      uint64_t master_seed, int frac_bits)
{
    (void)device; (void)nccl_id;
    if (!out) return ORACLE_MPC_ERR_ARG;
    *out = NULL;
    if (world_size < 1 || world_size > 16 || frac_bits < 1 || frac_bits > 30) return ORACLE_MPC_ERR_ARG;
    if (rank != -1) return ORACLE_MPC_ERR_UNSUPPORTED;       /* the oracle simulates every party */
    oracle_mpc_ctx c = (oracle_mpc_ctx)calloc(1, sizeof(oracle_mpc_ctx_s));
    if (!c) return ORACLE_MPC_ERR_ARG;
    c->P = world_size;
    c->frac = frac_bits;
    oracle_derive_keys(master_seed, world_size, c->k_party, &c->k_ttp);
    *out = c;
    return ORACLE_MPC_OK;
}

int oracle_mpc_destroy(oracle_mpc_ctx c) { if (!c) return ORACLE_MPC_ERR_ARG; free(c); return ORACLE_MPC_OK; }

int oracle_mpc_stats(oracle_mpc_ctx c, uint64_t* rounds, uint64_t* bytes_sent)
{
    if (!c) return ORACLE_MPC_ERR_ARG;
    if (rounds) *rounds = c->rounds;
    if (bytes_sent) *bytes_sent = c->bytes;
    return ORACLE_MPC_OK;
}

int oracle_mpc_encode(oracle_mpc_ctx c, const double* x, uint64_t* out, int64_t n)
{
    if (!c || n < 0) return ORACLE_MPC_ERR_ARG;
    return oracle_encode(x, out, n, c->frac) == ORACLE_OK ? ORACLE_MPC_OK : ORACLE_MPC_ERR_OVERFLOW;
}

int oracle_mpc_decode(oracle_mpc_ctx c, const uint64_t* v, double* out, int64_t n)
{
    if (!c || n < 0) return ORACLE_MPC_ERR_ARG;
    oracle_decode(v, out, n, c->frac);
    return ORACLE_MPC_OK;
}

int oracle_mpc_share(oracle_mpc_ctx c, const uint64_t* x, int src, uint64_t share_id, uint64_t* share_out, int64_t n)
{
    if (!c || n < 0 || src < 0 || src >= c->P || (n > 0 && (!x || !share_out))) return ORACLE_MPC_ERR_ARG;
    oracle_share(c->P, c->k_party, x, src, share_id, n, share_out);
    return ORACLE_MPC_OK;
}

int oracle_mpc_reveal(oracle_mpc_ctx c, const uint64_t* share, uint64_t* out, int64_t n)
{
    if (!c || n < 0 || (n > 0 && (!share || !out))) return ORACLE_MPC_ERR_ARG;
    c->rounds += 1;
    c->bytes += 8ull * (uint64_t)n * (uint64_t)c->P;
    oracle_reveal(c->P, share, n, out);
    return ORACLE_MPC_OK;
}

int oracle_mpc_ttp_triples(oracle_mpc_ctx c, uint64_t triple_id, int64_t M, int64_t K, int64_t N,
                           uint64_t* a, uint64_t* b, uint64_t* cc, void* workspace, size_t workspace_bytes)
{
    (void)workspace; (void)workspace_bytes;
    if (!c || M < 0 || K < 0 || N < 0) return ORACLE_MPC_ERR_SHAPE;
    oracle_ttp_triple(c->P, c->k_ttp, triple_id, M, K, N, NULL, 0, a, b, cc);
    return ORACLE_MPC_OK;
}

int oracle_mpc_ttp_wrap_pairs(oracle_mpc_ctx c, uint64_t wrap_id, int64_t n, uint64_t* r, uint64_t* theta_r)
{
    if (!c || n < 0) return ORACLE_MPC_ERR_ARG;
    oracle_wrap_pair(c->P, c->k_ttp, wrap_id, n, r, theta_r);
    return ORACLE_MPC_OK;
}

/* O6 (P <= 2) or O7 (P > 2) in place, the wrap pair regenerated from wrap_id (r, th NULL) or given */
static int oracle_mpc_truncate_impl(oracle_mpc_ctx c, uint64_t* x, int64_t n, int bits, uint64_t wrap_id,
                                    const uint64_t* r_in, const uint64_t* th_in)
{
    if (bits < 1 || bits > 62) return ORACLE_MPC_ERR_ARG;
    int64_t Pn = (int64_t)c->P * n;
    uint64_t* out = (uint64_t*)malloc((size_t)(Pn > 0 ? Pn : 1) * 8);
    int rc;
    if (c->P <= 2) {
        rc = oracle_truncate_local(c->P, x, n, bits, out);
    } else {
        uint64_t* r = (uint64_t*)r_in;
        uint64_t* th = (uint64_t*)th_in;
        if (!r_in) {
            r = (uint64_t*)malloc((size_t)(Pn > 0 ? Pn : 1) * 8);
            th = (uint64_t*)malloc((size_t)(Pn > 0 ? Pn : 1) * 8);
            oracle_wrap_pair(c->P, c->k_ttp, wrap_id, n, r, th);
        }
        rc = oracle_truncate_alg1(c->P, x, r, th, n, bits, out, NULL, NULL);
        if (!r_in) { free(r); free(th); }
        c->rounds += 1;
        c->bytes += 9ull * (uint64_t)n * (uint64_t)c->P;
    }
    if (rc == ORACLE_OK) memcpy(x, out, (size_t)Pn * 8);
    free(out);
    return rc == ORACLE_OK ? ORACLE_MPC_OK : ORACLE_MPC_ERR_ARG;
}

int oracle_mpc_truncate(oracle_mpc_ctx c, uint64_t* x, int64_t n, int bits, uint64_t wrap_id)
{
    if (!c || n < 0 || (n > 0 && !x)) return ORACLE_MPC_ERR_ARG;
    return oracle_mpc_truncate_impl(c, x, n, bits, wrap_id, NULL, NULL);
}

int oracle_mpc_truncate_pairs(oracle_mpc_ctx c, uint64_t* x, int64_t n, int bits, const uint64_t* r,
                              const uint64_t* theta_r)
{
    if (!c || n < 0 || (n > 0 && (!x || (c->P > 2 && (!r || !theta_r))))) return ORACLE_MPC_ERR_ARG;
    return oracle_mpc_truncate_impl(c, x, n, bits, 0, r, theta_r);
}

int oracle_mpc_beaver_matmul(oracle_mpc_ctx c, const uint64_t* x, const uint64_t* y, const uint64_t* a,
                             const uint64_t* b, const uint64_t* cc, uint64_t* z, int64_t M, int64_t K, int64_t N,
                             int truncate, uint64_t wrap_id, void* workspace, size_t workspace_bytes)
{
    (void)workspace; (void)workspace_bytes;
    if (!c || M < 0 || K < 0 || N < 0) return ORACLE_MPC_ERR_SHAPE;
    c->rounds += 1;                                            /* eps || delta */
    c->bytes += 8ull * (uint64_t)(M * K + K * N) * (uint64_t)c->P;
    if (M == 0 || N == 0) return ORACLE_MPC_OK;
    oracle_beaver_matmul(c->P, x, y, a, b, cc, M, K, N, NULL, NULL, NULL, NULL, z);
    if (truncate) return oracle_mpc_truncate_impl(c, z, M * N, c->frac, wrap_id, NULL, NULL);
    return ORACLE_MPC_OK;
}

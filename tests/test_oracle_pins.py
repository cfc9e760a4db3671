"""Pins of the CPU oracle against things other than itself (-m "not gpu").

Each test names what fixes the expected value: a published known-answer
vector, a value printed in PAPER.md / SPEC.md, a closed form, an independent
library routine (numpy's wrapping uint64 matmul), Python big integers, or the
paper's own §4.3 float64 block decomposition.  A plausible slip in the oracle
(dropped term, wrong sign, transposed operand, wrong party, wrong rounding)
fails at least one of them.
"""
import os

import numpy as np
import pytest

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")
MASTER = synth.MASTER_SEED
Q = 1 << 64


def _signed(v: int) -> int:
    v &= Q - 1
    return v - Q if v >= (1 << 63) else v


# ----------------------------------------------------------------- O1 PRG
def test_philox_known_answer_vectors():
    n = 0
    for line in open(os.path.join(GOLD, "philox4x32_10_kat.txt")):
        if line.startswith("#") or not line.strip():
            continue
        w = [int(t, 16) for t in line.split()]
        assert oracle.philox4x32_10(w[0:4], w[4:6]) == w[6:10]
        n += 1
    assert n == 3


def test_prg_frozen_table():
    tags = dict(PRZS=1, A=2, B=3, C=4, R=5, THETA=6)
    kp, kt = oracle.derive_keys(MASTER, 3)
    keys = {"k_0": int(kp[0]), "k_1": int(kp[1]), "k_2": int(kp[2]), "k_ttp": kt}
    seen = 0
    for line in open(os.path.join(GOLD, "prg_frozen.txt")):
        if line.startswith("#") or not line.strip():
            continue
        t = line.split()
        if t[0] == "key":
            assert keys[t[1]] == int(t[2], 16), t[1]
        else:
            stream = oracle.stream_id(tags[t[2]], int(t[3]), int(t[4]))
            got = oracle.prg(keys[t[1]], stream, 4)
            assert [int(v) for v in got] == [int(h, 16) for h in t[5:9]]
        seen += 1
    assert seen == 7


def test_prg_offset_and_parity_of_index():
    s = oracle.stream_id(2, 1, 99)
    full = oracle.prg(12345, s, 11)
    for start in range(0, 9):
        assert np.array_equal(oracle.prg(12345, s, 3, start=start), full[start:start + 3])


# ----------------------------------------------------------------- O2 encode/decode
def test_encode_decode_spec_examples():
    # SPEC S:48-50
    assert int(oracle.encode([1.0])[0]) == 65536
    assert int(oracle.encode([0.0])[0]) == 0
    assert int(oracle.encode([-0.5])[0]) == Q - 32768
    assert oracle.decode(np.array([65536], dtype=np.uint64))[0] == 1.0
    assert oracle.decode(np.array([Q - 32768], dtype=np.uint64))[0] == -0.5
    x = np.array([3.14159, -2.71828, 1e-9, -7.999, 123456.789])
    assert np.max(np.abs(oracle.decode(oracle.encode(x)) - x)) <= 2.0 ** -17


def test_encode_ties_and_overflow():
    # ties: half away from zero (reading R2); 2^-17 is exactly half an ulp
    h = 2.0 ** -17
    assert int(oracle.encode([h])[0]) == 1
    assert int(oracle.encode([-h])[0]) == Q - 1
    assert int(oracle.encode([3 * h])[0]) == 2
    with pytest.raises(OverflowError):
        oracle.encode([2.0 ** 47])          # 2^47 * 2^16 = 2^63
    with pytest.raises(OverflowError):
        oracle.encode([float("nan")])
    assert int(oracle.encode([2.0 ** 46])[0]) == 1 << 62


# ----------------------------------------------------------------- O3/O8 share/reveal
@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("n", [0, 1, 7, 4096])
def test_share_reveal_roundtrip(P, n):
    x = synth.uniform_ring((n,), seed=P * 100 + n)
    for src in {0, P - 1}:
        s = oracle.share(P, MASTER, x, src=src, share_id=5 + src)
        assert s.shape == (P, n)
        assert np.array_equal(oracle.reveal(s), x)


def test_share_p1_is_plaintext_and_przs_sums_to_zero():
    x = synth.uniform_ring((33,), seed=1)
    assert np.array_equal(oracle.share(1, MASTER, x, 0, 3)[0], x)
    for P in (2, 3, 5):
        z = oracle.share(P, MASTER, np.zeros(33, dtype=np.uint64), 0, 9)
        assert not np.any(z[0] == 0)                       # genuinely random
        assert np.array_equal(oracle.reveal(z), np.zeros(33, dtype=np.uint64))


def test_share_neighbour_rule_explicit():
    # [x]_p = G(k_p) − G(k_{p−1}) + [p=src]x, written out with the raw PRG
    P, n, sid = 3, 5, 77
    x = synth.uniform_ring((n,), seed=2)
    kp, _ = oracle.derive_keys(MASTER, P)
    st = oracle.stream_id(oracle.TAG_PRZS, 0, sid)
    g = [oracle.prg(int(kp[p]), st, n) for p in range(P)]
    s = oracle.share(P, MASTER, x, src=1, share_id=sid)
    for p in range(P):
        exp = g[p] - g[(p - 1) % P] + (x if p == 1 else 0)
        assert np.array_equal(s[p], exp.astype(np.uint64))


def test_fig2_worked_example():
    rows = {}
    for line in open(os.path.join(GOLD, "fig2_example.txt")):
        if line.startswith("#") or not line.strip():
            continue
        t = line.split()
        rows[t[0]] = np.array([float(v) for v in t[1:]])
    for P in (1, 2, 3):
        xs = oracle.share(P, MASTER, oracle.encode(rows["x"]), 0, 1)
        ys = oracle.share(P, MASTER, oracle.encode(rows["y"]), 0, 2)
        assert np.allclose(oracle.decode(oracle.reveal(xs)), rows["x"])
        zs = (xs + ys).astype(np.uint64)                   # private addition
        assert np.allclose(oracle.decode(oracle.reveal(zs)), rows["x_plus_y"])


# ----------------------------------------------------------------- ring GEMM
def test_ring_matmul_vs_numpy_wrapping():
    A = synth.uniform_ring((37, 53), 3)
    B = synth.uniform_ring((53, 29), 4)
    assert np.array_equal(oracle.ring_matmul(A, B), A @ B)


def test_ring_matmul_vs_bigint_bruteforce():
    A = synth.uniform_ring((5, 7), 5)
    B = synth.uniform_ring((7, 3), 6)
    C = oracle.ring_matmul(A, B)
    for i in range(5):
        for j in range(3):
            exact = sum(int(A[i, k]) * int(B[k, j]) for k in range(7))
            assert int(C[i, j]) == exact % Q


def test_ring_matmul_closed_forms():
    # (2^64−1)·(2^64−1) ≡ 1, so an all-ones-bits K-inner product is K mod 2^64
    K = 1000
    A = np.full((3, K), Q - 1, dtype=np.uint64)
    B = np.full((K, 4), Q - 1, dtype=np.uint64)
    assert np.all(oracle.ring_matmul(A, B) == K)
    # 2^32 · 2^32 = 2^64 ≡ 0
    assert int(oracle.ring_matmul([[1 << 32]], [[1 << 32]])[0, 0]) == 0
    # identity
    X = synth.uniform_ring((6, 6), 7)
    assert np.array_equal(oracle.ring_matmul(X, np.eye(6, dtype=np.uint64)), X)


def _paper_float64_block_gemm(A, B):
    """PAPER.md §4.3: split each u64 into four 16-bit blocks, compute
    the 10 block products with float64 GEMMs, shift-add mod 2^64.  Exact while
    K * (2^16-1)^2 < 2^53."""
    A = A.astype(np.uint64)
    B = B.astype(np.uint64)
    assert A.shape[1] * (2 ** 16 - 1) ** 2 < 2 ** 53
    Ab = [((A >> np.uint64(16 * i)) & np.uint64(0xFFFF)).astype(np.float64) for i in range(4)]
    Bb = [((B >> np.uint64(16 * j)) & np.uint64(0xFFFF)).astype(np.float64) for j in range(4)]
    out = np.zeros((A.shape[0], B.shape[1]), dtype=np.uint64)
    products = 0
    for i in range(4):
        for j in range(4 - i):
            P = (Ab[i] @ Bb[j]).astype(np.uint64)          # exact integer < 2^53
            out += P << np.uint64(16 * (i + j))
            products += 1
    assert products == 10                                   # "summing 10 pairwise products"
    return out


def test_ring_matmul_vs_paper_float64_blocks():
    A = synth.uniform_ring((64, 300), 8)
    B = synth.uniform_ring((300, 48), 9)
    assert np.array_equal(oracle.ring_matmul(A, B), _paper_float64_block_gemm(A, B))


# ----------------------------------------------------------------- O4 triples
@pytest.mark.parametrize("P", [1, 2, 3, 5])
def test_triple_defining_property(P):
    M, K, N = 9, 13, 7
    a, b, c = oracle.ttp_triple(P, MASTER, 42, M, K, N)
    A, B, C = oracle.reveal(a), oracle.reveal(b), oracle.reveal(c)
    assert np.array_equal(C, A @ B)                          # P:577, S:202 (numpy, not the oracle GEMM)
    if P > 1:   # c_p for p >= 1 are raw PRG streams (reading R6)
        _, kt = oracle.derive_keys(MASTER, P)
        for p in range(1, P):
            assert np.array_equal(c[p].ravel(), oracle.prg(kt, oracle.stream_id(oracle.TAG_C, p, 42), M * N))
            assert np.array_equal(a[p].ravel(), oracle.prg(kt, oracle.stream_id(oracle.TAG_A, p, 42), M * K))


def test_triple_row_sample_matches_full():
    P, M, K, N = 3, 20, 11, 6
    a, b, c = oracle.ttp_triple(P, MASTER, 5, M, K, N)
    rows = [0, 7, 19, 3]
    a2, b2, c2 = oracle.ttp_triple(P, MASTER, 5, M, K, N, rows=rows)
    assert np.array_equal(a2, a[:, rows])
    assert np.array_equal(b2, b)
    assert np.array_equal(c2, c[:, rows])


# ----------------------------------------------------------------- O5 Beaver
def _shared_inputs(P, M, K, N, seed, tid=1):
    X = synth.uniform_fixed((M, K), seed)
    Y = synth.uniform_fixed((K, N), seed + 1)
    xs = oracle.share(P, MASTER, X, 0, 100 * tid)
    ys = oracle.share(P, MASTER, Y, 1 % P, 100 * tid + 1)
    a, b, c = oracle.ttp_triple(P, MASTER, tid, M, K, N)
    return X, Y, xs, ys, a, b, c


@pytest.mark.parametrize("P", [1, 2, 3, 4])
def test_beaver_identity_exact(P):
    # Σ_p z_p = x@y mod 2^64 exactly (derivation P:584-588); numpy as the independent GEMM
    X, Y, xs, ys, a, b, c = _shared_inputs(P, 17, 23, 11, seed=10 + P)
    z, im = oracle.beaver_matmul(xs, ys, a, b, c, want_intermediates=True)
    assert np.array_equal(oracle.reveal(z), X @ Y)
    assert np.array_equal(im["eps"], X - oracle.reveal(a))
    assert np.array_equal(im["delta"], Y - oracle.reveal(b))


def test_beaver_party0_gets_eps_delta():
    # reading R7: exactly party 0 adds ε@δ; all others: c_p + ε@b_p + a_p@δ
    P = 3
    X, Y, xs, ys, a, b, c = _shared_inputs(P, 4, 5, 6, seed=3)
    z, im = oracle.beaver_matmul(xs, ys, a, b, c, want_intermediates=True)
    e, d = im["eps"], im["delta"]
    for p in range(P):
        exp = c[p] + e @ b[p] + a[p] @ d + (e @ d if p == 0 else 0)
        assert np.array_equal(z[p], exp.astype(np.uint64))


def test_beaver_spec_scalar_examples():
    for P in (1, 2, 3):
        xs = oracle.share(P, MASTER, oracle.encode([[2.0]]), 0, 1)
        ys = oracle.share(P, MASTER, oracle.encode([[3.0]]), 0, 2)
        a, b, c = oracle.ttp_triple(P, MASTER, 11, 1, 1, 1)
        z = oracle.truncate(oracle.beaver_matmul(xs, ys, a, b, c), 16, MASTER, wrap_id=3)
        assert abs(oracle.decode(oracle.reveal(z))[0, 0] - 6.0) <= 2.0 ** -16
        y0 = oracle.share(P, MASTER, np.zeros((1, 1), dtype=np.uint64), 0, 4)
        z0 = oracle.truncate(oracle.beaver_matmul(xs, y0, a, b, c), 16, MASTER, wrap_id=4)
        assert abs(oracle.decode(oracle.reveal(z0))[0, 0]) <= 2.0 ** -16


def test_p1_closed_form_fixed_point_matmul():
    # P = 1 runs the protocol on unencrypted data: the truncated result
    # is the textbook fixed-point product round_half_up(X@Y / 2^16), in big ints.
    M, K, N = 6, 9, 5
    X, Y, xs, ys, a, b, c = _shared_inputs(1, M, K, N, seed=21)
    zt = oracle.truncate(oracle.beaver_matmul(xs, ys, a, b, c), 16)
    for i in range(M):
        for j in range(N):
            s = sum(_signed(int(X[i, k])) * _signed(int(Y[k, j])) for k in range(K))
            exp = (s + (1 << 15)) >> 16            # floor((s + 2^15)/2^16) = round half up
            assert int(zt[0, i, j]) == exp % Q


# ----------------------------------------------------------------- O6/O7 truncation
def test_wrap_count_vs_bigint_and_spec_example():
    # shares {2^63, 2^63, 5} of x = 5.  With signed representatives
    # (reading R9) Σ signed = −2^64 + 5, so θ = −1.
    x = np.array([[1 << 63], [1 << 63], [5]], dtype=np.uint64)
    assert int(oracle.wrap_count(x)[0]) == -1
    s = synth.uniform_ring((4, 300), 31)
    th = oracle.wrap_count(s)
    for i in range(300):
        tot = sum(_signed(int(s[p, i])) for p in range(4))
        assert (tot - _signed(tot % Q)) // Q == int(th[i])
    assert np.all(oracle.wrap_count(s[:1]) == 0)                     # P=1: θ = 0


def test_truncate_local_p2_error_bound_and_failures():
    # P=2 local truncation: within ±1 ulp of x/2^16 unless θ_x ≠ 0 (prob |x|/Q)
    rng = np.random.default_rng(5)
    n = 20000
    xv = rng.integers(-(1 << 40), 1 << 40, size=n, dtype=np.int64)
    xs = oracle.share(2, MASTER, synth.to_ring(xv), 0, 8)
    out, dg = oracle.truncate(xs, 16, diagnostics=True)
    rv = oracle.reveal(out).view(np.int64)
    exact = xv / 65536.0
    ok = dg["theta"] == 0
    assert np.all(np.abs(rv[ok] - exact[ok]) <= 1.0)
    assert np.sum(~ok) <= 3          # expected ≈ Σ|x|/2^64 ≈ 6e-4


def test_truncate_local_is_floor_plus_bit15():
    v = np.array([[0, 1 << 15, (1 << 15) - 1, Q - (1 << 15), Q - (1 << 15) - 1, Q - 1, (3 << 16) + 5]], dtype=np.uint64)
    out = oracle.truncate_local(v, 16)[0]
    for vi, oi in zip(v[0], out):
        s = _signed(int(vi))
        assert _signed(int(oi)) == (s + (1 << 15)) >> 16


@pytest.mark.parametrize("P", [3, 4, 8])
def test_alg1_identity_and_accuracy(P):
    # Alg. 1 + correction with η skipped.
    rng = np.random.default_rng(P)
    n = 5000
    xv = rng.integers(-(1 << 40), 1 << 40, size=n, dtype=np.int64)
    xs = oracle.share(P, MASTER, synth.to_ring(xv), 0, 12)
    r, th_r = oracle.wrap_pair(P, MASTER, 77, n)
    # wrap pair: revealed θ_r equals the exact wrap count of r's shares (big-int oracle)
    th_exact = oracle.wrap_count(r)
    assert np.array_equal(oracle.reveal(th_r).view(np.int64), th_exact)
    out, dg = oracle.truncate_alg1(xs, r, th_r, 16, diagnostics=True)
    rv = oracle.reveal(out).view(np.int64)
    good = dg["eta"] == 0
    # with η = 0 the correction is exact: error of the per-share rounding only, ≤ P/2 ulp
    assert np.all(np.abs(rv[good] - xv[good] / 65536.0) <= P / 2)
    # η ≠ 0 has probability |x|/Q: here ≤ 2^40/2^64 — essentially never
    assert np.sum(~good) <= 2
    # θ_x identity element-wise: θ_x = θ_z + β − θ_r − η
    xsum = [sum(_signed(int(xs[p, i])) for p in range(P)) for i in range(50)]
    for i in range(50):
        tx = (xsum[i] - int(xv[i])) // Q
        z = int(dg["z"][i])
        zsh = [(int(xs[p, i]) + int(r[p, i])) % Q for p in range(P)]
        beta = sum((_signed(int(xs[p, i])) + _signed(int(r[p, i])) - _signed(zsh[p])) // Q for p in range(P))
        theta_z = (sum(_signed(v) for v in zsh) - _signed(z)) // Q
        eta = (int(xv[i]) + _signed(sum(int(r[p, i]) for p in range(P)) % Q) - _signed(z)) // Q
        assert tx == theta_z + beta - int(th_exact[i]) - eta


def test_alg1_failure_rate_matches_paper():
    # P(η ≠ 0) = |x|/Q regardless of |P|: at |x| = 2^60 that is 1/16
    P, n = 4, 40000
    xv = np.full(n, 1 << 60, dtype=np.int64)
    xs = oracle.share(P, MASTER, synth.to_ring(xv), 0, 13)
    r, th_r = oracle.wrap_pair(P, MASTER, 78, n)
    _, dg = oracle.truncate_alg1(xs, r, th_r, 16, diagnostics=True)
    rate = float(np.mean(dg["eta"] != 0))
    sigma = (0.0625 * 0.9375 / n) ** 0.5
    assert abs(rate - 0.0625) < 6 * sigma


def test_sampled_triple_and_shares_match_full():
    P, M, K, N = 3, 12, 9, 10
    a, b, c = oracle.ttp_triple(P, MASTER, 6, M, K, N)
    rows, cols = [11, 0, 5], [9, 2]
    a2, b2, c2 = oracle.ttp_triple_sampled(P, MASTER, 6, M, K, N, rows, cols)
    assert np.array_equal(a2, a[:, rows])
    assert np.array_equal(b2, b[:, :, cols])
    assert np.array_equal(c2, c[:, rows][:, :, cols])
    Y = synth.uniform_ring((K, N), 4)
    full = oracle.share(P, MASTER, Y, 2, 33)
    idx = np.array([[k * N + j for j in cols] for k in range(K)])
    part = oracle.share_indices(P, MASTER, Y.ravel()[idx.ravel()], 2, 33, idx)
    assert np.array_equal(part.reshape(P, K, len(cols)), full[:, :, cols])


def test_wrap_pair_indices_match_full():
    r, th = oracle.wrap_pair(4, MASTER, 17, 50)
    idx = [49, 3, 0, 17]
    r2, th2 = oracle.wrap_pair_indices(4, MASTER, 17, idx)
    assert np.array_equal(r2, r[:, idx]) and np.array_equal(th2, th[:, idx])


def test_share_range_matches_full():
    x = synth.uniform_ring((10, 7), seed=3)
    full = oracle.share(3, MASTER, x, 1, 21)
    part = oracle.share(3, MASTER, x[4:6], 1, 21, start=4 * 7)
    assert np.array_equal(part, full[:, 4:6])

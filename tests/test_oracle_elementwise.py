"""Pins of the oracle's elementwise Beaver multiplication and square (SURVEY
§8(f) NEXT-1; App. A.1.1) against things other than itself:
Python big-integer arithmetic (the ring Z/2^64 written out), the closed forms
the paper states (c = ab, b = a^2, [x][y] = [c] + ε[b] + [a]δ + εδ,
[x^2] = [b] + 2ε[a] + ε^2), SPEC's printed examples (mul(2.0, 3.0) = 6.0,
square(3.0) = 9.0, products with 0), and the float64 product of the decoded
values.  A dropped or doubled term, a term added by every party instead of
party 0, or a wrong factor (ε[a] instead of 2ε[a]) fails one of them.
"""
import numpy as np
import pytest

import oracle
import synth

MASTER = synth.MASTER_SEED
Q = 1 << 64


def _ints(a):
    return [int(v) for v in np.asarray(a, dtype=np.uint64).ravel()]


def _shares(P, X, share_id):
    return oracle.share(P, MASTER, X, 0, share_id)


@pytest.mark.parametrize("P", [1, 2, 3, 8])
def test_mul_triple_defining_property_bigint(P):
    a, b, c = oracle.ttp_mul_triple(P, MASTER, 11, (5, 7))
    A = [sum(col) % Q for col in zip(*[_ints(a[p]) for p in range(P)])]
    B = [sum(col) % Q for col in zip(*[_ints(b[p]) for p in range(P)])]
    C = [sum(col) % Q for col in zip(*[_ints(c[p]) for p in range(P)])]
    assert C == [(x * y) % Q for x, y in zip(A, B)]          # c = ab
    if P > 1:   # a, b uniform-looking (not all-zero / equal across parties)
        assert len(set(_ints(a[0])) | set(_ints(a[1]))) == 70


@pytest.mark.parametrize("P", [1, 2, 5])
def test_square_pair_defining_property_bigint(P):
    a, b = oracle.ttp_square_pair(P, MASTER, 12, (33,))
    A = [sum(col) % Q for col in zip(*[_ints(a[p]) for p in range(P)])]
    B = [sum(col) % Q for col in zip(*[_ints(b[p]) for p in range(P)])]
    assert B == [(x * x) % Q for x in A]                    # b = a^2


def test_triple_streams_follow_the_layout():
    """a_p / b_p / c_p (p >= 1) are the PRG streams A||p||id, B||p||id, C||p||id
    (R6; the PRG itself is pinned by the Philox KAT and the frozen table)."""
    P, tid = 3, 77
    _, kt = oracle.derive_keys(MASTER, P)
    a, b, c = oracle.ttp_mul_triple(P, MASTER, tid, (9,))
    for p in range(P):
        assert np.array_equal(a[p], oracle.prg(kt, oracle.stream_id(oracle.TAG_A, p, tid), 9))
        assert np.array_equal(b[p], oracle.prg(kt, oracle.stream_id(oracle.TAG_B, p, tid), 9))
        if p:
            assert np.array_equal(c[p], oracle.prg(kt, oracle.stream_id(oracle.TAG_C, p, tid), 9))


@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
def test_beaver_mul_identity_bigint(P):
    """Before truncation Σ_p z_p = x·y mod 2^64 exactly (App. A.1.1 identity)."""
    rng = np.random.default_rng(P)
    X = rng.integers(0, 2**64 - 1, size=(4, 6), dtype=np.uint64, endpoint=True)
    Y = rng.integers(0, 2**64 - 1, size=(4, 6), dtype=np.uint64, endpoint=True)
    a, b, c = oracle.ttp_mul_triple(P, MASTER, 20 + P, X.shape)
    z = oracle.beaver_mul(_shares(P, X, 1), oracle.share(P, MASTER, Y, 1 % P, 2), a, b, c)
    Z = [sum(col) % Q for col in zip(*[_ints(z[p]) for p in range(P)])]
    assert Z == [(x * y) % Q for x, y in zip(_ints(X), _ints(Y))]


@pytest.mark.parametrize("P", [1, 2, 3, 8])
def test_beaver_square_identity_bigint(P):
    rng = np.random.default_rng(100 + P)
    X = rng.integers(0, 2**64 - 1, size=(37,), dtype=np.uint64, endpoint=True)
    a, b = oracle.ttp_square_pair(P, MASTER, 40 + P, X.shape)
    z = oracle.beaver_square(_shares(P, X, 3), a, b)
    Z = [sum(col) % Q for col in zip(*[_ints(z[p]) for p in range(P)])]
    assert Z == [(x * x) % Q for x in _ints(X)]


def test_only_party_zero_adds_the_public_term():
    """With ε, δ fixed, parties p >= 1 hold c_p + ε b_p + a_p δ (no εδ) and
    party 0 additionally εδ; the square's parties p >= 1 hold b_p + 2ε a_p.
    Recomputed with Python big integers from the oracle's revealed ε, δ."""
    P = 3
    rng = np.random.default_rng(5)
    X = rng.integers(0, 2**64 - 1, size=(8,), dtype=np.uint64, endpoint=True)
    Y = rng.integers(0, 2**64 - 1, size=(8,), dtype=np.uint64, endpoint=True)
    xs, ys = _shares(P, X, 5), oracle.share(P, MASTER, Y, 1, 6)
    a, b, c = oracle.ttp_mul_triple(P, MASTER, 50, X.shape)
    z, it = oracle.beaver_mul(xs, ys, a, b, c, want_intermediates=True)
    eps = [sum(v) % Q for v in zip(*[[int(t) for t in xs[p] - a[p]] for p in range(P)])]
    dlt = [sum(v) % Q for v in zip(*[[int(t) for t in ys[p] - b[p]] for p in range(P)])]
    assert _ints(it["eps"]) == eps and _ints(it["delta"]) == dlt
    for p in range(P):
        want = [(int(c[p][i]) + eps[i] * int(b[p][i]) + int(a[p][i]) * dlt[i] + (eps[i] * dlt[i] if p == 0 else 0)) % Q
                for i in range(8)]
        assert _ints(z[p]) == want
    a2, b2 = oracle.ttp_square_pair(P, MASTER, 51, X.shape)
    z2, it2 = oracle.beaver_square(xs, a2, b2, want_intermediates=True)
    e2 = _ints(it2["eps"])
    for p in range(P):
        want = [(int(b2[p][i]) + 2 * e2[i] * int(a2[p][i]) + (e2[i] * e2[i] if p == 0 else 0)) % Q for i in range(8)]
        assert _ints(z2[p]) == want


def test_p1_closed_form():
    """P = 1: the protocol on unencrypted data (R16) gives z = x·y exactly."""
    X = synth.uniform_fixed((50,), 7)
    Y = synth.uniform_fixed((50,), 8)
    a, b, c = oracle.ttp_mul_triple(1, MASTER, 60, X.shape)
    z = oracle.beaver_mul(X[None], Y[None], a, b, c)
    assert np.array_equal(z[0], X * Y)
    a2, b2 = oracle.ttp_square_pair(1, MASTER, 61, X.shape)
    assert np.array_equal(oracle.beaver_square(X[None], a2, b2)[0], X * X)


@pytest.mark.parametrize("P", [2, 4])
def test_spec_examples_mul_and_square(P):
    """mul(enc 2.0, enc 3.0) -> 6.0 ± 2^-16, mul by 0 -> 0,
    square(enc 3.0) -> 9.0, square(0) -> 0 (after truncation; Alg. 1 for P > 2)."""
    X = oracle.encode(np.array([2.0, 0.0, -1.5, 3.0]))
    Y = oracle.encode(np.array([3.0, 5.0, 0.0, -3.0]))
    a, b, c = oracle.ttp_mul_triple(P, MASTER, 70, X.shape)
    z = oracle.beaver_mul(_shares(P, X, 7), oracle.share(P, MASTER, Y, 1, 8), a, b, c)
    got = oracle.decode(oracle.reveal(oracle.truncate(z, 16, MASTER, wrap_id=3)))
    assert np.all(np.abs(got - np.array([6.0, 0.0, 0.0, -9.0])) <= 2.0 ** -16 * P / 2)
    a2, b2 = oracle.ttp_square_pair(P, MASTER, 71, X.shape)
    z2 = oracle.beaver_square(_shares(P, X, 9), a2, b2)
    got2 = oracle.decode(oracle.reveal(oracle.truncate(z2, 16, MASTER, wrap_id=4)))
    assert np.all(np.abs(got2 - np.array([4.0, 0.0, 2.25, 9.0])) <= 2.0 ** -16 * P / 2)


@pytest.mark.parametrize("P", [2, 3, 8])
def test_decoded_accuracy_vs_float64(P):
    """Inputs in [-8, 8]: every decoded product within 2^-14 of the float64
    product (exact: |x y| 2^32 < 2^53), except the oracle-flagged wrap events
    (θ != 0 for P = 2, η != 0 for Alg. 1), whose count is tiny."""
    n = 20000
    X = synth.uniform_fixed((n,), 300 + P)
    Y = synth.uniform_fixed((n,), 400 + P)
    a, b, c = oracle.ttp_mul_triple(P, MASTER, 80 + P, (n,))
    z = oracle.beaver_mul(_shares(P, X, 10), oracle.share(P, MASTER, Y, 1, 11), a, b, c)
    zt, dg = oracle.truncate(z, 16, MASTER, wrap_id=5, diagnostics=True)
    got = oracle.decode(oracle.reveal(zt))
    exact = (X.view(np.int64).astype(np.float64) / 65536) * (Y.view(np.int64).astype(np.float64) / 65536)
    fail = (dg["theta"] != 0) if P <= 2 else (dg["eta"] != 0)
    assert np.all(np.abs(got - exact)[~fail] <= 2.0 ** -14)
    assert fail.sum() <= 2
    # square == mul(x, x) after reveal, bit for bit before truncation (S:275 cross-check)
    a2, b2 = oracle.ttp_square_pair(P, MASTER, 90 + P, (n,))
    zs = oracle.beaver_square(_shares(P, X, 12), a2, b2)
    a3, b3, c3 = oracle.ttp_mul_triple(P, MASTER, 95 + P, (n,))
    zm = oracle.beaver_mul(_shares(P, X, 13), _shares(P, X, 14), a3, b3, c3)
    assert np.array_equal(oracle.reveal(zs), oracle.reveal(zm))

"""Pins of the oracle's ReLU path: binary sharing, the
bitwise AND with binary Beaver triples (App. A.1.2), the Kogge-Stone ring adder,
A2B (§4.1 / A.1.3), single-bit B2A (Alg. 2) and ReLU([x]) = [x][x >= 0]
(§4.2, A.1.4) — against numpy's plaintext bit operations and wrapping adds,
exhaustive truth tables, SPEC's printed examples and the exact relu of the
two's-complement integers.  A wrong shift direction, a missing carry level, a
public term on every party or B2A's 2[r]z term with the wrong sign fails one."""
import itertools

import numpy as np
import pytest

import oracle
import synth

MASTER = synth.MASTER_SEED
ONES = np.uint64(0xFFFFFFFFFFFFFFFF)


def _rand(n, seed):
    return synth.uniform_ring((n,), seed)


@pytest.mark.parametrize("P", [1, 2, 3, 8])
def test_binary_share_reveal_and_zero_share(P):
    X = _rand(100, 1)
    s = oracle.bshare(P, MASTER, X, P - 1, 5)
    assert np.array_equal(oracle.breveal(s), X)                   # x = ⊕ shares
    assert not np.any(oracle.breveal(oracle.bshare(P, MASTER, None, 0, 6, shape=(50,))))   # zero-share
    if P == 1:
        assert np.array_equal(s[0], X)


@pytest.mark.parametrize("P", [1, 2, 4])
def test_binary_and_matches_plaintext(P):
    X, Y = _rand(500, 2), _rand(500, 3)
    a, b, c = oracle.ttp_binary_triple(P, MASTER, 9, X.shape)
    assert np.array_equal(oracle.breveal(c), oracle.breveal(a) & oracle.breveal(b))   # c = a ⊗ b
    xs, ys = oracle.bshare(P, MASTER, X, 0, 1), oracle.bshare(P, MASTER, Y, P - 1, 2)
    assert np.array_equal(oracle.breveal(oracle.binary_and(xs, ys, a, b, c)), X & Y)
    zero, ones = oracle.bshare(P, MASTER, np.zeros_like(X), 0, 3), oracle.bshare(P, MASTER, np.full_like(X, ONES), 0, 4)
    assert not np.any(oracle.breveal(oracle.binary_and(xs, zero, a, b, c)))            # x AND 0 = 0
    assert np.array_equal(oracle.breveal(oracle.binary_and(xs, ones, a, b, c)), X)     # x AND 1...1 = x


def test_de_morgan_bruteforce_4bit():
    """NOT(x AND y) == (NOT x) OR (NOT y), OR composed as a ⊕ b ⊕ (a AND b), over
    all 4-bit pairs at P = 2 (SPEC bin_share invariant)."""
    P = 2
    pairs = np.array(list(itertools.product(range(16), range(16))), dtype=np.uint64)
    X, Y = pairs[:, 0].copy(), pairs[:, 1].copy()
    xs, ys = oracle.bshare(P, MASTER, X, 0, 1), oracle.bshare(P, MASTER, Y, 1, 2)
    t1 = oracle.ttp_binary_triple(P, MASTER, 1, X.shape)
    t2 = oracle.ttp_binary_triple(P, MASTER, 2, X.shape)
    notx, noty = xs.copy(), ys.copy()
    notx[0] ^= np.uint64(15)
    noty[0] ^= np.uint64(15)
    lhs = oracle.binary_and(xs, ys, *t1)
    lhs[0] ^= np.uint64(15)
    rhs = notx ^ noty ^ oracle.binary_and(notx, noty, *t2)
    assert np.array_equal(oracle.breveal(lhs), oracle.breveal(rhs))
    assert np.array_equal(oracle.breveal(lhs), (~(X & Y)) & np.uint64(15))


@pytest.mark.parametrize("P", [1, 2, 3])
def test_add_ring_matches_wrapping_add(P):
    X, Y = _rand(2000, 4), _rand(2000, 5)
    X[:3] = [ONES, 0, 1 << 63]
    Y[:3] = [1, 0, 1 << 63]          # 2^64-1 + 1 -> 0 (SPEC add_ring), 0 + 0, 2^63 + 2^63 -> 0
    xs, ys = oracle.bshare(P, MASTER, X, 0, 1), oracle.bshare(P, MASTER, Y, P - 1, 2)
    got = oracle.breveal(oracle.add_ring(P, MASTER, 7, xs, ys))
    assert np.array_equal(got, X + Y)
    assert got[0] == 0 and got[2] == 0


@pytest.mark.parametrize("P", [1, 2, 3, 4, 5, 8])
def test_a2b_reveals_twos_complement_bits(P):
    X = _rand(3000, 6)
    xs = oracle.share(P, MASTER, X, 0, 1)
    assert np.array_equal(oracle.breveal(oracle.a2b(MASTER, 11, xs)), X)
    enc = oracle.encode(np.array([-1.0, 0.0, 2.5]))
    b = oracle.breveal(oracle.a2b(MASTER, 12, oracle.share(P, MASTER, enc, 0, 2)))
    assert [int(v) >> 63 for v in b] == [1, 0, 0]                 # encode(-1.0) has the sign bit set


@pytest.mark.parametrize("P", [2, 3, 4])
def test_b2a_bit_truth_table_exhaustive(P):
    """All (b, r) combinations, with hand-made shares of b and of the bit pair
    (r arithmetic and binary) — Alg. 2 must return arithmetic shares of b."""
    rng = np.random.default_rng(P)
    for bv, rv in itertools.product((0, 1), (0, 1)):
        n = 64
        bsh = rng.integers(0, 2**63, size=(P, n), dtype=np.uint64)           # random high bits, ignored
        bsh[0] ^= (np.bitwise_xor.reduce(bsh, axis=0) & np.uint64(1)) ^ np.uint64(bv)
        rB = rng.integers(0, 2, size=(P, n), dtype=np.uint64)
        rB[0] ^= np.bitwise_xor.reduce(rB, axis=0) ^ np.uint64(rv)
        rA = rng.integers(0, 2**64 - 1, size=(P, n), dtype=np.uint64, endpoint=True)
        rA[0] -= rA.sum(axis=0, dtype=np.uint64) - np.uint64(rv)
        out, z = oracle.b2a_bit(bsh, rA, rB, want_z=True)
        assert np.all(oracle.reveal(out) == bv)
        assert np.all(z == bv ^ rv)                                            # revealed mask bit


@pytest.mark.parametrize("P", [2, 3])
def test_bit_pair_consistency(P):
    rA, rB = oracle.ttp_bit_pair(P, MASTER, 5, (1000,))
    r = oracle.breveal(rB)
    assert set(np.unique(r)) <= {0, 1} and np.array_equal(oracle.reveal(rA), r)
    assert 400 < int(r.sum()) < 600                                            # a random bit


@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
def test_relu_exact_and_rounds(P):
    X = _rand(4000, 7)
    X[:5] = [0, 1, ONES, 1 << 63, (1 << 63) - 1]                  # 0, 1, -1, INT64_MIN, INT64_MAX
    xs = oracle.share(P, MASTER, X, 0, 1)
    out, d = oracle.relu(MASTER, 21, xs, diagnostics=True)
    xi = X.view(np.int64)
    assert np.array_equal(oracle.reveal(out).view(np.int64), np.maximum(xi, 0))     # exact: scale-1 indicator
    assert np.array_equal(oracle.reveal(d["sign"]), (xi < 0).astype(np.uint64))
    levels = int(np.ceil(np.log2(P))) if P > 1 else 0
    assert d["rounds"] == 7 * levels + 2                           # A2B adders + B2A + multiplication


def test_relu_spec_examples():
    """SPEC compare_logic: relu(enc -2.0) -> 0, relu(enc 2.0) -> 2.0 (P = 2)."""
    enc = oracle.encode(np.array([-2.0, 2.0, 0.0, -0.5, 7.25]))
    out = oracle.relu(MASTER, 22, oracle.share(2, MASTER, enc, 0, 9))
    assert np.array_equal(oracle.decode(oracle.reveal(out)), np.array([0.0, 2.0, 0.0, 0.0, 7.25]))

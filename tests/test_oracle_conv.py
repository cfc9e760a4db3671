"""Pins of the oracle's ring convolution and Beaver convolution (SURVEY §8(f)
NEXT-2; "the same procedure ... matrix multiplication and
convolution") against things other than itself: PyTorch's float64 conv2d on
small integers (exact), an im2col + numpy wrapping-uint64 matmul written here,
the triple's defining property, the Beaver identity, the P = 1 closed form and
the decoded accuracy.  A swapped stride/padding axis, a transposed weight, a
dropped term or a public term added by every party fails one of them."""
import numpy as np
import pytest
import torch

import oracle
import synth

MASTER = synth.MASTER_SEED
GEOMS = [  # (B, C, H, W, Cout, kh, kw, stride, padding)
    (1, 3, 11, 11, 4, 7, 7, 2, 3),       # ResNet conv1 shape family (7x7 / 2, pad 3)
    (2, 5, 6, 7, 3, 3, 3, 1, 1),         # 3x3 same padding, batch 2, W != H
    (1, 4, 9, 8, 6, 1, 1, 2, 0),         # 1x1 stride-2 downsample
    (1, 2, 5, 9, 3, 2, 4, (1, 2), (0, 1)),  # rectangular kernel, per-axis stride / padding
]


def _im2col_conv(x, w, g):
    """Reference written here: explicit zero padding, im2col by slicing, then
    numpy's wrapping uint64 matmul (a different construction from the oracle's loops)."""
    B, C, H, W = x.shape
    Cout = w.shape[0]
    Bo, _, Ho, Wo = oracle.conv_out_shape(g)
    xp = np.zeros((B, C, H + 2 * g.ph, W + 2 * g.pw), dtype=np.uint64)
    xp[:, :, g.ph:g.ph + H, g.pw:g.pw + W] = x
    cols = np.zeros((B, Ho, Wo, C, g.kh, g.kw), dtype=np.uint64)
    for ky in range(g.kh):
        for kx in range(g.kw):
            cols[:, :, :, :, ky, kx] = xp[:, :, ky:ky + g.sh * Ho:g.sh, kx:kx + g.sw * Wo:g.sw].transpose(0, 2, 3, 1)
    out = cols.reshape(B * Ho * Wo, -1) @ w.reshape(Cout, -1).T
    return out.reshape(B, Ho, Wo, Cout).transpose(0, 3, 1, 2)


def _geom(t):
    return oracle.conv_geom(*t)


@pytest.mark.parametrize("t", GEOMS)
def test_conv2d_matches_torch_float64_on_small_integers(t):
    g = _geom(t)
    rng = np.random.default_rng(1)
    x = rng.integers(-300, 300, (g.B, g.C, g.H, g.W))
    w = rng.integers(-300, 300, (g.Cout, g.C, g.kh, g.kw))
    got = oracle.conv2d(synth.to_ring(x), synth.to_ring(w), g).view(np.int64)
    ref = torch.nn.functional.conv2d(torch.tensor(x, dtype=torch.float64), torch.tensor(w, dtype=torch.float64),
                                     stride=(g.sh, g.sw), padding=(g.ph, g.pw)).numpy()
    assert np.array_equal(got, ref.astype(np.int64))


@pytest.mark.parametrize("t", GEOMS)
def test_conv2d_matches_im2col_uint64_matmul_full_range(t):
    g = _geom(t)
    rng = np.random.default_rng(2)
    x = rng.integers(0, 2**64 - 1, (g.B, g.C, g.H, g.W), dtype=np.uint64, endpoint=True)
    w = rng.integers(0, 2**64 - 1, (g.Cout, g.C, g.kh, g.kw), dtype=np.uint64, endpoint=True)
    assert np.array_equal(oracle.conv2d(x, w, g), _im2col_conv(x, w, g))


@pytest.mark.parametrize("P", [1, 2, 3])
def test_conv_triple_defining_property(P):
    g = _geom(GEOMS[1])
    a, b, c = oracle.ttp_conv_triple(P, MASTER, 5, g)
    assert np.array_equal(oracle.reveal(c), _im2col_conv(oracle.reveal(a), oracle.reveal(b), g))


@pytest.mark.parametrize("P", [1, 2, 3, 4])
@pytest.mark.parametrize("t", GEOMS[:3])
def test_beaver_conv_identity(P, t):
    """Before truncation Σ_p z_p = conv(X, Y) mod 2^64, ε / δ revealed at the
    input / weight shapes (R22)."""
    g = _geom(t)
    rng = np.random.default_rng(P)
    X = rng.integers(0, 2**64 - 1, (g.B, g.C, g.H, g.W), dtype=np.uint64, endpoint=True)
    Y = rng.integers(0, 2**64 - 1, (g.Cout, g.C, g.kh, g.kw), dtype=np.uint64, endpoint=True)
    xs, ys = oracle.share(P, MASTER, X, 0, 1), oracle.share(P, MASTER, Y, 1 % P, 2)
    a, b, c = oracle.ttp_conv_triple(P, MASTER, 6, g)
    z, it = oracle.beaver_conv2d(xs, ys, a, b, c, g, want_intermediates=True)
    assert np.array_equal(oracle.reveal(z), _im2col_conv(X, Y, g))
    assert it["eps"].shape == X.shape and np.array_equal(it["eps"], oracle.reveal(xs - a))
    assert it["delta"].shape == Y.shape and np.array_equal(it["delta"], oracle.reveal(ys - b))


def test_public_term_only_on_party_zero():
    P, g = 3, _geom(GEOMS[2])
    X = synth.uniform_fixed((g.B, g.C, g.H, g.W), 3)
    Y = synth.uniform_fixed((g.Cout, g.C, g.kh, g.kw), 4)
    xs, ys = oracle.share(P, MASTER, X, 0, 1), oracle.share(P, MASTER, Y, 1, 2)
    a, b, c = oracle.ttp_conv_triple(P, MASTER, 7, g)
    z, it = oracle.beaver_conv2d(xs, ys, a, b, c, g, want_intermediates=True)
    eps, dlt = it["eps"], it["delta"]
    for p in range(P):
        want = c[p] + _im2col_conv(eps, b[p], g) + _im2col_conv(a[p], dlt, g)
        if p == 0:
            want = want + _im2col_conv(eps, dlt, g)
        assert np.array_equal(z[p], want)


def test_p1_closed_form():
    g = _geom(GEOMS[0])
    X = synth.uniform_fixed((g.B, g.C, g.H, g.W), 5)
    Y = synth.uniform_fixed((g.Cout, g.C, g.kh, g.kw), 6)
    a, b, c = oracle.ttp_conv_triple(1, MASTER, 8, g)
    assert np.array_equal(oracle.beaver_conv2d(X[None], Y[None], a, b, c, g)[0], _im2col_conv(X, Y, g))


@pytest.mark.parametrize("P", [2, 3])
def test_decoded_accuracy_vs_float64(P):
    g = _geom((1, 8, 12, 12, 6, 3, 3, 1, 1))
    X = synth.gaussian_fixed((g.B, g.C, g.H, g.W), 9, 1.0, 0, 8, absval=True)
    Y = synth.gaussian_fixed((g.Cout, g.C, g.kh, g.kw), 10, (2.0 / 72) ** 0.5, -8, 8)
    xs, ys = oracle.share(P, MASTER, X, 0, 1), oracle.share(P, MASTER, Y, 1, 2)
    a, b, c = oracle.ttp_conv_triple(P, MASTER, 9, g)
    z, dg = oracle.truncate(oracle.beaver_conv2d(xs, ys, a, b, c, g), 16, MASTER, wrap_id=2, diagnostics=True)
    got = oracle.decode(oracle.reveal(z))
    ref = torch.nn.functional.conv2d(torch.tensor(X.view(np.int64) / 65536.0), torch.tensor(Y.view(np.int64) / 65536.0),
                                     stride=1, padding=1).numpy()
    fail = (dg["theta"] != 0) if P <= 2 else (dg["eta"] != 0)
    assert np.all(np.abs(got - ref)[~fail] <= 2.0 ** -14)
    assert fail.sum() <= 1


# ---------------------------------------------------------------- 1-D (Wav2Letter)
CONV1D = [  # (B, C, L, Cout, k, stride, padding)
    (1, 1, 400, 5, 25, 16, 4),            # Wav2Letter conv1 family (waveform front end, 250 / 160 / 45)
    (2, 6, 30, 4, 8, 2, 3),               # conv2 family (k 48, stride 2, pad 23)
    (1, 5, 12, 7, 7, 1, 3),               # conv3-9 (k 7, same padding)
    (3, 9, 11, 6, 1, 1, 0),               # 1x1 layers
]


def _conv1d_loops(x, w, stride, pad):
    """1-D ring convolution written out here (explicit loops, wrapping via Python ints)."""
    B, C, L = x.shape
    Cout, _, k = w.shape
    Lo = (L + 2 * pad - k) // stride + 1
    out = np.zeros((B, Cout, Lo), dtype=np.uint64)
    for bi in range(B):
        for co in range(Cout):
            for o in range(Lo):
                acc = 0
                for ci in range(C):
                    for t in range(k):
                        pos = o * stride - pad + t
                        if 0 <= pos < L:
                            acc += int(x[bi, ci, pos]) * int(w[co, ci, t])
                out[bi, co, o] = acc % 2 ** 64
    return out


@pytest.mark.parametrize("t", CONV1D)
def test_conv1d_as_h1_conv2d(t):
    """The 1-D geometry (H = kh = 1) of the oracle's conv2d equals a 1-D convolution
    written out with loops on full-range ring elements, and PyTorch's float64 conv1d
    on small integers."""
    B, C, L, Cout, k, st, pd = t
    g = oracle.conv1d_geom(*t)
    rng = np.random.default_rng(sum(t))
    x = synth.uniform_ring((B, C, L), 11 + L)
    w = synth.uniform_ring((Cout, C, k), 12 + k)
    got = oracle.conv2d(x.reshape(B, C, 1, L), w.reshape(Cout, C, 1, k), g)
    Lo = (L + 2 * pd - k) // st + 1
    assert got.shape == (B, Cout, 1, Lo)
    assert np.array_equal(got.reshape(B, Cout, Lo), _conv1d_loops(x, w, st, pd))
    xs = rng.integers(-300, 300, (B, C, L))
    ws = rng.integers(-300, 300, (Cout, C, k))
    ref = torch.nn.functional.conv1d(torch.from_numpy(xs).double(), torch.from_numpy(ws).double(), stride=st,
                                     padding=pd).numpy().astype(np.int64)
    got2 = oracle.conv2d(synth.to_ring(xs).reshape(B, C, 1, L), synth.to_ring(ws).reshape(Cout, C, 1, k), g)
    assert np.array_equal(got2.view(np.int64).reshape(B, Cout, Lo), ref)


def test_wav2letter_geometry_matches_the_gemm_shapes():
    """synth.WAV2LETTER_CONV1D reproduces the im2col GEMM shapes of WAV2LETTER_B1
    (M = L_out, K = C * k, N = Cout), i.e. torchaudio's waveform Wav2Letter on 1 s
    of 16 kHz audio."""
    shapes = []
    for name, C, L, Co, k, st, pd, cnt in synth.WAV2LETTER_CONV1D:
        Lo = (L + 2 * pd - k) // st + 1
        shapes.append((name, Lo, C * k, Co, cnt))
    assert shapes == [tuple(s) for s in synth.WAV2LETTER_B1]

"""GPU parity of the private 2-D convolution with conv triples (SURVEY §8(f)
NEXT-2) against the oracle, bit for bit: the TTP conv triples, the
fused all-parties path (implicit im2col limb split + ring GEMM with the NCHW
epilogue, transposed GEMM for one small image), the one-party kernels (mask at
the input / weight shapes -> caller's reveal -> finish), the 1-rank NCCL path,
and truncation (local and Alg. 1).  Geometries cover 7x7/2 pad 3, 3x3 pad 1,
1x1/2, rectangular kernels with per-axis stride/padding, batch 2, ResNet-50's
conv1 and a layer-4 conv at full size."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu
MASTER = synth.MASTER_SEED
GEOMS = [  # (B, C, H, W, Cout, kh, kw, stride, padding)
    (1, 3, 23, 23, 8, 7, 7, 2, 3),
    (2, 5, 9, 10, 7, 3, 3, 1, 1),
    (1, 16, 14, 14, 40, 1, 1, 2, 0),
    (1, 6, 7, 12, 300, 2, 4, (1, 2), (0, 1)),       # Cout >> pixels: transposed GEMM
    (3, 4, 5, 5, 3, 5, 5, 1, 2),
    (2, 6, 1, 30, 4, 1, 8, (1, 2), (0, 3)),         # a 1-D convolution (H = kh = 1): Wav2Letter's conv2 family
]


@pytest.fixture(scope="module")
def mpc():
    from paper_2109_00984_b200 import build
    build.build()
    import paper_2109_00984_b200 as m
    assert torch.cuda.is_available(), "GPU tests need a B200"
    return m


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).cuda().view(torch.uint64)


def host(t):
    return t.view(torch.int64).cpu().numpy().view(np.uint64)


def _inputs(g, seed):
    X = synth.gaussian_fixed((g.B, g.C, g.H, g.W), seed, 1.0, 0, 8, absval=True)
    Y = synth.gaussian_fixed((g.Cout, g.C, g.kh, g.kw), seed + 1, (2.0 / (g.C * g.kh * g.kw)) ** 0.5, -8, 8)
    return X, Y


@pytest.mark.parametrize("t", GEOMS)
@pytest.mark.parametrize("P", [1, 2, 3])
def test_ttp_conv_triples_parity(mpc, t, P):
    c = mpc.Context(P, mpc.ALL_PARTIES, device=0, master_seed=MASTER)
    g = c.conv_geom(*t)
    a, b, cc = c.ttp_conv_triples(4, g)
    ea, eb, ec = oracle.ttp_conv_triple(P, MASTER, 4, oracle.conv_geom(*t))
    assert np.array_equal(host(a), ea) and np.array_equal(host(b), eb) and np.array_equal(host(cc), ec)
    for r in range(P):      # one-party contexts: own slice; rank 0 also forms c_0
        cr = mpc.Context(P, r, device=0, master_seed=MASTER)
        ar, br, crr = cr.ttp_conv_triples(4, g)
        assert np.array_equal(host(ar), ea[r]) and np.array_equal(host(br), eb[r]) and np.array_equal(host(crr), ec[r])


@pytest.mark.parametrize("t", GEOMS)
@pytest.mark.parametrize("P", [1, 2, 3, 4])
@pytest.mark.parametrize("truncate", [False, True])
def test_beaver_conv2d_parity(mpc, t, P, truncate):
    c = mpc.Context(P, mpc.ALL_PARTIES, device=0, master_seed=MASTER)
    g, og = c.conv_geom(*t), oracle.conv_geom(*t)
    X, Y = _inputs(g, 7)
    gx, gy = c.share(dev(X), 0, 11), c.share(dev(Y), 1 % P, 12)
    ga, gb, gc = c.ttp_conv_triples(5, g)
    z = host(c.beaver_conv2d(g, gx, gy, ga, gb, gc, truncate=truncate, wrap_id=3))
    xs, ys = oracle.share(P, MASTER, X, 0, 11), oracle.share(P, MASTER, Y, 1 % P, 12)
    ez = oracle.beaver_conv2d(xs, ys, *oracle.ttp_conv_triple(P, MASTER, 5, og), og)
    if truncate:
        ez = oracle.truncate(ez, 16, MASTER, wrap_id=3)
    else:
        assert np.array_equal(oracle.reveal(z), oracle.conv2d(X, Y, og))     # Beaver identity
    assert np.array_equal(z, ez)


@pytest.mark.parametrize("P", [2, 3])
@pytest.mark.parametrize("t", [GEOMS[1], GEOMS[3]])
def test_one_party_contexts_conv(mpc, P, t):
    """One-party kernels: mask at the input / weight shapes, the reveal done here
    as a uint64 sum, then beaver_conv2d_finish on every party."""
    og = oracle.conv_geom(*t)
    X, Y = _inputs(og, 9)
    xs, ys = oracle.share(P, MASTER, X, 0, 1), oracle.share(P, MASTER, Y, 1, 2)
    a, b, cc = oracle.ttp_conv_triple(P, MASTER, 6, og)
    ctxs = [mpc.Context(P, r, device=0, master_seed=MASTER) for r in range(P)]
    g = ctxs[0].conv_geom(*t)
    eds = [ctxs[r].mask(dev(xs[r]), dev(a[r]), dev(ys[r]), dev(b[r])) for r in range(P)]
    ed = eds[0].clone()
    for e in eds[1:]:
        ed = (ed.view(torch.int64) + e.view(torch.int64)).view(torch.uint64)
    trunc = P <= 2
    zs = np.stack([host(ctxs[r].beaver_conv2d_finish(g, ed, dev(a[r]), dev(b[r]), dev(cc[r]), truncate=trunc))
                   for r in range(P)])
    ez = oracle.beaver_conv2d(xs, ys, a, b, cc, og)
    assert np.array_equal(zs, oracle.truncate(ez, 16) if trunc else ez)


def test_one_party_nccl_conv(mpc):
    t = GEOMS[0]
    og = oracle.conv_geom(*t)
    c = mpc.Context(1, 0, device=0, master_seed=MASTER, nccl_id=mpc.nccl_unique_id())
    g = c.conv_geom(*t)
    X, Y = _inputs(og, 13)
    a, b, cc = oracle.ttp_conv_triple(1, MASTER, 7, og)
    z = host(c.beaver_conv2d(g, dev(X), dev(Y), dev(a[0]), dev(b[0]), dev(cc[0]), truncate=True))
    assert np.array_equal(z, oracle.truncate(oracle.beaver_conv2d(X[None], Y[None], a, b, cc, og), 16)[0])


@pytest.mark.parametrize("name,t", [
    ("resnet50.conv1", (1, 3, 224, 224, 64, 7, 7, 2, 3)),
    ("resnet50.l4.c2", (1, 512, 7, 7, 512, 3, 3, 1, 1)),
    ("resnet50.l2.ds", (1, 256, 56, 56, 512, 1, 1, 2, 0)),
])
def test_resnet_layers_full_parity(mpc, name, t):
    """Full-size ResNet-50 convolutions, 2 parties, truncated: every share equals
    the oracle's; decoded within 2^-14 of torch's float64 conv2d (except flagged
    wraps)."""
    P = 2
    c = mpc.Context(P, mpc.ALL_PARTIES, device=0, master_seed=MASTER)
    g, og = c.conv_geom(*t), oracle.conv_geom(*t)
    X, Y = _inputs(og, 21)
    gx, gy = c.share(dev(X), 0, 1), c.share(dev(Y), 1, 2)
    ga, gb, gc = c.ttp_conv_triples(8, g)
    z = host(c.beaver_conv2d(g, gx, gy, ga, gb, gc, truncate=True))
    xs, ys = oracle.share(P, MASTER, X, 0, 1), oracle.share(P, MASTER, Y, 1, 2)
    ez, dg = oracle.truncate(oracle.beaver_conv2d(xs, ys, *oracle.ttp_conv_triple(P, MASTER, 8, og), og), 16,
                             diagnostics=True)
    assert np.array_equal(z, ez), name
    got = oracle.decode(oracle.reveal(z))
    ref = torch.nn.functional.conv2d(torch.tensor(X.view(np.int64) / 65536.0), torch.tensor(Y.view(np.int64) / 65536.0),
                                     stride=(og.sh, og.sw), padding=(og.ph, og.pw)).numpy()
    ok = dg["theta"] == 0
    assert np.all(np.abs(got - ref)[ok] <= 2.0 ** -14)


# ---------------------------------------------------------------- 1-D convolutions (Wav2Letter)
def _inputs1d(g, seed):
    X = synth.gaussian_fixed((g.B, g.C, g.W), seed, 1.0, -8, 8)
    Y = synth.gaussian_fixed((g.Cout, g.C, g.kw), seed + 1, (2.0 / (g.C * g.kw)) ** 0.5, -8, 8)
    return X, Y


@pytest.mark.parametrize("B", [1, 4])
@pytest.mark.parametrize("layer", synth.WAV2LETTER_CONV1D, ids=[l[0] for l in synth.WAV2LETTER_CONV1D])
def test_wav2letter_conv1d_full_parity(mpc, layer, B):
    """Every Wav2Letter layer as a true private 1-D convolution at full
    size (batch 1 and 4), 2 parties, truncated: every share equals the oracle's
    (eps, delta revealed at the activation / weight shapes), and the decoded output
    is within 2^-14 of torch's float64 conv1d except the flagged wraps."""
    name, C, L, Co, k, st, pd, _ = layer
    if B > 1 and C * k > 2000:
        pytest.skip("oracle time: batch 4 only for K <= 2000")
    P = 2
    c = mpc.Context(P, mpc.ALL_PARTIES, device=0, master_seed=MASTER)
    g, og = c.conv1d_geom(B, C, L, Co, k, st, pd), oracle.conv1d_geom(B, C, L, Co, k, st, pd)
    X, Y = _inputs1d(g, 31 + k)
    gx, gy = c.share(dev(X), 0, 1), c.share(dev(Y), 1, 2)
    ga, gb, gc = c.ttp_conv1d_triples(9, g)
    assert tuple(ga.shape) == (P, B, C, L) and tuple(gb.shape) == (P, Co, C, k)
    z = host(c.beaver_conv1d(g, gx, gy, ga, gb, gc, truncate=True))
    Lo = (L + 2 * pd - k) // st + 1
    assert z.shape == (P, B, Co, Lo)
    X4, Y4 = X.reshape(B, C, 1, L), Y.reshape(Co, C, 1, k)
    xs, ys = oracle.share(P, MASTER, X4, 0, 1), oracle.share(P, MASTER, Y4, 1, 2)
    ez, dg = oracle.truncate(oracle.beaver_conv2d(xs, ys, *oracle.ttp_conv_triple(P, MASTER, 9, og), og), 16,
                             diagnostics=True)
    assert np.array_equal(z, ez.reshape(z.shape)), name
    got = oracle.decode(oracle.reveal(z))
    ref = torch.nn.functional.conv1d(torch.tensor(X.view(np.int64) / 65536.0), torch.tensor(Y.view(np.int64) / 65536.0),
                                     stride=st, padding=pd).numpy()
    ok = (dg["theta"] == 0).reshape(got.shape)
    assert np.all(np.abs(got - ref)[ok] <= 2.0 ** -14)


def test_conv1d_one_party_group_alg1(mpc):
    """A 1-D convolution through the one-party schedule (3 parties as threads,
    reveals through the in-process group) with Alg. 1 truncation."""
    from test_gpu_local_group import run_parties
    P, t = 3, (2, 250, 50, 250, 7, 1, 3)
    og = oracle.conv1d_geom(*t)
    X, Y = _inputs1d(og, 41)
    X4, Y4 = X.reshape(t[0], t[1], 1, t[2]), Y.reshape(t[3], t[1], 1, t[4])
    xs, ys = oracle.share(P, MASTER, X4, 0, 1), oracle.share(P, MASTER, Y4, 1, 2)
    a, b, cc = oracle.ttp_conv_triple(P, MASTER, 10, og)

    def body(ctx, r):
        g = ctx.conv1d_geom(*t)
        lead = (t[0], t[1], t[2])
        z = ctx.beaver_conv1d(g, dev(xs[r]).view(lead), dev(ys[r]).view(t[3], t[1], t[4]), dev(a[r]).view(lead),
                              dev(b[r]).view(t[3], t[1], t[4]), dev(cc[r]).view(t[0], t[3], -1), truncate=True,
                              wrap_id=12)
        return host(z)

    got = np.stack([z.reshape(cc.shape[1:]) for z in run_parties(mpc, P, body)])
    ez = oracle.truncate(oracle.beaver_conv2d(xs, ys, a, b, cc, og), 16, MASTER, wrap_id=12)
    assert np.array_equal(got, ez)


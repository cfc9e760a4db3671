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

"""GPU parity of the elementwise private multiplication and square (SURVEY
§8(f) NEXT-1; App. A.1.1) against the oracle, bit for bit: TTP
triples / Beaver pairs, the fused all-parties kernels, the one-party kernels
(mask -> caller's reveal -> finish), the 1-rank NCCL path, truncation (local
and Alg. 1) and the batched reveal.  Sizes span odd/even lengths (vector and
scalar paths), empty inputs and a multi-million element case."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu
MASTER = synth.MASTER_SEED


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


def ctx(mpc, P, rank=None):
    return mpc.Context(P, mpc.ALL_PARTIES if rank is None else rank, device=0, master_seed=MASTER)


@pytest.mark.parametrize("P", [1, 2, 3, 8])
@pytest.mark.parametrize("n", [1, 2, 7, 4096, 100001])
def test_ttp_elementwise_parity(mpc, P, n):
    c = ctx(mpc, P)
    a, b, cc = c.ttp_mul_triples(3, (n,))
    ea, eb, ec = oracle.ttp_mul_triple(P, MASTER, 3, (n,))
    assert np.array_equal(host(a), ea) and np.array_equal(host(b), eb) and np.array_equal(host(cc), ec)
    a2, b2 = c.ttp_square_pairs(4, (n,))
    fa, fb = oracle.ttp_square_pair(P, MASTER, 4, (n,))
    assert np.array_equal(host(a2), fa) and np.array_equal(host(b2), fb)
    # one-party contexts produce their own party's slice (rank 0 also forms c_0)
    for r in range(P):
        cr = ctx(mpc, P, rank=r)
        ar, br, cr_ = cr.ttp_mul_triples(3, (n,))
        assert np.array_equal(host(ar), ea[r]) and np.array_equal(host(br), eb[r]) and np.array_equal(host(cr_), ec[r])
        ar2, br2 = cr.ttp_square_pairs(4, (n,))
        assert np.array_equal(host(ar2), fa[r]) and np.array_equal(host(br2), fb[r])


@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("shape", [(1,), (7,), (64, 33), (1000, 1001)])
@pytest.mark.parametrize("truncate", [False, True])
def test_beaver_mul_and_square_parity(mpc, P, shape, truncate):
    c = ctx(mpc, P)
    X = synth.uniform_fixed(shape, 11)
    Y = synth.uniform_fixed(shape, 12)
    gx, gy = c.share(dev(X), 0, 21), c.share(dev(Y), 1 % P, 22)
    ga, gb, gc = c.ttp_mul_triples(5, shape)
    z = host(c.beaver_mul(gx, gy, ga, gb, gc, truncate=truncate, wrap_id=9))
    xs, ys = oracle.share(P, MASTER, X, 0, 21), oracle.share(P, MASTER, Y, 1 % P, 22)
    a, b, cc = oracle.ttp_mul_triple(P, MASTER, 5, shape)
    ez = oracle.beaver_mul(xs, ys, a, b, cc)
    if truncate:
        ez = oracle.truncate(ez, 16, MASTER, wrap_id=9)
    assert np.array_equal(z, ez)
    ga2, gb2 = c.ttp_square_pairs(6, shape)
    z2 = host(c.beaver_square(gx, ga2, gb2, truncate=truncate, wrap_id=10))
    a2, b2 = oracle.ttp_square_pair(P, MASTER, 6, shape)
    ez2 = oracle.beaver_square(xs, a2, b2)
    if truncate:
        ez2 = oracle.truncate(ez2, 16, MASTER, wrap_id=10)
    assert np.array_equal(z2, ez2)
    if not truncate:    # identities, numpy wrapping uint64 products
        assert np.array_equal(oracle.reveal(z), X * Y) and np.array_equal(oracle.reveal(z2), X * X)


def test_empty_and_rounds(mpc):
    c = ctx(mpc, 2)
    e = torch.empty((2, 0), dtype=torch.uint64, device="cuda")
    assert c.beaver_mul(e, e, e, e, e).numel() == 0
    r0, _ = c.stats()
    x = c.share(dev(synth.uniform_fixed((10,), 1)), 0, 1)
    a, b, cc = c.ttp_mul_triples(1, (10,))
    c.beaver_mul(x, x, a, b, cc)
    a2, b2 = c.ttp_square_pairs(2, (10,))
    c.beaver_square(x, a2, b2)
    r1, _ = c.stats()
    assert r1 - r0 == 2                     # one round each (P = 2: truncation is local)
    c.reveal_batch([x, x, x])
    assert c.stats()[0] - r1 == 1          # three tensors, one round


@pytest.mark.parametrize("P", [2, 3])
@pytest.mark.parametrize("n", [5, 4098])
def test_one_party_contexts_mul_and_square(mpc, P, n):
    """The one-party kernels: mask (mpc_beaver_mask with M=1, K=n, N=1 / N=0),
    the reveal done here as a uint64 sum, then *_finish on every party."""
    X = synth.uniform_fixed((n,), 31)
    Y = synth.uniform_fixed((n,), 32)
    xs, ys = oracle.share(P, MASTER, X, 0, 1), oracle.share(P, MASTER, Y, 1, 2)
    a, b, cc = oracle.ttp_mul_triple(P, MASTER, 7, (n,))
    a2, b2 = oracle.ttp_square_pair(P, MASTER, 8, (n,))
    ctxs = [ctx(mpc, P, rank=r) for r in range(P)]
    trunc = P <= 2
    eds = [ctxs[r].beaver_mask(dev(xs[r]).view(1, n), dev(ys[r]).view(n, 1), dev(a[r]).view(1, n),
                               dev(b[r]).view(n, 1)) for r in range(P)]
    ed = eds[0].clone()
    for e in eds[1:]:
        ed = (ed.view(torch.int64) + e.view(torch.int64)).view(torch.uint64)
    zs = np.stack([host(ctxs[r].beaver_mul_finish(ed, dev(a[r]), dev(b[r]), dev(cc[r]), truncate=trunc))
                   for r in range(P)])
    ez = oracle.beaver_mul(xs, ys, a, b, cc)
    assert np.array_equal(zs, oracle.truncate(ez, 16) if trunc else ez)
    es = [ctxs[r].beaver_mask(dev(xs[r]).view(1, n), torch.empty((n, 0), dtype=torch.uint64, device="cuda"),
                              dev(a2[r]).view(1, n), torch.empty((n, 0), dtype=torch.uint64, device="cuda"))
          for r in range(P)]
    e = es[0].clone()
    for t in es[1:]:
        e = (e.view(torch.int64) + t.view(torch.int64)).view(torch.uint64)
    zs2 = np.stack([host(ctxs[r].beaver_square_finish(e, dev(a2[r]), dev(b2[r]), truncate=trunc)) for r in range(P)])
    ez2 = oracle.beaver_square(xs, a2, b2)
    assert np.array_equal(zs2, oracle.truncate(ez2, 16) if trunc else ez2)


def test_one_party_nccl_mul_square_and_batch_reveal(mpc):
    """A 1-rank NCCL context runs the production one-party path (mask, NCCL
    reveal of [eps | delta], finish with the fused truncation) and the grouped
    batched reveal."""
    P, n = 1, 10001
    c = mpc.Context(P, 0, device=0, master_seed=MASTER, nccl_id=mpc.nccl_unique_id())
    X = synth.uniform_fixed((n,), 41)
    Y = synth.uniform_fixed((n,), 42)
    a, b, cc = oracle.ttp_mul_triple(P, MASTER, 9, (n,))
    z = host(c.beaver_mul(dev(X), dev(Y), dev(a[0]), dev(b[0]), dev(cc[0]), truncate=True))
    assert np.array_equal(z, oracle.truncate(oracle.beaver_mul(X[None], Y[None], a, b, cc), 16)[0])
    a2, b2 = oracle.ttp_square_pair(P, MASTER, 10, (n,))
    z2 = host(c.beaver_square(dev(X), dev(a2[0]), dev(b2[0]), truncate=True))
    assert np.array_equal(z2, oracle.truncate(oracle.beaver_square(X[None], a2, b2), 16)[0])
    outs = c.reveal_batch([dev(X), dev(Y), dev(X[:7])])
    assert np.array_equal(host(outs[0]), X) and np.array_equal(host(outs[1]), Y) and np.array_equal(host(outs[2]), X[:7])


def test_large_sampled_accuracy(mpc):
    """16.8 M elements (4096^2), 2 parties, truncated: bit-exact with the oracle
    on the full tensor, and decoded within 2^-14 of float64 except flagged wraps."""
    P, shape = 2, (4096, 4096)
    c = ctx(mpc, P)
    X = synth.uniform_fixed(shape, 51)
    Y = synth.uniform_fixed(shape, 52)
    gx, gy = c.share(dev(X), 0, 1), c.share(dev(Y), 1, 2)
    ga, gb, gc = c.ttp_mul_triples(11, shape)
    z = host(c.beaver_mul(gx, gy, ga, gb, gc, truncate=True))
    xs, ys = oracle.share(P, MASTER, X, 0, 1), oracle.share(P, MASTER, Y, 1, 2)
    a, b, cc = oracle.ttp_mul_triple(P, MASTER, 11, shape)
    ez, dg = oracle.truncate(oracle.beaver_mul(xs, ys, a, b, cc), 16, diagnostics=True)
    assert np.array_equal(z, ez)
    got = oracle.decode(oracle.reveal(z))
    exact = (X.view(np.int64).astype(np.float64) / 65536) * (Y.view(np.int64).astype(np.float64) / 65536)
    ok = dg["theta"] == 0
    assert np.all(np.abs(got - exact)[ok] <= 2.0 ** -14)

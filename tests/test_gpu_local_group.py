"""The one-party-per-GPU schedule with P > 1 parties on ONE GPU.

P one-party contexts joined by an in-process group (mpc_create_local; reveals
are host rendezvous + one reduction kernel, stream-ordered with events) are
driven by P host threads, each on its own CUDA stream — the same entry points,
kernels, comm stream and overlap as the NCCL deployment (one process per party,
P:377-378), which needs P GPUs.  Every party's shares are compared bit for bit
with the oracle (all parties simulated in one process):
  * Beaver matmul through the overlapped schedule (delta, then eps reveal on the
    comm stream; phase-1 / phase-2 GEMMs), P = 2, 3, 4, with the P <= 2 local
    truncation and Alg. 1 (u64 + int8 reveals) for P > 2;
  * ReLU round by round: 7 XOR reveals per adder-tree
    height, the packed B2A bit reveal and the multiplication's sum reveal;
  * elementwise product / square, convolution, reveal and reveal_batch;
  * the collective contract: mismatched sizes fail on every party.
"""
import os
import threading

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu
MASTER = synth.MASTER_SEED
os.environ.setdefault("MPC_GROUP_TIMEOUT_S", "60")


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


def run_parties(mpc, P, body, master=MASTER):
    """body(ctx, rank) on P threads, one one-party context and one stream each;
    returns the per-rank results (exceptions re-raised)."""
    g = mpc.Group(P)
    ctxs = [mpc.Context(P, r, device=0, master_seed=master, group=g) for r in range(P)]
    results, errors = [None] * P, []

    def worker(r):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                results[r] = body(ctxs[r], r)
                s.synchronize()
        except BaseException as e:  # noqa: BLE001
            errors.append((r, e))

    th = [threading.Thread(target=worker, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    torch.cuda.synchronize()
    for c in ctxs:
        c.close()
    g.close()
    if errors:
        raise errors[0][1]
    return results


# ------------------------------------------------------------------ Beaver matmul
@pytest.mark.parametrize("P", [2, 3, 4])
@pytest.mark.parametrize("M,K,N", [(64, 64, 64), (300, 100, 260), (49, 700, 300), (1, 45, 3)])
def test_beaver_overlapped_schedule_parity(mpc, P, M, K, N):
    X = synth.uniform_fixed((M, K), M + K)
    Y = synth.uniform_fixed((K, N), N + 1)
    xs = oracle.share(P, MASTER, X, 0, 101)
    ys = oracle.share(P, MASTER, Y, 1, 102)
    a, b, cc = oracle.ttp_triple(P, MASTER, 7, M, K, N)

    def body(c, r):
        ga, gb, gc = c.ttp_triples(7, M, K, N)              # rank 0 also forms c_0 (the TTP)
        gx = c.share(dev(X) if r == 0 else None, 0, 101, shape=(M, K))
        gy = c.share(dev(Y) if r == 1 else None, 1, 102, shape=(K, N))
        z = c.beaver_matmul(gx, gy, ga, gb, gc, truncate=True, wrap_id=5)
        out = c.reveal(z)
        return host(ga), host(gc), host(gx), host(z), host(out), c.stats()

    res = run_parties(mpc, P, body)
    assert np.array_equal(np.stack([r[0] for r in res]), a)
    assert np.array_equal(np.stack([r[1] for r in res]), cc)
    assert np.array_equal(np.stack([r[2] for r in res]), xs)
    ez = oracle.truncate(oracle.beaver_matmul(xs, ys, a, b, cc), 16, MASTER, wrap_id=5)
    assert np.array_equal(np.stack([r[3] for r in res]), ez)
    for r in res:
        assert np.array_equal(r[4], oracle.reveal(ez))
        assert r[5][0] == (3 if P > 2 else 2)             # matmul (+ Alg. 1) + output reveal


@pytest.mark.parametrize("P", [2, 3])
@pytest.mark.parametrize("chunks", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("M,K,N", [(1024, 300, 520), (2100, 64, 130), (4096, 96, 384)])
def test_beaver_chunked_eps_reveal(mpc, P, chunks, M, K, N):
    """The eps reveal in row chunks (each chunk's eps @ b_p GEMM starts as soon as
    that chunk is revealed): shares bit-identical to the oracle for
    every chunk count, ragged last chunk (2100 rows = 9 tiles), chunks > tiles."""
    X = synth.uniform_fixed((M, K), M + chunks)
    Y = synth.uniform_fixed((K, N), N + chunks)
    xs = oracle.share(P, MASTER, X, 0, 111)
    ys = oracle.share(P, MASTER, Y, 1, 112)
    a, b, cc = oracle.ttp_triple(P, MASTER, 8, M, K, N)

    def body(c, r):
        c.set_reveal_chunks(chunks)
        z = c.beaver_matmul(dev(xs[r]), dev(ys[r]), dev(a[r]), dev(b[r]), dev(cc[r]), truncate=True, wrap_id=9)
        return host(z), c.stats()[0]

    res = run_parties(mpc, P, body)
    ez = oracle.truncate(oracle.beaver_matmul(xs, ys, a, b, cc), 16, MASTER, wrap_id=9)
    assert np.array_equal(np.stack([r[0] for r in res]), ez)
    assert all(r[1] == (2 if P > 2 else 1) for r in res)  # the chunked eps || delta reveal is ONE round


def test_beaver_untruncated_identity(mpc):
    P, M, K, N = 3, 130, 90, 70
    X = synth.uniform_ring((M, K), 1)
    Y = synth.uniform_ring((K, N), 2)
    xs, ys = oracle.share(P, MASTER, X, 0, 1), oracle.share(P, MASTER, Y, 2, 2)
    a, b, cc = oracle.ttp_triple(P, MASTER, 3, M, K, N)
    res = run_parties(mpc, P, lambda c, r: host(c.beaver_matmul(dev(xs[r]), dev(ys[r]), dev(a[r]), dev(b[r]),
                                                                 dev(cc[r]), truncate=False)))
    z = np.stack(res)
    assert np.array_equal(z, oracle.beaver_matmul(xs, ys, a, b, cc))
    assert np.array_equal(oracle.reveal(z), X @ Y)          # Beaver identity (numpy wraps mod 2^64)


# ------------------------------------------------------------------ ReLU
@pytest.mark.parametrize("P", [1, 2, 3, 4, 5, 8])
@pytest.mark.parametrize("n", [1, 2, 7, 1000, 65537])
def test_relu_one_party_parity(mpc, P, n):
    X = synth.uniform_ring((n,), 300 + n)
    edge = np.array([0, 1, 2**64 - 1, 1 << 63, (1 << 63) - 1], dtype=np.uint64)
    X[:min(n, 5)] = edge[:min(n, 5)]
    xs = oracle.share(P, MASTER, X, 0, 1)

    def body(c, r):
        r0, b0 = c.stats()
        z, sign = c.relu(dev(xs[r]), relu_id=77, want_sign=True)
        r1, b1 = c.stats()
        return host(z), host(sign), r1 - r0, b1 - b0

    res = run_parties(mpc, P, body)
    ez, dg = oracle.relu(MASTER, 77, xs, diagnostics=True)
    assert np.array_equal(np.stack([r[0] for r in res]), ez)
    assert np.array_equal(np.stack([r[1] for r in res]), dg["sign"])
    assert np.array_equal(oracle.reveal(ez).view(np.int64), np.maximum(X.view(np.int64), 0))
    levels = int(np.ceil(np.log2(P))) if P > 1 else 0
    for r in res:
        assert r[2] == dg["rounds"] == 7 * levels + 2
        assert r[3] > 0


def test_relu_one_party_matches_all_parties_kernel(mpc):
    P, n = 4, 100003
    X = synth.gaussian_fixed((n,), 8, 1.0, -8, 8)
    xs = oracle.share(P, MASTER, X, 0, 9)
    ca = mpc.Context(P, mpc.ALL_PARTIES, device=0, master_seed=MASTER)
    za = host(ca.relu(dev(xs), relu_id=12))
    res = run_parties(mpc, P, lambda c, r: host(c.relu(dev(xs[r]), relu_id=12)))
    assert np.array_equal(np.stack(res), za)
    got = oracle.decode(oracle.reveal(za))
    assert np.array_equal(got, np.maximum(X.view(np.int64), 0) / 65536.0)


# ------------------------------------------------------------------ elementwise, conv, reveals
@pytest.mark.parametrize("P", [2, 3])
def test_elementwise_mul_square(mpc, P):
    n = 30001
    X = synth.uniform_fixed((n,), 41)
    Y = synth.uniform_fixed((n,), 42)
    xs, ys = oracle.share(P, MASTER, X, 0, 3), oracle.share(P, MASTER, Y, 1, 4)
    a, b, cc = oracle.ttp_mul_triple(P, MASTER, 9, (n,))
    sa, sb = oracle.ttp_square_pair(P, MASTER, 10, (n,))

    def body(c, r):
        z = c.beaver_mul(dev(xs[r]), dev(ys[r]), dev(a[r]), dev(b[r]), dev(cc[r]), truncate=True, wrap_id=1)
        s = c.beaver_square(dev(xs[r]), dev(sa[r]), dev(sb[r]), truncate=True, wrap_id=2)
        return host(z), host(s)

    res = run_parties(mpc, P, body)
    ez = oracle.truncate(oracle.beaver_mul(xs, ys, a, b, cc), 16, MASTER, wrap_id=1)
    es = oracle.truncate(oracle.beaver_square(xs, sa, sb), 16, MASTER, wrap_id=2)
    assert np.array_equal(np.stack([r[0] for r in res]), ez)
    assert np.array_equal(np.stack([r[1] for r in res]), es)


def test_conv2d(mpc):
    P, t = 2, (2, 3, 17, 13, 8, 3, 3, 2, 1)
    og = oracle.conv_geom(*t)
    X = synth.gaussian_fixed((og.B, og.C, og.H, og.W), 3, 1.0, 0, 8, absval=True)
    Y = synth.gaussian_fixed((og.Cout, og.C, og.kh, og.kw), 4, 0.2, -8, 8)
    xs, ys = oracle.share(P, MASTER, X, 0, 1), oracle.share(P, MASTER, Y, 1, 2)
    a, b, cc = oracle.ttp_conv_triple(P, MASTER, 6, og)

    def body(c, r):
        g = c.conv_geom(*t)
        return host(c.beaver_conv2d(g, dev(xs[r]), dev(ys[r]), dev(a[r]), dev(b[r]), dev(cc[r]), truncate=True))

    z = np.stack(run_parties(mpc, P, body))
    assert np.array_equal(z, oracle.truncate(oracle.beaver_conv2d(xs, ys, a, b, cc, og), 16))


def test_reveal_and_batch(mpc):
    P = 4
    A = synth.uniform_ring((5000,), 1)
    B = synth.uniform_ring((3, 7), 2)
    sa, sb = oracle.share(P, MASTER, A, 2, 1), oracle.share(P, MASTER, B, 3, 2)

    def body(c, r):
        r0, _ = c.stats()
        one = c.reveal(dev(sa[r]))
        two = c.reveal_batch([dev(sa[r]), dev(sb[r])])
        return host(one), [host(t) for t in two], c.stats()[0] - r0

    for one, two, rounds in run_parties(mpc, P, body):
        assert np.array_equal(one, A) and np.array_equal(two[0], A) and np.array_equal(two[1], B)
        assert rounds == 2


def test_collective_contract_mismatch_fails_everywhere(mpc):
    P = 2

    def body(c, r):
        try:
            c.reveal(torch.zeros(4 + r, dtype=torch.uint64, device="cuda"))
        except mpc.MpcError as e:
            return e.status
        return 0

    assert run_parties(mpc, P, body) == [2, 2]                 # MPC_ERR_SHAPE on both parties


@pytest.mark.parametrize("P", [2, 3])
@pytest.mark.parametrize("M,K,N", [(64, 64, 64), (300, 100, 260), (49, 700, 300)])
def test_beaver_prepared_one_party(mpc, P, M, K, N):
    """Weight side prepared (delta reveal) ahead, then eps revealed on the comm
    stream overlapping a_p @ delta: the one-call shares bit for bit."""
    X = synth.uniform_fixed((M, K), M + 5)
    Y = synth.uniform_fixed((K, N), N + 6)
    xs, ys = oracle.share(P, MASTER, X, 0, 11), oracle.share(P, MASTER, Y, 1, 12)
    a, b, cc = oracle.ttp_triple(P, MASTER, 13, M, K, N)

    def body(c, r):
        prep = c.beaver_prepare(dev(ys[r]), dev(b[r]), M)
        z = c.beaver_matmul_prepared(dev(xs[r]), dev(a[r]), dev(cc[r]), prep, truncate=True, wrap_id=4)
        return host(z)

    z = np.stack(run_parties(mpc, P, body))
    assert np.array_equal(z, oracle.truncate(oracle.beaver_matmul(xs, ys, a, b, cc), 16, MASTER, wrap_id=4))


def test_relu_one_party_sixteen_parties(mpc):
    """P = 16 (the context maximum): four adder-tree heights, 8 adders at the first."""
    P, n = 16, 4099
    X = synth.uniform_ring((n,), 16)
    xs = oracle.share(P, MASTER, X, 3, 5)
    res = run_parties(mpc, P, lambda c, r: (host(c.relu(dev(xs[r]), relu_id=21)), c.stats()[0]))
    ez, dg = oracle.relu(MASTER, 21, xs, diagnostics=True)
    assert np.array_equal(np.stack([r[0] for r in res]), ez)
    assert all(r[1] == dg["rounds"] == 7 * 4 + 2 for r in res)


def test_beaver_eight_parties_alg1(mpc):
    """Eight one-party contexts: overlapped schedule + Alg. 1 (u64 and int8 reveals)."""
    P, M, K, N = 8, 70, 90, 50
    X = synth.uniform_fixed((M, K), 81)
    Y = synth.uniform_fixed((K, N), 82)
    xs, ys = oracle.share(P, MASTER, X, 0, 1), oracle.share(P, MASTER, Y, 7, 2)
    a, b, cc = oracle.ttp_triple(P, MASTER, 8, M, K, N)
    res = run_parties(mpc, P, lambda c, r: host(c.beaver_matmul(dev(xs[r]), dev(ys[r]), dev(a[r]), dev(b[r]),
                                                                 dev(cc[r]), truncate=True, wrap_id=9)))
    assert np.array_equal(np.stack(res), oracle.truncate(oracle.beaver_matmul(xs, ys, a, b, cc), 16, MASTER,
                                                         wrap_id=9))


@pytest.mark.parametrize("P", [2, 3])
def test_beaver_matmul_batched_one_party(mpc, P):
    B, M, K, N = 6, 70, 64, 90
    X = np.stack([synth.uniform_fixed((M, K), 10 + i) for i in range(B)])
    Y = np.stack([synth.uniform_fixed((K, N), 20 + i) for i in range(B)])
    xs, ys = oracle.share(P, MASTER, X, 0, 31), oracle.share(P, MASTER, Y, 1, 32)
    tr = [oracle.ttp_triple(P, MASTER, 40 + i, M, K, N) for i in range(B)]
    a, b, cc = (np.ascontiguousarray(np.stack([t[j] for t in tr], axis=1)) for j in range(3))

    def body(c, r):
        return host(c.beaver_matmul_batched(dev(xs[r]), dev(ys[r]), dev(a[r]), dev(b[r]), dev(cc[r]),
                                            truncate=True, wrap_id=3)), c.stats()[0]

    res = run_parties(mpc, P, body)
    ez = np.stack([oracle.beaver_matmul(xs[:, i], ys[:, i], a[:, i], b[:, i], cc[:, i]) for i in range(B)], axis=1)
    assert np.array_equal(np.stack([r[0] for r in res]), oracle.truncate(ez, 16, MASTER, wrap_id=3))
    assert all(r[1] == 1 + (P > 2) for r in res)

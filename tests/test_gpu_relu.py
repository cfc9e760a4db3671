"""GPU parity of the fused ReLU path (A2B by a Kogge-Stone
adder tree with binary Beaver ANDs, sign bit, Alg. 2 B2A, Beaver multiplication)
against the oracle, bit for bit, for P = 1..8, odd / even lengths, edge values
(0, ±1, INT64_MIN/MAX), plus the exact plaintext relu and round accounting."""
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


@pytest.mark.parametrize("P", [1, 2, 3, 4, 5, 8])
@pytest.mark.parametrize("n", [1, 2, 7, 1000, 65537])
def test_relu_parity(mpc, P, n):
    X = synth.uniform_ring((n,), 100 + n)
    edge = np.array([0, 1, 2**64 - 1, 1 << 63, (1 << 63) - 1], dtype=np.uint64)
    X[:min(n, 5)] = edge[:min(n, 5)]
    c = mpc.Context(P, mpc.ALL_PARTIES, device=0, master_seed=MASTER)
    xs = c.share(dev(X), 0, 1)
    r0, _ = c.stats()
    z, sign = c.relu(xs, relu_id=77, want_sign=True)
    rounds = c.stats()[0] - r0
    ez, dg = oracle.relu(MASTER, 77, oracle.share(P, MASTER, X, 0, 1), diagnostics=True)
    assert np.array_equal(host(z), ez)
    assert np.array_equal(host(sign), dg["sign"])
    assert np.array_equal(oracle.reveal(host(z)).view(np.int64), np.maximum(X.view(np.int64), 0))
    assert rounds == dg["rounds"]


def test_relu_fixed_point_activations(mpc):
    """Decoded: relu of fixed-point activations N(0, 1) at 2^16 (exact, R25)."""
    P, n = 2, 1 << 20
    X = synth.gaussian_fixed((n,), 5, 1.0, -8, 8)
    c = mpc.Context(P, mpc.ALL_PARTIES, device=0, master_seed=MASTER)
    z = c.relu(c.share(dev(X), 0, 3), relu_id=5)
    got = oracle.decode(oracle.reveal(host(z)))
    assert np.array_equal(got, np.maximum(X.view(np.int64), 0) / 65536.0)

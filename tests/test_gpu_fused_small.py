"""The fused 2-party small-output Beaver matmul (csrc/ring_gemm_fused.cu: mask,
local reveal, limb split and limb GEMM in one kernel; SURVEY §8(f) NEXT-4's
wide-K text matmul runs on it) against the oracle, bit for bit.

In-process cases use the default launch (split-K over the SMs + finalize);
subprocess cases force the knobs read once per process: one CTA (no split-K,
z written by the kernel), one 32-K block per CTA, short drained TMEM units
(the multi-unit path the full-size text matmul needs only past 4.9 M K), two
converter groups instead of one, contiguous K ranges, bulk prefetches and
MPC_FUSED_SMALL=0 (the planes-based path) — every variant must give the
oracle's shares.  Shapes with even K and N run the TMA-staged kernel, the others
the register path.
"""
import hashlib
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MASTER = synth.MASTER_SEED
P = 2


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


def _oracle_z(M, K, N, gen, tid, truncate=True):
    X, Y = gen((M, K), 41), gen((K, N), 42)
    a, b, c = oracle.ttp_triple(P, MASTER, tid, M, K, N)
    z = oracle.beaver_matmul(oracle.share(P, MASTER, X, 0, 1), oracle.share(P, MASTER, Y, 1, 2), a, b, c)
    return X, Y, (oracle.truncate(z, 16) if truncate else z)


@pytest.mark.parametrize("M,K,N", [(32, 2048, 32),      # exactly 64 32-K blocks, full tile (TMA-staged)
                                   (32, 70001, 32),     # ragged K tail, 148 CTAs (odd K: register path)
                                   (32, 70002, 32),     # the same on the TMA-staged kernel
                                   (20, 9000, 30),      # ragged rows / columns / K tail, TMA-staged
                                   (7, 4096, 2),        # TMA boxes mostly out of bounds (zero-filled)
                                   (17, 4099, 5),       # ragged rows / columns
                                   (1, 6000, 32),       # a single row
                                   (32, 5000, 1)])      # a single column
@pytest.mark.parametrize("gen", ["uniform_fixed", "uniform_ring"])
def test_fused_small_parity(mpc, M, K, N, gen):
    g = getattr(synth, gen)
    truncate = gen == "uniform_fixed"
    X, Y, ez = _oracle_z(M, K, N, g, 5, truncate)
    c = mpc.Context(P, mpc.ALL_PARTIES, device=0, master_seed=MASTER)
    x, y = c.share(dev(X), 0, 1), c.share(dev(Y), 1, 2)
    a, b, cc = c.ttp_triples(5, M, K, N)
    torch.cuda.synchronize()
    n0 = c.launch_count()
    z = c.beaver_matmul(x, y, a, b, cc, truncate=truncate)
    torch.cuda.synchronize()
    assert c.launch_count() - n0 == 1, "expected one fused launch (the planes path makes two: split, GEMM)"
    assert np.array_equal(host(z), ez)


def test_fused_small_all_ones_carries(mpc):
    """All-0xFF shares: every limb product is 255^2, the largest accumulator entry."""
    M, K, N = 32, 33 * 1024 + 7, 32
    c = mpc.Context(P, mpc.ALL_PARTIES, device=0, master_seed=MASTER)
    ones = np.full((P, M, K), np.uint64(2 ** 64 - 1), dtype=np.uint64)
    onesy = np.full((P, K, N), np.uint64(2 ** 64 - 1), dtype=np.uint64)
    zero_mk = np.zeros((P, M, K), dtype=np.uint64)
    zero_kn = np.zeros((P, K, N), dtype=np.uint64)
    cz = np.zeros((P, M, N), dtype=np.uint64)
    # x_p = y_p = all ones, a = b = c = 0: eps = delta = 2 * (2^64 - 1), b'_0 = delta
    z = c.beaver_matmul(dev(ones), dev(onesy), dev(zero_mk), dev(zero_kn), dev(cz), truncate=False)
    ez = oracle.beaver_matmul(ones, onesy, zero_mk, zero_kn, cz)
    assert np.array_equal(host(z), ez)


SCRIPT = r"""
import hashlib, sys
import numpy as np, torch
sys.path.insert(0, {root!r})
import synth
import paper_2109_00984_b200 as m
M, K, N = {M}, {K}, {N}
c = m.Context(2, m.ALL_PARTIES, device=0, master_seed=synth.MASTER_SEED)
dev = lambda a: torch.from_numpy(a.view(np.int64)).cuda().view(torch.uint64)
x = c.share(dev(synth.uniform_ring((M, K), 41)), 0, 1)
y = c.share(dev(synth.uniform_ring((K, N), 42)), 1, 2)
a, b, cc = c.ttp_triples(5, M, K, N)
z = c.beaver_matmul(x, y, a, b, cc, truncate=False)
print(hashlib.sha256(z.view(torch.int64).cpu().numpy().tobytes()).hexdigest())
"""


@pytest.mark.parametrize("env", [{"MPC_FUSED_CTAS": "1"}, {"MPC_FUSED_CTAS": "148"},
                                 {"MPC_FUSED_UNIT": "3"}, {"MPC_FUSED_UNIT": "7", "MPC_FUSED_CTAS": "5"},
                                 {"MPC_FUSED_GROUPS": "2"}, {"MPC_FUSED_GROUPS": "2", "MPC_FUSED_UNIT": "3"},
                                 {"MPC_FUSED_CYCLIC": "0", "MPC_FUSED_UNIT": "5"}, {"MPC_FUSED_PF": "2"},
                                 {"MPC_FUSED_TMA": "0"}, {"MPC_FUSED_SMALL": "0"}],
                         ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()))
@pytest.mark.parametrize("shape", [(29, 9000, 31), (30, 9002, 32)],
                         ids=["register-path", "tma-staged"])
def test_fused_small_launch_variants(mpc, env, shape):
    M, K, N = shape                         # 282 32-K blocks, ragged (odd N: register path; even: TMA)
    _, _, ez = _oracle_z(M, K, N, synth.uniform_ring, 5, truncate=False)
    want = hashlib.sha256(np.ascontiguousarray(ez).view(np.int64).tobytes()).hexdigest()
    out = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT, M=M, K=K, N=N)], capture_output=True,
                         text=True, env={**os.environ, **env}, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    assert out.stdout.strip().splitlines()[-1] == want

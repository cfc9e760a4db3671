"""Determinism across launch configurations (SURVEY.md §8(c) pin table,
"Determinism": same seeds => identical shares across chunk counts and tile
configs; ring addition is associative, so any order is exact).

Each configuration runs in its own process because the GEMM's tuning knobs
(K-chunk length MPC_GEMM_KC, split-K factor MPC_GEMM_SPLITS, programmatic
dependent launch MPC_NO_PDL, transposed GEMM for small M MPC_NO_SWAP / MPC_SWAP_GAIN, the
2-CTA GEMM's operand producer MPC_GEMM_TMA, its tile order MPC_GEMM_PARTY_MAJOR /
MPC_GEMM_GROUPM / MPC_GEMM_SERPENTINE) are
read once per process.  Every run must
produce the oracle's shares bit for bit.
"""
import hashlib
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = 2
SHAPES = [(300, 3000, 700),           # 94 K-blocks per segment, 2 x 6 output tiles, ragged tails
          (49, 2000, 700),            # small M: the ring GEMM runs transposed (unless MPC_NO_SWAP)
          (20, 3000, 300),            # M <= 32: the stacked-plane kernel (unless MPC_GEMM_SMALL=0)
          (300, 2000, 24)]            # N <= 32: transposed onto the stacked-plane kernel

SCRIPT = r"""
import hashlib, sys
import numpy as np, torch
sys.path.insert(0, {root!r})
import synth
import paper_2109_00984_b200 as m
M, K, N, P = {M}, {K}, {N}, {P}
c = m.Context(P, m.ALL_PARTIES, device=0, master_seed=synth.MASTER_SEED)
dev = lambda a: torch.from_numpy(a.view(np.int64)).cuda().view(torch.uint64)
x = c.share(dev(synth.uniform_fixed((M, K), 31)), 0, 1)
y = c.share(dev(synth.uniform_fixed((K, N), 32)), 1, 2)
a, b, cc = c.ttp_triples(4, M, K, N)
z = c.beaver_matmul(x, y, a, b, cc, truncate=True)
print(hashlib.sha256(z.view(torch.int64).cpu().numpy().tobytes()).hexdigest())
"""


@pytest.fixture(scope="module", params=SHAPES, ids=lambda s: "x".join(map(str, s)))
def case(request):
    from paper_2109_00984_b200 import build
    build.build()
    M, K, N = request.param
    X = synth.uniform_fixed((M, K), 31)
    Y = synth.uniform_fixed((K, N), 32)
    a, b, c = oracle.ttp_triple(P, synth.MASTER_SEED, 4, M, K, N)
    z = oracle.beaver_matmul(oracle.share(P, synth.MASTER_SEED, X, 0, 1), oracle.share(P, synth.MASTER_SEED, Y, 1, 2),
                             a, b, c)
    z = oracle.truncate(z, 16)
    return (M, K, N), hashlib.sha256(np.ascontiguousarray(z).view(np.int64).tobytes()).hexdigest()


@pytest.mark.parametrize("env", [
    {},
    {"MPC_GEMM_KC": "8"},
    {"MPC_GEMM_KC": "33"},
    {"MPC_GEMM_SPLITS": "3"},
    {"MPC_GEMM_SPLITS": "7", "MPC_GEMM_KC": "5"},
    {"MPC_NO_PDL": "1"},
    {"MPC_NO_SWAP": "1"},
    {"MPC_SWAP_GAIN": "1.0"},               # the plain model: small-M shapes run transposed
    {"MPC_SWAP_GAIN": "100"},               # transposed wherever allowed
    {"MPC_GEMM_SMALL": "0"},
    {"MPC_GEMM_SMALL": "1"},
    {"MPC_GEMM_TMA": "0"},                  # bulk-copy producer with the peer relay everywhere
    {"MPC_GEMM_TMA": "1"},                  # 2-CTA tensor-TMA producer everywhere
    {"MPC_GEMM_TMA": "1", "MPC_GEMM_TMA_L2": "1"},
    {"MPC_GEMM_PARTY_MAJOR": "1"},          # instance-major tile order (the > 2 GiB default)
    {"MPC_GEMM_PARTY_MAJOR": "1", "MPC_GEMM_GROUPM": "3"},
    # K-serpentine (the default): odd items of a cluster walk their units backwards
    {"MPC_GEMM_SERPENTINE": "0"},
    {"MPC_GEMM_SERPENTINE": "1", "MPC_GEMM_TMA": "0"},
    {"MPC_GEMM_SERPENTINE": "1", "MPC_GEMM_TMA": "0", "MPC_GEMM_SPLITS": "7", "MPC_GEMM_KC": "5"},
], ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()) or "default")
def test_same_shares_under_every_launch_config(case, env):
    (M, K, N), expected = case
    full = dict(os.environ)
    for k in ("MPC_GEMM_KC", "MPC_GEMM_SPLITS", "MPC_NO_PDL", "MPC_NO_SWAP", "MPC_GEMM_DEBUG", "MPC_GEMM_SMALL",
              "MPC_GEMM_TMA", "MPC_GEMM_TMA_L2", "MPC_GEMM_PARTY_MAJOR", "MPC_GEMM_GROUPM", "MPC_GEMM_SERPENTINE", "MPC_SWAP_GAIN"):
        full.pop(k, None)
    full.update(env)
    out = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT, M=M, K=K, N=N, P=P)], env=full,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    assert out.stdout.strip().splitlines()[-1] == expected, env


def test_mbarrier_watchdog_traps_instead_of_hanging():
    """A stage whose bulk copies are dropped (MPC_GEMM_FAULT_INJECT=1) never
    completes its mbarrier; the wait watchdog (2^34 cycles) traps, so the call
    fails with a CUDA error in seconds instead of hanging the GPU."""
    script = r"""
import sys; sys.path.insert(0, {root!r})
import torch, synth
import paper_2109_00984_b200 as m
c = m.Context(1, m.ALL_PARTIES, device=0)
A = torch.zeros((300, 300), dtype=torch.uint64, device="cuda")
try:
    C = c.ring_matmul(A, A)
    torch.cuda.synchronize()
except Exception as e:
    print("FAILED:", type(e).__name__)
    sys.exit(3)
print("NO-TRAP")
""".format(root=ROOT)
    env = dict(os.environ, MPC_GEMM_FAULT_INJECT="1")
    out = subprocess.run([sys.executable, "-c", script], env=env, capture_output=True, text=True, timeout=180)
    assert out.returncode != 0 and "NO-TRAP" not in out.stdout, (out.stdout, out.stderr[-2000:])

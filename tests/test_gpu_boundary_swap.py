"""The parity harness of SURVEY §8(b): ONE protocol script (encode, share, TTP
triples, Beaver matmul with truncation, Alg. 1 / local truncation with an offline
wrap pair, reveal, decode — tests/boundary_backends.py) run against both
libraries behind the same boundary — libmpc_ring.so's mpc_* on CUDA tensors and
the CPU oracle's oracle_mpc_* on host arrays — and every output compared bit for
bit, including the round / byte accounting of mpc_stats."""
import numpy as np
import pytest
import torch

import synth
from boundary_backends import GpuBackend, OracleBackend, run_protocol

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def built():
    from paper_2109_00984_b200 import build
    build.build()
    assert torch.cuda.is_available(), "GPU tests need a B200"


@pytest.mark.parametrize("P,M,K,N", [(1, 64, 64, 64), (2, 64, 64, 64), (2, 300, 100, 260), (3, 129, 257, 70),
                                     (4, 40, 1000, 33), (8, 260, 96, 130)])
def test_same_script_both_libraries(built, P, M, K, N):
    rng = np.random.default_rng(7 * P + M)
    Xf = rng.uniform(-8, 8, (M, K))
    Yf = rng.uniform(-8, 8, (K, N))
    got = run_protocol(GpuBackend(), P, M, K, N, Xf, Yf, synth.MASTER_SEED)
    ref = run_protocol(OracleBackend(), P, M, K, N, Xf, Yf, synth.MASTER_SEED)
    for k in ("x", "y", "a", "b", "c", "z", "z2", "r", "th", "zr"):
        assert np.array_equal(got[k], ref[k]), k
    assert np.array_equal(got["dec"], ref["dec"])
    assert got["stats"] == ref["stats"]

"""The oracle's boundary (oracle_mpc_*, host pointers) composes its pinned steps
exactly as include/mpc_ring.h specifies the calls of the same names: a protocol
script through oracle_mpc_* equals the same steps called one by one
(tests/test_oracle_pins.py pins those), with Table 3's round counts
and the ABI's status codes.  tests/test_gpu_boundary_swap.py runs the SAME
script against libmpc_ring.so on the GPU."""
import ctypes

import numpy as np
import pytest

import oracle
import synth
from boundary_backends import OracleBackend, run_protocol

MASTER = synth.MASTER_SEED


@pytest.mark.parametrize("P,M,K,N", [(1, 5, 7, 3), (2, 9, 17, 11), (3, 8, 5, 6), (4, 3, 33, 2)])
def test_oracle_boundary_script(P, M, K, N):
    rng = np.random.default_rng(P * 100 + M)
    Xf = rng.uniform(-8, 8, (M, K))
    Yf = rng.uniform(-8, 8, (K, N))
    out = run_protocol(OracleBackend(), P, M, K, N, Xf, Yf, MASTER)
    X, Y = oracle.encode(Xf), oracle.encode(Yf)
    xs, ys = oracle.share(P, MASTER, X, 0, 1), oracle.share(P, MASTER, Y, 1 % P, 2)
    a, b, c = oracle.ttp_triple(P, MASTER, 1, M, K, N)
    assert np.array_equal(out["x"], xs) and np.array_equal(out["y"], ys)
    assert np.array_equal(out["a"], a) and np.array_equal(out["b"], b) and np.array_equal(out["c"], c)
    z = oracle.truncate(oracle.beaver_matmul(xs, ys, a, b, c), 16, MASTER, wrap_id=3)
    assert np.array_equal(out["z"], z)
    r, th = oracle.wrap_pair(P, MASTER, 4, M * N)
    z2 = (oracle.truncate_alg1(z.reshape(P, -1), r, th, 8) if P > 2 else oracle.truncate_local(z, 8))
    assert np.array_equal(out["z2"].reshape(P, -1), np.asarray(z2).reshape(P, -1))
    assert np.array_equal(out["zr"], oracle.reveal(z))
    assert np.array_equal(out["dec"], oracle.decode(oracle.reveal(z)))
    # rounds: beaver 1 (+1 Alg. 1), truncate_pairs 0 / 1, reveal 1 (Table 3)
    assert out["stats"][0] == 2 + 2 * (P > 2)


def test_oracle_boundary_status_codes():
    be = OracleBackend()
    L = be.L
    h = ctypes.c_void_p()
    assert L.oracle_mpc_create(ctypes.byref(h), 2, 0, 0, None, 1, 16) == 7       # one party: unsupported
    assert L.oracle_mpc_create(ctypes.byref(h), 0, -1, 0, None, 1, 16) == 1      # P = 0
    be.create(2, MASTER)
    x = np.zeros(4, dtype=np.uint64)
    out = np.zeros((2, 4), dtype=np.uint64)
    assert be.call("share", x.ctypes.data, 2, 1, out.ctypes.data, 4) == 1         # src out of range
    big = np.array([2.0 ** 47], dtype=np.float64)
    enc = np.zeros(1, dtype=np.uint64)
    assert be.call("encode", big.ctypes.data, enc.ctypes.data, 1) == 3            # MPC_ERR_OVERFLOW
    be.close()

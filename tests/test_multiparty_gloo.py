"""World-size-2 (and 4) multi-process tests on CPU with the gloo backend.

They cover the host logic of the one-party-per-GPU path (rank -> session /
party layout, NCCL unique-id exchange, max-over-ranks timing) and the
distributed decomposition of the protocol that the NCCL path implements: each
process holds ONE party's shares, reveals eps || delta with a sum-allreduce of
the uint64 bits viewed as int64 (two's-complement addition = addition mod
2^64, as ncclUint64/ncclSum), and forms its own z_p.  The result must equal
the single-process all-parties oracle bit-exactly.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2109_00984_b200 import dist as mdist

MASTER = synth.MASTER_SEED


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(world, fn, *args):
    oracle.build()          # once, before the workers import it
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, fn, args)) for r in range(world)]
    for p in procs:
        p.start()
    results = {}
    for _ in range(world):
        r, out = q.get(timeout=240)
        results[r] = out
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return results


def _worker(rank, world, port, q, fn, args):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = fn(rank, world, *args)
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def _ring_allreduce(u: np.ndarray) -> np.ndarray:
    """Reveal: sum-allreduce of uint64 shares through their int64 view."""
    t = torch.from_numpy(np.ascontiguousarray(u).view(np.int64).copy())
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t.numpy().view(np.uint64)


# ---------------------------------------------------------------------------
def _layout_and_id(rank, world):
    lay = mdist.layout(rank, world, 2)
    groups = mdist.session_groups(lay)
    uid = mdist.exchange_unique_id(lay, groups, lambda: bytes([lay.session]) * 128)
    t = mdist.max_over_ranks(float(rank) * 1.5)
    return lay.session, lay.party, uid, t


def test_layout_unique_id_and_max_over_ranks():
    res = _run(4, _layout_and_id)
    for r in range(4):
        session, party, uid, t = res[r]
        assert (session, party) == (r // 2, r % 2)
        assert uid == bytes([session]) * 128          # same id within a session, distinct across
        assert t == 4.5                               # max over ranks


def test_layout_rejects_odd_world():
    with pytest.raises(ValueError):
        mdist.layout(0, 3, 2)


# ---------------------------------------------------------------------------
def _party_beaver(rank, world, M, K, N):
    P = world
    X = synth.uniform_fixed((M, K), 31)
    Y = synth.uniform_fixed((K, N), 32)
    # this party's shares (the oracle deals all parties; each process keeps its own)
    xs = oracle.share(P, MASTER, X, 0, 7)[rank]
    ys = oracle.share(P, MASTER, Y, 1 % P, 8)[rank]
    a, b, c = (t[rank] for t in oracle.ttp_triple(P, MASTER, 9, M, K, N))
    # mask, then ONE reveal of eps || delta (one round)
    ed = np.concatenate([(xs - a).ravel(), (ys - b).ravel()])
    ed = _ring_allreduce(ed)
    eps, delta = ed[:M * K].reshape(M, K), ed[M * K:].reshape(K, N)
    # z_p = c_p + eps@b_p + a_p@delta + [p=0] eps@delta, in the folded form the kernel uses
    bprime = b + (delta if rank == 0 else np.uint64(0))
    z = c + a @ delta + eps @ bprime
    return z, eps, delta


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_beaver_equals_oracle(world):
    M, K, N = 9, 17, 6
    res = _run(world, _party_beaver, M, K, N)
    X = synth.uniform_fixed((M, K), 31)
    Y = synth.uniform_fixed((K, N), 32)
    xs = oracle.share(world, MASTER, X, 0, 7)
    ys = oracle.share(world, MASTER, Y, 1 % world, 8)
    a, b, c = oracle.ttp_triple(world, MASTER, 9, M, K, N)
    ez, im = oracle.beaver_matmul(xs, ys, a, b, c, want_intermediates=True)
    for r in range(world):
        z, eps, delta = res[r]
        assert np.array_equal(z, ez[r])
        assert np.array_equal(eps, im["eps"]) and np.array_equal(delta, im["delta"])
    assert np.array_equal(oracle.reveal(np.stack([res[r][0] for r in range(world)])), X @ Y)


def _party_trunc(rank, world, n):
    # Alg. 1 one-party decomposition (R12): z_p = x_p + r_p revealed with a u64 sum
    # and the top nibble h_p = signed(z_p) >> 60 with a small-integer sum.
    P = world
    xv = np.random.default_rng(3).integers(-(1 << 44), 1 << 44, size=n, dtype=np.int64)
    x = oracle.share(P, MASTER, synth.to_ring(xv), 0, 5)[rank]
    r, th = oracle.wrap_pair(P, MASTER, 11, n)
    r, th = r[rank], th[rank]
    z = x + r
    zsum = _ring_allreduce(z)
    h = torch.from_numpy((z.view(np.int64) >> 60).astype(np.int64))
    dist.all_reduce(h, op=dist.ReduceOp.SUM)
    H = h.numpy()
    def sgn(v):
        v = int(v)
        return v - (1 << 64) if v >= (1 << 63) else v
    beta = [(sgn(xi) + sgn(ri) - sgn(zi)) >> 64 for xi, ri, zi in zip(x, r, z)]
    out = np.zeros(n, dtype=np.uint64)
    for i in range(n):
        th_z = 0
        if rank == 0:
            zz = int(zsum[i])
            kappa = ((zz >> 60) - int(H[i])) % 16
            S = (int(H[i]) + kappa) * (1 << 60) + (zz & ((1 << 60) - 1))
            szz = zz - (1 << 64) if zz >= (1 << 63) else zz
            th_z = (S - szz) >> 64
        theta_x = (int(beta[i]) - int(th[i]) + th_z) % (1 << 64)
        xi = int(x[i])
        sx = xi - (1 << 64) if xi >= (1 << 63) else xi
        y = (sx >> 16) + ((xi >> 15) & 1)
        out[i] = (y - theta_x * (1 << 48)) % (1 << 64)
    return out


def test_distributed_alg1_truncation_equals_oracle():
    world, n = 3, 400
    res = _run(world, _party_trunc, n)
    xv = np.random.default_rng(3).integers(-(1 << 44), 1 << 44, size=n, dtype=np.int64)
    xs = oracle.share(world, MASTER, synth.to_ring(xv), 0, 5)
    r, th = oracle.wrap_pair(world, MASTER, 11, n)
    exp = oracle.truncate_alg1(xs, r, th, 16)
    for p in range(world):
        assert np.array_equal(res[p], exp[p])


# ---------------------------------------------------------------------------
def _party_elementwise(rank, world, n):
    """One party of the elementwise product and square:
    mask, ONE reveal of [eps | delta] (mpc_beaver_mul's batched round), z_p with
    the public term on party 0; the square reveals eps alone."""
    P = world
    X = synth.uniform_fixed((n,), 61)
    Y = synth.uniform_fixed((n,), 62)
    xs = oracle.share(P, MASTER, X, 0, 3)[rank]
    ys = oracle.share(P, MASTER, Y, 1 % P, 4)[rank]
    a, b, c = (t[rank] for t in oracle.ttp_mul_triple(P, MASTER, 5, (n,)))
    ed = _ring_allreduce(np.concatenate([xs - a, ys - b]))
    eps, delta = ed[:n], ed[n:]
    z = c + eps * b + a * delta + (eps * delta if rank == 0 else np.uint64(0))
    a2, b2 = (t[rank] for t in oracle.ttp_square_pair(P, MASTER, 6, (n,)))
    e2 = _ring_allreduce(xs - a2)
    z2 = b2 + np.uint64(2) * e2 * a2 + (e2 * e2 if rank == 0 else np.uint64(0))
    return z, z2


@pytest.mark.parametrize("world", [2, 4])
def test_distributed_elementwise_mul_square_equal_oracle(world):
    n = 257
    res = _run(world, _party_elementwise, n)
    X = synth.uniform_fixed((n,), 61)
    Y = synth.uniform_fixed((n,), 62)
    xs = oracle.share(world, MASTER, X, 0, 3)
    ys = oracle.share(world, MASTER, Y, 1 % world, 4)
    ez = oracle.beaver_mul(xs, ys, *oracle.ttp_mul_triple(world, MASTER, 5, (n,)))
    ez2 = oracle.beaver_square(xs, *oracle.ttp_square_pair(world, MASTER, 6, (n,)))
    for r in range(world):
        assert np.array_equal(res[r][0], ez[r]) and np.array_equal(res[r][1], ez2[r])

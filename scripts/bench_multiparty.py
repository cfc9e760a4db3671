"""One party per GPU: the P-party Beaver private matmul with fixed-point truncation
as each party runs it (the paper's setup, one process and one GPU per party,
P:377-378), shared by bench.py's two ways of running it:

  * N GPUs (torchrun): party = rank, reveals over NCCL (ncclUint64 sum), barriers
    through torch.distributed; timing is the max over ranks;
  * one GPU: the SAME per-party code on P host threads, each with its own
    one-party context (mpc_create_local) and CUDA stream, the reveals through the
    in-process group (mpc_group) — so the multi-GPU path runs, and is checked,
    on the one GPU a test box has.

A step is one online Beaver matmul (mask, eps reveal in row chunks overlapped
with eps @ b_p, delta reveal, a'_p @ delta) plus the truncation: fused local
for P <= 2, Alg. 1 for P > 2 with the wrap pair materialised in the
offline phase (mpc_ttp_wrap_pairs -> mpc_truncate_pairs).  Inputs already
shared, triple and wrap pair pre-generated (t_online); one triple
is reused by every timed step (ring time is data-independent).

After the timed region each party's shares at a seeded sample of outputs are
compared bit for bit with the CPU oracle on party 0 (outside the timed region).
"""
from __future__ import annotations

import os
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

SEED_X, SEED_Y, TRIPLE_ID, WRAP_ID = 1005, 1006, 3, 7          # the C5 recipe


def _dev(a, device):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).to(device).view(torch.uint64)


def sample_indices(P, M, N, rows=2, cols=64):
    rng = np.random.default_rng(1000 + P)
    r = np.sort(rng.choice(M, min(rows, M), replace=False)).astype(np.int64)
    c = np.sort(rng.choice(N, min(cols, N), replace=False)).astype(np.int64)
    return r, c


def party_run(ctx, party, P, M, K, N, steps, warmup, barrier, device, master, chunks=0):
    """Everything one party does (its own context, its current CUDA stream).
    barrier(): all parties meet (host side).  Returns this party's timing,
    kernel-class breakdown and its z shares at the sample outputs."""
    stream = torch.cuda.current_stream(device)
    if chunks:
        ctx.set_reveal_chunks(chunks)
    X = synth.uniform_fixed((M, K), SEED_X) if party == 0 else None
    Y = synth.uniform_fixed((K, N), SEED_Y) if party == 1 % P else None
    t_setup = time.perf_counter()
    x = ctx.share(_dev(X, device) if X is not None else None, 0, 1, shape=(M, K))
    y = ctx.share(_dev(Y, device) if Y is not None else None, 1 % P, 2, shape=(K, N))
    del X, Y
    a, b, c = ctx.ttp_triples(TRIPLE_ID, M, K, N)                 # offline (rank 0 also the TTP)
    r = th = None
    if P > 2:
        r, th = ctx.ttp_wrap_pairs(WRAP_ID, M * N)                 # offline: Alg. 1's [r], [theta_r]
    z = torch.empty((M, N), dtype=torch.uint64, device=device)

    def step():
        ctx.beaver_matmul(x, y, a, b, c, truncate=P <= 2, out=z)
        if P > 2:
            ctx.truncate_pairs(z.view(-1), r, th)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize(device)
    setup_s = time.perf_counter() - t_setup
    ctx.profile_enable(True)
    for cls in ("gemm", "split", "trunc", "comm"):
        ctx.profile_read(cls)
    r0 = ctx.stats()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize(device)
    ms = e0.elapsed_time(e1) / steps
    r1 = ctx.stats()
    brk = {cls: ctx.profile_read(cls)[0] / steps for cls in ("gemm", "split", "trunc", "comm")}
    ctx.profile_enable(False)
    rows, cols = sample_indices(P, M, N)
    zi = z.view(torch.int64)
    zs = zi[torch.from_numpy(rows).to(device)][:, torch.from_numpy(cols).to(device)].cpu().numpy().view(np.uint64)
    barrier()
    out = {"ms": ms, "breakdown_ms": brk, "rounds_per_step": (r1[0] - r0[0]) / steps,
           "bytes_sent_per_step": (r1[1] - r0[1]) / steps, "setup_s": setup_s, "z_sample": zs}
    del x, y, a, b, c, z, r, th
    return out


def oracle_check(P, M, K, N, z_samples, master, seed_x=SEED_X, seed_y=SEED_Y, triple_id=TRIPLE_ID,
                 wrap_id=WRAP_ID, rows_cols=None):
    """Party 0: every party's sampled shares against the CPU oracle, bit for bit.
    The oracle computes those outputs one by one from the rows of x, a and the
    columns of y, b (the seeded inputs are regenerated from their recipe; x is
    shared by party 0 with share id 1, y by party 1 % P with share id 2)."""
    import oracle
    rows, cols = rows_cols if rows_cols is not None else sample_indices(P, M, N)
    t = time.perf_counter()
    X = synth.uniform_fixed((M, K), seed_x)[rows]
    Yc = synth.uniform_fixed((K, N), seed_y)[:, cols]
    xs = oracle.share_indices(P, master, X.ravel(), 0, 1, (rows[:, None] * K + np.arange(K)[None, :]).ravel())
    ys = oracle.share_indices(P, master, Yc.ravel(), 1 % P, 2, (np.arange(K)[:, None] * N + cols[None, :]).ravel())
    a, b, cc = oracle.ttp_triple_sampled(P, master, triple_id, M, K, N, rows, cols)
    zraw = oracle.beaver_matmul(xs.reshape(P, len(rows), K), ys.reshape(P, K, len(cols)), a, b, cc)
    if P > 2:
        r, th = oracle.wrap_pair_indices(P, master, wrap_id, (rows[:, None] * N + cols[None, :]).ravel())
        ez = oracle.truncate_alg1(zraw.reshape(P, -1), r, th, 16).reshape(zraw.shape)
    else:
        ez = oracle.truncate(zraw, 16)
    got = np.stack(z_samples)
    return {"bit_exact": bool(np.array_equal(got, ez)), "outputs_per_party": int(len(rows) * len(cols)),
            "sample": f"{len(rows)} rows x {len(cols)} seeded columns of every party's z share",
            "oracle_s": time.perf_counter() - t}


def summarise(P, M, K, N, results, check, mode):
    ms = max(r["ms"] for r in results)
    ops = 2.0 * M * N * K
    line = {"workload": f"{P}-party Beaver ring GEMM {M}x{K}x{N} + " + ("Alg. 1 truncation (wrap pair offline)" if P > 2
                                                                        else "local truncation"),
            "mode": mode, "ms_per_private_matmul": ms, "ring_TOPS": ops / (ms * 1e-3) / 1e12,
            "per_party_ms": [r["ms"] for r in results],
            "breakdown_ms_max_over_parties": {k: max(r["breakdown_ms"][k] for r in results)
                                              for k in results[0]["breakdown_ms"]},
            "rounds_per_step": results[0]["rounds_per_step"],
            "bytes_sent_per_party_per_step": results[0]["bytes_sent_per_step"],
            "check": check}
    return line


def run_local_group(P, M, K, N, steps=3, warmup=2, chunks=0, check=True):
    """All P parties as threads on this GPU (in-process group): the multi-GPU code path."""
    import paper_2109_00984_b200 as mpc
    dev = torch.device("cuda", torch.cuda.current_device())
    g = mpc.Group(P)
    ctxs = [mpc.Context(P, r, device=dev.index, master_seed=synth.MASTER_SEED, group=g) for r in range(P)]
    bar = threading.Barrier(P)
    results, errors = [None] * P, []

    def worker(r):
        try:
            torch.cuda.set_device(dev)
            s = torch.cuda.Stream(dev)
            with torch.cuda.stream(s):
                results[r] = party_run(ctxs[r], r, P, M, K, N, steps, warmup, bar.wait, dev, synth.MASTER_SEED,
                                       chunks)
        except BaseException as e:  # noqa: BLE001
            errors.append(e)
            bar.abort()

    th = [threading.Thread(target=worker, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    torch.cuda.synchronize()
    for c in ctxs:
        c.close()
    g.close()
    if errors:
        raise errors[0]
    chk = oracle_check(P, M, K, N, [r["z_sample"] for r in results], synth.MASTER_SEED) if check else None
    out = summarise(P, M, K, N, results, chk, f"{P} one-party contexts on ONE GPU through the in-process group "
                                             "(the multi-GPU schedule and kernels; the parties share one GPU, so "
                                             "the time is not a per-GPU number)")
    torch.cuda.empty_cache()
    return out


def per_gpu_baseline(M, K, N, steps=5, warmup=2):
    """One party alone on one GPU through the one-party schedule (1-rank NCCL
    communicator: every reveal is a local copy): the per-GPU compute floor of the
    one-party-per-GPU runs, i.e. the no-communication variant of SURVEY §8(d)."""
    import paper_2109_00984_b200 as mpc
    dev = torch.device("cuda", torch.cuda.current_device())
    ctx = mpc.Context(1, 0, device=dev.index, master_seed=synth.MASTER_SEED, nccl_id=mpc.nccl_unique_id())
    res = party_run(ctx, 0, 1, M, K, N, steps, warmup, lambda: None, dev, synth.MASTER_SEED)
    ctx.close()
    torch.cuda.empty_cache()
    ms = res["ms"]
    return {"workload": f"1 party {M}x{K}x{N} Beaver (one-party schedule, 1-rank NCCL communicator)",
            "ms_per_private_matmul": ms, "ring_TOPS": 2.0 * M * N * K / (ms * 1e-3) / 1e12,
            "breakdown_ms": res["breakdown_ms"]}


if __name__ == "__main__":
    import json
    P = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
    print(json.dumps(run_local_group(P, n, n, n)))

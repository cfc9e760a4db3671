"""Where the e2e step's time goes (bench.py's e2e loop, 2-party 4096^3, one GPU):
the same loop (a) as bench.py runs it — H2D of the f64 inputs from pinned memory,
encode, share, Beaver on a pre-generated single-use triple, reveal, decode, D2H
of the f64 product, copies on their own streams, double-buffered; (b) without
the H2D / D2H copies (inputs and outputs stay in device memory); (c) with the
copies but no compute (the copies alone, the transfer floor)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2109_00984_b200 as mpc  # noqa: E402

P, M, K, N = 2, 4096, 4096, 4096
dev = torch.device("cuda", 0)
ctx = mpc.Context(P, mpc.ALL_PARTIES, device=0, master_seed=synth.MASTER_SEED)
X = synth.uniform_fixed((M, K), 1002)
Y = synth.uniform_fixed((K, N), 1003)
hX = torch.from_numpy(X.view(np.int64).astype(np.float64) / 65536.0).pin_memory()
hY = torch.from_numpy(Y.view(np.int64).astype(np.float64) / 65536.0).pin_memory()
hout = [torch.empty((M, N), dtype=torch.float64).pin_memory() for _ in range(2)]
dX = [hX.to(dev) for _ in range(2)]
dY = [hY.to(dev) for _ in range(2)]
dout = [torch.empty((M, N), dtype=torch.float64, device=dev) for _ in range(2)]
xe = torch.empty((M, K), dtype=torch.uint64, device=dev)
ye = torch.empty((K, N), dtype=torch.uint64, device=dev)
zr = torch.empty((M, N), dtype=torch.uint64, device=dev)
x = torch.empty((P, M, K), dtype=torch.uint64, device=dev)
y = torch.empty((P, K, N), dtype=torch.uint64, device=dev)
z = torch.empty((P, M, N), dtype=torch.uint64, device=dev)
steps = 12
pool = [ctx.ttp_triples((3 << 20) + j, M, K, N) for j in range(steps + 2)]
stream = torch.cuda.current_stream(dev)
h2d_s, d2h_s = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
ev = lambda: torch.cuda.Event()  # noqa: E731
loaded, done, freed = [ev(), ev()], [ev(), ev()], [ev(), ev()]


def loop(n, copies=True, compute=True):
    for i in range(n):
        s = i % 2
        with torch.cuda.stream(h2d_s):
            if i >= 2:
                h2d_s.wait_event(done[s])
            if copies:
                dX[s].copy_(hX, non_blocking=True)
                dY[s].copy_(hY, non_blocking=True)
            loaded[s].record(h2d_s)
        ta, tb, tc = pool[i % len(pool)]
        stream.wait_event(loaded[s])
        if compute:
            ctx.share(ctx.encode(dX[s], out=xe, check=False), 0, 2 * i, shape=(M, K), out=x)
            ctx.share(ctx.encode(dY[s], out=ye, check=False), 1, 2 * i + 1, shape=(K, N), out=y)
        done[s].record(stream)
        if compute:
            ctx.beaver_matmul(x, y, ta, tb, tc, truncate=True, out=z)
        if i >= 2:
            stream.wait_event(freed[s])
        if compute:
            ctx.decode(ctx.reveal(z, out=zr), out=dout[s])
        with torch.cuda.stream(d2h_s):
            d2h_s.wait_stream(stream)
            if copies:
                hout[s].copy_(dout[s], non_blocking=True)
            freed[s].record(d2h_s)
    stream.wait_stream(d2h_s)
    stream.wait_stream(h2d_s)


def timed(**kw):
    loop(2, **kw)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(stream)
    h2d_s.wait_event(e0)
    loop(steps, **kw)
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


out = {}
for rep in range(2):
    out["a_e2e_ms"] = timed(copies=True, compute=True)
    out["b_no_copies_ms"] = timed(copies=False, compute=True)
    out["c_copies_only_ms"] = timed(copies=True, compute=False)
print(json.dumps(out))

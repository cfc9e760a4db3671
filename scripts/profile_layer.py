"""One 2-party Beaver private matmul of a given shape, repeated, for ncu captures
of the small-layer kernels (all parties on one GPU):

  ncu --set full -k regex:ring_gemm_kernel --launch-skip 2 --launch-count 1 \\
      python scripts/profile_layer.py 197 768 3072
(launch 0 is the TTP's c = a @ b, launches 1.. the Beaver GEMMs)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2109_00984_b200 as mpc  # noqa: E402

M, K, N = (int(v) for v in sys.argv[1:4])
ctx = mpc.Context(2, mpc.ALL_PARTIES, device=0, master_seed=synth.MASTER_SEED)
dev = lambda a: torch.from_numpy(a.view(np.int64)).cuda().view(torch.uint64)  # noqa: E731
x = ctx.share(dev(synth.uniform_fixed((M, K), 41)), 0, 1)
y = ctx.share(dev(synth.uniform_fixed((K, N), 42)), 1, 2)
a, b, c = ctx.ttp_triples(5, M, K, N)
z = torch.empty_like(c)
for _ in range(4):
    ctx.beaver_matmul(x, y, a, b, c, truncate=True, out=z)
torch.cuda.synchronize()
print("done", M, K, N)

"""Per-layer timeline of the 2-CTA ring GEMM on small model layers
(MPC_GEMM_DEBUG=1 prints setup / MMA-end / epilogue-end times per launch).

  MPC_GEMM_DEBUG=1 python scripts/small_gemm_debug.py
"""
import sys, os
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2109_00984_b200 as m  # noqa: E402

c = m.Context(2, m.ALL_PARTIES, device=0, master_seed=synth.MASTER_SEED)
shapes = [(3136, 64, 256), (784, 128, 512), (196, 256, 1024), (3136, 64, 64), (3136, 576, 64), (784, 1152, 128), (196, 2304, 256), (49, 4608, 512),
          (197, 768, 768), (197, 768, 3072), (197, 3072, 768), (12544, 147, 64), (1, 2048, 1000)]
for (M, K, N) in shapes:
    dev = lambda a: torch.from_numpy(a.view(np.int64)).cuda().view(torch.uint64)  # noqa: E731
    x = c.share(dev(synth.uniform_fixed((M, K), 31)), 0, 1)
    y = c.share(dev(synth.uniform_fixed((K, N), 32)), 1, 2)
    a, b, cc = c.ttp_triples(4, M, K, N)
    print(f"--- {M}x{K}x{N}", file=sys.stderr, flush=True)
    for _ in range(3):
        z = c.beaver_matmul(x, y, a, b, cc, truncate=True)
    torch.cuda.synchronize()

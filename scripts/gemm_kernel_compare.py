"""Ring-GEMM kernel time of a 2-party Beaver matmul on the 256 x 128 kernel vs
the stacked-plane kernel (MPC_GEMM_SMALL=0 / 1, set by the caller), from the
library's own launch profiling (CUDA events around each GEMM launch).

  MPC_GEMM_SMALL=1 python scripts/gemm_kernel_compare.py
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2109_00984_b200 as mpc  # noqa: E402

SHAPES = [(1, 2048, 1000), (1, 768, 1000), (32, 519820, 32), (16, 4096, 256), (32, 1024, 2048), (8, 8192, 8192),
          (32, 4096, 4096), (2048, 1024, 24)]
MID = [(64, 64, 64), (49, 4608, 512), (49, 512, 2048), (49, 1024, 2048), (49, 2048, 512), (196, 2304, 256),
       (196, 256, 1024), (100, 250, 250), (50, 12000, 250), (50, 1750, 250), (51, 8000, 2000), (51, 2000, 2000),
       (51, 2000, 29), (197, 768, 768), (128, 1024, 1024)]
if os.environ.get("SHAPES") == "mid":
    SHAPES = MID


def main():
    c = mpc.Context(2, mpc.ALL_PARTIES, device=0, master_seed=synth.MASTER_SEED)
    dev = lambda a: torch.from_numpy(a.view(np.int64)).cuda().view(torch.uint64)  # noqa: E731
    out = {}
    for M, K, N in SHAPES:
        x = c.share(dev(synth.uniform_fixed((M, K), 1)), 0, 1)
        y = c.share(dev(synth.uniform_fixed((K, N), 2)), 1, 2)
        a, b, cc = c.ttp_triples(3, M, K, N)
        z = torch.empty_like(cc)
        for _ in range(3):
            c.beaver_matmul(x, y, a, b, cc, truncate=True, out=z)
        torch.cuda.synchronize()
        c.profile_enable(True)
        c.profile_read("gemm")
        c.profile_read("split")
        reps = 20
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(reps):
            c.beaver_matmul(x, y, a, b, cc, truncate=True, out=z)
        e1.record()
        torch.cuda.synchronize()
        g, gn = c.profile_read("gemm")
        s, _ = c.profile_read("split")
        c.profile_enable(False)
        out[f"{M}x{K}x{N}"] = {"step_us": e0.elapsed_time(e1) / reps * 1e3, "gemm_us": g / reps * 1e3,
                               "gemm_launches_per_step": gn / reps, "split_us": s / reps * 1e3}
        print(f"{M}x{K}x{N}", json.dumps(out[f'{M}x{K}x{N}']), flush=True)
        del x, y, a, b, cc, z
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

"""configs[4]'s GEMM: the P-party 8192^3 Beaver matmul (all parties on one GPU),
repeated, for ncu DRAM-traffic captures of the ring GEMM under the tile-order /
unit-length knobs (MPC_GEMM_KC, MPC_GEMM_GROUPM, MPC_GEMM_TMA):

  MPC_GEMM_KC=32 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum \\
      -k regex:ring_gemm_kernel --launch-skip 2 --launch-count 1 python scripts/profile_c5.py 4
(launch 0 is the TTP's c = a @ b, launches 1.. the Beaver GEMMs); without ncu it
prints the CUDA-event time per Beaver GEMM step."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2109_00984_b200 as mpc  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 4
n = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
ctx = mpc.Context(P, mpc.ALL_PARTIES, device=0, master_seed=synth.MASTER_SEED)
g = torch.Generator(device="cuda").manual_seed(5)
x = torch.randint(-(1 << 62), 1 << 62, (P, n, n), dtype=torch.int64, device="cuda", generator=g).view(torch.uint64)
y = torch.randint(-(1 << 62), 1 << 62, (P, n, n), dtype=torch.int64, device="cuda", generator=g).view(torch.uint64)
a, b, c = ctx.ttp_triples(3, n, n, n)
z = torch.empty_like(c)
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
ctx.beaver_matmul(x, y, a, b, c, truncate=False, out=z)
torch.cuda.synchronize()
ctx.profile_enable(True)
ctx.profile_read("gemm")
e0.record()
for _ in range(reps):
    ctx.beaver_matmul(x, y, a, b, c, truncate=False, out=z)
e1.record()
torch.cuda.synchronize()
gm, _ = ctx.profile_read("gemm")
print(f"P={P} n={n} KC={os.environ.get('MPC_GEMM_KC', '-')} GROUPM={os.environ.get('MPC_GEMM_GROUPM', '-')} "
      f"TMA={os.environ.get('MPC_GEMM_TMA', '-')}: step {e0.elapsed_time(e1) / reps:.2f} ms, gemm {gm / reps:.2f} ms")

"""The HBM / Philox-bound elementwise kernels at the bench sizes, each launched a
few times, for ncu captures (all parties on one GPU):

  ncu --set full -k regex:trunc_alg1_all --launch-skip 1 --launch-count 1 \\
      python scripts/profile_elementwise.py alg1 8
  ncu --set full -k regex:share_kernel --launch-skip 1 --launch-count 1 \\
      python scripts/profile_elementwise.py share 2

alg1 P: Alg. 1 truncation of P parties x 8192^2 shares (wrap pair from its id,
then from memory); share P: P-party sharing of 4096^2 elements; relu P: the fused
all-parties ReLU of 2^24 elements (NEXT-3, Philox-bound)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2109_00984_b200 as mpc  # noqa: E402

what, P = sys.argv[1], int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
ctx = mpc.Context(P, mpc.ALL_PARTIES, device=0, master_seed=synth.MASTER_SEED)
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
if what == "alg1":
    n = 8192 * 8192
    x = torch.randint(-(1 << 62), 1 << 62, (P, n), dtype=torch.int64, device="cuda").view(torch.uint64)
    r, th = ctx.ttp_wrap_pairs(7, n)
    for mode in ("id", "pairs"):
        for i in range(reps + 1):
            if i == 1:
                torch.cuda.synchronize(); e0.record()
            if mode == "id":
                ctx.truncate(x, 16, wrap_id=7)
            else:
                ctx.truncate_pairs(x, r, th, 16)
        e1.record(); torch.cuda.synchronize()
        print(f"alg1 {mode} P={P}: {e0.elapsed_time(e1) / reps:.3f} ms per launch")
elif what == "share":
    n = 4096 * 4096
    x = torch.randint(-(1 << 62), 1 << 62, (n,), dtype=torch.int64, device="cuda").view(torch.uint64)
    out = torch.empty((P, n), dtype=torch.uint64, device="cuda")
    for i in range(reps + 1):
        if i == 1:
            torch.cuda.synchronize(); e0.record()
        ctx.share(x, 0, 1, out=out)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"share P={P}: {ms:.4f} ms, {(8 * n * (P + 1)) / ms / 1e6:.0f} GB/s")
elif what == "relu":
    n = 1 << 24
    x = torch.randint(-(1 << 40), 1 << 40, (P, n), dtype=torch.int64, device="cuda").view(torch.uint64)
    z = torch.empty_like(x)
    for i in range(reps + 1):
        if i == 1:
            torch.cuda.synchronize(); e0.record()
        ctx.relu(x, relu_id=9, out=z)
    e1.record(); torch.cuda.synchronize()
    print(f"relu P={P}: {e0.elapsed_time(e1) / reps:.4f} ms per call")

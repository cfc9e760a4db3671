"""Elementwise private multiplication / square on one GPU,
all parties on the device: ms per op, achieved HBM bandwidth from the
algorithmic bytes, fraction of the measured copy peak (MEASURED_PEAKS.json).

Algorithmic bytes per element (P parties, u64 shares):
  mul:    read x_p, y_p, a_p, b_p, c_p, write z_p  -> 48 P B
  square: read x_p, a_p, b_p,           write z_p  -> 32 P B
  TTP triple: write a_p, b_p, c_p -> 24 P B;  TTP pair: 16 P B
  Alg. 1 truncation (P > 2): read + write x_p -> 16 P B (plus Philox for r_p, theta_r)
  ReLU (fused A2B + B2A + multiplication): read x_p, write out_p -> 16 P B; bound by the
    Philox expansions of its triples (relu_philox_per_elem)

  python scripts/bench_elementwise.py [--n 16777216] [--parties 2] [--reps 50]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
import paper_2109_00984_b200 as mpc  # noqa: E402


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except (OSError, ValueError, KeyError):
        return 6443.5


def timed(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def run(n, P, reps):
    ctx = mpc.Context(P, mpc.ALL_PARTIES, device=0, master_seed=synth.MASTER_SEED)
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.randint(-2**20, 2**20, (P, n), device="cuda", generator=g).view(torch.uint64)
    y = torch.randint(-2**20, 2**20, (P, n), device="cuda", generator=g).view(torch.uint64)
    a, b, c = ctx.ttp_mul_triples(1, (n,))
    a2, b2 = ctx.ttp_square_pairs(2, (n,))
    z = torch.empty_like(x)
    peak = hbm_peak()
    out = {"n": n, "parties": P, "hbm_peak_gbs": peak}
    # the Beaver kernels alone (P <= 2: with the fused local truncation); for P > 2 the
    # Alg. 1 truncation (1 round, Philox-heavy) is timed as its own line
    tr = P <= 2
    cases = {
        "mul": (lambda: ctx.beaver_mul(x, y, a, b, c, truncate=tr, out=z), 48 * P),
        "square": (lambda: ctx.beaver_square(x, a2, b2, truncate=tr, out=z), 32 * P),
        "ttp_mul_triple": (lambda: ctx.ttp_mul_triples(3, (n,), out=(a, b, c)), 24 * P),
        "ttp_square_pair": (lambda: ctx.ttp_square_pairs(4, (n,), out=(a2, b2)), 16 * P),
    }
    if P > 2:
        cases["trunc_alg1"] = (lambda: ctx.truncate(z, 16, wrap_id=5), 16 * P)
    if P <= 8:   # the fused ReLU path (Philox / ALU bound; bytes = x_p in, out_p out)
        cases["relu"] = (lambda: ctx.relu(x, relu_id=9, out=z), 16 * P)
    for name, (fn, bpe) in cases.items():
        ms = timed(fn, reps)
        gbs = bpe * n / (ms * 1e-3) / 1e9
        out[name] = {"ms": ms, "bytes_per_elem": bpe, "achieved_gbs": gbs, "frac_of_hbm": gbs / peak,
                     "Gelem_per_s": n / (ms * 1e-3) / 1e9}
    if "relu" in out:
        # Philox4x32-10 blocks per element (each block serves an element pair): binary zero-shares
        # P per leaf, per AND gate 3P - 1, ceil(log2 P) * 12 gates per adder path... counted exactly:
        levels, q = 0, 1
        while q < P:
            q, levels = q * 2, levels + 1
        adders = P - 1                               # a tree over P leaves has P - 1 adders
        blocks = P * P + adders * 12 * (3 * P - 1) + (1 + 2 * (P - 1)) + (3 * P - 1)
        out["relu"]["philox_blocks_per_elem"] = blocks / 2.0
        out["relu"]["philox_blocks_per_s"] = blocks / 2.0 * n / (out["relu"]["ms"] * 1e-3)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=4096 * 4096)
    ap.add_argument("--parties", type=int, default=2)
    ap.add_argument("--reps", type=int, default=50)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    print(json.dumps(run(args.n, args.parties, args.reps)))


if __name__ == "__main__":
    main()

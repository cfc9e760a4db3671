"""Kernel timeline of one CUDA-graph replay of a model chain (scripts/bench_layers.py
--chain), read from CUPTI through torch.profiler: per kernel class the summed
device time, and the idle gaps between consecutive kernels — what a layer costs
in the real back-to-back replay (ncu serialises and cold-starts every kernel).

  python scripts/chain_timeline.py [--model resnet50|vit|...] [--prepared-offline] [--out FILE]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))

import synth  # noqa: E402
import paper_2109_00984_b200 as mpc  # noqa: E402
import bench_layers as bl  # noqa: E402


def short(name):
    for k in ("split_both", "split_left", "split_right", "split_conv", "ring_gemm_small", "ring_gemm_kernel",
              "finalize", "trunc", "mask", "share", "encode", "decode"):
        if k in name:
            return k
    return name[:40]


def timeline(g, replays=3):
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(replays):
            g.replay()
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    ks = sorted(((e.time_range.start, e.time_range.end, e.name) for e in evs), key=lambda t: t[0])
    return ks


def summarize(ks, replays):
    cls, gaps = {}, []
    for i, (t0, t1, n) in enumerate(ks):
        c = cls.setdefault(short(n), {"n": 0, "us": 0.0})
        c["n"] += 1
        c["us"] += t1 - t0
        if i:
            gaps.append(t0 - ks[i - 1][1])
    span = ks[-1][1] - ks[0][0]
    for c in cls.values():
        c["n"] /= replays
        c["us"] /= replays
    neg = sum(g for g in gaps if g < 0) / replays
    pos = sum(g for g in gaps if g > 0 and g < 200) / replays   # big gaps = between replays
    return {"span_us_per_replay": span / replays, "classes": cls, "idle_gap_us": pos, "overlap_us": -neg}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="resnet50")
    ap.add_argument("--offline", action="store_true", help="weight sides prepared before timing")
    ap.add_argument("--replays", type=int, default=3)
    ap.add_argument("--out", default=None)
    ap.add_argument("--per-kernel", action="store_true")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    ctx = mpc.Context(2, mpc.ALL_PARTIES, device=0, master_seed=synth.MASTER_SEED)
    res = {}

    def hook(g):
        ks = timeline(g, args.replays)
        res["summary"] = summarize(ks, args.replays)
        if args.per_kernel:
            n = len(ks) // args.replays
            t0 = ks[0][0]
            res["kernels"] = [(short(k[2]), round(k[0] - t0, 2), round(k[1] - k[0], 2)) for k in ks[:n]]

    ms = bl.run_chain(ctx, synth.MODELS[args.model], 10, offline=args.offline, hook=hook)
    res["chain_ms_events"] = ms
    res["model"] = args.model + (" (weights prepared offline)" if args.offline else "")
    s = json.dumps(res, indent=1)
    print(s)
    if args.out:
        with open(args.out, "w") as f:
            f.write(s)


if __name__ == "__main__":
    main()

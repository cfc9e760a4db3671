"""The other BASELINE.json configs, measured in the same run as bench.py's
headline (configs[1]), all parties on one GPU:

  C1  configs[0]: 2-party Beaver 64x64x64 (latency: us per private matmul, one CUDA graph)
  C3  configs[2]: 2-party ResNet-50 b1 linear/conv layers as im2col ring GEMMs + truncation
                  (54 private matmuls in one CUDA graph)
  C4  configs[3]: 2-party ViT-B/16 linear layers (50 private matmuls in one CUDA graph)
  C5  configs[4]: 4- and 8-party Beaver 8192^3 (Alg. 1 truncation), all parties on one GPU
  NEXT-4:         the 32 x 519,820 x 32 text-embedding matmul (stacked-plane GEMM)

Each line gives ms, ring-TOPS (2*M*N*K per private matmul) and the fraction of
the limb-GEMM roofline (144*M*N*K int8 ops per party at bench.py's int8 peak);
chains also give the fraction of the per-layer max(tensor time, HBM floor)
(bench_layers.t_hbm_ms: the x, a, y, b, c reads and z write of every party).

  python scripts/bench_configs.py [--skip-c5]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))

import synth  # noqa: E402
import paper_2109_00984_b200 as mpc  # noqa: E402
import bench_layers  # noqa: E402


def _events_ms(fn, reps, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def c1_latency(reps=200):
    P, M, K, N = 2, 64, 64, 64
    ctx = mpc.Context(P, mpc.ALL_PARTIES, device=0, master_seed=synth.MASTER_SEED)
    dev = lambda a: torch.from_numpy(a.view(np.int64)).cuda().view(torch.uint64)  # noqa: E731
    x = ctx.share(dev(synth.uniform_fixed((M, K), 1001)), 0, 1)
    y = ctx.share(dev(synth.uniform_fixed((K, N), 1002)), 1, 2)
    a, b, c = ctx.ttp_triples(1, M, K, N)
    z = torch.empty_like(c)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        ctx.beaver_matmul(x, y, a, b, c, truncate=True, out=z)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(10):
                ctx.beaver_matmul(x, y, a, b, c, truncate=True, out=z)
    ms = _events_ms(g.replay, reps // 10) / 10
    return {"workload": "configs[0] 2-party 64^3 Beaver + truncation", "us_per_private_matmul": ms * 1e3,
            "graph": "10 matmuls per CUDA graph replay"}


def chain(name, reps=10, offline_variant=False):
    ctx = mpc.Context(2, mpc.ALL_PARTIES, device=0, master_seed=synth.MASTER_SEED)
    layers = synth.MODELS[name]
    ms = bench_layers.run_chain(ctx, layers, reps)
    ops, tg, n = bench_layers.layer_totals(layers)
    rl = bench_layers.layer_rooflines(layers)
    out = {"private_matmuls": n, "chain_ms": ms, "ring_TOPS": ops / (ms * 1e-3) / 1e12,
           "roofline_ms": tg, "roofline_frac": tg / ms,
           "roofline_tensor_or_hbm_ms": rl, "roofline_tensor_or_hbm_frac": rl / ms}
    if offline_variant:
        # weight sides (delta reveal + splits) prepared with the triples, before the input arrives
        mo = bench_layers.run_chain(ctx, layers, reps, offline=True)
        out["weights_prepared_offline"] = {"chain_ms": mo, "ring_TOPS": ops / (mo * 1e-3) / 1e12,
                                           "roofline_frac": tg / mo, "roofline_tensor_or_hbm_frac": rl / mo,
                                           "note": "delta = w - b revealed in the offline phase (mpc_beaver_prepare); "
                                                   "the timed chain holds the eps reveal, x-side split and GEMM"}
    return out


def c5(P, n=8192, steps=3):
    ctx = mpc.Context(P, mpc.ALL_PARTIES, device=0, master_seed=synth.MASTER_SEED)
    gen = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randint(-8 << 16, 8 << 16, (P, n, n), device="cuda", generator=gen).view(torch.uint64)
    y = torch.randint(-8 << 16, 8 << 16, (P, n, n), device="cuda", generator=gen).view(torch.uint64)
    a, b, c = ctx.ttp_triples(1, n, n, n)
    z = torch.empty_like(c)
    ctx.profile_enable(True)
    ms = _events_ms(lambda: ctx.beaver_matmul(x, y, a, b, c, truncate=True, wrap_id=1, out=z), steps, warm=1)
    gemm_ms, gl = ctx.profile_read("gemm")
    trunc_ms, _ = ctx.profile_read("trunc")
    split_ms, _ = ctx.profile_read("split")
    ctx.profile_enable(False)
    k = steps + 1
    tg = bench_layers.t_gemm_ms(n, n, n, parties=P)
    hbm = bench_layers.hbm_gbs()
    t_ms, s_ms = trunc_ms / k, split_ms / k
    out = {"ms_per_private_matmul": ms, "ring_TOPS": 2.0 * n ** 3 / (ms * 1e-3) / 1e12,
           "gemm_ms": gemm_ms / k, "alg1_truncation_ms": t_ms, "split_ms": s_ms,
           # Alg. 1 (seeded TTP): reads and writes every party's share, 16 P B per element
           "alg1_hbm_frac": 16.0 * P * n * n / (t_ms * 1e-3) / (hbm * 1e9) if t_ms > 0 else None,
           # mask + local reveal + split: (3P + 1) x 8 B per element of both operands
           "split_hbm_frac": 2 * (3 * P + 1) * 8.0 * n * n / (s_ms * 1e-3) / (hbm * 1e9) if s_ms > 0 else None,
           "roofline_ms": tg, "roofline_frac": tg / ms,
           "note": f"all {P} parties on one GPU (the GEMM work is P x 144 n^3); one party per GPU is the NCCL path"}
    del x, y, a, b, c, z
    torch.cuda.empty_cache()
    return out


def one_party_schedule(n=4096, steps=10):
    """One party per GPU, as the N-GPU bench runs it, on this GPU: a 1-rank NCCL
    communicator (its allreduces are copies, so no NVLink time is measured) runs
    the overlapped schedule — mask, eps (row chunks) then delta reveal on the comm
    stream, b_p split + per-chunk eps split and phase-1 GEMM (eps @ b_p) on 132 SMs,
    delta split + phase-2 GEMM (a'_p @ delta) — against the fused single-GEMM
    schedule of a context without communicator (P = 1 both).  The difference is
    what the overlap structure itself costs (chunked phase-1 launches, 16 SMs left
    to NCCL during phase 1)."""
    gen = torch.Generator(device="cuda").manual_seed(7)
    x = torch.randint(-8 << 16, 8 << 16, (n, n), device="cuda", generator=gen).view(torch.uint64)
    y = torch.randint(-8 << 16, 8 << 16, (n, n), device="cuda", generator=gen).view(torch.uint64)
    out = {}
    for label, uid in (("fused_no_comm", None), ("overlapped_nccl_1rank", mpc.nccl_unique_id())):
        ctx = mpc.Context(1, 0, device=0, master_seed=synth.MASTER_SEED, nccl_id=uid)
        a, b, c = ctx.ttp_triples(1, n, n, n)
        z = torch.empty_like(c)
        out[label + "_ms"] = _events_ms(lambda: ctx.beaver_matmul(x, y, a, b, c, truncate=True, out=z), steps)
        del ctx, a, b, c, z
    out["schedule_overhead_frac"] = out["overlapped_nccl_1rank_ms"] / out["fused_no_comm_ms"] - 1.0
    out["workload"] = f"1 party {n}^3 Beaver + truncation"
    torch.cuda.empty_cache()
    return out


def run(skip_c5=False):
    out = {"C1": c1_latency(), "one_party_schedule": one_party_schedule()}
    for key, name in (("C3_resnet50", "resnet50"), ("C4_vit_b16", "vit"), ("C4_vit_b16_with_attention", "vit_attn"),
                      ("NEXT4_text", "text")):
        out[key] = chain(name, offline_variant=name in ("resnet50", "vit"))
        torch.cuda.empty_cache()
    # the convolutional models as true private convolutions (conv triples, reveal at the
    # activation / weight shapes): ResNet-50 b1 (2-D) and Wav2Letter b1 / b32 (1-D)
    ctx = mpc.Context(2, mpc.ALL_PARTIES, device=0, master_seed=synth.MASTER_SEED)
    ms, rb = bench_layers.run_conv_chain(ctx, synth.CONV_MODELS["resnet50"], 20)
    out["NEXT2_resnet50_conv2d"] = {"chain_ms": ms, "reveal_MB_per_party": rb / 1e6,
                                    "reveal_MB_im2col_shape": sum(8 * (M * K + K * N) * c
                                                                  for _, M, K, N, c in synth.RESNET50_B1) / 1e6}
    out["NEXT2_wav2letter_conv1d"] = bench_layers.wav2letter_conv1d_report(ctx)
    del ctx
    torch.cuda.empty_cache()
    if not skip_c5:
        out["C5_p4_8192"] = c5(4)
        out["C5_p8_8192"] = c5(8)
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-c5", action="store_true")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    print(json.dumps(run(args.skip_c5), indent=1))

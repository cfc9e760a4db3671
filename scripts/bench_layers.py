"""Per-layer 2-party Beaver matmul timings for the paper's model workloads
(configs[2]/[3]: ResNet-50 batch 1 im2col GEMMs, ViT-B/16 linear layers; also
ResNet-18, the model the paper times, and Wav2Letter), both parties on one GPU,
truncation fused.  Reports µs per private matmul, ring-TOPS and the share of
the layer time spent in the tcgen05 GEMM.  --chain captures every layer of a
model (each repeated `count` times, in order) in ONE CUDA graph and times the
whole chain, as a private inference would run them back to back.

  python scripts/bench_layers.py [--model resnet50|vit|resnet18|wav2letter|text|all] [--reps 20]
                                 [--graph] [--chain] [--conv]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
import paper_2109_00984_b200 as mpc  # noqa: E402


def run_layer(ctx, M, K, N, reps, graph):
    dev = torch.device("cuda", 0)
    X = synth.uniform_fixed((M, K), 11)
    Y = synth.uniform_fixed((K, N), 12)
    x = ctx.share(torch.from_numpy(X.view(np.int64)).to(dev).view(torch.uint64), 0, 1)
    y = ctx.share(torch.from_numpy(Y.view(np.int64)).to(dev).view(torch.uint64), 1, 2)
    a, b, c = ctx.ttp_triples(1, M, K, N)
    z = torch.empty_like(c)
    ctx.beaver_matmul(x, y, a, b, c, truncate=True, out=z)
    torch.cuda.synchronize()
    if graph:
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            ctx.beaver_matmul(x, y, a, b, c, truncate=True, out=z)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                ctx.beaver_matmul(x, y, a, b, c, truncate=True, out=z)
        step = g.replay
    else:
        def step():
            ctx.beaver_matmul(x, y, a, b, c, truncate=True, out=z)
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    ctx.profile_enable(True)
    ctx.profile_read("gemm")
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        step()
    e1.record()
    torch.cuda.synchronize()
    gemm_ms, _ = ctx.profile_read("gemm")
    ctx.profile_enable(False)
    ms = e0.elapsed_time(e1) / reps
    return ms, (gemm_ms / reps if not graph else None)


def run_chain(ctx, layers, reps, prepared=False, offline=False, hook=None):
    """All layers of one model in one CUDA graph; returns ms per pass.

    prepared: the weight side of every private matmul (delta reveal, delta and
    b'_p splits: mpc_beaver_prepare) runs on a second stream, in layer order,
    beside the activation chain (mpc_beaver_matmul_prepared, which waits for its
    layer's prepare) — all inside the same graph and timed region.
    offline: the weight sides are prepared once before timing (they depend only
    on the weights and the pre-generated triples, so they belong to the offline
    phase with the triples); the timed graph holds the x sides only."""
    dev = torch.device("cuda", 0)
    bufs = []
    batched = []                      # (x, y, a, b, c, z, count) of batched entries (attention heads)
    for i, layer in enumerate(layers):
        _, M, K, N, count = layer[:5]
        if len(layer) > 5:            # a batch of independent matmuls (6th field), one batched call
            B = layer[5]
            X = synth.uniform_fixed((B, M, K), 100 + i)
            Y = synth.uniform_fixed((B, K, N), 200 + i)
            x = ctx.share(torch.from_numpy(X.view(np.int64)).to(dev).view(torch.uint64), 0, 1 + 2 * i)
            y = ctx.share(torch.from_numpy(Y.view(np.int64)).to(dev).view(torch.uint64), 1, 2 + 2 * i)
            tr = [ctx.ttp_triples(1000 * (i + 1) + h, M, K, N) for h in range(B)]
            a, b, c = (torch.stack([t[j] for t in tr], dim=1).contiguous() for j in range(3))
            batched.append((x, y, a, b, c, torch.empty_like(c), count))
            continue
        X = synth.uniform_fixed((M, K), 100 + i)
        Y = synth.uniform_fixed((K, N), 200 + i)
        x = ctx.share(torch.from_numpy(X.view(np.int64)).to(dev).view(torch.uint64), 0, 1 + 2 * i)
        y = ctx.share(torch.from_numpy(Y.view(np.int64)).to(dev).view(torch.uint64), 1, 2 + 2 * i)
        a, b, c = ctx.ttp_triples(1 + i, M, K, N)
        preps = [ctx.beaver_prepare(y, b, M) for _ in range(count)] if (prepared or offline) else None
        bufs.append((x, y, a, b, c, torch.empty_like(c), count, preps))

    def run_batched():
        for x, y, a, b, c, z, count in batched:
            for _ in range(count):
                ctx.beaver_matmul_batched(x, y, a, b, c, truncate=True, out=z)

    side = torch.cuda.Stream(priority=0) if prepared else None

    if offline:
        for x, y, a, b, c, z, count, preps in bufs:
            for r in range(count):
                ctx.beaver_prepare(y, b, x.shape[-2], out=preps[r])
        torch.cuda.synchronize()

    def chain():
        run_batched()
        if offline:
            for x, y, a, b, c, z, count, preps in bufs:
                for r in range(count):
                    ctx.beaver_matmul_prepared(x, a, c, preps[r], truncate=True, out=z)
            return
        if not prepared:
            for x, y, a, b, c, z, count, _ in bufs:
                for _ in range(count):
                    ctx.beaver_matmul(x, y, a, b, c, truncate=True, out=z)
            return
        main = torch.cuda.current_stream()
        side.wait_stream(main)
        evs = []
        with torch.cuda.stream(side):
            for x, y, a, b, c, z, count, preps in bufs:
                for r in range(count):
                    ctx.beaver_prepare(y, b, x.shape[-2], out=preps[r])
                    e = torch.cuda.Event()
                    e.record(side)
                    evs.append(e)
        k = 0
        for x, y, a, b, c, z, count, preps in bufs:
            for r in range(count):
                main.wait_event(evs[k])
                k += 1
                ctx.beaver_matmul_prepared(x, a, c, preps[r], truncate=True, out=z)
        main.wait_stream(side)

    chain()
    torch.cuda.synchronize()
    s = torch.cuda.Stream(priority=-1) if prepared else torch.cuda.Stream()
    with torch.cuda.stream(s):
        chain()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            chain()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    if hook is not None:              # e.g. a kernel timeline of one replay (scripts/chain_timeline.py)
        hook(g)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


# Limb-GEMM roofline of one 2-party private matmul on one GPU:
# 144*M*N*K int8 ops per party at the int8 peak bench.py uses (2 x measured
# sustained bf16, MEASURED_PEAKS.json; 2 x 1407 TOPS if the file is absent).
def int8_peak_tops():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        for k in ("bf16_tflops_sustained", "bf16_tflops"):
            if k in d:
                return 2.0 * float(d[k])
    except (OSError, ValueError):
        pass
    return 2.0 * 1407.2


def t_gemm_ms(M, K, N, parties=2):
    return 144.0 * M * N * K * parties / (int8_peak_tops() * 1e12) * 1e3


def layer_totals(layers):
    """(ring ops 2*M*N*K, limb-GEMM roofline ms, private matmuls) of a layer list
    whose entries are (name, M, K, N, count[, batch])."""
    ops = tg = n = 0.0
    for layer in layers:
        _, M, K, N, cnt = layer[:5]
        B = layer[5] if len(layer) > 5 else 1
        ops += 2.0 * M * K * N * cnt * B
        tg += t_gemm_ms(M, K, N) * cnt * B
        n += cnt * B
    return ops, tg, int(n)


def hbm_gbs():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except (OSError, ValueError, KeyError):
        return 6650.0


def t_hbm_ms(M, K, N, parties=2):
    """HBM floor of one private matmul with all parties on one GPU: the bytes the
    protocol cannot avoid — read x_p, a_p (M x K), y_p, b_p (K x N), c_p (M x N)
    and write z_p, 8 B each, for every party (limb planes excluded: they are this
    design's intermediate, not the method's)."""
    return parties * 8.0 * (2 * M * K + 2 * K * N + 2 * M * N) / (hbm_gbs() * 1e9) * 1e3


def layer_rooflines(layers):
    """Per-layer max(limb-GEMM tensor time, HBM floor), summed over the chain:
    the roofline of a chain whose small layers are HBM-bound rather than
    tensor-bound (reported beside the tensor-only figure)."""
    tot = 0.0
    for layer in layers:
        _, M, K, N, cnt = layer[:5]
        B = layer[5] if len(layer) > 5 else 1
        tot += max(t_gemm_ms(M, K, N), t_hbm_ms(M, K, N)) * cnt * B
    return tot


def run_conv_chain(ctx, layers, reps):
    """All convolutions of one model as TRUE private convolutions (conv triples,
    eps/delta revealed at the input/weight shapes) in one CUDA graph."""
    dev = torch.device("cuda", 0)
    bufs, reveal_bytes = [], 0
    for i, (_, C, H, W, Co, k, st, pd, count) in enumerate(layers):
        g = ctx.conv_geom(1, C, H, W, Co, k, k, st, pd)
        X = synth.gaussian_fixed((1, C, H, W), 100 + i, 1.0, 0, 8, absval=True)
        Y = synth.gaussian_fixed((Co, C, k, k), 200 + i, (2.0 / (C * k * k)) ** 0.5, -8, 8)
        x = ctx.share(torch.from_numpy(X.view(np.int64)).to(dev).view(torch.uint64), 0, 1 + 2 * i)
        y = ctx.share(torch.from_numpy(Y.view(np.int64)).to(dev).view(torch.uint64), 1, 2 + 2 * i)
        a, b, c = ctx.ttp_conv_triples(1 + i, g)
        bufs.append((g, x, y, a, b, c, torch.empty_like(c), count))
        reveal_bytes += 8 * (X.size + Y.size) * count

    def chain():
        for g, x, y, a, b, c, z, count in bufs:
            for _ in range(count):
                ctx.beaver_conv2d(g, x, y, a, b, c, truncate=True, out=z)

    chain()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        chain()
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=s):
            chain()
    for _ in range(3):
        gr.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        gr.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, reveal_bytes


def run_conv1d_chain(ctx, layers, B, reps):
    """Wav2Letter's convolutions as TRUE private 1-D convolutions (eps / delta revealed at
    the activation / weight shapes) in one CUDA graph; returns (ms, reveal bytes per party,
    im2col-shape reveal bytes per party, ring ops)."""
    dev = torch.device("cuda", 0)
    bufs, rb, rb_im2col, ops = [], 0, 0, 0.0
    for i, (_, C, L, Co, k, st, pd, count) in enumerate(layers):
        g = ctx.conv1d_geom(B, C, L, Co, k, st, pd)
        Lo = (L + 2 * pd - k) // st + 1
        X = synth.gaussian_fixed((B, C, L), 300 + i, 1.0, -8, 8)
        Y = synth.gaussian_fixed((Co, C, k), 400 + i, (2.0 / (C * k)) ** 0.5, -8, 8)
        x = ctx.share(torch.from_numpy(X.view(np.int64)).to(dev).view(torch.uint64), 0, 1 + 2 * i)
        y = ctx.share(torch.from_numpy(Y.view(np.int64)).to(dev).view(torch.uint64), 1, 2 + 2 * i)
        a, b, c = ctx.ttp_conv1d_triples(1 + i, g)
        bufs.append((g, x, y, a, b, c, torch.empty_like(c), count))
        rb += 8 * (X.size + Y.size) * count
        M, K = B * Lo, C * k
        rb_im2col += 8 * (M * K + K * Co) * count
        ops += 2.0 * M * K * Co * count

    def chain():
        for g, x, y, a, b, c, z, count in bufs:
            for _ in range(count):
                ctx.beaver_conv1d(g, x, y, a, b, c, truncate=True, out=z)

    chain()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        chain()
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=s):
            chain()
    for _ in range(3):
        gr.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        gr.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, rb, rb_im2col, ops


def wav2letter_conv1d_report(ctx, reps=20):
    out = {}
    for B in (1, 32):
        ms, rb, rbi, ops = run_conv1d_chain(ctx, synth.WAV2LETTER_CONV1D, B, reps)
        layers = [(n, B * ((L + 2 * pd - k) // st + 1), C * k, Co, cnt)
                  for n, C, L, Co, k, st, pd, cnt in synth.WAV2LETTER_CONV1D]
        tg = sum(t_gemm_ms(M, K, N) * cnt for _, M, K, N, cnt in layers)
        rl = layer_rooflines(layers)
        out[f"b{B}"] = {"chain_ms": ms, "private_convs": sum(l[-1] for l in synth.WAV2LETTER_CONV1D),
                        "ring_TOPS": ops / (ms * 1e-3) / 1e12, "roofline_ms": tg, "roofline_frac": tg / ms,
                        "roofline_tensor_or_hbm_frac": rl / ms,
                        "reveal_MB_per_party": rb / 1e6, "reveal_MB_im2col_shape": rbi / 1e6,
                        "graph": "one CUDA graph per model; true 1-D convolutions (conv triples)"}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="all", choices=list(synth.MODELS) + ["all"])
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--graph", action="store_true")
    ap.add_argument("--chain", action="store_true")
    ap.add_argument("--conv", action="store_true", help="true private convolutions (conv triples) for CNNs")
    ap.add_argument("--prepared", action="store_true",
                    help="chain: weight sides prepared on a second stream beside the activation chain")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    ctx = mpc.Context(2, mpc.ALL_PARTIES, device=0, master_seed=synth.MASTER_SEED)
    out = {}
    for name, layers in synth.MODELS.items():
        if args.model not in (name, "all"):
            continue
        if args.conv:
            if name == "wav2letter":
                out["wav2letter_conv1d"] = r = wav2letter_conv1d_report(ctx, args.reps)
                for bk, v in r.items():
                    print(f"wav2letter {bk} (true 1-D convs): {v['chain_ms']:.3f} ms ({v['ring_TOPS']:.2f} ring-TOPS), "
                          f"reveal {v['reveal_MB_per_party']:.0f} MB/party (im2col shape "
                          f"{v['reveal_MB_im2col_shape']:.0f} MB)", flush=True)
                continue
            if name not in synth.CONV_MODELS:
                continue
            ms, rb = run_conv_chain(ctx, synth.CONV_MODELS[name], args.reps)
            ops = sum(2.0 * M * K * N * cnt for _, M, K, N, cnt in layers)
            tg = sum(t_gemm_ms(M, K, N) * cnt for _, M, K, N, cnt in layers)
            n = sum(cnt for *_, cnt in layers)
            rb_im2col = sum(8 * (M * K + K * N) * cnt for _, M, K, N, cnt in layers)
            out[name + "_conv"] = {"chain_ms": ms, "private_convs": n, "ring_TOPS": ops / (ms * 1e-3) / 1e12,
                                   "roofline_ms": tg, "roofline_frac": tg / ms, "reveal_MB_per_party": rb / 1e6,
                                   "reveal_MB_im2col_shape": rb_im2col / 1e6, "graph": "one CUDA graph per model"}
            print(f"{name} (true convs): chain of {n} private convolutions {ms:.3f} ms "
                  f"({out[name + '_conv']['ring_TOPS']:.2f} ring-TOPS), reveal {rb / 1e6:.0f} MB/party "
                  f"(im2col-shape reveal would be {rb_im2col / 1e6:.0f} MB)", flush=True)
            continue
        if args.chain:
            ms = run_chain(ctx, layers, args.reps, prepared=args.prepared)
            ops, tg, n = layer_totals(layers)
            key = name + ("_prepared" if args.prepared else "")
            rl = layer_rooflines(layers)
            out[key] = {"chain_ms": ms, "private_matmuls": n, "ring_TOPS": ops / (ms * 1e-3) / 1e12,
                        "roofline_ms": tg, "roofline_frac": tg / ms,
                        "roofline_tensor_or_hbm_ms": rl, "roofline_tensor_or_hbm_frac": rl / ms,
                        "graph": "one CUDA graph per model" + (
                            "; weight sides (delta reveal + splits) on a second stream" if args.prepared else "")}
            print(f"{key}: chain of {n} private matmuls {ms:.3f} ms ({out[key]['ring_TOPS']:.2f} ring-TOPS, "
                  f"limb-GEMM roofline {tg:.3f} ms = {tg / ms:.3f}; per-layer max(tensor, HBM) {rl:.3f} ms "
                  f"= {rl / ms:.3f})", flush=True)
            continue
        rows, total_ms, total_ops = [], 0.0, 0.0
        for lname, M, K, N, count in layers:
            ms, gms = run_layer(ctx, M, K, N, args.reps, args.graph)
            total_ms += ms * count
            total_ops += 2.0 * M * K * N * count
            rows.append({"layer": lname, "M": M, "K": K, "N": N, "count": count, "us": ms * 1e3,
                         "gemm_us": None if gms is None else gms * 1e3,
                         "ring_TOPS": 2.0 * M * K * N / (ms * 1e-3) / 1e12,
                         "roofline_frac": t_gemm_ms(M, K, N) / ms})
            print(f"{name:9s} {lname:12s} {M:6d}x{K:5d}x{N:5d} x{count:2d}  {ms * 1e3:9.1f} us"
                  + ("" if gms is None else f"  (gemm {gms * 1e3:8.1f} us)")
                  + f"  {rows[-1]['ring_TOPS']:7.2f} ring-TOPS  roofline {rows[-1]['roofline_frac']:.3f}", flush=True)
        out[name] = {"layers": rows, "total_ms": total_ms, "ring_TOPS": total_ops / (total_ms * 1e-3) / 1e12,
                     "graph": args.graph}
        print(f"{name}: total {total_ms:.3f} ms per private inference's linear layers "
              f"({out[name]['ring_TOPS']:.2f} ring-TOPS)", flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()

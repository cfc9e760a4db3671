"""bench.py's multi-process path (torchrun, one process per party) on ONE GPU:
two ranks with --parties 1 form two 1-party sessions (each with its own 1-rank
NCCL communicator, so no communicator spans processes sharing the device) and
run everything the N-GPU bench runs — gloo rendezvous, session groups, NCCL
unique-id exchange, one-party contexts with the overlapped schedule, e2e,
exposed-communication probe, max-over-ranks timing — and rank 0 prints exactly
one JSON line on stdout."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_torchrun_two_ranks_one_json_line():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29561", os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--parties", "1", "--steps", "3", "--warmup", "3", "--M", "512", "--K", "768", "--N", "640"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["sessions"] == 2 and d["config"]["mode"] == "one party per GPU"
    assert d["check"]["max_abs_err_sampled_rows"] <= 2.0 ** -14
    assert d["e2e"]["max_abs_err_sampled_rows"] <= 2.0 ** -14
    assert d["gpu_launches"] > 0 and "exposed_comm" in d
    chk = d["check"]["bit_exact_vs_oracle"]          # the timed shares of session 0, gathered to rank 0
    assert chk["bit_exact"] and chk["outputs_per_party"] == 2 * 128


def test_multiparty_emulation_matches_oracle():
    """bench_multiparty's per-party code (the N-GPU schedule: chunked eps reveal,
    offline wrap pairs, Alg. 1 over u64 + int8 reveals) for P parties as threads on
    one GPU, at a small size, bit-exact on its seeded sample."""
    sys.path.insert(0, os.path.join(ROOT, "scripts"))
    import bench_multiparty as bmp
    for P, n in ((2, 1024), (3, 1100), (5, 640)):
        out = bmp.run_local_group(P, n, n // 2, n + 64, steps=2, warmup=1, chunks=3)
        assert out["check"]["bit_exact"], (P, n)
        assert out["rounds_per_step"] == (2 if P > 2 else 1)
    base = bmp.per_gpu_baseline(512, 512, 512, steps=2)
    assert base["ms_per_private_matmul"] > 0

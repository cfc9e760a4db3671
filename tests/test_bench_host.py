"""Host logic of bench.py that runs without a GPU: the reference arm (the CPU
oracle timed on a bounded row sample) and its JSON line, alone and
under torchrun with two ranks (rank 0 alone prints; the others exit 0), and the
oracle's thread-count knob used for the one-thread cpu_baseline (timing only:
results must not depend on it)."""
import json
import os
import subprocess
import sys

import numpy as np

import oracle
import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ref_cmd(*extra):
    return [os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "2", "--warmup", "1",
            "--M", "256", "--K", "192", "--N", "160", *extra]


def _one_line(stdout):
    lines = [l for l in stdout.splitlines() if l.strip()]
    assert len(lines) == 1, stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, *_ref_cmd("--sample-rows", "32")], capture_output=True, text=True,
                         timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    d = _one_line(out.stdout)
    assert d["impl"] == "reference" and d["value"] > 0 and d["steps"] == 2 and d["warmup"] == 1
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert "8 of 256 output rows" in d["cpu_baseline"]["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["higher_is_better"] is True and d["vs_baseline"] is None


def test_reference_arm_sized_sample():
    """--sample-rows 0 (the default) sizes the sample from two calibration runs."""
    out = subprocess.run([sys.executable, *_ref_cmd()], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    d = _one_line(out.stdout)
    rows = int(d["config"]["workload"].split("oracle on a ")[1].split("-row")[0])
    assert 4 <= rows <= 256


def test_reference_arm_two_ranks_rank0_prints():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29573", *_ref_cmd("--sample-rows", "16", "--gpus", "2")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    d = _one_line(out.stdout)
    assert d["impl"] == "reference" and d["n_gpus"] == 2


def test_oracle_threads_do_not_change_results():
    P, M, K, N = 2, 37, 29, 23
    X = synth.uniform_fixed((M, K), 71)
    Y = synth.uniform_fixed((K, N), 72)
    n0 = oracle.get_threads()
    outs = []
    try:
        for t in (1, 3):
            oracle.set_threads(t)
            assert oracle.get_threads() == t
            x = oracle.share(P, synth.MASTER_SEED, X, 0, 1)
            y = oracle.share(P, synth.MASTER_SEED, Y, 1, 2)
            a, b, c = oracle.ttp_triple(P, synth.MASTER_SEED, 3, M, K, N)
            outs.append(oracle.truncate(oracle.beaver_matmul(x, y, a, b, c), 16))
    finally:
        oracle.set_threads(n0)
    assert np.array_equal(outs[0], outs[1])

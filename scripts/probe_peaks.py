"""Measure int8 / bf16 dense tensor peaks of this B200 with cuBLAS(Lt) through
torch (8192^3): burst = best of 10; sustained = back-to-back for ~4 s (clocks
sampled by a background nvidia-smi), the recipe MEASURED_PEAKS.json uses for
bf16.  Writes profiles/r01/peaks_cublas.json."""
import json
import os
import statistics
import subprocess
import threading
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class Clocks:
    def __init__(self):
        self.rows = []

    def __enter__(self):
        self.p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active",
                                   "--format=csv,noheader,nounits", "-lms", "100"],
                                  stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        self.t = threading.Thread(target=lambda: [self.rows.append(l.strip()) for l in self.p.stdout], daemon=True)
        self.t.start()
        return self

    def __exit__(self, *a):
        self.p.terminate()
        self.t.join(timeout=5)

    def median_sm(self):
        v = [float(r.split(",")[0]) for r in self.rows if r and r.split(",")[0].strip().replace(".", "").isdigit()]
        return statistics.median(v) if v else None


def measure(fn, ops):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    n = max(10, int(4000 / best))
    with Clocks() as clk:
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        for _ in range(n):
            fn()
        e.record(); torch.cuda.synchronize()
    return {"burst_tops": ops / best / 1e9, "sustained_tops": ops * n / s.elapsed_time(e) / 1e9,
            "sustained_s": s.elapsed_time(e) / 1e3, "sm_mhz_median_sustained": clk.median_sm()}


def main():
    n = 8192
    a = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda")
    b = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda").t().contiguous().t()
    x = torch.randn(n, n, dtype=torch.bfloat16, device="cuda")
    y = torch.randn(n, n, dtype=torch.bfloat16, device="cuda")
    res = {"int8 torch._int_mm (cuBLASLt)": measure(lambda: torch._int_mm(a, b), 2.0 * n ** 3),
           "bf16 torch.matmul (cuBLAS)": measure(lambda: x @ y, 2.0 * n ** 3)}
    for k, v in res.items():
        print(k, v, flush=True)
    os.makedirs(os.path.join(ROOT, "profiles", "r01"), exist_ok=True)
    json.dump(res, open(os.path.join(ROOT, "profiles", "r01", "peaks_cublas.json"), "w"), indent=1)


if __name__ == "__main__":
    main()

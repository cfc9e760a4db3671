"""Measure the int8 dense tensor-core peak of this B200 with cuBLASLt through
torch._int_mm (8192^3, burst = best of 10, sustained = back-to-back for ~4 s),
the same recipe MEASURED_PEAKS.json uses for bf16.  Writes profiles/int8_peak.json."""
import json
import os
import subprocess
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def clocks():
    try:
        out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active",
                              "--format=csv,noheader"], capture_output=True, text=True, timeout=5).stdout.strip()
        return out
    except Exception as e:
        return str(e)


def main():
    n = 8192
    a = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda")
    b = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda").t().contiguous().t()
    res = {}
    for name, fn, ops in (("int8 _int_mm", lambda: torch._int_mm(a, b), 2.0 * n ** 3),
                          ("bf16 matmul", None, 2.0 * n ** 3)):
        if fn is None:
            x = torch.randn(n, n, dtype=torch.bfloat16, device="cuda")
            y = torch.randn(n, n, dtype=torch.bfloat16, device="cuda")
            fn = lambda: x @ y  # noqa: E731
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(10):
            s, e = torch.cuda.Event(True), torch.cuda.Event(True)
            s.record(); fn(); e.record(); torch.cuda.synchronize()
            best = min(best, s.elapsed_time(e))
        t0 = time.time(); cnt = 0
        s = torch.cuda.Event(True); e = torch.cuda.Event(True)
        s.record()
        while time.time() - t0 < 4.0:
            for _ in range(10):
                fn()
            cnt += 10
            if cnt % 50 == 0:
                mid = clocks()
        e.record(); torch.cuda.synchronize()
        sus = s.elapsed_time(e) / cnt
        res[name] = {"burst_tops": ops / best / 1e9, "sustained_tops": ops / sus / 1e9, "clocks_during": mid}
        print(name, res[name], flush=True)
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    json.dump(res, open(os.path.join(ROOT, "profiles", "int8_peak.json"), "w"), indent=1)


if __name__ == "__main__":
    main()

"""Host <-> device copy bandwidth from pinned memory (the e2e leg's transfer
roofline): H2D alone, D2H alone, and both at once on two streams, for the
e2e step's sizes (268 MB in, 134 MB out at 4096^2 f64)."""
import json
import torch

dev = torch.device("cuda", 0)
n_in, n_out = 2 * 4096 * 4096, 4096 * 4096
h_in = torch.empty(n_in, dtype=torch.float64).pin_memory()
h_out = torch.empty(n_out, dtype=torch.float64).pin_memory()
d_in = torch.empty(n_in, dtype=torch.float64, device=dev)
d_out = torch.empty(n_out, dtype=torch.float64, device=dev)
s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def both():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


t_h2d = timed(lambda: d_in.copy_(h_in, non_blocking=True))
t_d2h = timed(lambda: h_out.copy_(d_out, non_blocking=True))
t_both = timed(both)
print(json.dumps({"h2d_ms": t_h2d, "h2d_GBps": 8 * n_in / t_h2d / 1e6, "d2h_ms": t_d2h,
                  "d2h_GBps": 8 * n_out / t_d2h / 1e6, "both_ms": t_both,
                  "bytes_in": 8 * n_in, "bytes_out": 8 * n_out}))

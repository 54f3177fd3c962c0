"""Calibration probe: torch fill (write-only) and sum (read-only) bandwidth on
a 64 GB f64 buffer, CUDA-event timed (best of 5). Context for the build
(write-bound) and matrix-sweep (read-bound) roofline fractions."""
import json

import torch

n = 8 * 1024 ** 3  # 8 Gi doubles = 64 GiB
x = torch.empty(n, dtype=torch.float64, device="cuda")
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
res = {}
for name, fn, bytes_ in (("write_fill", lambda: x.fill_(0.5), n * 8), ("read_sum", lambda: x.sum(), n * 8),
                         ("copy_half", lambda: x[: n // 2].copy_(x[n // 2:]), n * 8)):
    best = 1e9
    for _ in range(5):
        a, b = ev(), ev()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    res[name] = {"GB/s": bytes_ / (best / 1e3) / 1e9, "ms": best}
print(json.dumps(res))

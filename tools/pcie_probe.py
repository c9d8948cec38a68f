"""PCIe floor of the e2e number: pinned H2D of the 10M inputs (160 MB xy + 640 MB int64
triangles) and D2H of the 10M output CSR (131 MB), CUDA events, best of 5."""
import json

import torch


def best(fn, k=5):
    ts = []
    for _ in range(k):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts)


h_in = torch.empty(800_000_000, dtype=torch.uint8).pin_memory()
d_in = torch.empty(800_000_000, dtype=torch.uint8, device="cuda")
h_out = torch.empty(131_500_000, dtype=torch.uint8).pin_memory()
d_out = torch.empty(131_500_000, dtype=torch.uint8, device="cuda")
t_in = best(lambda: d_in.copy_(h_in, non_blocking=True))
t_out = best(lambda: h_out.copy_(d_out, non_blocking=True))
print(json.dumps({"h2d_ms": round(t_in, 3), "h2d_gbs": round(0.8 / t_in * 1e3, 1), "d2h_ms": round(t_out, 3),
                  "d2h_gbs": round(0.1315 / t_out * 1e3, 1), "floor_ms": round(t_in + t_out, 3)}))

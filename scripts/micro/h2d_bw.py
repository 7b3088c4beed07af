"""Host link bandwidth on this box: pinned H2D / D2H copies of 1-64 MB (CUDA events)."""
import json

import torch

for mb in (1, 2, 8, 32):
    n = mb << 20
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    res = {"MB": mb}
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            fn()
        e1.record()
        torch.cuda.synchronize()
        res[name + "_GBps"] = round(n * 20 / (e0.elapsed_time(e1) * 1e-3) / 1e9, 1)
    print(json.dumps(res), flush=True)

"""Sweep pa_hbm_read_probe (bulk-copy read-only stream) configurations on one GPU and
print the best read GB/s per (chunk, stages, ctas-per-SM); 4 GiB buffer, best of 5."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2309_06180_b200 as pa  # noqa: E402

dev = torch.device("cuda", 0)
sms = torch.cuda.get_device_properties(dev).multi_processor_count
buf = torch.empty(4 << 30, dtype=torch.uint8, device=dev)
buf.fill_(1)
sink = torch.zeros(16 * sms, dtype=torch.int32, device=dev)
res = []
for chunk in (8192, 16384, 32768, 65536):
    for stages in (2, 3, 4, 6, 8, 12):
        if stages * chunk > 200 * 1024:
            continue
        for cps in (1, 2, 3, 4, 6, 8):
            if cps * (stages * chunk + 1024) > 228 * 1024:
                continue
            best = 0.0
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                pa.hbm_read_probe(buf, sink, chunk=chunk, stages=stages, ctas=cps * sms)
                e1.record()
                torch.cuda.synchronize()
                best = max(best, buf.numel() / (e0.elapsed_time(e1) * 1e-3) / 1e9)
            res.append({"chunk": chunk, "stages": stages, "ctas_per_sm": cps, "inflight_kb": cps * stages * chunk // 1024,
                        "gbs": round(best, 1)})
            print(json.dumps(res[-1]), flush=True)
res.sort(key=lambda r: -r["gbs"])
print("BEST", json.dumps(res[:5]))
x = torch.ones(2 << 30, dtype=torch.float16, device=dev)
best = 0
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); x.sum(dtype=torch.float32); e1.record(); torch.cuda.synchronize()
    best = max(best, x.numel() * 2 / (e0.elapsed_time(e1) * 1e-3) / 1e9)
print("torch sum GB/s", round(best, 1))
y = torch.empty_like(x)
best = 0
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); y.copy_(x); e1.record(); torch.cuda.synchronize()
    best = max(best, 2 * x.numel() * 2 / (e0.elapsed_time(e1) * 1e-3) / 1e9)
print("torch copy GB/s (read+write)", round(best, 1))

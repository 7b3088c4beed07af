"""Timing experiment (variant build -DPA_PREFILL_TRACE, PA_LIB_VARIANT=trace, PA_PREFILL=5):
per-tile clock64 events of the first work item of CTAs 0..63: S ready / P arrive for
both query tiles' first warp group."""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2309_06180_b200 as pa  # noqa: E402
from paper_2309_06180_b200 import _lib  # noqa: E402
from prefill_bench import build  # noqa: E402
from synth.prefill import make_prefill  # noqa: E402

c = make_prefill(sys.argv[1] if len(sys.argv) > 1 else "p_2k")
q, kc, vc, bt, cl, qs = build(c)
out = torch.empty_like(q)
for _ in range(3):
    pa.paged_prefill_attention(out, q, kc, vc, bt, cl, qs, 0.088, max_query_len=int(c["qlen"].max()))
torch.cuda.synchronize()
buf = np.zeros(64 * 256, np.int64)
f = _lib.raw().pa_debug_prefill_trace_read
f.argtypes = [ctypes.c_void_p, ctypes.c_int]
assert f(buf.ctypes.data, buf.size) == 0
t = buf.reshape(64, 256)
res = {"x0": [], "p2s0": [], "x1": [], "p2s1": [], "offset": []}
for cta in range(64):
    r = t[cta]
    for j in range(1, 30):
        s0, p0, s0n = r[2 * j], r[2 * j + 1], r[2 * j + 2]
        s1, p1, s1n = r[129 + 2 * j], r[128 + 2 * j], r[129 + 2 * j + 2]
        if s0 and p0 and s0n and s0n > p0:
            res["x0"].append(p0 - s0)
            res["p2s0"].append(s0n - p0)
        if s1 and p1 and s1n and s1n > p1:
            res["x1"].append(p1 - s1)
            res["p2s1"].append(s1n - p1)
        if s0 and s1:
            res["offset"].append(s1 - s0)
print(json.dumps({k: float(np.median(v)) if v else None for k, v in res.items()}))
print("nonzero per cta:", [(int(np.count_nonzero(t[c, :128])), int(np.count_nonzero(t[c, 128:]))) for c in range(8)])
print("cta0 first:", t[0, :8].tolist(), t[0, 128:136].tolist())
d = [(t[c, 200] - t[c, 6], t[c, 201] - t[c, 200], t[c, 202] - t[c, 201], t[c, 203] - t[c, 202], t[c, 7] - t[c, 203])
     for c in range(64) if t[c, 200] and t[c, 7]]
print("tile3 phases (ld, max+bar, emit, odone+rescale, tail):", np.median(np.array(d), axis=0).tolist() if d else None)

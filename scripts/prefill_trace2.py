"""Timing experiment (variant build -DPA_PREFILL_TRACE, PA_LIB_VARIANT=ptrace, PA_PREFILL=2):
per-tile clock64 events of the first work item of CTAs 0..63 in the v2 prefill kernel.
  softmax group t (slots t*64 + 4j + {0: S ready, 1: S loaded, 2: P emitted, 3: P arrived})
  MMA warp (128 + 4j + {0: V(j) landed, 1: PV_0(j) issued, 2: K(j+1) landed, 3: P_1(j) seen})
  TMA warp (192 + 4j + {0: K(j) issued, 1: V(j) issued})
Prints median per-tile phase lengths in SM cycles."""
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
T = buf.reshape(64, 256)
ph = {k: [] for k in ("ld0", "cmp0", "tail0", "wait0", "per0", "ld1", "cmp1", "tail1", "wait1", "per1",
                      "vfull_minus_p0", "pv0_issue_minus_p0", "kfull_wait", "p1_wait", "k_lead", "v_lead")}
for cta in range(64):
    r = T[cta]
    for j in range(2, 14):
        for t in (0, 1):
            b = t * 64 + 4 * j
            a0, a1, a2, a3, n0 = r[b], r[b + 1], r[b + 2], r[b + 3], r[b + 4]
            if a0 and a1 and a2 and a3 and n0 and n0 > a3:
                ph[f"ld{t}"].append(a1 - a0)
                ph[f"cmp{t}"].append(a2 - a1)
                ph[f"tail{t}"].append(a3 - a2)
                ph[f"wait{t}"].append(n0 - a3)
                ph[f"per{t}"].append(n0 - a0)
        m = 128 + 4 * j
        p0 = r[4 * j + 3]
        if r[m] and p0:
            ph["vfull_minus_p0"].append(r[m] - p0)  # > 0: V(j) landed after P_0(j) arrived
        if r[m + 1] and p0:
            ph["pv0_issue_minus_p0"].append(r[m + 1] - p0)
        if r[m + 2] and r[m + 1]:
            ph["kfull_wait"].append(r[m + 2] - r[m + 1])  # MMA warp blocked on K(j+1)
        if r[m + 3] and r[m + 2]:
            ph["p1_wait"].append(r[m + 3] - r[m + 2])  # ... then on P_1(j)
        if r[192 + 4 * j] and r[4 * j]:
            ph["k_lead"].append(r[128 + 4 * (j - 1) + 2] - r[192 + 4 * j])  # K(j) landed minus issued
        if r[192 + 4 * j + 1] and r[128 + 4 * j]:
            ph["v_lead"].append(r[128 + 4 * j] - r[192 + 4 * j + 1])  # V(j) landed minus V(j) issued
res = {k: (float(np.median(v)) if v else None) for k, v in ph.items()}
res["samples"] = len(ph["per0"])
print(json.dumps(res))
print("cta0 WG0 S-ready times (rel):", (T[0, 0:64:4] - T[0, 0]).tolist())
print("cta0 WG1 S-ready times (rel):", (T[0, 64:128:4] - T[0, 0]).tolist())
print("cta0 MMA V landed (rel):", (T[0, 128:192:4] - T[0, 0]).tolist())

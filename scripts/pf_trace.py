"""Per-item timeline of the packed prompt kernel (variant build with -DPA_PREFILL_TRACE):
clock64 stamps of CTAs 0..63, 14 slots per item (items 0..17 of the CTA):
softmax thread 0 -- 0 table seen, 1..5 S(j) seen (j < 5), 6 epilogue start (last P V done),
7 epilogue end; MMA thread -- 8 Q ready, 9 O free (previous epilogue done), 10..13 P(j)
released (j < 4).
  make clean && make NVXFLAGS=-DPA_PREFILL_TRACE && python scripts/pf_trace.py p_prefix5"""
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

name = sys.argv[1] if len(sys.argv) > 1 else "p_prefix5"
c = make_prefill(name)
q, kc, vc, bt, cl, qs = build(c)
out = torch.empty_like(q)
ws = torch.empty(16, dtype=torch.uint8, device="cuda")
hqs = np.concatenate([[0], np.cumsum(c["qlen"])]).astype(np.int32)
for _ in range(3):
    pa.paged_prefill_attention_packed(out, q, kc, vc, bt, cl, qs, 1.0 / np.sqrt(128), hqs,
                                      c["ctx"].astype(np.int32), c["shared"].astype(np.int32),
                                      max_query_len=int(c["qlen"].max()), workspace=ws)
torch.cuda.synchronize()
buf = np.zeros(64 * 256, np.int64)
L = _lib.raw()
L.pa_debug_prefill_trace_read.restype = ctypes.c_int
assert L.pa_debug_prefill_trace_read(buf.ctypes.data, 64 * 256) == 0
tr = buf.reshape(64, 256)[:, :18 * 14].reshape(64, 18, 14).astype(np.float64)
tr[tr == 0] = np.nan
base = np.nanmin(tr[:, 0, :], axis=1)
rel = tr - base[:, None, None]
d = lambda a, b: float(np.nanmedian(rel[:, 1:16, b] - rel[:, 1:16, a]))  # noqa: E731
period = np.nanmedian(np.diff(rel[:, :17, 0], axis=1))
print(json.dumps({
    "config": name, "item_period_cyc": float(period),
    "table_to_S0": d(0, 1), "S0_to_S1": d(1, 2), "S1_to_S2": d(2, 3), "S2_to_S3": d(3, 4),
    "S0_to_P0": d(1, 10), "P0_to_P1": d(10, 11), "P1_to_P2": d(11, 12), "P2_to_P3": d(12, 13),
    "lastP_to_epi": float(np.nanmedian(rel[:, 1:16, 6] - np.nanmax(rel[:, 1:16, 10:14], axis=2))),
    "epilogue": d(6, 7), "epi_end_to_next_table": float(np.nanmedian(rel[:, 2:17, 0] - rel[:, 1:16, 7])),
    "q_ready_to_o_free": d(8, 9), "o_free_to_P0": d(9, 10)}))
for i in range(6):
    print(i, [int(v) if v == v else -1 for v in rel[0, i]])

"""Per-tile timeline of the tcgen05 grouped decode (variant build with -DPA_TC_TRACE):
clock64 stamps of CTAs 0..7 for every tile -- producer acquired/published (0/1), MMA saw
the tile (2) and issued its P V (3), softmax warp 0 saw S (4), wrote P (5), released P (6).
  make clean && make NVXFLAGS=-DPA_TC_TRACE && python scripts/tc_trace.py c5_beam 4"""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2309_06180_b200 as pa  # noqa: E402
from paper_2309_06180_b200 import _lib  # noqa: E402
from synth import make_config, materialize_torch, tables_torch  # noqa: E402

name, gs = (sys.argv[1] if len(sys.argv) > 1 else "c5_beam"), int(sys.argv[2]) if len(sys.argv) > 2 else 4
wl = make_config(name)
# bench.py's conditions: the traced launch reads a cache no recent launch touched (cold L2)
R = int(os.environ.get("TC_TRACE_CACHES", "1"))
xs = [materialize_torch(wl, "cuda") for _ in range(R)]
x = xs[0]
tb = tables_torch(wl, "cuda")
out = torch.empty_like(x["query"])
plan = pa.decode_plan(wl.context_lens)  # bench.py's longest-first order
for _ in range(3):
    pa.paged_attention_decode_grouped(out, x["query"], x["key"], x["value"], x["key_cache"], x["value_cache"],
                                      tb["block_tables"], tb["context_lens"], wl.scale, gs,
                                      max_context_len=wl.max_context_len, seq_order=plan)
for y in xs[1:]:  # evict x's cache from L2 (each copy > L2 / R)
    pa.paged_attention_decode_grouped(out, y["query"], y["key"], y["value"], y["key_cache"], y["value_cache"],
                                      tb["block_tables"], tb["context_lens"], wl.scale, gs,
                                      max_context_len=wl.max_context_len, seq_order=plan)
torch.cuda.synchronize()
L = _lib.raw()
L.pa_debug_tc_trace_reset.restype = ctypes.c_int
assert L.pa_debug_tc_trace_reset() == 0
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
pa.paged_attention_decode_grouped(out, x["query"], x["key"], x["value"], x["key_cache"], x["value_cache"],
                                  tb["block_tables"], tb["context_lens"], wl.scale, gs,
                                  max_context_len=wl.max_context_len, seq_order=plan)
e1.record()
torch.cuda.synchronize()
span = np.zeros(1024 * 8, np.uint64)
L.pa_debug_tc_span.restype = ctypes.c_int
assert L.pa_debug_tc_span(span.ctypes.data, span.nbytes) == 0
sp = span.reshape(1024, 8).astype(np.int64)
sp = sp[sp[:, 0] > 0]
t0 = sp[:, 0].min()
print(json.dumps({"launch_event_us": e0.elapsed_time(e1) * 1e3, "ctas": len(sp),
                  "entry_us_max": float((sp[:, 0].max() - t0) / 1e3),
                  "pdl_wait_us_max": float((sp[:, 1] - sp[:, 0]).max() / 1e3),
                  "exit_us": [float(np.percentile(sp[:, 2] - t0, q) / 1e3) for q in (0, 10, 50, 90, 100)],
                  "items_per_cta": [int(np.percentile(sp[:, 3], q)) for q in (0, 50, 100)],
                  "tiles_per_cta": [int(np.percentile(sp[:, 4], q)) for q in (0, 10, 50, 90, 100)],
                  "first_tile_published_us": [float(np.percentile(sp[:, 5] - t0, q) / 1e3) for q in (0, 50, 100)],
                  "kernel_entry_us": [float(np.percentile(sp[:, 6] - t0, q) / 1e3) for q in (0, 50, 100)],
                  "prologue_done_us": [float(np.percentile(sp[:, 1] - t0, q) / 1e3) for q in (0, 50, 100)],
                  "first_list_published_us": [float(np.percentile(sp[:, 7] - t0, q) / 1e3) for q in (0, 50, 100)],
                  "exit_us_vs_tiles": [[int(a), float((b - t0) / 1e3)] for a, b in
                                       sorted(zip(sp[:, 4], sp[:, 2]))[:: max(1, len(sp) // 12)]]}))
NT = 1024
buf = np.zeros(8 * NT * 8, np.int64)
L.pa_debug_tc_trace.restype = ctypes.c_int
assert L.pa_debug_tc_trace(buf.ctypes.data, buf.nbytes) == 0
tr = buf.reshape(8, NT, 8)
res = {}
for c in range(8):
    t = tr[c]
    n = int((t[:, 2] > 0).sum())
    ns = int((t[:, 4] > 0).sum())
    d = lambda a, b, m: np.median(t[:m, b] - t[:m, a]) if m > 1 else None  # noqa: E731
    per = np.diff(t[:n, 2])
    res[c] = {"tiles": n, "s_tiles": ns,
              "span_us": float((t[n - 1, 2] - t[0, 2]) / 1.9e3) if n > 1 else None,
              "tile_period_cyc_med": float(np.median(per)) if n > 2 else None,
              "prod_issue_cyc_med(0->1)": float(d(0, 1, n)),
              "publish_to_mma_cyc_med(1->2)": float(d(1, 2, n)),
              "s_seen_to_P_cyc_med(4->5)": float(d(4, 5, ns)),
              "P_to_release_cyc_med(5->6)": float(d(5, 6, ns)),
              "release_to_pv_cyc_med(6->3)": float(d(6, 3, ns)),
              "s_seen_period_cyc_med": float(np.median(np.diff(t[:ns, 4]))) if ns > 2 else None,
              "s_issue_cyc_med(2->7)": float(d(2, 7, n))}
    print(json.dumps({"cta": c, **res[c]}))
# first 40 tiles of CTA 0, cycles relative to the first stamp
t0 = tr[0][tr[0] > 0].min()
for i in range(40):
    print(i, [int(v - t0) if v > 0 else -1 for v in tr[0, i, :8]])
# epilogue stamps of the softmax warps (items 0..63 of CTAs 0..7): start, o_last seen, O
# stored + o_free, job published; relative to the tile trace's first stamp
ep = np.zeros(8 * 64 * 8, np.int64)
L.pa_debug_tc_ep.restype = ctypes.c_int
assert L.pa_debug_tc_ep(ep.ctypes.data, ep.nbytes) == 0
ep = ep.reshape(8, 64, 8)
d01, d12, d23, d14 = [], [], [], []
for c in range(8):
    for it in range(64):
        e = ep[c, it]
        if (e[:5] > 0).all():
            d01.append(e[1] - e[0]); d12.append(e[2] - e[1]); d23.append(e[3] - e[2]); d14.append(e[4] - e[1])
print(json.dumps({"epilogue_items": len(d01), "wait_o_last_cyc_med": float(np.median(d01)) if d01 else None,
                  "o_store_cyc_med": float(np.median(d12)) if d12 else None,
                  "split_publish_cyc_med": float(np.median(d23)) if d23 else None,
                  "o_tmem_ld_cyc_med": float(np.median(d14)) if d14 else None}))
for it in range(6):
    print("ep", it, [int(v - t0) if v > 0 else -1 for v in ep[0, it, :5]])
# where CTA 0..7's time goes: per-tile MMA-saw periods, excess over the median period
gaps = []
for c in range(8):
    t = tr[c]
    n = int((t[:, 2] > 0).sum())
    per = np.diff(t[:n, 2])
    med = np.median(per)
    ex = per - med
    top = np.argsort(-ex)[:8]
    gaps.append({"cta": c, "tiles": n, "span_cyc": int(t[n - 1, 2] - t[0, 2]), "median": float(med),
                 "excess_total": int(ex[ex > 0].sum()), "excess_over_2x": int(ex[per > 2 * med].sum()),
                 "top": [(int(i), int(per[i])) for i in top]})
for g in gaps:
    print(json.dumps(g))

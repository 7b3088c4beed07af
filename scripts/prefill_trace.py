"""Timing experiment: clock64 event trace of the prefill kernel (pa_debug_prefill_trace).

Needs the trace build: scripts/build_variant.sh trace -DPA_PREFILL_TRACE, then run with
PA_LIB_VARIANT=trace."""
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


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "p_2k"
    c = make_prefill(cfg)
    q, kc, vc, bt, cl, qs = build(c)
    out = torch.empty_like(q)
    mql = int(c["qlen"].max())
    for _ in range(3):
        pa.paged_prefill_attention(out, q, kc, vc, bt, cl, qs, 0.088, max_query_len=mql)
    ctas = 40000
    buf = torch.zeros((ctas, 64), dtype=torch.int64, device="cuda")
    _lib.raw().pa_debug_prefill_trace(ctypes.c_void_p(buf.data_ptr()), ctas)
    pa.paged_prefill_attention(out, q, kc, vc, bt, cl, qs, 0.088, max_query_len=mql)
    torch.cuda.synchronize()
    _lib.raw().pa_debug_prefill_trace(None, 0)
    t = buf.cpu().numpy()
    t = t[t[:, 0] != 0]
    n = t[:, 53]
    res = {"config": cfg, "ctas": int(len(t))}
    res["setup"] = float(np.median(t[:, 1] - t[:, 0]))
    res["q_wait"] = float(np.median(t[:, 2] - t[:, 1]))
    res["first_S"] = float(np.median(t[:, 19] - t[:, 1]))
    per_tile, smx, wait_s = [], [], []
    for r in t:
        k = int(min(r[53], 16))
        for j in range(k):
            smx.append(r[35 + j] - r[19 + j])
            if j + 1 < k:
                per_tile.append(r[19 + j + 1] - r[19 + j])
                wait_s.append(r[19 + j + 1] - r[35 + j])
    res["tile_period_med"] = float(np.median(per_tile)) if per_tile else None
    res["softmax_med"] = float(np.median(smx))
    res["p_to_next_S_med"] = float(np.median(wait_s)) if wait_s else None
    sel = t[t[:, 53] >= 4]
    if len(sel):
        res["t2_ldS"] = float(np.median(sel[:, 55] - sel[:, 21]))
        res["t2_max"] = float(np.median(sel[:, 56] - sel[:, 55]))
        res["t2_emit"] = float(np.median(sel[:, 57] - sel[:, 56]))
        res["t2_rescale"] = float(np.median(sel[:, 58] - sel[:, 57]))
        res["t2_tail"] = float(np.median(sel[:, 37] - sel[:, 58]))
    res["epilogue"] = float(np.median(t[:, 52] - t[:, 51]))
    res["cta_total_med"] = float(np.median(t[:, 52] - t[:, 0]))
    res["tiles_mean"] = float(n.mean())
    # per SM: busy fraction = sum of CTA spans / (last end - first start)
    busy = []
    for sm in np.unique(t[:, 54]):
        rr = t[t[:, 54] == sm]
        span = rr[:, 52].max() - rr[:, 0].min()
        busy.append((rr[:, 52] - rr[:, 0]).sum() / span)
    res["sm_busy_frac_med"] = float(np.median(busy))
    res["sm_span_cycles_med"] = float(np.median([t[t[:, 54] == sm][:, 52].max() - t[t[:, 54] == sm][:, 0].min()
                                                 for sm in np.unique(t[:, 54])]))
    print(json.dumps(res))


if __name__ == "__main__":
    main()

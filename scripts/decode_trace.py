"""Timing experiment (variant build -DPA_DECODE_TRACE, PA_LIB_VARIANT=dtrace): per-CTA
globaltimer events of the coop decode kernel (start after griddepcontrol.wait, first
stage full, end) -> concurrency / bandwidth timeline, CTA lifetimes, head and tail.
  PA_LIB_VARIANT=dtrace python scripts/decode_trace.py c2_alpaca c2_sharegpt"""
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


def main():
    f = _lib.raw().pa_debug_decode_trace_read
    f.argtypes = [ctypes.c_void_p, ctypes.c_int]
    for name in sys.argv[1:] or ["c2_alpaca"]:
        wl = make_config(name)
        x = materialize_torch(wl, "cuda")
        tb = tables_torch(wl, "cuda")
        out = torch.empty_like(x["query"])
        ws = torch.zeros(max(16, pa.paged_attention_workspace_size(wl.S, wl.H, wl.D, wl.max_context_len)),
                         dtype=torch.uint8, device="cuda")
        for _ in range(5):
            pa.paged_attention_decode(out, x["query"], x["key"], x["value"], x["key_cache"], x["value_cache"],
                                      tb["block_tables"], tb["context_lens"], wl.scale,
                                      max_context_len=wl.max_context_len, workspace=ws)
        torch.cuda.synchronize()
        n = 1 << 17
        buf = np.zeros(n * 4, np.uint64)
        assert f(buf.ctypes.data, buf.size) == 0
        t = buf.reshape(n, 4).astype(np.int64)
        live = (t[:, 0] > 0) & (t[:, 2] >= t[:, 0])
        last = t[live, 2].max()
        # every launch of the same grid rewrites the same rows: keep the last launch's
        # (rows of an earlier, larger grid are older than 5 ms)
        live &= t[:, 0] > last - 5_000_000
        T0 = t[live, 0].min()
        tt = t[live]
        t0, t1, t2 = tt[:, 0] - T0, tt[:, 1] - T0, tt[:, 2] - T0
        sm = tt[:, 3] & 0xFFFF
        nt = (tt[:, 3] >> 16) & 0xFFFF
        span = t2.max()
        tile_bytes = 2 * min(4, wl.H) * 16 * wl.D * (4 if wl.dtype == "f32" else 2)
        life = t2 - t0
        lat = np.where(t1 >= t0, t1 - t0, 0)
        step = 1000
        bins = np.arange(0, span + step, step)
        act = np.array([((t0 <= b) & (t2 > b)).sum() for b in bins])
        gbs = np.zeros(len(bins))
        for a, b_, nb in zip(t1, t2, nt):
            if b_ <= a or nb == 0:
                continue
            rate = nb * tile_bytes / (b_ - a)  # bytes per ns, spread over [first data, end]
            for i in range(int(a // step), min(int(b_ // step) + 1, len(bins))):
                lo, hi = max(a, i * step), min(b_, (i + 1) * step)
                if hi > lo:
                    gbs[i] += rate * (hi - lo) / step
        cmax = act.max()
        full_from = int(np.argmax(act >= 0.9 * cmax))
        tail_from = len(act) - 1 - int(np.argmax(act[::-1] >= 0.9 * cmax))
        res = {"config": name, "ctas": int(live.sum()), "span_us": round(span / 1e3, 2), "last_end": int(last - T0),
               "sms": int(len(np.unique(sm))), "max_concurrent": int(cmax),
               "ramp_us_to_90pct": full_from, "tail_us_below_90pct": len(act) - 1 - tail_from,
               "life_us_mean": round(life.mean() / 1e3, 2), "life_us_p50": round(np.median(life) / 1e3, 2),
               "life_us_max": round(life.max() / 1e3, 2),
               "first_data_us_mean": round(lat.mean() / 1e3, 2),
               "first_data_us_p90": round(np.percentile(lat, 90) / 1e3, 2),
               "tiles_mean": round(float(nt.mean()), 2), "tiles_max": int(nt.max()),
               "bytes_GB": round(nt.sum() * tile_bytes / 1e9, 4),
               "avg_GBps_over_span": round(nt.sum() * tile_bytes / span, 1),
               "timeline_1us_active": act.tolist(), "timeline_1us_GBps": [round(g) for g in gbs.tolist()]}
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()

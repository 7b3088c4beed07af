"""Kernel-level ablations of the default decode: attention
launch time and algorithmic GB/s of pa_paged_attention_decode under
  * block size B in {1, 8, 16, 32}            (Fig.18b analogue)
  * sorted vs shuffled physical placement     (Fig.18a analogue: block-table indirection)
  * grid order: generator order vs longest-first sequences (tail effect; scheduling only)
Each case: R layer caches rotated (R x K/V per launch >= 4 x L2), 300 timed launches
after 10 warm-up, CUDA events around every launch; prints one JSON line per case.
  python scripts/ablate.py [block_size|placement|order] [config ...]
"""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2309_06180_b200 as pa  # noqa: E402
from synth import make_config, materialize_torch, subset, tables_torch  # noqa: E402


def time_decode(wl, iters=300, warm=10):
    dev = torch.device("cuda", 0)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    kv = wl.logical_kv_bytes()
    R = min(8, max(2, math.ceil(4 * l2 / kv)))
    tb = tables_torch(wl, dev)
    layers = [materialize_torch(wl, dev, layer=r) for r in range(R)]
    out = torch.empty_like(layers[0]["query"])
    ws = torch.zeros(max(16, pa.paged_attention_workspace_size(wl.S, wl.H, wl.D, wl.max_context_len, 0)),
                     dtype=torch.uint8, device=dev)
    calls = [pa.prepare(pa.paged_attention_decode, out, L["query"], L["key"], L["value"], L["key_cache"],
                        L["value_cache"], tb["block_tables"], tb["context_lens"], wl.scale,
                        max_context_len=wl.max_context_len, workspace=ws) for L in layers]
    for i in range(warm):
        calls[i % R]()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
    torch.cuda.synchronize()
    torch.cuda._sleep(20_000_000)
    for i in range(iters):
        ev[i][0].record()
        calls[i % R]()
        ev[i][1].record()
    torch.cuda.synchronize()
    t = np.array([a.elapsed_time(b) for a, b in ev]) * 1e3
    sb = wl.step_bytes()
    byts = sb["kv_logical"] + sb["q_out"] + sb["tables"] + sb["cache_write"] // 2
    del layers
    return {"us_mean": round(float(t.mean()), 2), "us_p10": round(float(np.percentile(t, 10)), 2),
            "us_p50": round(float(np.percentile(t, 50)), 2), "us_p90": round(float(np.percentile(t, 90)), 2),
            "gbs": round(byts / (t.mean() * 1e-6) / 1e9, 1), "alg_bytes": byts, "layers": R}


def main():
    mode = sys.argv[1] if len(sys.argv) > 1 else "block_size"
    names = sys.argv[2:] or ["c2_sharegpt", "c2_alpaca"]
    for name in names:
        if mode == "block_size":
            for B in (1, 8, 16, 32):
                wl = make_config(name, B=B)
                print(json.dumps({"mode": mode, "config": name, "B": B, **time_decode(wl)}), flush=True)
        elif mode == "placement":
            for pl in ("shuffled", "sorted", "shuffled", "sorted"):
                wl = make_config(name, placement=pl)
                print(json.dumps({"mode": mode, "config": name, "placement": pl, **time_decode(wl)}), flush=True)
        elif mode == "order":
            wl = make_config(name)
            lf = subset(wl, np.argsort(-wl.context_lens.astype(np.int64), kind="stable"))
            for tag, w in (("generator", wl), ("longest_first", lf), ("generator", wl), ("longest_first", lf)):
                print(json.dumps({"mode": mode, "config": name, "order": tag, **time_decode(w)}), flush=True)
        else:
            raise SystemExit(f"unknown mode {mode}")
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

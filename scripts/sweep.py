"""Launch-shape sweep for pa_paged_attention (tuning only; not a bench line).

For each config: materialise once, then time the attention call alone with CUDA events
for every (PA_HPC, PA_STG, partition_tokens) setting.  Prints one JSON per setting.
  python scripts/sweep.py c2_sharegpt c2_alpaca c4_long
"""
import itertools
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2309_06180_b200 as pa  # noqa: E402
from synth import make_config, materialize_torch, tables_torch  # noqa: E402

SHAPES = [(4, 3), (4, 2), (4, 4), (2, 4), (2, 6), (8, 2), (8, 3), (1, 8), (1, 4)]
PTS = [256, 512, 1024]
if os.environ.get("SWEEP_SHAPES"):
    SHAPES = [tuple(int(v) for v in x.split(",")) for x in os.environ["SWEEP_SHAPES"].split(";")]
if os.environ.get("SWEEP_PTS"):
    PTS = [int(x) for x in os.environ["SWEEP_PTS"].split(",")]


def main():
    for name in sys.argv[1:] or ["c2_sharegpt"]:
        wl = make_config(name)
        x = materialize_torch(wl, "cuda")
        tb = tables_torch(wl, "cuda")
        out = torch.empty_like(x["query"])
        kv = wl.logical_kv_bytes()
        for (hpc, stg), pt in itertools.product(SHAPES, PTS):
            os.environ["PA_HPC"], os.environ["PA_STG"] = str(hpc), str(stg)
            ws = torch.zeros(max(16, pa.paged_attention_workspace_size(wl.S, wl.H, wl.D, wl.max_context_len, pt)),
                             dtype=torch.uint8, device="cuda")

            def call():
                pa.paged_attention(out, x["query"], x["key_cache"], x["value_cache"], tb["block_tables"],
                                   tb["context_lens"], wl.scale, max_context_len=wl.max_context_len,
                                   partition_tokens=pt, workspace=ws)
            try:
                for _ in range(5):
                    call()
                torch.cuda.synchronize()
            except Exception as e:  # unsupported shape (smem)
                print(json.dumps({"config": name, "hpc": hpc, "stg": stg, "pt": pt, "error": str(e)[:120]}))
                continue
            n = 50
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(n):
                call()
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) / n * 1e3
            print(json.dumps({"config": name, "hpc": hpc, "stg": stg, "pt": pt, "us": round(us, 2),
                              "kv_GBps": round(kv / us / 1e3, 1)}), flush=True)
        os.environ.pop("PA_HPC", None)
        os.environ.pop("PA_STG", None)
        del x


if __name__ == "__main__":
    main()

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

# (scheduler, warps per CTA, stages per warp, heads per warp)
SHAPES = [("grid", 4, 2, 1), ("grid", 4, 2, 2), ("grid", 4, 2, 5), ("grid", 4, 3, 2), ("grid", 2, 2, 2),
          ("persistent", 4, 2, 1)]
PTS = [512]
if os.environ.get("SWEEP_SHAPES"):
    SHAPES = []
    for x in os.environ["SWEEP_SHAPES"].split(";"):
        f = x.split(",")
        SHAPES.append((f[0], int(f[1]), int(f[2]), int(f[3])))
if os.environ.get("SWEEP_PTS"):
    PTS = [int(x) for x in os.environ["SWEEP_PTS"].split(",")]


def main():
    for name in sys.argv[1:] or ["c2_sharegpt"]:
        wl = make_config(name)
        x = materialize_torch(wl, "cuda")
        tb = tables_torch(wl, "cuda")
        out = torch.empty_like(x["query"])
        kv = wl.logical_kv_bytes()
        for (sched, hpc, stg, hpw), pt in itertools.product(SHAPES, PTS):
            os.environ["PA_SCHED"] = "coop" if sched.startswith("shared") else sched
            os.environ["PA_HPC"], os.environ["PA_STG"] = str(hpc), str(stg)
            os.environ["PA_HPW"] = str(hpw)
            os.environ["PA_PPC"] = str(hpw)  # 4th field doubles as coop partitions-per-CTA
            if sched.startswith("shared"):  # sharedG: heads per CTA and block slots per stage
                os.environ["PA_SHARED_HPC"], os.environ["PA_SHARED_SLOTS"] = str(hpc), str(hpw)
            ws = torch.zeros(max(16, pa.paged_attention_workspace_size(wl.S, wl.H, wl.D, wl.max_context_len, pt)),
                             dtype=torch.uint8, device="cuda")

            def call():
                if sched.startswith("shared"):  # sharing-aware entry, group size in the name
                    pa.paged_attention_decode_shared(out, x["query"], x["key"], x["value"], x["key_cache"],
                                                     x["value_cache"], tb["block_tables"], tb["context_lens"],
                                                     wl.scale, int(sched[6:] or 4),
                                                     max_context_len=wl.max_context_len, workspace=ws)
                elif os.environ.get("SWEEP_PTS"):  # explicit partition size: unfused entry
                    pa.paged_attention(out, x["query"], x["key_cache"], x["value_cache"], tb["block_tables"],
                                       tb["context_lens"], wl.scale, max_context_len=wl.max_context_len,
                                       partition_tokens=pt, workspace=ws)
                else:
                    pa.paged_attention_decode(out, x["query"], x["key"], x["value"], x["key_cache"],
                                              x["value_cache"], tb["block_tables"], tb["context_lens"], wl.scale,
                                              max_context_len=wl.max_context_len, workspace=ws)
            try:
                for _ in range(5):
                    call()
                torch.cuda.synchronize()
            except Exception as e:  # unsupported shape (smem)
                print(json.dumps({"config": name, "sched": sched, "hpc": hpc, "stg": stg, "hpw": hpw, "pt": pt,
                                  "error": str(e)[:120]}))
                continue
            n = 50
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(n):
                call()
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) / n * 1e3
            print(json.dumps({"config": name, "sched": sched, "hpc": hpc, "stg": stg, "hpw": hpw, "pt": pt,
                              "us": round(us, 2),
                              "kv_GBps": round(kv / us / 1e3, 1)}), flush=True)
        for k in ("PA_HPC", "PA_STG", "PA_HPW", "PA_SCHED", "PA_PPC", "PA_SHARED_HPC", "PA_SHARED_SLOTS"):
            os.environ.pop(k, None)
        del x


if __name__ == "__main__":
    main()

"""Tiny sharing-aware decode steps (pa_paged_attention_decode_shared, N1 stage stream) for
compute-sanitizer: beam groups with shared and diverged blocks, a split context, block
sizes 16 / 32 / 8, one and several slots per stage."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2309_06180_b200 as pa  # noqa: E402
from synth import make_config, materialize_torch, tables_torch  # noqa: E402

for slots in ("1", "2"):
    os.environ["PA_SHARED_SLOTS"] = slots
    pa.reload_tuning()
    for name, over, gs in (("c5_beam", dict(S=8, H=4, H_kv=4), 4), ("c5_beam", dict(S=6, H=2, H_kv=2, B=32), 3),
                           ("c3_fork", dict(S=12, H=2, H_kv=2, B=8), 6), ("c4_long", dict(S=4, H=2, H_kv=2), 2)):
        wl = make_config(name, **over)
        x = materialize_torch(wl, "cuda")
        tb = tables_torch(wl, "cuda")
        if len(wl.block_mapping):
            pa.copy_blocks([x["key_cache"]], [x["value_cache"]], tb["block_mapping"])
        out = torch.empty_like(x["query"])
        pa.paged_attention_decode_shared(out, x["query"], x["key"], x["value"], x["key_cache"], x["value_cache"],
                                         tb["block_tables"], tb["context_lens"], wl.scale, gs,
                                         max_context_len=wl.max_context_len)
torch.cuda.synchronize()
print("sanitize shared workload done")

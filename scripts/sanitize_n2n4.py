"""Small prefill (both kernels) and fused-TP steps for compute-sanitizer."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2309_06180_b200 as pa  # noqa: E402
from paper_2309_06180_b200.tp import FusedTP  # noqa: E402
from synth import make_config, materialize_torch, shard, tables_torch  # noqa: E402
from tests.test_gpu_prefill import prefill_problem  # noqa: E402

for v in ("2", "3"):
    os.environ["PA_PREFILL"] = v
    pa.reload_tuning()
    for B in (1, 16):
        q, kc, vc, bt, cl, qs = prefill_problem([300, 5, 130, 64], [140, 5, 2, 64], B, 4, 2, "bf16")
        out = torch.empty_like(q)
        pa.paged_prefill_attention(out, q, kc, vc, bt, cl, qs, 0.1)
torch.cuda.synchronize()
os.environ.pop("PA_PREFILL")
pa.reload_tuning()
wl = make_config("c2_sharegpt", S=6, H=4, H_kv=4)
ranks = FusedTP.local_group(2, wl.S, wl.H, wl.D, torch.float16)
streams = [torch.cuda.Stream() for _ in range(2)]
ins = []
for r in range(2):
    sh = shard(wl, r, 2)
    ins.append((sh, materialize_torch(sh, "cuda"), tables_torch(sh, "cuda")))
torch.cuda.synchronize()
for r in range(2):
    sh, x, tb = ins[r]
    with torch.cuda.stream(streams[r]):
        ranks[r].decode(x["query"], x["key"], x["value"], x["key_cache"], x["value_cache"], tb["block_tables"],
                        tb["context_lens"], sh.scale, max_context_len=sh.max_context_len)
torch.cuda.synchronize()
print("status", [int(rk.status.item()) for rk in ranks])
for rk in ranks:
    rk.close()
print("sanitize n2/n4 workload done")

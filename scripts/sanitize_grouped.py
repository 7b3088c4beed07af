"""Small grouped (N1 tensor-core) decode steps for compute-sanitizer: beams (shared
blocks), unrelated sequences, split contexts, multi-stage tiles (1 slot per stage)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2309_06180_b200 as pa  # noqa: E402

from synth import make_config  # noqa: E402
from tests.test_gpu_grouped import grouped_step  # noqa: E402

for slots in ("2", "1"):
    os.environ["PA_GROUP_SLOTS"] = slots
    pa.reload_tuning()
    for name, over, gs in (("c5_beam", dict(S=8, H=2, H_kv=2), 4), ("c3_fork", dict(S=12, H=2, H_kv=2), 6),
                           ("c4_long", dict(S=4, H=2, H_kv=2), 2)):
        out, _ = grouped_step(make_config(name, **over), gs)
        assert not torch.isnan(out).any()
torch.cuda.synchronize()
print("sanitize grouped workload done")

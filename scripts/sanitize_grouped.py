"""Small grouped (N1, tcgen05) decode steps for compute-sanitizer: beams (shared pieces),
parallel samples at the fork step (CoW'd last blocks), unrelated sequences, long contexts,
GQA, block size 32 and a ragged head quad (H % 4 != 0)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from synth import make_config  # noqa: E402
from tests.test_gpu_grouped import grouped_step  # noqa: E402

for name, over, gs in (("c5_beam", dict(S=8, H=4, H_kv=4), 4), ("c3_fork", dict(S=12, H=4, H_kv=4), 6),
                       ("c4_long", dict(S=4, H=4, H_kv=4), 2), ("c5_beam", dict(S=8, H=4, H_kv=2), 4),
                       ("c5_beam", dict(S=8, H=2, H_kv=2, B=32), 4), ("c2_sharegpt", dict(S=6, H=6, H_kv=6), 3)):
    out, _ = grouped_step(make_config(name, **over), gs)
    assert not torch.isnan(out).any()
torch.cuda.synchronize()
print("sanitize grouped workload done")

"""Tiny decode steps for compute-sanitizer (memcheck / racecheck / synccheck): the coop
kernel with 1 and 2 partitions per CTA, fused and unfused paths, copy_blocks, block sizes
1 and 16, a split context."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from synth import make_config  # noqa: E402
from tests.pathutil import gpu_step  # noqa: E402

import paper_2309_06180_b200 as pa  # noqa: E402

for ppc in sys.argv[1:] or ["1", "2"]:
    os.environ["PA_PPC"] = ppc
    pa.reload_tuning()
    for name, over in (("c1_tiny", {}), ("c3_fork", dict(S=12, H=4, H_kv=4)),
                       ("explicit", dict(ctx=[0, 1, 17, 600], H=4, H_kv=4, D=128, B=1, dtype="f16", seed=3))):
        wl = make_config(name, **over)
        gpu_step(wl)
        gpu_step(wl, fused=True)
torch.cuda.synchronize()
print("sanitize workload done")

"""Fig.19 analogue: swap bandwidth vs block size, GPU <-> pinned CPU pool.

For each block size the same 512 MiB of KV (OPT-13B shape: 40 kv heads, D=128, fp16, one
layer, K+V) moves GPU->CPU (swap-out) and CPU->GPU (swap-in), either as ONE pa_swap_blocks
launch (GPU threads read/write mapped host memory) or as one cudaMemcpyAsync per block
(pa_swap_blocks_memcpy, what per-block swapping costs).  Prints one JSON line per point.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2309_06180_b200 as pa  # noqa: E402

H_KV, D = 40, 128
TOTAL = 512 << 20  # bytes of K+V moved per call


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best * 1e-3


def main():
    for B in (1, 2, 4, 8, 16, 32, 64, 128, 256):
        blk = H_KV * B * D * 2
        nblocks = TOTAL // (2 * blk)
        gk = torch.randn((nblocks, H_KV, B, D), device="cuda", dtype=torch.float16)
        gv = torch.randn_like(gk)
        ck = torch.empty((nblocks, H_KV, B, D), dtype=torch.float16).pin_memory()
        cv = torch.empty_like(ck).pin_memory()
        perm = np.random.default_rng(B).permutation(nblocks)
        mp = np.stack([np.arange(nblocks), perm], 1).astype(np.int64)
        mdev, mhost = torch.from_numpy(mp).cuda(), torch.from_numpy(mp)
        res = {"block_size": B, "block_bytes_per_kv": blk, "blocks": int(nblocks), "bytes": TOTAL}
        res["out_kernel_GBps"] = TOTAL / timed(lambda: pa.swap_blocks([ck], [cv], [gk], [gv], mdev)) / 1e9
        res["in_kernel_GBps"] = TOTAL / timed(lambda: pa.swap_blocks([gk], [gv], [ck], [cv], mdev)) / 1e9
        reps = 2 if nblocks > 20000 else 5
        res["out_memcpy_GBps"] = TOTAL / timed(lambda: pa.swap_blocks_memcpy([ck], [cv], [gk], [gv], mhost),
                                                reps) / 1e9
        res["in_memcpy_GBps"] = TOTAL / timed(lambda: pa.swap_blocks_memcpy([gk], [gv], [ck], [cv], mhost),
                                               reps) / 1e9
        print(json.dumps({k: (round(v, 2) if isinstance(v, float) else v) for k, v in res.items()}), flush=True)
        del gk, gv, ck, cv


if __name__ == "__main__":
    main()

"""Tensor-parallel head sharding of the decode attention.

Megatron-style SPMD: rank r of P owns the contiguous query heads [r*H/P, (r+1)*H/P)
and the matching kv heads; every rank holds the same block tables, context lengths and
slot mapping (the paper's single KV cache manager) and its own
[NB][H_kv/P][B][D] caches.  The only exchange is an all-gather of the per-rank output
head slices (BJ:north_star), NCCL over NVLink on B200s; any torch.distributed backend
works (gloo in the CPU tests).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def head_range(num_heads: int, world: int, rank: int):
    """[first, last) query heads of `rank` (contiguous, Megatron convention, reading c14)."""
    if num_heads % world:
        raise ValueError(f"{num_heads} heads do not split over {world} ranks")
    h = num_heads // world
    return rank * h, (rank + 1) * h


def gather_heads(out_local: torch.Tensor, group=None, buffer: torch.Tensor | None = None) -> torch.Tensor:
    """All-gather [S][H/P][D] head slices into the full [S][H][D] output.

    One all_gather_into_tensor into a [P*S][H/P][D] buffer (rank-major), then a permute;
    rank order equals head order because ranks own contiguous head ranges."""
    world = dist.get_world_size(group)
    S, h, D = out_local.shape
    if buffer is None:
        buffer = torch.empty((world * S, h, D), dtype=out_local.dtype, device=out_local.device)
    dist.all_gather_into_tensor(buffer, out_local.contiguous(), group=group)
    return buffer.view(world, S, h, D).permute(1, 0, 2, 3).reshape(S, world * h, D)

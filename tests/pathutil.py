"""Test helpers: run one decode step through the CUDA path (C ABI via the torch binding)
and through the fp64 oracle on the same generated inputs.  The two share only the
input generator (synth)."""
from __future__ import annotations

import numpy as np

TOL = {"f32": 1e-5, "f16": 2e-3, "bf16": 1e-2}  # BJ:north_star max-abs tolerances


def bits(t) -> np.ndarray:
    """Raw storage bits of a torch tensor (any device) as numpy uint16/uint32."""
    import torch
    t = t.detach().contiguous().cpu()
    if t.dtype == torch.float32:
        return t.view(torch.int32).numpy().view(np.uint32)
    return t.view(torch.int16).numpy().view(np.uint16)


def as_f64(t) -> np.ndarray:
    import torch
    return t.detach().to(torch.float64).cpu().numpy()


def gpu_step(wl, device="cuda", partition_tokens=0, inputs=None, run_copy=True, run_write=True, fused=False):
    """copy_blocks -> reshape_and_cache -> paged_attention on the device (fused=True:
    copy_blocks -> paged_attention_decode, the cache write inside the attention kernel).
    Returns (out, key_cache, value_cache, inputs)."""
    import torch

    import paper_2309_06180_b200 as pa
    from synth import materialize_torch, tables_torch
    x = inputs or materialize_torch(wl, device)
    tb = tables_torch(wl, device)
    kc, vc = x["key_cache"], x["value_cache"]
    if run_copy and len(wl.block_mapping):
        pa.copy_blocks([kc], [vc], tb["block_mapping"])
    out = torch.empty_like(x["query"])
    if fused:
        pa.paged_attention_decode(out, x["query"], x["key"], x["value"], kc, vc, tb["block_tables"],
                                  tb["context_lens"], wl.scale, max_context_len=wl.max_context_len)
        torch.cuda.synchronize()
        return out, kc, vc, x
    if run_write:
        pa.reshape_and_cache(x["key"], x["value"], kc, vc, tb["slot_mapping"])
    pa.paged_attention(out, x["query"], kc, vc, tb["block_tables"], tb["context_lens"], wl.scale,
                       max_context_len=wl.max_context_len, partition_tokens=partition_tokens)
    torch.cuda.synchronize()
    return out, kc, vc, x


def oracle_step(wl, run_copy=True, run_write=True):
    """The same step in the fp64 oracle.  Returns (out fp64, key_cache bits, value_cache bits)."""
    import oracle
    from synth import materialize_numpy
    n = materialize_numpy(wl)
    kc, vc = n["key_cache"], n["value_cache"]
    if run_copy and len(wl.block_mapping):
        kcs, vcs = oracle.copy_blocks([kc], [vc], wl.block_mapping, wl.dtype)
        kc, vc = kcs[0], vcs[0]
    if run_write:
        kc, vc = oracle.reshape_and_cache(n["key"], n["value"], kc, vc, wl.slot_mapping, wl.B, wl.dtype)
    out = oracle.paged_attention(n["query"], kc, vc, wl.block_tables, wl.context_lens, wl.scale, wl.B, wl.H_kv,
                                 wl.dtype)
    return out, kc, vc


def max_abs(gpu_out, ref) -> float:
    g = as_f64(gpu_out)
    assert not np.isnan(g).any(), "NaN in GPU output (poisoned slot read?)"
    return float(np.max(np.abs(g - ref))) if ref.size else 0.0

"""Seeded synthetic workloads for the multi-token (prompt-phase) path, SURVEY §8(f) N4.

No arithmetic of the method lives here -- only lengths and block placement, shared by the
tests and scripts/prefill_bench.py.

Configurations (reading c23):
  p_sharegpt  whole prompts of a ShareGPT-length trace (P:536-540 length mix, the LogNormal
              fit of synth.workload) until the batch holds >= 8192 query tokens;
              LLaMA-13B attention shape H = H_kv = 40, D = 128, f16, B = 16.
  p_2k        8 prompts of 2048 tokens (the model's maximum context), same shape.
  p_chunk256  chunked prefill: 64 prompts whose next 256 tokens are computed after 768
              already cached ones (a 1024-token prompt in four chunks).
  p_prefix1 / p_prefix5
              the shared-prefix translation workload of P:604-618: a cached prefix of 80
              (one-shot) / 341 (five-shot) tokens reserved once, 256 requests whose
              user-specific suffix (a WMT16 sentence, LogNormal mean 30 tokens, sigma 0.5 --
              the paper gives no length statistics) is the only prompt-phase work.
"""
from __future__ import annotations

import numpy as np

from . import rng as R
from .workload import request_pool, _lognormal

PREFILL_CONFIGS = {
    "p_sharegpt": dict(kind="trace", mix="sharegpt", tokens=8192, H=40, H_kv=40, B=16, dtype="f16", seed=1101),
    "p_2k": dict(kind="uniform", n=8, length=2048, H=40, H_kv=40, B=16, dtype="f16", seed=1102),
    "p_prefix1": dict(kind="prefix", prefix=80, n=256, H=40, H_kv=40, B=16, dtype="f16", seed=1103),
    "p_prefix5": dict(kind="prefix", prefix=341, n=256, H=40, H_kv=40, B=16, dtype="f16", seed=1104),
    "p_chunk256": dict(kind="chunk", n=64, chunk=256, done=768, H=40, H_kv=40, B=16, dtype="f16", seed=1105),
}


def make_prefill(name: str, **over) -> dict:
    """Returns dict(ctx, qlen, block_tables, num_blocks, H, H_kv, B, dtype, seed, name);
    keyword arguments override configuration fields (e.g. B=128)."""
    c = dict(PREFILL_CONFIGS[name])
    c.update(over)
    B = c["B"]
    if c["kind"] == "trace":
        prompt, _ = request_pool(c["seed"], c["mix"])
        n = int(np.searchsorted(np.cumsum(prompt), c["tokens"]) + 1)
        ctx = prompt[:n].astype(np.int64)
        qlen = ctx.copy()
    elif c["kind"] == "chunk":  # chunked prefill: the next `chunk` prompt tokens after `done` cached ones
        ctx = np.full(c["n"], c["done"] + c["chunk"], np.int64)
        qlen = np.full(c["n"], c["chunk"], np.int64)
    elif c["kind"] == "uniform":
        ctx = np.full(c["n"], c["length"], np.int64)
        qlen = ctx.copy()
    else:
        k = R.key(c["seed"], R.STREAM_LEN)
        suf = np.clip(np.rint(_lognormal(k, np.arange(c["n"], dtype=np.int64), 30.0, 0.5)), 1, 512).astype(np.int64)
        ctx = c["prefix"] + suf
        qlen = suf
    S = len(ctx)
    nb = (ctx + B - 1) // B
    W = int(nb.max())
    bt = np.full((S, W), -1, np.int32)
    if c["kind"] == "prefix":
        # full prefix blocks are shared physical blocks; the partial last prefix block is
        # copied per request (copy-on-write) and the suffix follows in private blocks
        full = c["prefix"] // B
        nid = full
        for s in range(S):
            bt[s, :full] = np.arange(full)
            bt[s, full:nb[s]] = np.arange(nid, nid + nb[s] - full)
            nid += nb[s] - full
        NB = nid
    else:
        NB = int(nb.sum())
        ids = np.argsort(R.bits_np(R.key(c["seed"], R.STREAM_PERM), np.arange(NB, dtype=np.int64)), kind="stable")
        off = 0
        for s in range(S):
            bt[s, :nb[s]] = ids[off:off + nb[s]]
            off += nb[s]
    # per sequence: leading cached tokens shared (same physical blocks) with the previous
    # sequence -- the host-side hint of pa_paged_prefill_attention_packed
    shared = np.zeros(S, np.int64)
    if c["kind"] == "prefix" and S > 1:
        shared[1:] = (c["prefix"] // B) * B
    c.update(name=name, ctx=ctx, qlen=qlen, block_tables=bt, num_blocks=NB, shared=shared)
    return c


def algorithmic_flops(ctx: np.ndarray, qlen: np.ndarray, H: int, D: int) -> int:
    """4*D flops (q.k and p*v, 2 each per dim) per (query row, head, attended token);
    query row i of a sequence attends to ctx - qlen + i + 1 tokens (causal)."""
    tot = 0
    for c, q in zip(ctx.tolist(), qlen.tolist()):
        base = c - q
        # sum_{i<q} (base + i + 1)
        tot += q * (base + 1) + q * (q - 1) // 2
    return 4 * D * H * tot

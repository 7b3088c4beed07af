"""Seeded synthetic decode-step workloads with the shapes of the paper's experiments.

Holds NO arithmetic of the method.  It decides *which* tokens exist and *where* they
live (context lengths, block tables, slot mapping, copy-on-write pairs) and draws the
values of q, the new k/v and the cached K/V from the counter-based streams of
``synth.rng``.  Both the oracle side (numpy, raw bits) and the CUDA side (torch
tensors on the device) materialise inputs from here; neither computes them from the
other.

Shapes (BJ:configs):
  c1_tiny       4 seqs, 2 heads, D 64, B 16, fp32, ctx U{1..100}, shuffled pool x2
  c2_sharegpt   OPT-13B: 256 seqs, 40 heads, D 128, B 16, fp16, ShareGPT-like ctx
  c2_alpaca     same, Alpaca-like ctx
  c3_parallel   LLaMA-13B: 42 requests x n=6 samples sharing prompt blocks, bf16
  c3_fork       the same at the fork step (first append -> copy-on-write pairs)
  c4_sharegpt   OPT-66B: 256 seqs, 72 heads, ShareGPT-like ctx
  c4_long       OPT-66B: ctx U{1024..2048}
  c5_beam       OPT-175B: 64 requests x beam width 4, random-survivor beam tree, 96 heads

Length model: LogNormal prompt/output lengths whose means
keep the ShareGPT/Alpaca ratios of P:511 (8.4x inputs, 5.8x outputs), clipped to the
2048-token OPT limit; a decode snapshot picks requests with probability
proportional to their output length and a uniform generated count g < output.
Physical blocks come from a seeded shuffled free list (Fig.7).
"""
from __future__ import annotations

import math
from collections import deque
from dataclasses import dataclass, field, replace

import numpy as np

from . import rng as R

MAX_LEN = 2048

LENGTH_MIXES = {
    # name: (prompt mean, prompt sigma, output mean, output sigma)
    "sharegpt": (161.3, 1.0, 338.0, 0.8),
    "alpaca": (19.3, 0.5, 58.5, 0.7),
}


@dataclass
class Workload:
    name: str
    seed: int
    S: int
    H: int
    H_kv: int
    D: int
    B: int
    dtype: str
    scale: float
    context_lens: np.ndarray   # int32 [S]
    block_tables: np.ndarray   # int32 [S][W], -1 padded
    num_blocks: int
    slot_mapping: np.ndarray   # int64 [S]: slot of each sequence's current token (-1: none)
    block_mapping: np.ndarray  # int64 [P][2]: copy-on-write (src, dst) pairs of this step
    live: np.ndarray           # bool [NB][B]: slot holds a previous token's K/V before the step
    seq_origin: np.ndarray = None    # int64 [S]: sequence index in the parent workload
    block_origin: np.ndarray = None  # int64 [NB]: physical block id in the parent workload
    H_glob: int = 0
    Hkv_glob: int = 0
    q_head0: int = 0
    kv_head0: int = 0
    meta: dict = field(default_factory=dict)

    def __post_init__(self):
        if self.seq_origin is None:
            self.seq_origin = np.arange(self.S, dtype=np.int64)
        if self.block_origin is None:
            self.block_origin = np.arange(self.num_blocks, dtype=np.int64)
        if not self.H_glob:
            self.H_glob = self.H
        if not self.Hkv_glob:
            self.Hkv_glob = self.H_kv

    # ------------------------------------------------------------- derived sizes ---
    @property
    def W(self) -> int:
        return int(self.block_tables.shape[1])

    @property
    def elem_bytes(self) -> int:
        return R.ELEM_BYTES[self.dtype]

    @property
    def max_context_len(self) -> int:
        return int(self.context_lens.max()) if self.S else 0

    def logical_kv_bytes(self) -> int:
        """K+V bytes attention must read: sum_s ctx_s * H_kv * D * 2 * e."""
        return int(self.context_lens.astype(np.int64).sum()) * self.H_kv * self.D * 2 * self.elem_bytes

    def unique_kv_bytes(self) -> int:
        """K+V bytes of distinct physical (block, slot)s read by at least one sequence."""
        read = np.zeros((self.num_blocks, self.B), dtype=bool)
        for s in range(self.S):
            n = int(self.context_lens[s])
            if n <= 0:
                continue
            t = np.arange(n)
            read[self.block_tables[s, t // self.B], t % self.B] = True
        return int(read.sum()) * self.H_kv * self.D * 2 * self.elem_bytes

    def step_bytes(self) -> dict:
        """Algorithmic bytes of one decode step (one layer), per SURVEY §8(d)."""
        e = self.elem_bytes
        qo = 2 * self.S * self.H * self.D * e
        nblk = int(np.ceil(self.context_lens / self.B).sum())
        cache_write = 2 * 2 * int((self.slot_mapping >= 0).sum()) * self.H_kv * self.D * e
        cow = 2 * 2 * len(self.block_mapping) * self.H_kv * self.B * self.D * e
        return {"kv_logical": self.logical_kv_bytes(), "q_out": qo, "tables": 4 * nblk + 4 * self.S,
                "cache_write": cache_write, "copy_blocks": cow}

    def cache_shape(self):
        return (self.num_blocks, self.H_kv, self.B, self.D)


# ------------------------------------------------------------------ lengths --------

def _lognormal(k: int, idx: np.ndarray, mean: float, sigma: float) -> np.ndarray:
    u1 = 1.0 - R.uniform01_np(k, 2 * idx)
    u2 = R.uniform01_np(k, 2 * idx + 1)
    z = np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)
    mu = math.log(mean) - 0.5 * sigma * sigma
    return np.exp(mu + sigma * z)


def request_pool(seed: int, mix: str, n: int = 8192):
    """(prompt_len, output_len) int64 arrays of a synthetic request trace."""
    pm, ps, om, osd = LENGTH_MIXES[mix]
    k = R.key(seed, R.STREAM_LEN)
    idx = np.arange(n, dtype=np.int64)
    prompt = np.clip(np.rint(_lognormal(k, idx, pm, ps)), 1, MAX_LEN - 1).astype(np.int64)
    out = np.rint(_lognormal(k, idx + n, om, osd)).astype(np.int64)
    out = np.clip(out, 1, MAX_LEN - prompt)
    return prompt, out


def decode_snapshot(seed: int, mix: str, num: int):
    """Pick `num` requests in a decode iteration: probability proportional to output
    length (a request is present in that many iterations), g ~ U{0..out-1};
    returns (prompt, g, ctx = prompt + g + 1)."""
    prompt, out = request_pool(seed, mix)
    cum = np.cumsum(out).astype(np.float64)
    kp = R.key(seed, R.STREAM_PICK)
    u = R.uniform01_np(kp, np.arange(num, dtype=np.int64)) * cum[-1]
    pick = np.minimum(np.searchsorted(cum, u, side="right"), len(out) - 1)
    g = np.floor(R.uniform01_np(kp, np.arange(num, 2 * num, dtype=np.int64)) * out[pick]).astype(np.int64)
    g = np.minimum(g, out[pick] - 1)
    p = prompt[pick]
    return p, g, p + g + 1


def _perm(seed: int, n: int) -> np.ndarray:
    return np.argsort(R.bits_np(R.key(seed, R.STREAM_PERM), np.arange(n, dtype=np.int64)), kind="stable")


# ------------------------------------------------------------------ placement ------

def place_private(ctx: np.ndarray, B: int, seed: int, pool_factor: float = 1.1, min_extra: int = 0,
                  placement: str = "shuffled"):
    """Every sequence owns its blocks (no sharing).  Returns tables, NB, slot_mapping,
    live mask.  Blocks come from a shuffled pool of ceil(pool_factor * needed) ids
    (placement="sorted": ids handed out in order, each sequence's blocks consecutive --
    the contiguous-cache ablation, SURVEY §8(d) "Block placement")."""
    S = len(ctx)
    nb = (ctx + B - 1) // B
    need = int(nb.sum())
    NB = max(1, int(math.ceil(pool_factor * need)) + min_extra)
    if placement not in ("shuffled", "sorted"):
        raise ValueError(f"placement must be 'shuffled' or 'sorted' (got {placement!r})")
    perm = _perm(seed, NB) if placement == "shuffled" else np.arange(NB)
    W = max(1, int(nb.max()) if S else 1)
    bt = np.full((S, W), -1, dtype=np.int32)
    live = np.zeros((NB, B), dtype=bool)
    slots = np.full(S, -1, dtype=np.int64)
    off = 0
    for s in range(S):
        ids = perm[off: off + nb[s]]
        off += nb[s]
        bt[s, : nb[s]] = ids
        n = int(ctx[s])
        if n > 0:
            t = np.arange(n - 1)
            live[ids[t // B], t % B] = True
            slots[s] = int(ids[(n - 1) // B]) * B + (n - 1) % B
    return bt, NB, slots, live


class _Pool:
    """Fixture builder only: FIFO free list + refcounts + fork/append/free, enough to
    lay out shared prompt blocks and beam trees.  (The product allocator is pa_alloc_*;
    the oracle allocator is oracle/block_manager.py.)"""

    def __init__(self, order, B):
        self.fl = deque(int(b) for b in order)
        self.ref = np.zeros(len(order), dtype=np.int64)
        self.B = B
        self.t = {}
        self.n = 0

    def _pop(self):
        b = self.fl.popleft()
        self.ref[b] = 1
        return b

    def allocate(self, n):
        e, left = [], n
        while left > 0:
            f = min(self.B, left)
            e.append([self._pop(), f])
            left -= f
        h = self.n; self.n += 1
        self.t[h] = e
        return h

    def fork(self, h):
        e = [[b, f] for b, f in self.t[h]]
        for b, _ in e:
            self.ref[b] += 1
        c = self.n; self.n += 1
        self.t[c] = e
        return c

    def free(self, h):
        for b, _ in self.t.pop(h):
            self.ref[b] -= 1
            if self.ref[b] == 0:
                self.fl.append(b)

    def append(self, h):
        e = self.t[h]
        last = e[-1]
        if last[1] == self.B:
            b = self._pop()
            e.append([b, 1])
            return b * self.B, None
        b, f = last
        if self.ref[b] == 1:
            last[1] += 1
            return b * self.B + f, None
        d = self._pop()
        self.ref[b] -= 1
        last[0] = d
        last[1] += 1
        return d * self.B + f, (b, d)

    def live_mask(self, NB):
        live = np.zeros((NB, self.B), dtype=bool)
        for e in self.t.values():
            for b, f in e:
                live[b, :f] = True
        return live


def _export(pool, handles, B, W=None):
    rows = [[b for b, _ in pool.t[h]] for h in handles]
    ctx = np.array([sum(f for _, f in pool.t[h]) for h in handles], dtype=np.int32)
    W = W or max(len(r) for r in rows)
    bt = np.full((len(rows), W), -1, dtype=np.int32)
    for i, r in enumerate(rows):
        bt[i, : len(r)] = r
    return bt, ctx


def place_parallel_sampling(p, g, n, B, seed, fork_step: bool):
    """n samples per request fork the prompt.  Steady state: g >= 1 earlier
    appends already resolved copy-on-write; fork step: the timed append is the first,
    so every sample but the last copies the shared partial prompt block."""
    R_ = len(p)
    need = 0
    for r in range(R_):
        ctx = int(p[r] + g[r] + 1)
        need += p[r] // B + n * ((ctx + B - 1) // B - p[r] // B) + n
    NB = int(math.ceil(1.1 * need)) + 8
    pool = _Pool(_perm(seed, NB), B)
    seqs = []
    for r in range(R_):
        root = pool.allocate(int(p[r]))
        kids = [root] + [pool.fork(root) for _ in range(n - 1)]
        steps = 0 if fork_step else int(g[r])
        for _ in range(steps):
            for h in kids:
                pool.append(h)
        seqs.append(kids)
    live = pool.live_mask(NB)
    slots, pairs, handles = [], [], []
    for kids in seqs:
        for h in kids:
            s, cow = pool.append(h)
            slots.append(s)
            if cow is not None:
                pairs.append(cow)
            handles.append(h)
    bt, ctx = _export(pool, handles, B)
    return bt, ctx, NB, np.array(slots, np.int64), np.array(pairs, np.int64).reshape(-1, 2), live


def place_beam_search(p, g, k, B, seed, stickiness: float = 0.0):
    """Beam width k: each step draws k parents (with replacement) among the
    current candidates, forks them, frees the old candidates and appends one token.
    The last step is the timed one: its copy-on-write pairs form block_mapping."""
    R_ = len(p)
    need = sum(k * ((int(p[r] + g[r] + 1) + B - 1) // B + 1) for r in range(R_))
    NB = int(math.ceil(1.1 * need)) + 8
    pool = _Pool(_perm(seed, NB), B)
    kb = R.key(seed, R.STREAM_BEAM)
    beams = []
    for r in range(R_):
        root = pool.allocate(int(p[r]))
        cur = [pool.fork(root) for _ in range(k)]
        pool.free(root)
        for h in cur:
            pool.append(h)  # first generated token (g >= 0 more follow)
        beams.append(cur)

    def step(r, it):
        cur = beams[r]
        base = (r * (MAX_LEN + 2) + it) * k
        u = R.uniform01_np(kb, np.arange(base * 2, base * 2 + 2 * k, dtype=np.int64))
        parents = []
        for j in range(k):
            if u[2 * j] < stickiness:
                parents.append(cur[j])
            else:
                parents.append(cur[min(int(u[2 * j + 1] * k), k - 1)])
        new = [pool.fork(h) for h in parents]
        for h in cur:
            pool.free(h)
        beams[r] = new
        return new

    for r in range(R_):
        for it in range(int(g[r])):
            for h in step(r, it):
                pool.append(h)
    live = pool.live_mask(NB)
    slots, pairs, handles = [], [], []
    for r in range(R_):
        for h in step(r, int(g[r])):
            s, cow = pool.append(h)
            slots.append(s)
            if cow is not None:
                pairs.append(cow)
            handles.append(h)
    bt, ctx = _export(pool, handles, B)
    return bt, ctx, NB, np.array(slots, np.int64), np.array(pairs, np.int64).reshape(-1, 2), live


# ------------------------------------------------------------------ configs --------

CONFIGS = {
    # name: (seed, S or (requests, n), H, H_kv, D, B, dtype, kind, mix)
    "c1_tiny": dict(seed=1000, S=4, H=2, H_kv=2, D=64, B=16, dtype="f32", kind="uniform100"),
    "c2_sharegpt": dict(seed=1001, S=256, H=40, H_kv=40, D=128, B=16, dtype="f16", kind="snapshot", mix="sharegpt"),
    "c2_alpaca": dict(seed=1001, S=256, H=40, H_kv=40, D=128, B=16, dtype="f16", kind="snapshot", mix="alpaca"),
    "c3_parallel": dict(seed=1002, S=252, H=40, H_kv=40, D=128, B=16, dtype="bf16", kind="parallel", mix="sharegpt", n=6),
    "c3_fork": dict(seed=1002, S=252, H=40, H_kv=40, D=128, B=16, dtype="bf16", kind="parallel_fork", mix="sharegpt", n=6),
    "c4_sharegpt": dict(seed=1003, S=256, H=72, H_kv=72, D=128, B=16, dtype="f16", kind="snapshot", mix="sharegpt"),
    "c4_long": dict(seed=1003, S=256, H=72, H_kv=72, D=128, B=16, dtype="f16", kind="long"),
    "c5_beam": dict(seed=1004, S=256, H=96, H_kv=96, D=128, B=16, dtype="f16", kind="beam", mix="sharegpt", n=4),
}


def make_config(name: str, **over) -> Workload:
    """Build a named config; keyword overrides: seed, S, H, H_kv, D, B, dtype, mix,
    n, stickiness, ctx (explicit context lengths for 'explicit' kind), placement
    ('shuffled' default / 'sorted', private-block kinds only)."""
    c = dict(CONFIGS[name]) if name in CONFIGS else dict(kind="explicit", seed=0)
    c.update({k: v for k, v in over.items() if v is not None})
    seed, B, D, H, H_kv, dtype = c["seed"], c["B"], c["D"], c["H"], c["H_kv"], c["dtype"]
    kind = c["kind"]
    S = c.get("S")
    pairs = np.zeros((0, 2), np.int64)
    meta = {"kind": kind}
    if kind in ("uniform100", "snapshot", "long", "explicit"):
        if kind == "uniform100":
            ctx = 1 + np.floor(R.uniform01_np(R.key(seed, R.STREAM_MISC), np.arange(S)) * 100).astype(np.int64)
            pool_factor = 2.0
        elif kind == "snapshot":
            _, _, ctx = decode_snapshot(seed, c["mix"], S)
            pool_factor = 1.1
            meta["mix"] = c["mix"]
        elif kind == "long":
            ctx = 1024 + np.floor(R.uniform01_np(R.key(seed, R.STREAM_MISC), np.arange(S)) * 1025).astype(np.int64)
            pool_factor = 1.1
        else:
            ctx = np.asarray(c["ctx"], dtype=np.int64)
            S = len(ctx)
            pool_factor = c.get("pool_factor", 2.0)
        bt, NB, slots, live = place_private(ctx, B, seed, pool_factor, c.get("min_extra", 1),
                                            c.get("placement", "shuffled"))
        meta["placement"] = c.get("placement", "shuffled")
        ctx = ctx.astype(np.int32)
    elif kind in ("parallel", "parallel_fork"):
        n = c["n"]
        nreq = S // n
        p, g, _ = decode_snapshot(seed, c["mix"], nreq)
        if kind == "parallel":
            g = np.maximum(g, 1)
        bt, ctx, NB, slots, pairs, live = place_parallel_sampling(p, g, n, B, seed, kind == "parallel_fork")
        S = len(ctx)
        meta.update(n=n, requests=nreq)
    elif kind == "beam":
        n = c["n"]
        nreq = S // n
        p, g, _ = decode_snapshot(seed, c["mix"], nreq)
        g = np.minimum(g, MAX_LEN - 2 - p)
        bt, ctx, NB, slots, pairs, live = place_beam_search(p, np.maximum(g, 0), n, B, seed, c.get("stickiness", 0.0))
        S = len(ctx)
        meta.update(k=n, requests=nreq)
    else:
        raise ValueError(kind)
    scale = c.get("scale", 1.0 / math.sqrt(D))
    return Workload(name=name, seed=seed, S=S, H=H, H_kv=H_kv, D=D, B=B, dtype=dtype, scale=scale,
                    context_lens=ctx, block_tables=bt, num_blocks=NB, slot_mapping=slots,
                    block_mapping=pairs, live=live, meta=meta)


# ------------------------------------------------------------------ views ----------

def subset(wl: Workload, seqs) -> Workload:
    """The same values restricted to a few sequences, on a compact block pool: for
    oracle checks of sampled outputs at full size.  Values are drawn at the original
    counters (seq_origin / block_origin), so they equal the full workload's."""
    seqs = np.asarray(seqs, dtype=np.int64)
    bt = wl.block_tables[seqs]
    ctx = wl.context_lens[seqs]
    used = set()
    for i in range(len(seqs)):
        nb = (int(ctx[i]) + wl.B - 1) // wl.B
        used.update(int(b) for b in bt[i, :nb])
    slots = wl.slot_mapping[seqs]
    pairs = [tuple(pq) for pq in wl.block_mapping.tolist() if pq[1] in used]
    for s_, _ in pairs:
        used.add(int(s_))
    blocks = np.array(sorted(used), dtype=np.int64)
    remap = {int(b): i for i, b in enumerate(blocks)}
    nbt = np.full(bt.shape, -1, dtype=np.int32)
    for i in range(len(seqs)):
        nb = (int(ctx[i]) + wl.B - 1) // wl.B
        nbt[i, :nb] = [remap[int(b)] for b in bt[i, :nb]]
    nslots = np.array([remap[int(s) // wl.B] * wl.B + int(s) % wl.B if s >= 0 else -1 for s in slots], np.int64)
    npairs = np.array([(remap[a], remap[b]) for a, b in pairs], np.int64).reshape(-1, 2)
    return replace(wl, S=len(seqs), context_lens=ctx.copy(), block_tables=nbt, num_blocks=max(1, len(blocks)),
                   slot_mapping=nslots, block_mapping=npairs,
                   live=wl.live[blocks] if len(blocks) else np.zeros((1, wl.B), bool),
                   seq_origin=wl.seq_origin[seqs], block_origin=wl.block_origin[blocks] if len(blocks) else
                   np.zeros(1, np.int64), meta=dict(wl.meta, subset=True))


def shard(wl: Workload, rank: int, world: int) -> Workload:
    """Tensor-parallel head shard: rank r owns query heads
    [r*H/P, (r+1)*H/P) and kv heads [r*H_kv/P, ...); block tables are shared."""
    if wl.H % world or wl.H_kv % world:
        raise ValueError("heads must divide the world size")
    h, hk = wl.H // world, wl.H_kv // world
    return replace(wl, H=h, H_kv=hk, q_head0=wl.q_head0 + rank * h, kv_head0=wl.kv_head0 + rank * hk,
                   meta=dict(wl.meta, rank=rank, world=world))


# ------------------------------------------------------------------ values ---------

def _q_index(wl, s_idx, h_idx, d_idx):
    return (wl.seq_origin[s_idx] * wl.H_glob + wl.q_head0 + h_idx) * wl.D + d_idx


def _new_index(wl, s_idx, h_idx, d_idx):
    return (wl.seq_origin[s_idx] * wl.Hkv_glob + wl.kv_head0 + h_idx) * wl.D + d_idx


def materialize_numpy(wl: Workload, layer: int = 0, poison: bool = True) -> dict:
    """Raw-bit numpy arrays: query [S][H][D], key/value [S][H_kv][D] (this step's new
    token), key_cache/value_cache [NB][H_kv][B][D] (live slots drawn, others NaN)."""
    S, H, Hk, D, B = wl.S, wl.H, wl.H_kv, wl.D, wl.B
    s, h, d = np.meshgrid(np.arange(S), np.arange(H), np.arange(D), indexing="ij")
    q = R.f32_to_bits_np(R.uniform_f32_np(R.key(wl.seed, R.STREAM_Q, layer), _q_index(wl, s, h, d)), wl.dtype)
    s, h, d = np.meshgrid(np.arange(S), np.arange(Hk), np.arange(D), indexing="ij")
    idx = _new_index(wl, s, h, d)
    kn = R.f32_to_bits_np(R.uniform_f32_np(R.key(wl.seed, R.STREAM_KNEW, layer), idx), wl.dtype)
    vn = R.f32_to_bits_np(R.uniform_f32_np(R.key(wl.seed, R.STREAM_VNEW, layer), idx), wl.dtype)
    b, h, o, d = np.meshgrid(np.arange(wl.num_blocks), np.arange(Hk), np.arange(B), np.arange(D), indexing="ij")
    cidx = ((wl.block_origin[b] * wl.Hkv_glob + wl.kv_head0 + h) * B + o) * D + d
    out = {"query": q.reshape(S, H, D), "key": kn.reshape(S, Hk, D), "value": vn.reshape(S, Hk, D)}
    mask = wl.live[:, None, :, None] if poison else np.ones((1, 1, 1, 1), bool)
    nan = R.NAN_BITS[wl.dtype]
    for nm, st in (("key_cache", R.STREAM_KCACHE), ("value_cache", R.STREAM_VCACHE)):
        v = R.f32_to_bits_np(R.uniform_f32_np(R.key(wl.seed, st, layer), cidx), wl.dtype).reshape(cidx.shape)
        out[nm] = np.where(mask, v, v.dtype.type(nan)).astype(v.dtype)
    return out


def materialize_torch(wl: Workload, device, layer: int = 0, poison: bool = True,
                      chunk_blocks: int = 4096) -> dict:
    """Same values as materialize_numpy, generated by torch on `device`, as tensors of
    the storage dtype (the CUDA path's inputs)."""
    import torch
    S, H, Hk, D, B = wl.S, wl.H, wl.H_kv, wl.D, wl.B
    dev = torch.device(device)
    so = torch.as_tensor(wl.seq_origin, device=dev)

    def qlike(nheads, stream, hglob, h0):
        s = torch.arange(S, device=dev).view(S, 1, 1)
        h = torch.arange(nheads, device=dev).view(1, nheads, 1)
        d = torch.arange(D, device=dev).view(1, 1, D)
        idx = (so.view(S, 1, 1) * hglob + h0 + h) * D + d
        del s
        return R.f32_to_dtype_t(R.uniform_f32_t(R.key(wl.seed, stream, layer), idx), wl.dtype).contiguous()

    out = {"query": qlike(H, R.STREAM_Q, wl.H_glob, wl.q_head0),
           "key": qlike(Hk, R.STREAM_KNEW, wl.Hkv_glob, wl.kv_head0),
           "value": qlike(Hk, R.STREAM_VNEW, wl.Hkv_glob, wl.kv_head0)}
    tdt = R.torch_dtype(wl.dtype)
    bo = torch.as_tensor(wl.block_origin, device=dev)
    live = torch.as_tensor(wl.live, device=dev)
    nan_val = torch.tensor(float("nan"), dtype=tdt, device=dev)
    for nm, st in (("key_cache", R.STREAM_KCACHE), ("value_cache", R.STREAM_VCACHE)):
        cache = torch.empty(wl.cache_shape(), dtype=tdt, device=dev)
        k = R.key(wl.seed, st, layer)
        h = torch.arange(Hk, device=dev).view(1, Hk, 1, 1)
        o = torch.arange(B, device=dev).view(1, 1, B, 1)
        d = torch.arange(D, device=dev).view(1, 1, 1, D)
        for b0 in range(0, wl.num_blocks, chunk_blocks):
            b1 = min(wl.num_blocks, b0 + chunk_blocks)
            idx = ((bo[b0:b1].view(-1, 1, 1, 1) * wl.Hkv_glob + wl.kv_head0 + h) * B + o) * D + d
            v = R.f32_to_dtype_t(R.uniform_f32_t(k, idx), wl.dtype)
            if poison:
                v = torch.where(live[b0:b1].view(-1, 1, B, 1), v, nan_val)
            cache[b0:b1] = v
        out[nm] = cache
    return out


def tables_torch(wl: Workload, device) -> dict:
    import torch
    dev = torch.device(device)
    return {"block_tables": torch.as_tensor(wl.block_tables, device=dev).contiguous(),
            "context_lens": torch.as_tensor(wl.context_lens, device=dev).contiguous(),
            "slot_mapping": torch.as_tensor(wl.slot_mapping, device=dev).contiguous(),
            "block_mapping": torch.as_tensor(wl.block_mapping.reshape(-1, 2), device=dev).contiguous()}

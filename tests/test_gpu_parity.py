"""GPU parity: the CUDA path (libpagedattn.so through its C ABI) against the fp64 oracle
on identical generated inputs, plus the invariants BJ:north_star names.

Bars: cache writes, copy_blocks and block-table indexing bit-exact; attention max-abs
<= 1e-5 (fp32), 2e-3 (fp16), 1e-2 (bf16).  P:N = PAPER.md line N.
"""
import numpy as np
import pytest
import torch

import oracle
from synth import make_config, materialize_numpy, materialize_torch, shard, subset, tables_torch
from synth import rng as R
from synth.workload import place_private
from tests.pathutil import TOL, as_f64, bits, gpu_step, max_abs, oracle_step

pytestmark = pytest.mark.gpu
pa = pytest.importorskip("paper_2309_06180_b200")

SMALL = {
    "c1_tiny": {},
    "c2_sharegpt": dict(S=24, H=4, H_kv=4),
    "c2_alpaca": dict(S=40, H=4, H_kv=4),
    "c3_parallel": dict(S=24, H=2, H_kv=2),
    "c3_fork": dict(S=24, H=2, H_kv=2),
    "c4_sharegpt": dict(S=16, H=3, H_kv=3),
    "c4_long": dict(S=8, H=2, H_kv=2),
    "c5_beam": dict(S=16, H=2, H_kv=2),
}


def test_device_inputs_equal_oracle_inputs():
    wl = make_config("c3_fork", S=12, H=2, H_kv=2)
    n = materialize_numpy(wl)
    t = materialize_torch(wl, "cuda")
    for k in n:
        assert np.array_equal(n[k], bits(t[k])), k


@pytest.mark.parametrize("name", list(SMALL))
def test_step_parity_small(name):
    """copy_blocks + reshape_and_cache bitwise over the WHOLE cache (untouched slots
    included); attention within tolerance; no NaN from poisoned slots."""
    wl = make_config(name, **SMALL[name])
    out, kc, vc, _ = gpu_step(wl)
    ref, rkc, rvc = oracle_step(wl)
    assert np.array_equal(bits(kc), rkc) and np.array_equal(bits(vc), rvc)
    err = max_abs(out, ref)
    assert err <= TOL[wl.dtype], f"{name}: max-abs {err}"


@pytest.mark.parametrize("pt", [16, 32, 128, 512, 4096])
def test_partition_sizes(pt):
    wl = make_config("c2_sharegpt", S=24, H=4, H_kv=4)
    out, *_ = gpu_step(wl, partition_tokens=pt)
    ref, *_ = oracle_step(wl)
    assert max_abs(out, ref) <= TOL[wl.dtype]


def test_split_vs_single_pass():
    """Sequences with one partition are bitwise identical under any partition size;
    split ones agree within tolerance with the single-pass kernel."""
    wl = make_config("c2_sharegpt", S=32, H=4, H_kv=4)
    x = materialize_torch(wl, "cuda")
    a, *_ = gpu_step(wl, partition_tokens=512, inputs={k: v.clone() for k, v in x.items()})
    b, *_ = gpu_step(wl, partition_tokens=4096, inputs={k: v.clone() for k, v in x.items()})
    short = wl.context_lens <= 512
    assert short.any() and (~short).any()
    assert torch.equal(a[torch.as_tensor(short)], b[torch.as_tensor(short)])
    assert float((a.double() - b.double()).abs().max()) <= TOL[wl.dtype]


def test_determinism_bitwise():
    wl = make_config("c4_long", S=8, H=4, H_kv=4)
    x = materialize_torch(wl, "cuda")
    a, *_ = gpu_step(wl, inputs={k: v.clone() for k, v in x.items()})
    b, *_ = gpu_step(wl, inputs={k: v.clone() for k, v in x.items()})
    assert torch.equal(a, b)


# ------------------------------------------------ logical caches: B and placement ----

def logical_problem(ctx, B, place_seed, H, H_kv, D, dtype, seed=77):
    """The same LOGICAL q, K, V (drawn per (seq, head, token, dim)) placed into a
    [NB][H_kv][B][D] cache with block size B on shuffled blocks (test-side placement)."""
    ctx = np.asarray(ctx, np.int64)
    bt, NB, _, _ = place_private(ctx, B, place_seed, pool_factor=2.0, min_extra=3)
    S, T = len(ctx), int(max(1, ctx.max()))
    dev = "cuda"
    s = torch.arange(S, device=dev).view(S, 1, 1, 1)
    h = torch.arange(H_kv, device=dev).view(1, H_kv, 1, 1)
    t = torch.arange(T, device=dev).view(1, 1, T, 1)
    d = torch.arange(D, device=dev).view(1, 1, 1, D)
    idx = ((s * H_kv + h) * T + t) * D + d
    K = R.f32_to_dtype_t(R.uniform_f32_t(R.key(seed, R.STREAM_KCACHE), idx), dtype)
    V = R.f32_to_dtype_t(R.uniform_f32_t(R.key(seed, R.STREAM_VCACHE), idx), dtype)
    qi = (torch.arange(S, device=dev).view(S, 1, 1) * H + torch.arange(H, device=dev).view(1, H, 1)) * D + \
        torch.arange(D, device=dev).view(1, 1, D)
    q = R.f32_to_dtype_t(R.uniform_f32_t(R.key(seed, R.STREAM_Q), qi), dtype).contiguous()
    kc = torch.full((NB, H_kv, B, D), float("nan"), dtype=K.dtype, device=dev)
    vc = torch.full_like(kc, float("nan"))
    btt = torch.as_tensor(bt, device=dev)
    for si in range(S):
        n = int(ctx[si])
        if n == 0:
            continue
        tt = torch.arange(n, device=dev)
        blocks = btt[si, tt // B].long()
        kc[blocks, :, tt % B, :] = K[si, :, :n, :].permute(1, 0, 2)
        vc[blocks, :, tt % B, :] = V[si, :, :n, :].permute(1, 0, 2)
    cl = torch.as_tensor(ctx.astype(np.int32), device=dev)
    return q, kc, vc, btt, cl


def attend(q, kc, vc, bt, cl, scale, pt=0):
    out = torch.empty_like(q)
    pa.paged_attention(out, q, kc, vc, bt, cl, scale, max_context_len=int(cl.max()), partition_tokens=pt)
    torch.cuda.synchronize()
    return out


@pytest.mark.parametrize("dtype,D", [("f16", 128), ("bf16", 128), ("f32", 64), ("f16", 64), ("bf16", 64),
                                     ("f32", 128)])
def test_block_size_and_permutation_invariance_bitwise(dtype, D):
    """Same logical K/V, B in {1,2,4,8,16,32,64} and two physical placements: bitwise
    identical outputs (the kernel computes on 16-token logical tiles), and within
    tolerance of the oracle."""
    ctx = [1, 2, 15, 16, 17, 33, 100, 511, 512, 513, 700, 1100]
    H = H_kv = 2
    scale = 1.0 / np.sqrt(D)
    outs = []
    for B in (1, 2, 4, 8, 16, 32, 64):
        for ps in (11, 12):
            q, kc, vc, bt, cl = logical_problem(ctx, B, ps, H, H_kv, D, dtype)
            outs.append(attend(q, kc, vc, bt, cl, scale))
            if B in (1, 16) and ps == 11:
                ref = oracle.paged_attention(bits(q), bits(kc), bits(vc), bt.cpu().numpy(), cl.cpu().numpy(), scale,
                                             B, H_kv, dtype)
                assert max_abs(outs[-1], ref) <= TOL[dtype]
    for o in outs[1:]:
        assert torch.equal(o, outs[0])


def test_context_edge_cases():
    """ctx = 0 -> zeros; ctx = 1 -> the (just written) V row bit for bit; tile and
    partition boundaries within tolerance."""
    ctx = [0, 1, 2, 15, 16, 17, 31, 32, 33, 511, 512, 513, 1023, 1024, 1025, 2047, 2048]
    wl = make_config("explicit", ctx=ctx, H=4, H_kv=4, D=128, B=16, dtype="f16", seed=5)
    out, kc, vc, x = gpu_step(wl)
    ref, *_ = oracle_step(wl)
    assert max_abs(out, ref) <= TOL["f16"]
    assert torch.equal(out[0], torch.zeros_like(out[0]))
    assert torch.equal(out[1], x["value"][1])


def test_gqa():
    wl = make_config("c1_tiny", H=4, H_kv=2)
    out, *_ = gpu_step(wl)
    ref, *_ = oracle_step(wl)
    assert max_abs(out, ref) <= TOL["f32"]
    wl = make_config("c2_sharegpt", S=8, H=8, H_kv=2)
    out, *_ = gpu_step(wl)
    ref, *_ = oracle_step(wl)
    assert max_abs(out, ref) <= TOL["f16"]


def test_peaked_softmax_and_large_scores():
    """q x 8 (peaked softmax) within tolerance; scores spanning +-700 stay finite
    and within the bound derived in DESIGN.md (fp32 score rounding x max|v|)."""
    wl = make_config("c1_tiny", scale=8.0 / 8.0)
    out, *_ = gpu_step(wl)
    ref, *_ = oracle_step(wl)
    assert max_abs(out, ref) <= TOL["f32"]
    wl = make_config("c1_tiny", scale=60.0)
    out, *_ = gpu_step(wl)
    ref, *_ = oracle_step(wl)
    g = as_f64(out)
    assert np.isfinite(g).all()
    assert np.max(np.abs(g - ref)) <= 5e-2


@pytest.mark.parametrize("dtype", ["f16", "bf16"])
@pytest.mark.parametrize("qmul", [1.0, 8.0])
def test_peaked_softmax_16bit(dtype, qmul):
    """16-bit caches, D=128: the P.V product multiplies the softmax weight rounded to the
    storage dtype (DESIGN reading c25).  Flat and peaked (q x 8) softmax stay inside the
    north-star tolerance against the fp64 oracle, across tiles and split partitions."""
    wl = make_config("c1_tiny", dtype=dtype, D=128, H=4, H_kv=4, S=8, scale=qmul / 128 ** 0.5,
                     kind="explicit", ctx=[1, 15, 16, 17, 100, 513, 1100, 2048], seed=1077)
    out, *_ = gpu_step(wl)
    ref, *_ = oracle_step(wl)
    assert max_abs(out, ref) <= TOL[dtype]


# ------------------------------------------------------------ cache kernels ---------

def test_reshape_and_cache_prefill_shaped():
    """A multi-token slot_mapping (all prompt tokens of several sequences, as in the
    prompt phase) plus padding slots (-1): bitwise vs the oracle."""
    alloc = pa.BlockAllocator(64, 16, list(np.random.default_rng(3).permutation(64)))
    prompts = [7, 40, 16, 1, 33]
    slots = []
    for n in prompts:
        h = alloc.allocate(n)
        bt, _ = alloc.export([h], 8)
        slots += [int(bt[0, t // 16]) * 16 + t % 16 for t in range(n)]
    slots = np.array(slots[:30] + [-1] + slots[30:] + [-1], np.int64)
    T, H_kv, D = len(slots), 4, 64
    for dtype in ("f16", "bf16", "f32"):
        r = np.random.default_rng(4)
        npdt = np.uint32 if dtype == "f32" else np.uint16
        hi = 1 << (32 if dtype == "f32" else 16)
        key = r.integers(0, hi, (T, H_kv, D), dtype=np.uint64).astype(npdt)
        val = r.integers(0, hi, (T, H_kv, D), dtype=np.uint64).astype(npdt)
        kc0 = r.integers(0, hi, (64, H_kv, 16, D), dtype=np.uint64).astype(npdt)
        vc0 = r.integers(0, hi, (64, H_kv, 16, D), dtype=np.uint64).astype(npdt)
        ek, ev = oracle.reshape_and_cache(key, val, kc0, vc0, slots, 16, dtype)
        tdt = {"f32": torch.int32, "f16": torch.int16, "bf16": torch.int16}[dtype]
        view = R.torch_dtype(dtype)

        def dev(a):
            return torch.from_numpy(a.view(np.int32 if dtype == "f32" else np.int16)).to(tdt).cuda().view(view)
        kc, vc = dev(kc0), dev(vc0)
        pa.reshape_and_cache(dev(key), dev(val), kc, vc, torch.from_numpy(slots).cuda())
        torch.cuda.synchronize()
        assert np.array_equal(bits(kc), ek) and np.array_equal(bits(vc), ev), dtype


def test_copy_blocks_multilayer_bitwise():
    wl = make_config("c3_fork", S=30, H=2, H_kv=2)
    layers = [materialize_torch(wl, "cuda", layer=l) for l in range(3)]
    nl = [materialize_numpy(wl, layer=l) for l in range(3)]
    kcs = [x["key_cache"] for x in layers]
    vcs = [x["value_cache"] for x in layers]
    pa.copy_blocks(kcs, vcs, tables_torch(wl, "cuda")["block_mapping"])
    torch.cuda.synchronize()
    ek, ev = oracle.copy_blocks([n["key_cache"] for n in nl], [n["value_cache"] for n in nl], wl.block_mapping,
                                wl.dtype)
    for l in range(3):
        assert np.array_equal(bits(kcs[l]), ek[l]) and np.array_equal(bits(vcs[l]), ev[l])


@pytest.mark.parametrize("B", [1, 8, 16, 32])
def test_block_table_indexing_bitwise(B):
    """The attention kernel's own tile loader (block-table lookup + bulk copy) fetches
    exactly the oracle's logical rows (Fig.6)."""
    wl = make_config("c2_sharegpt", S=10, H=3, H_kv=3, B=B)
    x = materialize_torch(wl, "cuda")
    tb = tables_torch(wl, "cuda")
    mc = wl.max_context_len
    ko, vo = pa.debug_gather_kv(x["key_cache"], x["value_cache"], tb["block_tables"], tb["context_lens"], mc)
    n = materialize_numpy(wl)
    kb, vb = bits(ko), bits(vo)
    for s in range(wl.S):
        c = int(wl.context_lens[s])
        for h in range(wl.H_kv):
            rk, rv = oracle.gather_kv_bits(n["key_cache"], n["value_cache"], wl.block_tables[s], c, h, B, wl.dtype)
            assert np.array_equal(kb[s, h, :c], rk) and np.array_equal(vb[s, h, :c], rv)


def test_validate_tables():
    wl = make_config("c2_alpaca", S=16, H=2, H_kv=2)
    tb = tables_torch(wl, "cuda")
    assert pa.validate_tables(tb["block_tables"], tb["context_lens"], wl.B, wl.num_blocks) == -1
    bt = tb["block_tables"].clone()
    bt[3, 0] = wl.num_blocks
    assert pa.validate_tables(bt, tb["context_lens"], wl.B, wl.num_blocks) == 3 * wl.W
    cl = tb["context_lens"].clone()
    cl[5] = wl.W * wl.B + 1
    assert pa.validate_tables(tb["block_tables"], cl, wl.B, wl.num_blocks) == -6


@pytest.mark.parametrize("name", ["c3_fork", "c4_long"])
@pytest.mark.parametrize("mode", ["chunks4", "chunks4_1stream", "chunks1", "chunks7", "zerocopy", "split1241",
                                  "chunks4_graph"])
def test_decode_step_host_api_matches_device_api(mode, name, tuning_env):
    """pa_decode_step from pinned host buffers, in every transfer mode (copy-engine
    chunks on one or two compute streams, weighted chunks, captured-graph replay or eager
    enqueue, or zero-copy reads of q/k/v and writes of out by the kernel), equals the
    device API bit for bit (outputs and caches)."""
    if mode == "zerocopy":
        tuning_env("PA_E2E_MODE", "zerocopy")
    elif mode == "split1241":
        tuning_env("PA_E2E_SPLIT", "1,2,4,1")
    elif mode == "chunks4_graph":
        tuning_env("PA_E2E_GRAPH", "1")
    else:
        tuning_env("PA_E2E_CHUNKS", mode[6])
        tuning_env("PA_E2E_STREAMS", "1" if mode.endswith("1stream") else "2")
    wl = make_config(name, **SMALL[name])
    x = materialize_torch(wl, "cuda")
    ref, rk, rv, _ = gpu_step(wl, inputs={k: v.clone() for k, v in x.items()})
    kc, vc = x["key_cache"].clone(), x["value_cache"].clone()
    pin = {k: x[k].cpu().pin_memory() for k in ("query", "key", "value")}
    host = {k: torch.from_numpy(np.ascontiguousarray(v)).pin_memory() for k, v in
            dict(slot=wl.slot_mapping, bt=wl.block_tables, cl=wl.context_lens, bm=wl.block_mapping).items()}
    out = torch.empty(pin["query"].shape, dtype=pin["query"].dtype).pin_memory()
    st = torch.empty(pa.decode_step_staging_size(wl.S, wl.H, wl.H_kv, wl.D, wl.W, len(wl.block_mapping),
                                                 pin["query"].dtype), dtype=torch.uint8, device="cuda")
    ws_n = pa.paged_attention_workspace_size(wl.S, wl.H, wl.D, wl.max_context_len)
    ws = torch.zeros(max(ws_n, 16), dtype=torch.uint8, device="cuda")
    pa.decode_step(out, pin["query"], pin["key"], pin["value"], host["slot"], host["bt"], host["cl"], host["bm"],
                   kc, vc, wl.scale, st, ws, max_context_len=wl.max_context_len)
    torch.cuda.synchronize()
    assert torch.equal(out, ref.cpu())
    assert np.array_equal(bits(kc), bits(rk)) and np.array_equal(bits(vc), bits(rv))


@pytest.mark.parametrize("name", ["c3_fork", "c2_sharegpt"])
def test_decode_step_graph_replay_reads_current_host_data(name, tuning_env):
    """pa_decode_step (PA_E2E_GRAPH=1) captures a step into a CUDA graph keyed on its
    pointers and sizes and replays it: a replay must read the host buffers' CURRENT
    contents (new queries under the same pointers) and equal the device API on them, bit
    for bit; and a call with a different batch size (another key) must not replay the
    old graph."""
    tuning_env("PA_E2E_GRAPH", "1")
    wl = make_config(name, **SMALL[name])
    x = materialize_torch(wl, "cuda")
    kc, vc = x["key_cache"].clone(), x["value_cache"].clone()
    pin = {k: x[k].cpu().pin_memory() for k in ("query", "key", "value")}
    host = {k: torch.from_numpy(np.ascontiguousarray(v)).pin_memory() for k, v in
            dict(slot=wl.slot_mapping, bt=wl.block_tables, cl=wl.context_lens, bm=wl.block_mapping).items()}
    out = torch.empty(pin["query"].shape, dtype=pin["query"].dtype).pin_memory()
    st = torch.empty(pa.decode_step_staging_size(wl.S, wl.H, wl.H_kv, wl.D, wl.W, len(wl.block_mapping),
                                                 pin["query"].dtype), dtype=torch.uint8, device="cuda")
    ws = torch.zeros(max(pa.paged_attention_workspace_size(wl.S, wl.H, wl.D, wl.max_context_len), 16),
                     dtype=torch.uint8, device="cuda")

    def call():
        pa.decode_step(out, pin["query"], pin["key"], pin["value"], host["slot"], host["bt"], host["cl"],
                       host["bm"], kc, vc, wl.scale, st, ws, max_context_len=wl.max_context_len)
        torch.cuda.synchronize()
        return out.clone()

    first = call()
    ref1, _, _, _ = gpu_step(wl, inputs={k: v.clone() for k, v in x.items()})
    assert torch.equal(first, ref1.cpu())
    # same pointers, new contents: the queries reversed across sequences
    pin["query"].copy_(pin["query"].flip(0))
    x2 = {k: v.clone() for k, v in x.items()}
    x2["query"] = x["query"].flip(0).contiguous()
    ref2, rk, rv, _ = gpu_step(wl, inputs=x2)
    second = call()
    assert torch.equal(second, ref2.cpu())
    assert not torch.equal(second, first)
    assert np.array_equal(bits(kc), bits(rk)) and np.array_equal(bits(vc), bits(rv))
    tuning_env("PA_E2E_GRAPH", "0")
    assert torch.equal(call(), second)
    tuning_env("PA_E2E_GRAPH", "1")
    # a smaller batch under the same buffers is a different key: outputs of its rows only
    S2 = wl.S // 2
    out.zero_()
    pa.decode_step(out[:S2], pin["query"][:S2], pin["key"][:S2], pin["value"][:S2], host["slot"][:S2],
                   host["bt"][:S2], host["cl"][:S2], host["bm"][:0], kc, vc, wl.scale, st, ws,
                   max_context_len=wl.max_context_len)
    torch.cuda.synchronize()
    assert torch.equal(out[:S2], second[:S2])
    assert not out[S2:].any()


def test_cow_parent_unchanged():
    """Copy-on-write: the sample that keeps the shared block (writes in place)
    gets bitwise the same output whether or not its siblings copied and wrote."""
    wl = make_config("c3_fork", S=36, H=2, H_kv=2)
    full, *_ = gpu_step(wl)
    n = wl.meta["n"]
    keepers = [r * n + n - 1 for r in range(wl.S // n)]
    sub = subset(wl, keepers)
    alone, *_ = gpu_step(sub)
    assert torch.equal(full[keepers], alone)


def test_launch_counter():
    pa.take_launch_count()
    wl = make_config("c3_fork", S=12, H=2, H_kv=2)
    gpu_step(wl)
    assert pa.take_launch_count() >= 3


# ------------------------------------------------------------ full-size sampled -----

FULL = ["c2_sharegpt", "c2_alpaca", "c3_parallel", "c3_fork", "c4_long", "c5_beam"]


@pytest.mark.parametrize("name", FULL)
def test_full_size_sampled_parity(name):
    """BASELINE.json sizes in bench.py's launch configuration (default partitioning):
    sampled sequences x a head slice against the oracle; whole output NaN-free; the new
    token's K/V landed bit for bit."""
    wl = make_config(name)
    out, kc, vc, x = gpu_step(wl)
    assert not torch.isnan(out).any()
    rs = np.random.default_rng(len(name))
    seqs = sorted(set([int(np.argmax(wl.context_lens)), int(np.argmin(wl.context_lens))] +
                      rs.choice(wl.S, 4, replace=False).tolist()))
    world = wl.H // 4 if wl.H % 4 == 0 else 1
    rank = int(rs.integers(world))
    sub = shard(subset(wl, seqs), rank, world)
    ref, *_ = oracle_step(sub)
    h0 = sub.q_head0
    got = out[seqs][:, h0:h0 + sub.H]
    assert max_abs(got, ref) <= TOL[wl.dtype]
    slots = torch.as_tensor(wl.slot_mapping, device="cuda")
    B = wl.B
    assert torch.equal(kc[slots // B, :, slots % B, :], x["key"]) and torch.equal(vc[slots // B, :, slots % B, :],
                                                                                   x["value"])


def test_workspace_reuse_across_layouts():
    """One workspace (garbage-filled) serves calls with different partition counts and
    batch sizes: the call zeroes its own completion counters (pa.h contract)."""
    wl = make_config("c2_sharegpt", S=32, H=4, H_kv=4)
    x = materialize_torch(wl, "cuda")
    tb = tables_torch(wl, "cuda")
    pts = [16, 64, 512]
    need = max(pa.paged_attention_workspace_size(wl.S, wl.H, wl.D, wl.max_context_len, pt) for pt in pts)
    ws = torch.randint(0, 255, (need,), dtype=torch.uint8, device="cuda")
    pa.reshape_and_cache(x["key"], x["value"], x["key_cache"], x["value_cache"], tb["slot_mapping"])
    ref, *_ = oracle_step(wl)
    for pt, ns in [(16, 32), (64, 32), (512, 32), (16, 7), (64, 32), (16, 32)]:
        out = torch.empty_like(x["query"][:ns])
        pa.paged_attention(out, x["query"][:ns].contiguous(), x["key_cache"], x["value_cache"],
                           tb["block_tables"][:ns].contiguous(), tb["context_lens"][:ns].contiguous(), wl.scale,
                           max_context_len=wl.max_context_len, partition_tokens=pt, workspace=ws)
        torch.cuda.synchronize()
        assert max_abs(out, ref[:ns]) <= TOL[wl.dtype], (pt, ns)


@pytest.mark.parametrize("name", list(SMALL) + ["c2_sharegpt_full", "c5_beam_full"])
def test_fused_decode_equals_unfused_bitwise(name):
    """pa_paged_attention_decode (cache write fused into the attention kernel) leaves the
    same cache bytes and the same output bits as reshape_and_cache + paged_attention,
    and matches the oracle."""
    if name.endswith("_full"):
        wl = make_config(name[:-5])
    else:
        wl = make_config(name, **SMALL[name])
    x = materialize_torch(wl, "cuda")
    a, ka, va, _ = gpu_step(wl, inputs={k: v.clone() for k, v in x.items()})
    b, kb, vb, _ = gpu_step(wl, inputs={k: v.clone() for k, v in x.items()}, fused=True)
    assert torch.equal(a, b)
    assert torch.equal(ka.view(torch.int16 if ka.element_size() == 2 else torch.int32),
                       kb.view(torch.int16 if kb.element_size() == 2 else torch.int32))
    assert torch.equal(va.view(torch.int16 if va.element_size() == 2 else torch.int32),
                       vb.view(torch.int16 if vb.element_size() == 2 else torch.int32))
    if not name.endswith("_full"):
        ref, rkc, rvc = oracle_step(wl)
        assert np.array_equal(bits(kb), rkc) and np.array_equal(bits(vb), rvc)
        assert max_abs(b, ref) <= TOL[wl.dtype]


@pytest.mark.parametrize("B", [1, 8, 32])
def test_fused_decode_block_sizes(B):
    wl = make_config("c2_sharegpt", S=16, H=4, H_kv=4, B=B)
    out, kc, vc, _ = gpu_step(wl, fused=True)
    ref, rkc, rvc = oracle_step(wl)
    assert np.array_equal(bits(kc), rkc) and np.array_equal(bits(vc), rvc)
    assert max_abs(out, ref) <= TOL[wl.dtype]


def test_fused_decode_gqa():
    wl = make_config("c2_sharegpt", S=8, H=8, H_kv=2)
    out, kc, vc, _ = gpu_step(wl, fused=True)
    ref, rkc, rvc = oracle_step(wl)
    assert np.array_equal(bits(kc), rkc) and np.array_equal(bits(vc), rvc)
    assert max_abs(out, ref) <= TOL[wl.dtype]


@pytest.mark.parametrize("name", ["c1_tiny", "c2_alpaca", "c2_sharegpt", "c3_fork", "c4_long"])
def test_pdl_and_grid_order_bitwise_identical(name, tuning_env):
    """The coop kernel with programmatic dependent launch on/off and with the partition
    index slowest in the grid (PA_PZ) runs the same per-(sequence, head) tile arithmetic
    in the same order: outputs and cache writes are bit-identical, on repeated full-size
    runs (a stage-reuse or completion-word race would break this)."""
    wl = make_config(name)
    x = materialize_torch(wl, "cuda")
    ref = None
    for pdl, pz in (("1", "0"), ("0", "0"), ("1", "1"), ("1", "0")):
        tuning_env("PA_PDL", pdl)
        tuning_env("PA_PZ", pz)
        out, kc, vc, _ = gpu_step(wl, inputs={k: v.clone() for k, v in x.items()}, fused=True)
        if ref is None:
            ref = (out, kc, vc)
        else:
            assert torch.equal(out, ref[0]), (pdl, pz)
            assert torch.equal(kc.view(torch.int16), ref[1].view(torch.int16)), (pdl, pz)
            assert torch.equal(vc.view(torch.int16), ref[2].view(torch.int16)), (pdl, pz)


@pytest.mark.parametrize("B", [1, 16])
def test_swap_blocks_gpu_cpu_round_trip(B):
    """pa_swap_blocks: swap-out GPU -> pinned CPU pool and swap-in back, one
    launch each, bit-exact vs oracle_swap_blocks; the round trip restores the blocks."""
    wl = make_config("c2_alpaca", S=24, H=4, H_kv=4, B=B)
    x = materialize_torch(wl, "cuda")
    n = materialize_numpy(wl)
    NBc = 64
    rs = np.random.default_rng(B)
    src_blocks = rs.choice(wl.num_blocks, 40, replace=False)
    dst_blocks = rs.choice(NBc, 40, replace=False)
    out_map = np.stack([src_blocks, dst_blocks], 1).astype(np.int64)
    cpu_k = torch.zeros((NBc,) + x["key_cache"].shape[1:], dtype=x["key_cache"].dtype).pin_memory()
    cpu_v = torch.zeros_like(cpu_k).pin_memory()
    pa.swap_blocks([cpu_k], [cpu_v], [x["key_cache"]], [x["value_cache"]], torch.from_numpy(out_map).cuda())
    torch.cuda.synchronize()
    zk = np.zeros((NBc,) + n["key_cache"].shape[1:], n["key_cache"].dtype)
    ek, ev = oracle.swap_blocks([zk], [zk.copy()], [n["key_cache"]], [n["value_cache"]], out_map)
    assert np.array_equal(bits(cpu_k), ek[0]) and np.array_equal(bits(cpu_v), ev[0])
    back = torch.zeros_like(x["key_cache"])
    backv = torch.zeros_like(x["value_cache"])
    in_map = np.stack([dst_blocks, src_blocks], 1).astype(np.int64)
    pa.swap_blocks([back], [backv], [cpu_k], [cpu_v], torch.from_numpy(in_map).pin_memory())
    torch.cuda.synchronize()
    sb = torch.as_tensor(src_blocks, device="cuda")
    assert torch.equal(bits_t(back[sb]), bits_t(x["key_cache"][sb]))
    assert torch.equal(bits_t(backv[sb]), bits_t(x["value_cache"][sb]))
    # the per-block cudaMemcpyAsync baseline moves the same bytes
    cpu_k2, cpu_v2 = torch.zeros_like(cpu_k).pin_memory(), torch.zeros_like(cpu_v).pin_memory()
    pa.swap_blocks_memcpy([cpu_k2], [cpu_v2], [x["key_cache"]], [x["value_cache"]], torch.from_numpy(out_map))
    torch.cuda.synchronize()
    assert torch.equal(bits_t(cpu_k2), bits_t(cpu_k)) and torch.equal(bits_t(cpu_v2), bits_t(cpu_v))


def bits_t(t):
    return t.view(torch.int16) if t.element_size() == 2 else t.view(torch.int32)


@pytest.mark.parametrize("name", ["c2_sharegpt", "c4_long"])
def test_partitions_per_cta_bitwise_identical(name, tuning_env):
    """The coop scheduler may walk several 512-token partitions in one CTA (PA_PPC): each
    is finished and merged exactly as with one CTA per partition, so outputs and cache
    bytes are bit-identical for any PPC (TP / batch-composition invariance is kept)."""
    wl = make_config(name)
    x = materialize_torch(wl, "cuda")
    ref = None
    for ppc in ("1", "2", "3", "4"):
        tuning_env("PA_PPC", ppc)
        out, kc, vc, _ = gpu_step(wl, inputs={k: v.clone() for k, v in x.items()}, fused=True)
        if ref is None:
            ref = (out, kc)
        else:
            assert torch.equal(out, ref[0]), ppc
            assert torch.equal(kc.view(torch.int16), ref[1].view(torch.int16)), ppc


@pytest.mark.parametrize("name,gs,hpc,slots", [("c5_beam", 4, 0, 0), ("c3_parallel", 6, 0, 0), ("c3_fork", 6, 0, 0),
                                               ("c2_sharegpt", 4, 0, 0), ("c5_beam", 3, 0, 0), ("c3_parallel", 8, 0, 0),
                                               ("c5_beam", 4, 2, 1), ("c5_beam", 4, 1, 2), ("c3_fork", 6, 1, 1),
                                               ("c3_parallel", 4, 2, 3), ("c2_sharegpt", 2, 4, 1)])
def test_shared_decode_bitwise_equals_decode(name, gs, hpc, slots, tuning_env):
    """N1 sharing-aware entry: every distinct block of a sequence group is loaded once;
    outputs and cache bytes bit-identical to pa_paged_attention_decode at full size,
    including groups that do not align with the requests (gs 3 / 8), several heads per
    CTA, and stages with fewer block slots than members (a tile's distinct blocks then
    stream through several stages)."""
    import paper_2309_06180_b200 as pa
    if hpc:
        tuning_env("PA_SHARED_HPC", str(hpc))
    if slots:
        tuning_env("PA_SHARED_SLOTS", str(slots))
    wl = make_config(name)
    x = materialize_torch(wl, "cuda")
    tb = tables_torch(wl, "cuda")
    a, ka, va, _ = gpu_step(wl, inputs={k: v.clone() for k, v in x.items()}, fused=True)
    y = {k: v.clone() for k, v in x.items()}
    if len(wl.block_mapping):
        pa.copy_blocks([y["key_cache"]], [y["value_cache"]], tb["block_mapping"])
    b = torch.empty_like(y["query"])
    pa.paged_attention_decode_shared(b, y["query"], y["key"], y["value"], y["key_cache"], y["value_cache"],
                                     tb["block_tables"], tb["context_lens"], wl.scale, gs,
                                     max_context_len=wl.max_context_len)
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    assert torch.equal(bits_t(ka), bits_t(y["key_cache"])) and torch.equal(bits_t(va), bits_t(y["value_cache"]))


@pytest.mark.parametrize("B,slots", [(1, 0), (16, 0), (32, 0), (16, 1), (8, 2)])
def test_shared_decode_small_vs_oracle(B, slots, tuning_env):
    import paper_2309_06180_b200 as pa
    if slots:
        tuning_env("PA_SHARED_SLOTS", str(slots))
    wl = make_config("c5_beam", S=14, H=4, H_kv=4, B=B)
    x = materialize_torch(wl, "cuda")
    tb = tables_torch(wl, "cuda")
    if len(wl.block_mapping):
        pa.copy_blocks([x["key_cache"]], [x["value_cache"]], tb["block_mapping"])
    out = torch.empty_like(x["query"])
    pa.paged_attention_decode_shared(out, x["query"], x["key"], x["value"], x["key_cache"], x["value_cache"],
                                     tb["block_tables"], tb["context_lens"], wl.scale, 4,
                                     max_context_len=wl.max_context_len)
    torch.cuda.synchronize()
    ref, rkc, rvc = oracle_step(wl)
    assert np.array_equal(bits(x["key_cache"]), rkc) and np.array_equal(bits(x["value_cache"]), rvc)
    assert max_abs(out, ref) <= TOL[wl.dtype]


@pytest.mark.parametrize("name", ["c2_sharegpt_full", "c2_alpaca_full", "c4_long", "c3_fork"])
def test_grid_order_is_scheduling_only_bitwise(name):
    """A longest-first grid order (pa_decode_plan) or any other permutation changes which
    CTAs run first, never a result bit: fused decode and unfused attention outputs and the
    caches equal the natural-order run's."""
    wl = make_config(name[:-5]) if name.endswith("_full") else make_config(name, S=40, H=8, H_kv=8)
    x = materialize_torch(wl, "cuda")
    tb = tables_torch(wl, "cuda")
    plan = pa.decode_plan(wl.context_lens)
    assert np.all(np.diff(wl.context_lens[plan]) <= 0)
    rnd = np.random.default_rng(3).permutation(wl.S).astype(np.int32)
    outs, caches = [], []
    for order in (None, plan, rnd):
        y = {k: v.clone() for k, v in x.items()}
        if len(wl.block_mapping):
            pa.copy_blocks([y["key_cache"]], [y["value_cache"]], tb["block_mapping"])
        out = torch.empty_like(y["query"])
        pa.paged_attention_decode(out, y["query"], y["key"], y["value"], y["key_cache"], y["value_cache"],
                                  tb["block_tables"], tb["context_lens"], wl.scale, max_context_len=wl.max_context_len,
                                  seq_order=order)
        out2 = torch.empty_like(out)
        pa.paged_attention(out2, y["query"], y["key_cache"], y["value_cache"], tb["block_tables"], tb["context_lens"],
                           wl.scale, max_context_len=wl.max_context_len, seq_order=order)
        torch.cuda.synchronize()
        assert torch.equal(out, out2)
        outs.append(out)
        caches.append((y["key_cache"], y["value_cache"]))
    for o, (k, v) in zip(outs[1:], caches[1:]):
        assert torch.equal(o, outs[0])
        assert np.array_equal(bits(k), bits(caches[0][0])) and np.array_equal(bits(v), bits(caches[0][1]))
    if not name.endswith("_full"):
        ref, *_ = oracle_step(wl)
        assert max_abs(outs[1], ref) <= TOL[wl.dtype]


def _decode_fuzz(n=12, seed=180):
    rs = np.random.default_rng(seed)
    cases = []
    for i in range(n):
        dtype, D = [("f16", 128), ("bf16", 128), ("f32", 64), ("f16", 64), ("bf16", 64), ("f32", 128)][i % 6]
        H = int(rs.choice([1, 2, 3, 4, 5, 8]))
        H_kv = int(rs.choice([d for d in (1, 2, 4, 8) if H % d == 0 and d <= H]))
        S = int(rs.integers(1, 40))
        ctx = [int(c) for c in rs.choice([0, 1, 15, 16, 17, 200, 511, 512, 513, 1100, 2048], S)]
        cases.append((dict(ctx=ctx, H=H, H_kv=H_kv, D=D, B=int(rs.choice([1, 8, 16, 32])), dtype=dtype,
                           seed=int(rs.integers(1, 1 << 20))), bool(i % 2)))
    return cases


@pytest.mark.parametrize("over,fused", _decode_fuzz())
def test_decode_fuzz_vs_oracle(over, fused):
    """Seeded random decode steps through the coop kernel (fused cache write or not): 1..39
    sequences with contexts at the tile / partition edges (0, 1, 15-17, 511-513, 2048), 1..8
    query heads, GQA, head_dim 64 / 128, block size 1..32, f32 / f16 / bf16 -- every output
    vs the fp64 oracle, caches bit-exact."""
    wl = make_config("explicit", **over)
    out, kc, vc, _ = gpu_step(wl, fused=fused)
    ref, rkc, rvc = oracle_step(wl)
    assert np.array_equal(bits(kc), rkc) and np.array_equal(bits(vc), rvc)
    assert max_abs(out, ref) <= TOL[wl.dtype]

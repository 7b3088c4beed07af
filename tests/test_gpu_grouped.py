"""GPU parity of the sharing-aware decode step on the tcgen05 tensor cores (SURVEY 8(f) N1,
pa_paged_attention_decode_grouped): each distinct block piece of a group is loaded once and
Q K^T / P V run as tcgen05 MMAs over the group's rows.  Against the fp64 oracle on
identical generated inputs (max-abs <= 2e-3 fp16, 1e-2 bf16; caches bit-exact), at
small sizes spanning several tiles, split contexts, GQA, block sizes and unrelated
(non-sharing) groups, and at the full C3/C5 sizes on sampled sequences."""
import numpy as np
import pytest
import torch

from synth import make_config, materialize_torch, shard, subset, tables_torch
from tests.pathutil import TOL, bits, max_abs, oracle_step

pytestmark = pytest.mark.gpu
pa = pytest.importorskip("paper_2309_06180_b200")


def grouped_step(wl, gs, x=None, mcl=None):
    x = x or materialize_torch(wl, "cuda")
    tb = tables_torch(wl, "cuda")
    if len(wl.block_mapping):
        pa.copy_blocks([x["key_cache"]], [x["value_cache"]], tb["block_mapping"])
    out = torch.full_like(x["query"], float("nan"))
    pa.paged_attention_decode_grouped(out, x["query"], x["key"], x["value"], x["key_cache"], x["value_cache"],
                                      tb["block_tables"], tb["context_lens"], wl.scale, gs,
                                      max_context_len=wl.max_context_len if mcl is None else mcl)
    torch.cuda.synchronize()
    return out, x


@pytest.mark.parametrize("name,over,gs", [
    ("c5_beam", dict(S=14, H=4, H_kv=4), 4),            # beams: most blocks shared, last group ragged
    ("c5_beam", dict(S=16, H=4, H_kv=2), 4),            # GQA (c13)
    ("c5_beam", dict(S=16, H=2, H_kv=2, B=32), 4),      # 2 tiles per block
    ("c3_parallel", dict(S=24, H=2, H_kv=2), 6),        # parallel samples, bf16
    ("c3_fork", dict(S=24, H=2, H_kv=2), 6),            # fork step: CoW'd last blocks
    ("c3_parallel", dict(S=24, H=2, H_kv=2), 8),        # groups not aligned with requests
    ("c2_sharegpt", dict(S=24, H=4, H_kv=4), 4),        # unrelated sequences: no sharing
    ("c4_long", dict(S=8, H=2, H_kv=2), 2),             # split contexts (up to 4 partitions)
    ("c2_alpaca", dict(S=40, H=2, H_kv=2), 1),          # group of one
])
def test_grouped_decode_vs_oracle(name, over, gs):
    wl = make_config(name, **over)
    out, x = grouped_step(wl, gs)
    ref, rkc, rvc = oracle_step(wl)
    assert np.array_equal(bits(x["key_cache"]), rkc) and np.array_equal(bits(x["value_cache"]), rvc)
    assert not torch.isnan(out).any()
    assert max_abs(out, ref) <= TOL[wl.dtype]


def test_grouped_decode_context_edges():
    """ctx = 0 (zeros), ctx = 1 (the new token's V row), tile and partition boundaries,
    inside groups of unrelated sequences."""
    ctx = [0, 1, 2, 15, 16, 17, 31, 32, 33, 511, 512, 513, 1023, 1024, 1025, 2047, 2048]
    wl = make_config("explicit", ctx=ctx, H=4, H_kv=4, D=128, B=16, dtype="f16", seed=5)
    out, x = grouped_step(wl, 4)
    ref, rkc, rvc = oracle_step(wl)
    assert np.array_equal(bits(x["key_cache"]), rkc) and np.array_equal(bits(x["value_cache"]), rvc)
    assert max_abs(out, ref) <= TOL["f16"]
    assert not out[0].any()


@pytest.mark.parametrize("mcl", [512, 1000, 0])
def test_grouped_decode_split_parts_vs_oracle(mcl):
    """Split context (a6) in the tcgen05 kernel: parts of 512 tokens per group, the last part
    taking every position past the bound max_context_len gives (512: no split; 1000: two
    parts, the second absorbing contexts up to 2048; 0: W * B, four parts), members of one
    group with 1..4 parts of their own, merged by the last part to finish."""
    ctx = [2048, 1500, 600, 513, 512, 511, 100, 1, 1025, 1024, 0, 2000]
    wl = make_config("explicit", ctx=ctx, H=8, H_kv=8, D=128, B=16, dtype="f16", seed=11)
    out, x = grouped_step(wl, 4, mcl=mcl)
    ref, rkc, rvc = oracle_step(wl)
    assert np.array_equal(bits(x["key_cache"]), rkc) and np.array_equal(bits(x["value_cache"]), rvc)
    assert not torch.isnan(out).any()
    assert max_abs(out, ref) <= TOL["f16"]


@pytest.mark.parametrize("name,gs", [("c5_beam", 4), ("c3_parallel", 6)])
def test_grouped_decode_full_size_sampled(name, gs):
    """BASELINE.json sizes: whole output finite, sampled sequences x a head slice against
    the oracle, and every new token's K/V landed bit for bit."""
    wl = make_config(name)
    out, x = grouped_step(wl, gs)
    assert not torch.isnan(out).any()
    rs = np.random.default_rng(len(name))
    seqs = sorted(set([int(np.argmax(wl.context_lens))] + rs.choice(wl.S, 5, replace=False).tolist()))
    world = wl.H // 4
    rank = int(rs.integers(world))
    sub = shard(subset(wl, seqs), rank, world)
    ref, *_ = oracle_step(sub)
    got = out[seqs][:, sub.q_head0:sub.q_head0 + sub.H]
    assert max_abs(got, ref) <= TOL[wl.dtype]
    slots = torch.as_tensor(wl.slot_mapping, device="cuda")
    kc, vc, B = x["key_cache"], x["value_cache"], wl.B
    assert torch.equal(kc[slots // B, :, slots % B, :], x["key"])
    assert torch.equal(vc[slots // B, :, slots % B, :], x["value"])


def test_grouped_decode_rejects_unsupported():
    wl = make_config("c1_tiny")  # fp32, D = 64
    x = materialize_torch(wl, "cuda")
    tb = tables_torch(wl, "cuda")
    with pytest.raises(pa.PagedAttnError):
        pa.paged_attention_decode_grouped(torch.empty_like(x["query"]), x["query"], x["key"], x["value"],
                                          x["key_cache"], x["value_cache"], tb["block_tables"], tb["context_lens"],
                                          wl.scale, 4)


def test_grouped_decode_deterministic():
    """Full-size C5 three times: outputs bit-identical (the persistent CTAs draw work items
    in a different order every launch; a race between the producer, MMA and softmax warps
    over the tile buffers or tensor memory would show here)."""
    wl = make_config("c5_beam")
    x0 = materialize_torch(wl, "cuda")
    ref = None
    for _ in range(3):
        out, _ = grouped_step(wl, 4, x={k: v.clone() for k, v in x0.items()})
        if ref is None:
            ref = out
        else:
            assert torch.equal(out, ref)


@pytest.mark.parametrize("name,gs", [("c5_beam", 4), ("c3_fork", 6), ("c3_parallel", 6)])
def test_grouped_decode_full_size_full_output(name, gs):
    """BASELINE.json sizes, the WHOLE output against the oracle head slice by head slice
    (inputs from the seeded generator), caches bit-exact."""
    import oracle
    wl = make_config(name)
    out, x = grouped_step(wl, gs)
    got = out.double().cpu().numpy()
    hs = 8
    for r in range(wl.H // hs):
        sh = shard(wl, r, wl.H // hs)
        y = materialize_torch(sh, "cuda")
        n = {k: bits(v) for k, v in y.items()}
        kc, vc = n["key_cache"], n["value_cache"]
        if len(sh.block_mapping):
            kcs, vcs = oracle.copy_blocks([kc], [vc], sh.block_mapping, sh.dtype)
            kc, vc = kcs[0], vcs[0]
        kc, vc = oracle.reshape_and_cache(n["key"], n["value"], kc, vc, sh.slot_mapping, sh.B, sh.dtype)
        ref = oracle.paged_attention(n["query"], kc, vc, sh.block_tables, sh.context_lens, sh.scale, sh.B, sh.H_kv,
                                     sh.dtype)
        h0 = sh.q_head0
        err = float(np.max(np.abs(got[:, h0:h0 + sh.H] - ref)))
        assert err <= TOL[wl.dtype], (r, err)
        assert np.array_equal(bits(x["key_cache"][:, h0:h0 + sh.H]), kc)
        assert np.array_equal(bits(x["value_cache"][:, h0:h0 + sh.H]), vc)


@pytest.mark.parametrize("name,gs", [("c5_beam", 4), ("c3_parallel", 6)])
def test_grouped_decode_plan_order_is_scheduling_only(name, gs):
    """Walking the groups longest first (pa_decode_plan) changes which CTA computes an item,
    never a bit of it -- also with split contexts (c3_parallel: few items per SM, so parts of
    512 tokens, the empty parts skipped through the work counter, merges by the last part)."""
    wl = make_config(name)
    x0 = materialize_torch(wl, "cuda")
    tb = tables_torch(wl, "cuda")
    outs = []
    for order in (None, pa.decode_plan(wl.context_lens)):
        x = {k: v.clone() for k, v in x0.items()}
        if len(wl.block_mapping):
            pa.copy_blocks([x["key_cache"]], [x["value_cache"]], tb["block_mapping"])
        out = torch.empty_like(x["query"])
        pa.paged_attention_decode_grouped(out, x["query"], x["key"], x["value"], x["key_cache"], x["value_cache"],
                                          tb["block_tables"], tb["context_lens"], wl.scale, gs,
                                          max_context_len=wl.max_context_len, seq_order=order)
        torch.cuda.synchronize()
        outs.append(out)
    assert torch.equal(outs[0], outs[1])
    assert not torch.isnan(outs[1]).any()


def _fuzz_cases(n=10, seed=2309):
    rs = np.random.default_rng(seed)
    cases = []
    for i in range(n):
        name = ["c5_beam", "c3_parallel", "c3_fork"][i % 3]
        H = int(rs.choice([1, 2, 3, 4, 5, 6, 8]))
        H_kv = int(rs.choice([d for d in (1, 2, 4, 8) if H % d == 0 and d <= H]))
        S = 4 * int(rs.integers(1, 9)) if name == "c5_beam" else 6 * int(rs.integers(1, 6))  # whole requests (k=4 / n=6)
        over = dict(S=S, H=H, H_kv=H_kv, B=int(rs.choice([16, 32])), seed=int(rs.integers(1, 1 << 30)))
        if name == "c5_beam":
            over["stickiness"] = float(rs.choice([0.0, 0.5, 0.9]))
        cases.append((name, over, int(rs.integers(1, 9))))
    return cases


@pytest.mark.parametrize("name,over,gs", _fuzz_cases())
def test_grouped_decode_fuzz_vs_oracle(name, over, gs):
    """Seeded random shapes through the tcgen05 N1 kernel: group sizes 1..8 not aligned with
    the requests, 1..8 query heads (ragged head quads), GQA, block size 16 / 32, beam
    stickiness, ragged last groups -- every output vs the fp64 oracle, caches bit-exact."""
    wl = make_config(name, **over)
    out, x = grouped_step(wl, gs)
    ref, rkc, rvc = oracle_step(wl)
    assert np.array_equal(bits(x["key_cache"]), rkc) and np.array_equal(bits(x["value_cache"]), rvc)
    assert not torch.isnan(out).any()
    assert max_abs(out, ref) <= TOL[wl.dtype]

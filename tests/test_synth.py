"""The seeded input generator: both materialisations agree bit for bit, views (subset,
shard) draw the same values as the full workload, and the length mixes keep the
paper's ShareGPT/Alpaca ratios (8.4x longer inputs, 5.8x longer outputs)."""
import numpy as np
import pytest
import torch

from synth import make_config, materialize_numpy, materialize_torch, shard, subset
from synth import rng as R
from synth.workload import decode_snapshot, request_pool


def to_bits(t: torch.Tensor) -> np.ndarray:
    if t.dtype == torch.float32:
        return t.contiguous().view(torch.int32).numpy().view(np.uint32)
    return t.contiguous().view(torch.int16).numpy().view(np.uint16)


def test_numpy_and_torch_streams_agree():
    k = R.key(7, R.STREAM_Q)
    idx = np.arange(0, 1 << 18, dtype=np.int64) * 7919
    a = R.bits_np(k, idx)
    b = R.bits_t(k, torch.from_numpy(idx)).numpy().view(np.uint64)
    assert np.array_equal(a, b)
    fa = R.uniform_f32_np(k, idx)
    fb = R.uniform_f32_t(k, torch.from_numpy(idx)).numpy()
    assert np.array_equal(fa, fb)
    assert fa.min() >= -1.0 and fa.max() < 1.0
    for dt in ("f16", "bf16", "f32"):
        nb = R.f32_to_bits_np(fa, dt)
        tb = to_bits(R.f32_to_dtype_t(torch.from_numpy(fa), dt))
        assert np.array_equal(nb, tb), dt


def test_bf16_rounding_is_round_to_nearest_even():
    x = np.array([1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8, -1.0 - 2 ** -9, 1.0 + 2 ** -8 + 2 ** -20], np.float32)
    got = R.f32_to_bits_np(x, "bf16")
    ref = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("name", ["c1_tiny", "c3_fork"])
def test_materializations_identical(name):
    over = {} if name == "c1_tiny" else dict(S=18, H=2, H_kv=2)
    wl = make_config(name, **over)
    n = materialize_numpy(wl)
    t = materialize_torch(wl, "cpu", chunk_blocks=7)
    for key in ("query", "key", "value", "key_cache", "value_cache"):
        assert np.array_equal(n[key], to_bits(t[key])), key


def test_live_mask_and_slots():
    wl = make_config("c2_alpaca", S=32, H=2, H_kv=2)
    B = wl.B
    for s in range(wl.S):
        n = int(wl.context_lens[s])
        slot = int(wl.slot_mapping[s])
        assert slot == wl.block_tables[s, (n - 1) // B] * B + (n - 1) % B
        assert not wl.live[slot // B, slot % B]  # the current token is written by this step
        for t in range(n - 1):
            assert wl.live[wl.block_tables[s, t // B], t % B]
    n = materialize_numpy(wl)
    nan = R.NAN_BITS[wl.dtype]
    assert (n["key_cache"][~wl.live[:, None, :, None].repeat(wl.H_kv, 1).repeat(wl.D, 3)] == nan).all()


def test_subset_and_shard_draw_the_same_values():
    wl = make_config("c5_beam", S=24, H=4, H_kv=4)
    full = materialize_numpy(wl)
    seqs = [0, 5, 17, 23]
    sub = subset(wl, seqs)
    ns = materialize_numpy(sub)
    for i, s in enumerate(seqs):
        assert np.array_equal(ns["query"][i], full["query"][s])
        n = int(wl.context_lens[s])
        for t in range(n - 1):
            b_full = wl.block_tables[s, t // wl.B]
            b_sub = sub.block_tables[i, t // wl.B]
            assert np.array_equal(ns["key_cache"][b_sub, :, t % wl.B], full["key_cache"][b_full, :, t % wl.B])
    sh = shard(wl, 1, 2)
    nh = materialize_numpy(sh)
    assert np.array_equal(nh["query"], full["query"][:, 2:4])
    assert np.array_equal(nh["value_cache"], full["value_cache"][:, 2:4])


def test_length_mix_ratios_match_paper():
    ps, os_ = request_pool(1, "sharegpt", n=200000)
    pa, oa = request_pool(1, "alpaca", n=200000)
    assert abs(ps.mean() / pa.mean() - 8.4) < 0.4
    assert abs(os_.mean() / oa.mean() - 5.8) < 0.3
    assert ps.max() <= 2047 and (ps + os_).max() <= 2048


def test_snapshot_is_length_biased_and_bounded():
    p, g, ctx = decode_snapshot(1001, "sharegpt", 4096)
    assert ctx.max() <= 2048 and ctx.min() >= 2
    assert (g >= 0).all()
    wl = make_config("c2_sharegpt")
    assert wl.S == 256 and wl.H == 40 and wl.D == 128 and wl.dtype == "f16"
    assert 350 < wl.context_lens.mean() < 550


def test_sharing_fixtures():
    c3 = make_config("c3_fork")
    assert len(c3.block_mapping) > 150            # ~5 CoW pairs per request
    src, dst = c3.block_mapping[:, 0], c3.block_mapping[:, 1]
    assert len(set(dst.tolist())) == len(dst) and not (set(dst.tolist()) & set(src.tolist()))
    assert c3.unique_kv_bytes() < c3.logical_kv_bytes()
    c5 = make_config("c5_beam")
    assert c5.unique_kv_bytes() / c5.logical_kv_bytes() < 0.5   # beam trees share heavily
    src, dst = c5.block_mapping[:, 0], c5.block_mapping[:, 1]
    assert len(set(dst.tolist())) == len(dst) and not (set(dst.tolist()) & set(src.tolist()))


def test_determinism():
    a, b = make_config("c5_beam", S=16), make_config("c5_beam", S=16)
    assert np.array_equal(a.block_tables, b.block_tables) and np.array_equal(a.block_mapping, b.block_mapping)


def test_sorted_placement_is_consecutive():
    """placement='sorted' (the contiguous-cache ablation) hands out block ids in order:
    each sequence's blocks are consecutive, with the same lengths, pool size and live-slot
    count as the shuffled placement."""
    a = make_config("c2_alpaca", S=16, H=2, H_kv=2)
    b = make_config("c2_alpaca", S=16, H=2, H_kv=2, placement="sorted")
    assert np.array_equal(a.context_lens, b.context_lens) and a.num_blocks == b.num_blocks
    assert a.live.sum() == b.live.sum()
    off = 0
    for s in range(b.S):
        nb = -(-int(b.context_lens[s]) // b.B)
        assert np.array_equal(b.block_tables[s, :nb], np.arange(off, off + nb))
        off += nb
    with pytest.raises(ValueError):
        make_config("c2_alpaca", S=4, H=2, H_kv=2, placement="random")

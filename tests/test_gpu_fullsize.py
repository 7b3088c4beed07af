"""Full-size, full-output parity of bench.py's own entry points (SURVEY §8(c) parity
matrix, "attention | oracle fp64 | all").

Every BASELINE.json config at its full size, in the launch configuration bench.py times
(default partitioning, the cache write fused into the attention kernel; C5 on the
sharing-aware tcgen05 kernel, groups of 4): the WHOLE [S][H][D] output is compared element
by element with the fp64 oracle, and the caches after the step bit for bit.  The oracle
runs head slice by head slice (shard(): the same seeded values, generated for that slice
only) so host memory stays bounded; the oracle inputs come from the seeded generator
(synth), never from the CUDA path."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
import paper_2309_06180_b200 as pa
from synth import make_config, materialize_torch, shard, tables_torch
from tests.pathutil import TOL, as_f64, bits

pytestmark = pytest.mark.gpu

# bench.py's default decode entry per config (bench.py run_ours: the tcgen05 grouped kernel in
# beam groups of 4 on C5, the fused coop decode elsewhere)
DEFAULT_GROUPED = {"c5_beam": 4}
CONFIGS = ["c2_sharegpt", "c2_alpaca", "c3_parallel", "c3_fork", "c4_sharegpt", "c4_long", "c5_beam"]


def _bench_step(wl):
    """The step bench.py times, on the device: copy_blocks (CoW pairs) + the default decode."""
    x = materialize_torch(wl, "cuda")
    tb = tables_torch(wl, "cuda")
    kc, vc = x["key_cache"], x["value_cache"]
    if len(wl.block_mapping):
        pa.copy_blocks([kc], [vc], tb["block_mapping"])
    out = torch.empty_like(x["query"])
    g = DEFAULT_GROUPED.get(wl.name, 0)
    plan = pa.decode_plan(wl.context_lens)  # bench.py's longest-first grid order
    if g:
        pa.paged_attention_decode_grouped(out, x["query"], x["key"], x["value"], kc, vc, tb["block_tables"],
                                          tb["context_lens"], wl.scale, g, max_context_len=wl.max_context_len,
                                          seq_order=plan)
    else:
        pa.paged_attention_decode(out, x["query"], x["key"], x["value"], kc, vc, tb["block_tables"],
                                  tb["context_lens"], wl.scale, max_context_len=wl.max_context_len, seq_order=plan)
    torch.cuda.synchronize()
    return out, kc, vc


def _oracle_slice(sh):
    """The oracle's step on one head slice: inputs from the seeded generator (device-side
    torch streams, pinned equal to the numpy streams in tests/test_synth.py)."""
    x = materialize_torch(sh, "cuda")
    n = {k: bits(v) for k, v in x.items()}
    del x
    kc, vc = n["key_cache"], n["value_cache"]
    if len(sh.block_mapping):
        kcs, vcs = oracle.copy_blocks([kc], [vc], sh.block_mapping, sh.dtype)
        kc, vc = kcs[0], vcs[0]
    kc, vc = oracle.reshape_and_cache(n["key"], n["value"], kc, vc, sh.slot_mapping, sh.B, sh.dtype)
    out = oracle.paged_attention(n["query"], kc, vc, sh.block_tables, sh.context_lens, sh.scale, sh.B, sh.H_kv,
                                 sh.dtype)
    return out, kc, vc


@pytest.mark.parametrize("name", CONFIGS)
def test_full_size_full_output_parity(name):
    wl = make_config(name)
    out, kc, vc = _bench_step(wl)
    got = as_f64(out)
    assert not np.isnan(got).any(), "NaN in the output (a poisoned slot was read)"
    hs = 8  # heads per oracle slice: 40, 72 and 96 are multiples of 8
    world = wl.H // hs
    worst = 0.0
    for r in range(world):
        sh = shard(wl, r, world)
        ref, rkc, rvc = _oracle_slice(sh)
        h0, h1 = sh.q_head0, sh.q_head0 + sh.H
        err = float(np.max(np.abs(got[:, h0:h1] - ref)))
        worst = max(worst, err)
        assert err <= TOL[wl.dtype], f"{name} heads {h0}..{h1 - 1}: max-abs {err} > {TOL[wl.dtype]}"
        k0, k1 = sh.kv_head0, sh.kv_head0 + sh.H_kv
        assert np.array_equal(bits(kc[:, k0:k1]), rkc), f"{name}: key cache heads {k0}..{k1 - 1}"
        assert np.array_equal(bits(vc[:, k0:k1]), rvc), f"{name}: value cache heads {k0}..{k1 - 1}"
    print(f"{name}: {wl.S}x{wl.H} outputs, worst max-abs {worst:.3g} (tol {TOL[wl.dtype]})")


@pytest.mark.parametrize("name", ["c2_sharegpt", "c5_beam"])
def test_generator_on_cuda_equals_numpy(name):
    """The device-side generator the full-size oracle inputs come from draws the same bits
    as the numpy generator (integer counter hash + fp32 -> dtype rounding on the GPU)."""
    from synth import materialize_numpy
    wl = make_config(name, S=20, H=8, H_kv=8)
    sh = shard(wl, 1, 4)
    n = materialize_numpy(sh)
    t = materialize_torch(sh, "cuda")
    for key in ("query", "key", "value", "key_cache", "value_cache"):
        assert np.array_equal(n[key], bits(t[key])), key

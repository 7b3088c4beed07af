"""Fused tensor-parallel all-gather on one B200.

The attention kernel of rank r stores every output row of its heads into EVERY rank's
gather buffer, then a one-warp kernel exchanges completion flags
(`pa_paged_attention_decode_tp`).  With one GPU in this run, ranks are exercised two ways:
* simulated ranks in one process, each on its own CUDA stream (peers = local buffers);
* two processes sharing the GPU, buffers opened through CUDA IPC (the multi-GPU code
  path, minus NVLink).
The gathered output must equal the single-GPU decode bit for bit (the per-(sequence,
head) arithmetic does not depend on the head grouping) AND the fp64 oracle of the whole
(unsharded) step within the north-star tolerance (concatenating the heads'
outputs is the unsharded layer output).  The NCCL path (`gather_heads`) is exercised on
CUDA tensors too: a world-1 NCCL group in-process, and two processes over gloo."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _reference(wl):
    """Single-GPU decode step (copy_blocks, then the fused decode) of the whole workload."""
    from tests.pathutil import gpu_step
    out, kc, vc, _ = gpu_step(wl, fused=True)
    return out, kc, vc


def _assert_oracle(gathered, wl, what=""):
    """The gathered [S][H][D] output vs the fp64 oracle of the unsharded step."""
    from tests.pathutil import TOL, max_abs, oracle_step
    ref, _, _ = oracle_step(wl)
    err = max_abs(gathered, ref)
    assert err <= TOL[wl.dtype], f"{what}: max-abs {err} vs oracle > {TOL[wl.dtype]}"


def _rank_inputs(wl, rank, world):
    """Rank's head shard with its copy-on-write copies already applied (the step's
    copy_blocks runs on every rank's own cache slice before the attention)."""
    import paper_2309_06180_b200 as pa
    from synth import materialize_torch, shard, tables_torch
    sh = shard(wl, rank, world)
    x = materialize_torch(sh, "cuda")
    tb = tables_torch(sh, "cuda")
    if len(sh.block_mapping):
        pa.copy_blocks([x["key_cache"]], [x["value_cache"]], tb["block_mapping"])
    return sh, x, tb


@pytest.mark.parametrize("world,name", [(2, "c2_sharegpt"), (4, "c2_sharegpt"), (2, "c4_long"), (4, "c5_beam")])
def test_simulated_ranks_gather_bitwise(world, name):
    """Simulated ranks, one stream each, three consecutive steps (both gather buffers and
    epoch wrap of the alternation): every rank's gathered output == single-GPU decode."""
    from paper_2309_06180_b200.tp import FusedTP
    from synth import make_config
    wl = make_config(name, S=24, H=8, H_kv=8)
    ref, _, _ = _reference(wl)
    _assert_oracle(ref, wl, "single-GPU decode")
    ranks = FusedTP.local_group(world, wl.S, wl.H, wl.D, ref.dtype)
    try:
        ins = [_rank_inputs(wl, r, world) for r in range(world)]
        streams = [torch.cuda.Stream() for _ in range(world)]
        torch.cuda.synchronize()
        for step in range(3):
            outs = []
            for r in range(world):
                sh, x, tb = ins[r]
                if step > 0:  # fresh caches each step: the step writes its token into them
                    _, x, tb = _rank_inputs(wl, r, world)
                    ins[r] = (sh, x, tb)
                with torch.cuda.stream(streams[r]):
                    outs.append(ranks[r].decode(x["query"], x["key"], x["value"], x["key_cache"], x["value_cache"],
                                                tb["block_tables"], tb["context_lens"], sh.scale,
                                                max_context_len=sh.max_context_len))
            torch.cuda.synchronize()
            for r in range(world):
                assert int(ranks[r].status.item()) == 0, "flag wait timed out"
                assert torch.equal(outs[r], ref), f"step {step} rank {r}"
            _assert_oracle(outs[world - 1], wl, f"step {step} gathered on rank {world - 1}")
    finally:
        for rk in ranks:
            rk.close()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _ipc_worker(rank, world, port, name, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), PA_TP_TIMEOUT_MS="20000")
    import torch.distributed as dist

    from paper_2309_06180_b200.tp import FusedTP
    from synth import make_config
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ok = False
    try:
        torch.cuda.set_device(0)
        wl = make_config(name, S=24, H=8, H_kv=8)
        dt = {"f16": torch.float16, "bf16": torch.bfloat16, "f32": torch.float32}[wl.dtype]
        tp = FusedTP(None, wl.S, wl.H, wl.D, dt, "cuda:0")
        res = []
        for step in range(2):
            sh, x, tb = _rank_inputs(wl, rank, world)
            out = tp.decode(x["query"], x["key"], x["value"], x["key_cache"], x["value_cache"], tb["block_tables"],
                            tb["context_lens"], sh.scale, max_context_len=sh.max_context_len)
            torch.cuda.synchronize()
            res.append((out.cpu().view(torch.int16).numpy().copy(), int(tp.status.item())))  # numpy: pickled by value
            dist.barrier()  # both ranks done reading before the buffers are reused
        tp.close()
        q.put((rank, res))
        ok = True
    finally:
        if not ok:
            q.put((rank, None))
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["c2_sharegpt"])
def test_two_processes_ipc_gather_bitwise(name):
    """Two processes on the same GPU exchange IPC handles over gloo; each rank's kernel
    writes into both processes' buffers: both gathered outputs == single-GPU decode."""
    from synth import make_config
    wl = make_config(name, S=24, H=8, H_kv=8)
    ref, _, _ = _reference(wl)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, name, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    assert all(v is not None for v in got.values()), "a rank failed"
    ref_bits = ref.cpu().view(torch.int16).numpy()
    for r, res in got.items():
        for out, status in res:
            assert status == 0
            assert np.array_equal(out, ref_bits), f"rank {r}"
            _assert_oracle(torch.from_numpy(out).view(ref.dtype), wl, f"rank {r} (IPC)")


def test_nccl_gather_heads_world1_vs_oracle():
    """gather_heads through a real NCCL communicator on CUDA tensors (world 1: one GPU in
    this run) after the fused decode; the gathered output equals the oracle."""
    import torch.distributed as dist

    import paper_2309_06180_b200 as pa
    from paper_2309_06180_b200.tp import gather_heads
    from synth import make_config, materialize_torch, tables_torch
    wl = make_config("c2_sharegpt", S=16, H=8, H_kv=8)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        x = materialize_torch(wl, "cuda")
        tb = tables_torch(wl, "cuda")
        out = torch.empty_like(x["query"])
        pa.paged_attention_decode(out, x["query"], x["key"], x["value"], x["key_cache"], x["value_cache"],
                                  tb["block_tables"], tb["context_lens"], wl.scale, max_context_len=wl.max_context_len)
        full = gather_heads(out)
        torch.cuda.synchronize()
        assert full.is_cuda and torch.equal(full, out)
        _assert_oracle(full, wl, "NCCL world 1")
    finally:
        dist.destroy_process_group()


def _gloo_cuda_worker(rank, world, port, name, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    import paper_2309_06180_b200 as pa
    from paper_2309_06180_b200.tp import gather_heads
    from synth import make_config
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ok = False
    try:
        torch.cuda.set_device(0)
        wl = make_config(name, S=24, H=8, H_kv=8)
        sh, x, tb = _rank_inputs(wl, rank, world)
        out = torch.empty_like(x["query"])
        pa.paged_attention_decode(out, x["query"], x["key"], x["value"], x["key_cache"], x["value_cache"],
                                  tb["block_tables"], tb["context_lens"], sh.scale, max_context_len=sh.max_context_len)
        full = gather_heads(out)  # CUDA tensors through the torch.distributed all-gather
        torch.cuda.synchronize()
        if rank == 0:
            q.put(full.cpu().view(torch.int16).numpy().copy())
        ok = True
    finally:
        if not ok and rank == 0:
            q.put(None)
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["c2_sharegpt", "c5_beam"])
def test_two_processes_gather_heads_cuda_vs_oracle(name):
    """Two ranks (processes sharing the GPU), each running its head shard's decode on its
    own cache slice; gather_heads of the CUDA outputs == single-GPU decode bit for bit and
    == the fp64 oracle within tolerance."""
    from synth import make_config
    wl = make_config(name, S=24, H=8, H_kv=8)
    ref, _, _ = _reference(wl)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_cuda_worker, args=(r, 2, port, name, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
    assert got is not None, "a rank failed"
    assert np.array_equal(got, ref.cpu().view(torch.int16).numpy())
    _assert_oracle(torch.from_numpy(got).view(ref.dtype), wl, "gather_heads over 2 processes")

"""Head-sharded (tensor-parallel) decode on 2 CPU ranks over gloo: each rank runs the
fp64 oracle on its head shard of the same seeded workload (identical block tables,
its own kv-head slice of the cache) and the all-gather of the output head
slices (BJ:north_star) reassembles exactly the unsharded output."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, name, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    from paper_2309_06180_b200.tp import gather_heads, head_range
    from synth import make_config, shard
    from tests.pathutil import oracle_step
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ok = False
    try:
        wl = make_config(name, S=12, H=4, H_kv=4)
        sh = shard(wl, rank, world)
        assert (sh.q_head0, sh.q_head0 + sh.H) == head_range(wl.H, world, rank)
        out, kc, vc = oracle_step(sh)
        full = gather_heads(torch.from_numpy(out))
        if rank == 0:
            ref, _, _ = oracle_step(wl)
            q.put((full.numpy(), ref))
        ok = True
    finally:
        if not ok and rank == 0:
            q.put(None)
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["c2_sharegpt", "c5_beam"])
def test_two_rank_head_sharding_reassembles_bitwise(name):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got is not None
    full, ref = got
    assert np.array_equal(full, ref)


def test_head_range_rejects_uneven():
    from paper_2309_06180_b200.tp import head_range
    assert head_range(40, 8, 3) == (15, 20)
    with pytest.raises(ValueError):
        head_range(40, 3, 0)

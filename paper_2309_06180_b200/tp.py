"""Tensor-parallel head sharding of the decode attention.

Megatron-style SPMD: rank r of P owns the contiguous query heads [r*H/P, (r+1)*H/P)
and the matching kv heads; every rank holds the same block tables, context lengths and
slot mapping (the paper's single KV cache manager) and its own
[NB][H_kv/P][B][D] caches.  The only exchange is an all-gather of the per-rank output
head slices (BJ:north_star), NCCL over NVLink on B200s; any torch.distributed backend
works (gloo in the CPU tests).

`FusedTP` is the fused path: the attention kernel of every rank stores
its output rows straight into every rank's gather buffer through CUDA IPC peer pointers
(NVLink on a B200 node), followed by a one-warp flag handshake -- no NCCL call and no
permute on the hot path (`pa_paged_attention_decode_tp`, include/pa.h).  torch.distributed
is used once, at construction, to exchange the IPC handles.
"""
from __future__ import annotations

import ctypes

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


class _DevBuf:
    """A whole cudaMalloc allocation (IPC handles of it map to offset 0)."""

    def __init__(self, nbytes: int):
        from . import _lib
        self.ptr = ctypes.c_void_p()
        _lib.check(_lib.raw().pa_device_alloc(nbytes, ctypes.byref(self.ptr)), "pa_device_alloc")
        self.nbytes = nbytes

    def free(self):
        from . import _lib
        if self.ptr:
            _lib.check(_lib.raw().pa_device_free(self.ptr), "pa_device_free")
            self.ptr = ctypes.c_void_p()


def _as_tensor(ptr: int, shape, dtype, device) -> torch.Tensor:
    """Zero-copy torch view of device memory owned by this module (via __cuda_array_interface__)."""
    class _Holder:
        pass
    h = _Holder()
    typestr = {torch.float16: "<f2", torch.bfloat16: "<V2", torch.float32: "<f4", torch.int32: "<i4"}[dtype]
    h.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                  "version": 2, "strides": None}
    if dtype == torch.bfloat16:  # no numpy-style bf16 typestr: view int16 storage as bf16
        h.__cuda_array_interface__["typestr"] = "<i2"
        return torch.as_tensor(h, device=device).view(torch.bfloat16)
    return torch.as_tensor(h, device=device)


class FusedTP:
    """Fused tensor-parallel decode attention for `world` ranks (one per process, or, for
    tests, `world` simulated ranks in one process via `FusedTP.local_group`).

    Each rank owns two gather buffers [S][H_total][D] and an int32[world] flag array in
    whole cudaMalloc allocations; the handles are exchanged once over `group` (any
    torch.distributed backend) and opened with CUDA IPC.  decode(...) returns the gathered
    [S][H_total][D] output (a view of one of this rank's two alternating buffers)."""

    def __init__(self, group, S: int, H_total: int, D: int, dtype: torch.dtype, device=None,
                 _peer_ptrs=None, _rank=None, _world=None):
        from . import _lib
        self._lib = _lib
        self.device = torch.device(device or "cuda")
        self.world = _world if _world is not None else dist.get_world_size(group)
        self.rank = _rank if _rank is not None else dist.get_rank(group)
        self.S, self.H, self.D, self.dtype = S, H_total, D, dtype
        esz = torch.tensor([], dtype=dtype).element_size()
        self.out_bytes = S * H_total * D * esz
        self._opened = []
        if _peer_ptrs is None:
            # every rank takes part in every collective below even if its own step fails,
            # and all ranks agree on the outcome (raise everywhere or nowhere)
            self.bufs, mine, err = None, None, None
            try:
                self.bufs = [_DevBuf(self.out_bytes), _DevBuf(self.out_bytes), _DevBuf(4 * self.world + 4)]
                flags = _as_tensor(self.bufs[2].ptr.value, (self.world + 1,), torch.int32, self.device)
                flags.zero_()
                torch.cuda.synchronize(self.device)
                nb = _lib.raw().pa_ipc_handle_bytes()
                mine = []
                for b in self.bufs:
                    hb = ctypes.create_string_buffer(nb)
                    _lib.check(_lib.raw().pa_ipc_get_handle(b.ptr, hb), "pa_ipc_get_handle")
                    mine.append(hb.raw)
            except Exception as exc:  # noqa: BLE001 -- reported to every rank below
                err, mine = f"{type(exc).__name__}: {exc}", None
            allh = [None] * self.world
            dist.all_gather_object(allh, mine, group=group)
            peers = []
            if err is None and all(h is not None for h in allh):
                try:
                    nb = _lib.raw().pa_ipc_handle_bytes()
                    for k in range(self.world):
                        if k == self.rank:
                            peers.append([b.ptr.value for b in self.bufs])
                            continue
                        ptrs = []
                        for hbytes in allh[k]:
                            p = ctypes.c_void_p()
                            _lib.check(_lib.raw().pa_ipc_open_handle(ctypes.create_string_buffer(hbytes, nb),
                                                                      ctypes.byref(p)), "pa_ipc_open_handle")
                            self._opened.append(p)
                            ptrs.append(p.value)
                        peers.append(ptrs)
                except Exception as exc:  # noqa: BLE001
                    err = f"{type(exc).__name__}: {exc}"
            elif err is None:
                err = "a peer failed to create its buffers"
            errs = [None] * self.world
            dist.all_gather_object(errs, err, group=group)
            if any(e is not None for e in errs):
                self.close()
                raise RuntimeError("fused TP setup failed: " + "; ".join(f"rank {k}: {e}" for k, e in
                                                                         enumerate(errs) if e is not None))
        else:  # simulated ranks in one process: peers = [[gather_a, gather_b, flags_with_status], ...]
            self.bufs = None
            peers = _peer_ptrs
        self.peers = peers
        arr = lambda xs: (ctypes.c_void_p * self.world)(*xs)  # noqa: E731
        own_flags = peers[self.rank][2]
        self.status_ptr = own_flags + 4 * self.world  # int32 right after the flag array
        self.comm = _lib.raw().pa_tp_comm_create(self.world, self.rank, H_total, self.out_bytes,
                                                 arr([p[0] for p in peers]), arr([p[1] for p in peers]),
                                                 arr([p[2] for p in peers]), ctypes.c_void_p(self.status_ptr))
        if not self.comm:
            raise _lib.PagedAttnError(_lib.last_error())
        self.views = [_as_tensor(peers[self.rank][i], (S, H_total, D), dtype, self.device) for i in (0, 1)]
        self.status = _as_tensor(self.status_ptr, (1,), torch.int32, self.device)

    @staticmethod
    def local_group(world: int, S: int, H_total: int, D: int, dtype: torch.dtype, device=None):
        """`world` simulated ranks in ONE process on one GPU (tests): every rank's buffers
        are local allocations; rank k's FusedTP gets all of them as its peers."""
        esz = torch.tensor([], dtype=dtype).element_size()
        nbytes = S * H_total * D * esz
        bufs = [[_DevBuf(nbytes), _DevBuf(nbytes), _DevBuf(4 * world + 4)] for _ in range(world)]
        for b in bufs:
            _as_tensor(b[2].ptr.value, (world + 1,), torch.int32, torch.device(device or "cuda")).zero_()
        peers = [[b.ptr.value for b in bb] for bb in bufs]
        ranks = [FusedTP(None, S, H_total, D, dtype, device, _peer_ptrs=peers, _rank=r, _world=world)
                 for r in range(world)]
        ranks[0]._owned = bufs  # keep the allocations alive with rank 0
        return ranks

    def decode(self, query, key, value, key_cache, value_cache, block_tables, context_lens, scale: float,
               max_context_len: int = 0, workspace: torch.Tensor | None = None, stream=None,
               seq_order=None) -> torch.Tensor:
        """The decode step (cache write fused) on this rank's heads; returns the gathered
        [S][H_total][D] output, a view of one of the two alternating gather buffers.  It is
        valid until this rank's NEXT decode call: read it (on the same stream) before
        issuing that call (include/pa.h)."""
        from .ops import _code, _dev, _order, _stream, paged_attention_workspace_size
        S, H, D = query.shape
        if S > self.S or H * self.world != self.H or D != self.D or query.dtype != self.dtype:
            raise ValueError(f"FusedTP built for <= {self.S} sequences x {self.H} heads ({self.H // self.world} per "
                             f"rank) x {self.D} dims, {self.dtype}; got query {tuple(query.shape)} {query.dtype}")
        _, hk, B, _ = key_cache.shape
        W = block_tables.shape[1]
        mcl = max_context_len if max_context_len > 0 else W * B
        need = paged_attention_workspace_size(S, H, D, mcl, 0)
        if workspace is None and need > 0:
            workspace = torch.empty(need, dtype=torch.uint8, device=query.device)
        ws_ptr = _dev(workspace, "workspace") if workspace is not None else None
        ws_bytes = workspace.numel() * workspace.element_size() if workspace is not None else 0
        buf = ctypes.c_int(-1)
        self._lib.check(self._lib.raw().pa_paged_attention_decode_tp(
            self.comm, ctypes.byref(buf), _dev(query, "query"), _dev(key, "key"), _dev(value, "value"),
            _dev(key_cache, "key_cache"), _dev(value_cache, "value_cache"), _dev(block_tables, "block_tables"),
            _dev(context_lens, "context_lens"), float(scale), B, hk, S, H, D, W, int(mcl), _code(query),
            _order(seq_order, S), ws_ptr, ws_bytes, _stream(stream)), "pa_paged_attention_decode_tp")
        return self.views[buf.value][:S]

    def close(self):
        if getattr(self, "comm", None):
            self._lib.raw().pa_tp_comm_destroy(self.comm)
            self.comm = None
        for p in self._opened:
            self._lib.raw().pa_ipc_close_handle(p)
        self._opened = []
        if self.bufs:
            for b in self.bufs:
                b.free()
            self.bufs = None
        for bb in getattr(self, "_owned", []) or []:
            for b in bb:
                b.free()
        self._owned = None

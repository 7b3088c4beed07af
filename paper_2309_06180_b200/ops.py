"""Torch-tensor front end of libpagedattn.so -- argument marshalling only.

Same names as the C ABI (include/pa.h) without the ``pa_`` prefix.  Shapes are read
from the tensors, pointers and the current CUDA stream are passed through; every
computation happens in the library's sm_100a kernels.  P:N = PAPER.md line N.
"""
from __future__ import annotations

import ctypes
import threading

import torch

from . import _lib
from ._lib import check

_DT = {torch.float32: _lib.PA_F32, torch.float16: _lib.PA_F16, torch.bfloat16: _lib.PA_BF16}


def _code(t: torch.Tensor) -> int:
    try:
        return _DT[t.dtype]
    except KeyError:
        raise TypeError(f"unsupported dtype {t.dtype}") from None


def _dev(t: torch.Tensor, name: str) -> int:
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t.data_ptr()


def _check(dtype=None, idx32=(), idx64=(), **tensors):
    """Host-side type checks the C ABI cannot make (it sees raw pointers): every named
    value tensor in `tensors` has `dtype` (the query's) and the same head_dim (last dim);
    index tensors are int32 (block tables, context lengths) / int64 (slot and block
    mappings).  An int32 mapping read as int64 pairs would address garbage blocks."""
    D = None
    for name, t in tensors.items():
        if t is None:
            continue
        if dtype is not None and t.dtype != dtype:
            raise TypeError(f"{name} is {t.dtype}, expected {dtype} (query / caches share one dtype)")
        if D is None:
            D = t.shape[-1]
        elif t.shape[-1] != D:
            raise ValueError(f"{name} has head_dim {t.shape[-1]}, expected {D}")
    for name, t in idx32:
        if t.dtype != torch.int32:
            raise TypeError(f"{name} must be int32 (got {t.dtype})")
    for name, t in idx64:
        if t.dtype != torch.int64:
            raise TypeError(f"{name} must be int64 (got {t.dtype})")


_CAPTURE = threading.local()


def _call(name: str, args: tuple):
    """Issue C entry point `name` -- or, inside prepare(), hand the marshalled call back."""
    f = getattr(_lib.raw(), name)
    if getattr(_CAPTURE, "on", False):
        _CAPTURE.got = (f, args, name)
        return
    check(f(*args), name)


def prepare(fn, *args, **kwargs):
    """A zero-argument callable that re-issues ``fn(*args, **kwargs)`` -- one of this
    module's launch entry points -- with the Python-side checks and marshalling done once:
    same pointers, sizes and stream (captured now; the tensors are kept alive by the
    callable).  For launch-bound loops such as bench.py's timed region, where the
    per-call Python overhead would otherwise approach a short kernel's duration."""
    _CAPTURE.on, _CAPTURE.got = True, None
    try:
        fn(*args, **kwargs)
        got = _CAPTURE.got
    finally:
        _CAPTURE.on = False
    if got is None:
        raise ValueError(f"{getattr(fn, '__name__', fn)} issued no library call (nothing to prepare)")
    f, cargs, name = got
    keep = (args, kwargs)

    def run():
        st = f(*cargs)
        if st:
            raise _lib.PagedAttnError(st, name)
        return keep

    return run


def _stream(stream) -> int:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def paged_attention_workspace_size(num_seqs: int, num_heads: int, head_dim: int, max_context_len: int,
                                   partition_tokens: int = 0) -> int:
    return int(_lib.raw().pa_paged_attention_workspace_size(num_seqs, num_heads, head_dim, max_context_len,
                                                           partition_tokens))


def decode_plan(context_lens) -> "np.ndarray":
    """pa_decode_plan: the longest-first grid order (int32 numpy [S]) of a batch, from its
    HOST context lengths (numpy / CPU tensor / list).  Scheduling only: pass it as
    `seq_order` to the decode entries, once per decode iteration for every layer."""
    import numpy as np
    cl = np.ascontiguousarray(np.asarray(context_lens.cpu() if hasattr(context_lens, "cpu") else context_lens,
                                         dtype=np.int32))
    order = np.empty(cl.shape[0], dtype=np.int32)
    check(_lib.raw().pa_decode_plan(cl.ctypes.data, cl.shape[0], order.ctypes.data), "pa_decode_plan")
    return order


def _order(seq_order, S: int):
    """Host int32 copy of a grid order (kept alive by the marshalled arguments) or None."""
    if seq_order is None:
        return None
    vals = seq_order.cpu().tolist() if hasattr(seq_order, "cpu") else list(seq_order)
    if len(vals) != S:
        raise ValueError(f"seq_order has {len(vals)} entries for {S} sequences")
    return (ctypes.c_int32 * S)(*[int(v) for v in vals])


def paged_attention(out, query, key_cache, value_cache, block_tables, context_lens, scale: float,
                    block_size: int | None = None, num_kv_heads: int | None = None, max_context_len: int = 0,
                    partition_tokens: int = 0, workspace: torch.Tensor | None = None, stream=None, seq_order=None):
    """Eq.4 decode attention: out[s][h] = softmax(scale q.K^T) V over the
    block-table-addressed cache.  out/query [S][H][D]; caches [NB][H_kv][B][D];
    block_tables int32 [S][W]; context_lens int32 [S].  `workspace` (uint8, device, any
    content; see pa.h) is allocated when omitted and the context needs splitting.
    `seq_order`: optional host grid order (decode_plan); scheduling only."""
    _check(query.dtype, [("block_tables", block_tables), ("context_lens", context_lens)], out=out, query=query,
           key_cache=key_cache, value_cache=value_cache)
    S, H, D = query.shape
    _, hk, B, _ = key_cache.shape
    block_size = B if block_size is None else block_size
    num_kv_heads = hk if num_kv_heads is None else num_kv_heads
    W = block_tables.shape[1]
    mcl = max_context_len if max_context_len > 0 else W * block_size
    need = paged_attention_workspace_size(S, H, D, mcl, partition_tokens)
    if workspace is None and need > 0:
        workspace = torch.empty(need, dtype=torch.uint8, device=query.device)
    ws_ptr = _dev(workspace, "workspace") if workspace is not None else None
    ws_bytes = workspace.numel() * workspace.element_size() if workspace is not None else 0
    _call("pa_paged_attention_ex", (
        _dev(out, "out"), _dev(query, "query"), _dev(key_cache, "key_cache"), _dev(value_cache, "value_cache"),
        _dev(block_tables, "block_tables"), _dev(context_lens, "context_lens"), float(scale), int(block_size),
        int(num_kv_heads), S, H, D, W, int(mcl), _code(query), int(partition_tokens), _order(seq_order, S), ws_ptr,
        ws_bytes, _stream(stream)))
    return out


def paged_attention_decode(out, query, key, value, key_cache, value_cache, block_tables, context_lens, scale: float,
                           max_context_len: int = 0, workspace: torch.Tensor | None = None, stream=None,
                           seq_order=None):
    """The decode step's reshape_and_cache fused into paged_attention (pa.h): token s
    (key/value [S][H_kv][D]) is written at logical position ctx[s]-1 and attended.
    `seq_order`: optional host grid order (decode_plan); scheduling only."""
    _check(query.dtype, [("block_tables", block_tables), ("context_lens", context_lens)], out=out, query=query,
           key=key, value=value, key_cache=key_cache, value_cache=value_cache)
    S, H, D = query.shape
    _, hk, B, _ = key_cache.shape
    W = block_tables.shape[1]
    mcl = max_context_len if max_context_len > 0 else W * B
    need = paged_attention_workspace_size(S, H, D, mcl, 0)
    if workspace is None and need > 0:
        workspace = torch.empty(need, dtype=torch.uint8, device=query.device)
    ws_ptr = _dev(workspace, "workspace") if workspace is not None else None
    ws_bytes = workspace.numel() * workspace.element_size() if workspace is not None else 0
    _call("pa_paged_attention_decode", (
        _dev(out, "out"), _dev(query, "query"), _dev(key, "key"), _dev(value, "value"), _dev(key_cache, "key_cache"),
        _dev(value_cache, "value_cache"), _dev(block_tables, "block_tables"), _dev(context_lens, "context_lens"),
        float(scale), B, hk, S, H, D, W, int(mcl), _code(query), _order(seq_order, S), ws_ptr, ws_bytes,
        _stream(stream)))
    return out


def paged_attention_decode_shared(out, query, key, value, key_cache, value_cache, block_tables, context_lens,
                                  scale: float, group_size: int, max_context_len: int = 0,
                                  workspace: torch.Tensor | None = None, stream=None):
    """paged_attention_decode for sequence groups sharing blocks (parallel samples, beams):
    each distinct block of a group is read once per logical tile (pa.h)."""
    _check(query.dtype, [("block_tables", block_tables), ("context_lens", context_lens)], out=out, query=query,
           key=key, value=value, key_cache=key_cache, value_cache=value_cache)
    S, H, D = query.shape
    _, hk, B, _ = key_cache.shape
    W = block_tables.shape[1]
    mcl = max_context_len if max_context_len > 0 else W * B
    need = paged_attention_workspace_size(S, H, D, mcl, 0)
    if workspace is None and need > 0:
        workspace = torch.empty(need, dtype=torch.uint8, device=query.device)
    ws_ptr = _dev(workspace, "workspace") if workspace is not None else None
    ws_bytes = workspace.numel() * workspace.element_size() if workspace is not None else 0
    _call("pa_paged_attention_decode_shared", (
        _dev(out, "out"), _dev(query, "query"), _dev(key, "key"), _dev(value, "value"), _dev(key_cache, "key_cache"),
        _dev(value_cache, "value_cache"), _dev(block_tables, "block_tables"), _dev(context_lens, "context_lens"),
        float(scale), B, hk, S, H, D, W, int(mcl), int(group_size), _code(query), ws_ptr, ws_bytes, _stream(stream)))
    return out


def paged_attention_decode_grouped(out, query, key, value, key_cache, value_cache, block_tables, context_lens,
                                   scale: float, group_size: int, max_context_len: int = 0,
                                   workspace: torch.Tensor | None = None, stream=None, seq_order=None):
    """The sharing-aware decode step on the tcgen05 tensor cores (pa.h):
    groups of group_size consecutive sequences; each distinct block piece of a group is
    loaded once and Q K^T / P V run as tcgen05 MMAs over the group's rows.  f16/bf16,
    D = 128, block_size >= 16.  `seq_order`: optional host grid order (decode_plan)."""
    _check(query.dtype, [("block_tables", block_tables), ("context_lens", context_lens)], out=out, query=query,
           key=key, value=value, key_cache=key_cache, value_cache=value_cache)
    S, H, D = query.shape
    NB, hk, B, _ = key_cache.shape
    W = block_tables.shape[1]
    mcl = max_context_len if max_context_len > 0 else W * B
    need = paged_attention_workspace_size(S, H, D, mcl, 0)
    if workspace is None and need > 0:
        workspace = torch.empty(need, dtype=torch.uint8, device=query.device)
    ws_ptr = _dev(workspace, "workspace") if workspace is not None else None
    ws_bytes = workspace.numel() * workspace.element_size() if workspace is not None else 0
    _call("pa_paged_attention_decode_grouped", (
        _dev(out, "out"), _dev(query, "query"), _dev(key, "key"), _dev(value, "value"), _dev(key_cache, "key_cache"),
        _dev(value_cache, "value_cache"), _dev(block_tables, "block_tables"), _dev(context_lens, "context_lens"),
        float(scale), B, hk, NB, S, H, D, W, int(mcl), int(group_size), _code(query), _order(seq_order, S), ws_ptr,
        ws_bytes, _stream(stream)))
    return out


PREFILL_WORKSPACE_BYTES = 16


def _host_i32(x, name):
    import numpy as np
    a = np.ascontiguousarray(np.asarray(x.cpu() if hasattr(x, "cpu") else x, dtype=np.int32))
    return a


def paged_prefill_attention_packed(out, query, key_cache, value_cache, block_tables, context_lens, query_start,
                                   scale: float, host_query_start, host_context_lens, host_shared_prefix,
                                   max_query_len: int = 0, workspace: torch.Tensor | None = None, stream=None):
    """pa_paged_prefill_attention_packed (pa.h): requests sharing a cached prefix packed into
    128-row query tiles, the prefix attended once per tile (cascade).  The host_* arrays
    (numpy / CPU tensors / lists): query_start [S+1], context_lens [S], and per sequence the
    number of leading tokens it shares with the previous one (same physical blocks)."""
    _check(query.dtype, [("block_tables", block_tables), ("context_lens", context_lens),
                         ("query_start", query_start)], out=out, query=query, key_cache=key_cache,
           value_cache=value_cache)
    T, H, D = query.shape
    NB, hk, B, _ = key_cache.shape
    S, W = block_tables.shape
    hqs, hcl, hsp = (_host_i32(host_query_start, "host_query_start"), _host_i32(host_context_lens, "host_context_lens"),
                     _host_i32(host_shared_prefix, "host_shared_prefix"))
    if hqs.shape[0] != S + 1 or hcl.shape[0] != S or hsp.shape[0] != S:
        raise ValueError("host arrays must have S+1, S and S entries")
    if max_query_len <= 0:
        max_query_len = int((hqs[1:] - hqs[:-1]).max()) if S > 0 else 0
    if workspace is None:
        workspace = torch.empty(PREFILL_WORKSPACE_BYTES, dtype=torch.uint8, device=query.device)
    _call("pa_paged_prefill_attention_packed", (
        _dev(out, "out"), _dev(query, "query"), _dev(key_cache, "key_cache"), _dev(value_cache, "value_cache"),
        _dev(block_tables, "block_tables"), _dev(context_lens, "context_lens"), _dev(query_start, "query_start"),
        hqs.ctypes.data, hcl.ctypes.data, hsp.ctypes.data, float(scale), B, hk, NB, S, H, D, W, T,
        int(max_query_len), _code(query), _dev(workspace, "workspace"), workspace.numel() * workspace.element_size(),
        _stream(stream)))
    return out


def paged_prefill_attention(out, query, key_cache, value_cache, block_tables, context_lens, query_start,
                            scale: float, max_query_len: int = 0, workspace: torch.Tensor | None = None,
                            stream=None):
    """Causal multi-token attention over the paged cache (pa.h):
    query/out [T][H][D] with sequence s's rows in [query_start[s], query_start[s+1]), the
    last q_len of its context_lens[s] cached tokens.  tcgen05 tensor cores, f16/bf16, D=128.
    max_query_len sizes the grid; 0 reads it from query_start (a device->host sync).
    `workspace` (uint8 device tensor, >= 16 bytes, any content) holds the work-item
    counter; allocated per call when omitted."""
    _check(query.dtype, [("block_tables", block_tables), ("context_lens", context_lens),
                         ("query_start", query_start)], out=out, query=query, key_cache=key_cache,
           value_cache=value_cache)
    T, H, D = query.shape
    NB, hk, B, _ = key_cache.shape
    S, W = block_tables.shape
    if max_query_len <= 0:
        max_query_len = int((query_start[1:] - query_start[:-1]).max().item()) if S > 0 else 0
    if workspace is None:
        workspace = torch.empty(PREFILL_WORKSPACE_BYTES, dtype=torch.uint8, device=query.device)
    _call("pa_paged_prefill_attention", (
        _dev(out, "out"), _dev(query, "query"), _dev(key_cache, "key_cache"), _dev(value_cache, "value_cache"),
        _dev(block_tables, "block_tables"), _dev(context_lens, "context_lens"), _dev(query_start, "query_start"),
        float(scale), B, hk, NB, S, H, D, W, T, int(max_query_len), _code(query), _dev(workspace, "workspace"),
        workspace.numel() * workspace.element_size(), _stream(stream)))
    return out


def reshape_and_cache(key, value, key_cache, value_cache, slot_mapping, stream=None):
    """Fused reshape + block write: key/value [T][H_kv][D] into the caches at
    slot_mapping (int64 [T], -1 = skip)."""
    _check(key.dtype, idx64=[("slot_mapping", slot_mapping)], key=key, value=value, key_cache=key_cache,
           value_cache=value_cache)
    T, hk, D = key.shape
    B = key_cache.shape[2]
    _call("pa_reshape_and_cache", (
        _dev(key, "key"), _dev(value, "value"), _dev(key_cache, "key_cache"), _dev(value_cache, "value_cache"),
        _dev(slot_mapping, "slot_mapping"), T, hk, D, B, _code(key), _stream(stream)))


def copy_blocks(key_caches, value_caches, block_mapping, stream=None):
    """Fused copy-on-write block copy over every layer in one launch.
    block_mapping: int64 [P][2] (src, dst) on the device."""
    _check(key_caches[0].dtype, idx64=[("block_mapping", block_mapping)],
           **{f"key_caches[{i}]": k for i, k in enumerate(key_caches)},
           **{f"value_caches[{i}]": v for i, v in enumerate(value_caches)})
    L = len(key_caches)
    kp = (ctypes.c_void_p * L)(*[_dev(k, "key_caches[i]") for k in key_caches])
    vp = (ctypes.c_void_p * L)(*[_dev(v, "value_caches[i]") for v in value_caches])
    _, hk, B, D = key_caches[0].shape
    P = block_mapping.shape[0] if block_mapping.numel() else 0
    bm = _dev(block_mapping, "block_mapping") if P else None
    _call("pa_copy_blocks", (kp, vp, L, bm, P, hk, B, D, _code(key_caches[0]), _stream(stream)))


def _dev_or_pinned(t: torch.Tensor, name: str) -> int:
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if t.is_cuda or t.is_pinned():
        return t.data_ptr()
    raise ValueError(f"{name} must be a CUDA tensor or pinned host memory")


def swap_blocks(dst_key_caches, dst_value_caches, src_key_caches, src_value_caches, block_mapping, stream=None):
    """Swap blocks between pools: dst[l][d] <- src[l][s] for every (s, d) pair in
    block_mapping (int64 [P][2], device or pinned host) and layer, one launch.  Pools may be
    device tensors or pinned host tensors (the CPU swap pool)."""
    pools = list(dst_key_caches) + list(dst_value_caches) + list(src_key_caches) + list(src_value_caches)
    _check(dst_key_caches[0].dtype, idx64=[("block_mapping", block_mapping)],
           **{f"pool[{i}]": t for i, t in enumerate(pools)})
    L = len(dst_key_caches)
    arr = lambda xs, n: (ctypes.c_void_p * L)(*[_dev_or_pinned(x, n) for x in xs])  # noqa: E731
    _, hk, B, D = dst_key_caches[0].shape
    P = block_mapping.shape[0] if block_mapping.numel() else 0
    bm = _dev_or_pinned(block_mapping, "block_mapping") if P else None
    check(_lib.raw().pa_swap_blocks(arr(dst_key_caches, "dst_key"), arr(dst_value_caches, "dst_value"),
                                    arr(src_key_caches, "src_key"), arr(src_value_caches, "src_value"), L, bm, P, hk,
                                    B, D, _code(dst_key_caches[0]), _stream(stream)), "pa_swap_blocks")


def swap_blocks_memcpy(dst_key_caches, dst_value_caches, src_key_caches, src_value_caches, host_block_mapping,
                       stream=None):
    """Benchmark baseline: the same transfer as one cudaMemcpyAsync per (pair, layer, K/V)."""
    L = len(dst_key_caches)
    arr = lambda xs, n: (ctypes.c_void_p * L)(*[_dev_or_pinned(x, n) for x in xs])  # noqa: E731
    _, hk, B, D = dst_key_caches[0].shape
    bm = host_block_mapping.contiguous()
    check(_lib.raw().pa_swap_blocks_memcpy(arr(dst_key_caches, "dst_key"), arr(dst_value_caches, "dst_value"),
                                           arr(src_key_caches, "src_key"), arr(src_value_caches, "src_value"), L,
                                           bm.data_ptr(), bm.shape[0], hk, B, D, _code(dst_key_caches[0]),
                                           _stream(stream)), "pa_swap_blocks_memcpy")


def decode_step_staging_size(num_seqs, num_heads, num_kv_heads, head_dim, max_blocks_per_seq, num_pairs, dtype):
    return int(_lib.raw().pa_decode_step_staging_size(num_seqs, num_heads, num_kv_heads, head_dim,
                                                     max_blocks_per_seq, num_pairs, _DT[dtype]))


def _host(t: torch.Tensor, name: str) -> int:
    if t.is_cuda or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous host tensor")
    return t.data_ptr()


def decode_step(host_out, host_query, host_key, host_value, host_slot_mapping, host_block_tables,
                host_context_lens, host_block_mapping, key_cache, value_cache, scale: float, staging, workspace=None,
                max_context_len: int = 0, stream=None):
    """One decode step from HOST (pinned) inputs: H2D, copy_blocks, reshape_and_cache,
    paged_attention, D2H of out -- all enqueued on one stream (pa_decode_step)."""
    S, H, D = host_query.shape
    _, hk, B, _ = key_cache.shape
    W = host_block_tables.shape[1]
    P = host_block_mapping.shape[0] if host_block_mapping is not None and host_block_mapping.numel() else 0
    ws_ptr = _dev(workspace, "workspace") if workspace is not None else None
    ws_bytes = workspace.numel() if workspace is not None else 0
    check(_lib.raw().pa_decode_step(
        _host(host_out, "host_out"), _host(host_query, "host_query"), _host(host_key, "host_key"),
        _host(host_value, "host_value"), None,
        _host(host_block_tables, "host_block_tables"), _host(host_context_lens, "host_context_lens"),
        _host(host_block_mapping, "host_block_mapping") if P else None, P,
        _dev(key_cache, "key_cache"), _dev(value_cache, "value_cache"), float(scale), B, hk, S, H, D, W,
        int(max_context_len), _code(host_query), _dev(staging, "staging"), staging.numel(), ws_ptr, ws_bytes,
        _stream(stream)), "pa_decode_step")


def hbm_read_probe(buf: torch.Tensor, sink: torch.Tensor, chunk: int = 32768, stages: int = 4, ctas: int = 0,
                   stream=None):
    """Measurement helper (pa.h pa_hbm_read_probe): stream `buf` (device, contiguous,
    nbytes a multiple of `chunk`) into shared memory with bulk copies, writing only one
    word per CTA into `sink` (int32/uint32 device tensor with >= grid elements)."""
    nbytes = buf.numel() * buf.element_size()
    check(_lib.raw().pa_hbm_read_probe(_dev(buf, "buf"), nbytes, chunk, stages, ctas, _dev(sink, "sink"),
                                       _stream(stream)), "pa_hbm_read_probe")


def debug_gather_kv(key_cache, value_cache, block_tables, context_lens, max_ctx: int, stream=None):
    """Test-only: the logical K/V rows [S][H_kv][max_ctx][D] fetched by the attention
    kernel's own tile loader (block-table lookup + bulk copy)."""
    NB, hk, B, D = key_cache.shape
    S, W = block_tables.shape
    k_out = torch.zeros((S, hk, max_ctx, D), dtype=key_cache.dtype, device=key_cache.device)
    v_out = torch.zeros_like(k_out)
    check(_lib.raw().pa_debug_gather_kv(
        _dev(k_out, "k_out"), _dev(v_out, "v_out"), _dev(key_cache, "key_cache"), _dev(value_cache, "value_cache"),
        _dev(block_tables, "block_tables"), _dev(context_lens, "context_lens"), B, hk, S, D, W, max_ctx,
        _code(key_cache), _stream(stream)), "pa_debug_gather_kv")
    return k_out, v_out


def validate_tables(block_tables, context_lens, block_size: int, num_blocks: int, stream=None) -> int:
    S, W = block_tables.shape
    bad = ctypes.c_int64(-2)
    check(_lib.raw().pa_validate_tables(_dev(block_tables, "block_tables"), _dev(context_lens, "context_lens"), S, W,
                                        block_size, num_blocks, ctypes.byref(bad), _stream(stream)),
          "pa_validate_tables")
    return int(bad.value)


class BlockAllocator:
    """The paper's KV block manager in C++ (pa_alloc_*):
    allocate / append_slot / fork / free on a FIFO free list of physical block ids."""

    def __init__(self, num_blocks: int, block_size: int, initial_order=None):
        self.num_blocks, self.block_size = num_blocks, block_size
        arr = None
        if initial_order is not None:
            arr = (ctypes.c_int32 * num_blocks)(*[int(b) for b in initial_order])
        self._h = _lib.raw().pa_alloc_create(num_blocks, block_size, arr)
        if not self._h:
            raise ValueError("pa_alloc_create failed (bad sizes or initial_order not a permutation)")

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            _lib.raw().pa_alloc_destroy(h)
            self._h = None

    def allocate(self, num_tokens: int) -> int:
        out = ctypes.c_int(-1)
        check(_lib.raw().pa_alloc_allocate(self._h, num_tokens, ctypes.byref(out)), "pa_alloc_allocate")
        return out.value

    def append_slot(self, seq: int):
        """Returns (slot, cow) with cow = (src, dst) or None."""
        slot, src, dst = ctypes.c_int64(), ctypes.c_int(), ctypes.c_int()
        check(_lib.raw().pa_alloc_append_slot(self._h, seq, ctypes.byref(slot), ctypes.byref(src), ctypes.byref(dst)),
              "pa_alloc_append_slot")
        return slot.value, ((src.value, dst.value) if src.value >= 0 else None)

    def fork(self, parent: int) -> int:
        out = ctypes.c_int(-1)
        check(_lib.raw().pa_alloc_fork(self._h, parent, ctypes.byref(out)), "pa_alloc_fork")
        return out.value

    def free(self, seq: int) -> int:
        out = ctypes.c_int(0)
        check(_lib.raw().pa_alloc_free(self._h, seq, ctypes.byref(out)), "pa_alloc_free")
        return out.value

    def export(self, seqs, W: int):
        import numpy as np
        seqs = np.ascontiguousarray(seqs, dtype=np.int32)
        bt = np.empty((len(seqs), W), dtype=np.int32)
        cl = np.empty(len(seqs), dtype=np.int32)
        check(_lib.raw().pa_alloc_export(self._h, seqs.ctypes.data, len(seqs), W, bt.ctypes.data, cl.ctypes.data),
              "pa_alloc_export")
        return bt, cl

    def refcount(self, block: int) -> int:
        return int(_lib.raw().pa_alloc_refcount(self._h, block))

    def num_free(self) -> int:
        return int(_lib.raw().pa_alloc_num_free(self._h))

    def num_blocks_of(self, seq: int) -> int:
        return int(_lib.raw().pa_alloc_num_blocks_of(self._h, seq))

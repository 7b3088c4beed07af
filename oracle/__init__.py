"""fp64 CPU oracle for the PagedAttention decode hot path (arXiv 2309.06180).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this package.
It shares no code with the CUDA path (``paper_2309_06180_b200``) and never imports it.

The arithmetic lives in ``oracle.c`` (plain C, fp64, sequential loops); this module
only marshals numpy arrays into it.  ``block_manager.py`` is the plain-Python
reference of the paper's KV cache manager.

Functions and the passage they follow (P:N = PAPER.md line N):

- ``paged_attention``       Eq.4 over a block-table-addressed cache.
- ``contiguous_attention``  Eq.3 on already gathered K/V.
- ``gather_kv``             the contiguous K/V that Eq.3 assumes.
- ``split_attention``       per-partition (m, L, o~) + log-sum-exp merge (BJ:north_star).
- ``reshape_and_cache``     fused reshape + block write.
- ``copy_blocks``           fused block copy for copy-on-write.
- ``prefill_attention``     causal multi-token attention of the prompt phase / a shared
                            prefix's suffix over the paged cache.
- ``swap_blocks``           block transfers between the GPU pool and the CPU swap pool.
- ``decode``                storage dtype -> fp64, bit-exact (own fp16/bf16 decoders).

Parity pins: see tests/test_oracle.py; a function without a pin would be marked
"parity unpinned" here and in DESIGN.md -- every function above is pinned.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

F32, F16, BF16 = 0, 1, 2
_DT = {"f32": F32, "fp32": F32, "float32": F32, "f16": F16, "fp16": F16, "float16": F16,
       "bf16": BF16, "bfloat16": BF16}
_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so with gcc (fp64, -O2, OpenMP, no FMA contraction)."""
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        import subprocess
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-fPIC", "-shared", "-fopenmp",
                               "-ffp-contract=off", "-fno-fast-math", src, "-o", _LIB_PATH, "-lm"])
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        vp, i32, i64, d = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double
        L.oracle_decode.restype = d
        L.oracle_decode.argtypes = [ctypes.c_uint32, i32]
        L.oracle_decode_array.argtypes = [vp, i64, i32, vp]
        L.oracle_set_threads.argtypes = [i32]
        L.oracle_max_threads.restype = i32
        L.oracle_contiguous_attention.argtypes = [vp, vp, vp, vp, i32, i32, d]
        L.oracle_paged_attention.argtypes = [vp, vp, vp, vp, vp, vp, d, i32, i32, i32, i32, i32, i32, i32]
        L.oracle_split_attention.argtypes = [vp, vp, vp, vp, vp, vp, d, i32, i32, i32, i32, i32, i32, i32, i32]
        L.oracle_gather_kv.argtypes = [vp, vp, vp, vp, vp, i32, i32, i32, i32, i32, i32]
        L.oracle_gather_kv_bits.argtypes = [vp, vp, vp, vp, vp, i32, i32, i32, i32, i32, i32]
        L.oracle_reshape_and_cache.argtypes = [vp, vp, vp, vp, vp, i32, i32, i32, i32, i32]
        L.oracle_copy_blocks.argtypes = [vp, vp, i32, vp, i32, i32, i32, i32, i32, i32]
        L.oracle_swap_blocks.argtypes = [vp, vp, vp, vp, i32, vp, i32, i64]
        L.oracle_prefill_attention.argtypes = [vp, vp, vp, vp, vp, vp, vp, d, i32, i32, i32, i32, i32,
                                               i32, i32]
        _lib = L
    return _lib


def _dt(dtype) -> int:
    if isinstance(dtype, int):
        return dtype
    return _DT[str(dtype)]


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"], "oracle inputs must be C-contiguous"
    return a.ctypes.data_as(ctypes.c_void_p)


def _raw(a: np.ndarray) -> np.ndarray:
    """Storage arrays are passed as raw bit patterns (uint16 for f16/bf16, uint32/float32 for f32)."""
    return np.ascontiguousarray(a)


def set_threads(n: int) -> None:
    lib().oracle_set_threads(int(n))


def max_threads() -> int:
    return int(lib().oracle_max_threads())


def decode(bits: np.ndarray, dtype) -> np.ndarray:
    bits = _raw(bits)
    out = np.empty(bits.size, dtype=np.float64)
    lib().oracle_decode_array(_p(bits), bits.size, _dt(dtype), _p(out))
    return out.reshape(bits.shape)


def contiguous_attention(q: np.ndarray, K: np.ndarray, V: np.ndarray, scale: float) -> np.ndarray:
    q = np.ascontiguousarray(q, dtype=np.float64)
    K = np.ascontiguousarray(K, dtype=np.float64)
    V = np.ascontiguousarray(V, dtype=np.float64)
    n, D = K.shape if K.ndim == 2 else (0, q.shape[0])
    out = np.empty(q.shape[0], dtype=np.float64)
    lib().oracle_contiguous_attention(_p(out), _p(q), _p(K), _p(V), int(n), int(D), float(scale))
    return out


def paged_attention(query, key_cache, value_cache, block_tables, context_lens, scale,
                    block_size, num_kv_heads, dtype) -> np.ndarray:
    """Eq.4.  query [S][H][D], caches [NB][H_kv][B][D] (raw bits), block_tables [S][W] int32,
    context_lens [S] int32.  Returns fp64 [S][H][D]."""
    query, key_cache, value_cache = _raw(query), _raw(key_cache), _raw(value_cache)
    bt = np.ascontiguousarray(block_tables, dtype=np.int32)
    cl = np.ascontiguousarray(context_lens, dtype=np.int32)
    S, H, D = query.shape
    out = np.empty((S, H, D), dtype=np.float64)
    lib().oracle_paged_attention(_p(out), _p(query), _p(key_cache), _p(value_cache), _p(bt), _p(cl),
                                 float(scale), int(block_size), int(num_kv_heads), S, H, D,
                                 int(bt.shape[1]), _dt(dtype))
    return out


def prefill_attention(query, key_cache, value_cache, block_tables, context_lens, query_start, scale,
                      block_size, num_kv_heads, dtype) -> np.ndarray:
    """Causal multi-token attention (P:140-147, P:334-338 with Eq.4).  query [T][H][D] rows
    of sequence s in [query_start[s], query_start[s+1]); those are the last q_len tokens of its
    context_lens[s].  Returns fp64 [T][H][D]."""
    query, key_cache, value_cache = _raw(query), _raw(key_cache), _raw(value_cache)
    bt = np.ascontiguousarray(block_tables, dtype=np.int32)
    cl = np.ascontiguousarray(context_lens, dtype=np.int32)
    qs = np.ascontiguousarray(query_start, dtype=np.int32)
    T, H, D = query.shape
    S = cl.shape[0]
    assert qs.shape[0] == S + 1 and qs[-1] == T
    out = np.empty((T, H, D), dtype=np.float64)
    lib().oracle_prefill_attention(_p(out), _p(query), _p(key_cache), _p(value_cache), _p(bt), _p(cl),
                                   _p(qs), float(scale), int(block_size), int(num_kv_heads), S, H, D,
                                   int(bt.shape[1]), _dt(dtype))
    return out


def split_attention(query, key_cache, value_cache, block_tables, context_lens, scale,
                    block_size, num_kv_heads, dtype, partition_tokens: int) -> np.ndarray:
    query, key_cache, value_cache = _raw(query), _raw(key_cache), _raw(value_cache)
    bt = np.ascontiguousarray(block_tables, dtype=np.int32)
    cl = np.ascontiguousarray(context_lens, dtype=np.int32)
    S, H, D = query.shape
    out = np.empty((S, H, D), dtype=np.float64)
    lib().oracle_split_attention(_p(out), _p(query), _p(key_cache), _p(value_cache), _p(bt), _p(cl),
                                 float(scale), int(block_size), int(num_kv_heads), S, H, D,
                                 int(bt.shape[1]), _dt(dtype), int(partition_tokens))
    return out


def gather_kv(key_cache, value_cache, bt_row, n, kvh, block_size, dtype):
    """fp64 K[n][D], V[n][D] of one (sequence, kv head) in logical order."""
    key_cache, value_cache = _raw(key_cache), _raw(value_cache)
    bt_row = np.ascontiguousarray(bt_row, dtype=np.int32)
    _, H_kv, _, D = key_cache.shape
    K = np.empty((max(n, 1), D), dtype=np.float64)
    V = np.empty((max(n, 1), D), dtype=np.float64)
    lib().oracle_gather_kv(_p(K), _p(V), _p(key_cache), _p(value_cache), _p(bt_row), int(n), int(kvh),
                           int(block_size), int(H_kv), int(D), _dt(dtype))
    return K[:n], V[:n]


def gather_kv_bits(key_cache, value_cache, bt_row, n, kvh, block_size, dtype):
    """Raw-bit K[n][D], V[n][D] of one (sequence, kv head) in logical order."""
    key_cache, value_cache = _raw(key_cache), _raw(value_cache)
    bt_row = np.ascontiguousarray(bt_row, dtype=np.int32)
    _, H_kv, _, D = key_cache.shape
    K = np.empty((max(n, 1), D), dtype=key_cache.dtype)
    V = np.empty((max(n, 1), D), dtype=key_cache.dtype)
    lib().oracle_gather_kv_bits(_p(K), _p(V), _p(key_cache), _p(value_cache), _p(bt_row), int(n),
                                int(kvh), int(block_size), int(H_kv), int(D), _dt(dtype))
    return K[:n], V[:n]


def reshape_and_cache(key, value, key_cache, value_cache, slot_mapping, block_size, dtype):
    """In place on copies: returns (new_key_cache, new_value_cache)."""
    key, value = _raw(key), _raw(value)
    kc, vc = np.array(key_cache, copy=True), np.array(value_cache, copy=True)
    sm = np.ascontiguousarray(slot_mapping, dtype=np.int64)
    T, H_kv, D = key.shape
    lib().oracle_reshape_and_cache(_p(key), _p(value), _p(kc), _p(vc), _p(sm), int(T), int(H_kv),
                                   int(D), int(block_size), _dt(dtype))
    return kc, vc


def copy_blocks(key_caches, value_caches, block_mapping, dtype):
    """key_caches/value_caches: lists of [NB][H_kv][B][D] arrays (one per layer).
    Returns new lists with cache[dst] <- cache[src] for every pair (simultaneous semantics)."""
    kcs = [np.array(k, copy=True) for k in key_caches]
    vcs = [np.array(v, copy=True) for v in value_caches]
    bm = np.ascontiguousarray(np.asarray(block_mapping, dtype=np.int64).reshape(-1, 2))
    L = len(kcs)
    NB, H_kv, B, D = kcs[0].shape
    kp = (ctypes.c_void_p * L)(*[k.ctypes.data for k in kcs])
    vp = (ctypes.c_void_p * L)(*[v.ctypes.data for v in vcs])
    lib().oracle_copy_blocks(kp, vp, L, _p(bm), int(bm.shape[0]), int(H_kv), int(B), int(D), int(NB),
                             _dt(dtype))
    return kcs, vcs


def swap_blocks(dst_key, dst_value, src_key, src_value, block_mapping):
    """Lists (one per layer) of pools: returns new dst lists with dst[d] <- src[s] per pair."""
    dk = [np.array(x, copy=True) for x in dst_key]
    dv = [np.array(x, copy=True) for x in dst_value]
    sk = [np.ascontiguousarray(x) for x in src_key]
    sv = [np.ascontiguousarray(x) for x in src_value]
    bm = np.ascontiguousarray(np.asarray(block_mapping, dtype=np.int64).reshape(-1, 2))
    L = len(dk)
    block_bytes = dk[0][0].nbytes
    arr = lambda xs: (ctypes.c_void_p * L)(*[x.ctypes.data for x in xs])  # noqa: E731
    lib().oracle_swap_blocks(arr(dk), arr(dv), arr(sk), arr(sv), L, _p(bm), int(bm.shape[0]), int(block_bytes))
    return dk, dv

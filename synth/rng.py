"""Counter-based random numbers shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method: it only turns (seed, stream, index)
into bits.  Two implementations of the same SplitMix64 finaliser -- numpy (uint64)
and torch (int64 with logical shifts, runs on CPU or CUDA) -- produce identical bits
for identical counters, so each side can draw exactly the entries it needs.

    key(seed, stream)   = mix64(mix64(seed + G) ^ (stream * G))          (mod 2^64)
    bits(key, i)        = mix64(key + (i + 1) * G)
    uniform_f32(key, i) = ((bits >> 40) - 2^23) * 2^-23    in [-1, 1), exact in fp32

Values are then rounded to the storage dtype with round-to-nearest-even: fp16 by the
IEEE conversion (numpy/torch), bf16 by the integer rounding of the fp32 bit pattern.
"""
from __future__ import annotations

import numpy as np

G = 0x9E3779B97F4A7C15
M1 = 0xBF58476D1CE4E5B9
M2 = 0x94D049BB133111EB
MASK64 = (1 << 64) - 1

NAN_BITS = {"f32": 0x7FC00000, "f16": 0x7E00, "bf16": 0x7FC0}
ELEM_BYTES = {"f32": 4, "f16": 2, "bf16": 2}

# stream ids (never reuse a number for a different tensor)
STREAM_Q = 1
STREAM_KNEW = 2
STREAM_VNEW = 3
STREAM_KCACHE = 4
STREAM_VCACHE = 5
STREAM_LEN = 16
STREAM_PICK = 17
STREAM_PERM = 18
STREAM_BEAM = 19
STREAM_MISC = 20


def _mix_int(z: int) -> int:
    z &= MASK64
    z = ((z ^ (z >> 30)) * M1) & MASK64
    z = ((z ^ (z >> 27)) * M2) & MASK64
    return z ^ (z >> 31)


def key(seed: int, stream: int, layer: int = 0) -> int:
    s = stream + 4096 * layer
    return _mix_int(_mix_int(seed + G) ^ ((s * G) & MASK64))


# ---------------------------------------------------------------- numpy --------------

def mix64_np(z: np.ndarray) -> np.ndarray:
    z = z.astype(np.uint64, copy=True)
    z ^= z >> np.uint64(30)
    z *= np.uint64(M1)
    z ^= z >> np.uint64(27)
    z *= np.uint64(M2)
    z ^= z >> np.uint64(31)
    return z


def bits_np(k: int, idx: np.ndarray) -> np.ndarray:
    idx = np.asarray(idx, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (idx + np.uint64(1)) * np.uint64(G) + np.uint64(k)
    return mix64_np(z)


def uniform01_np(k: int, idx) -> np.ndarray:
    """fp64 uniform in [0, 1) from the top 53 bits."""
    return (bits_np(k, idx) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def uniform_f32_np(k: int, idx) -> np.ndarray:
    top = (bits_np(k, idx) >> np.uint64(40)).astype(np.int64) - (1 << 23)
    return (top.astype(np.float32) * np.float32(2.0 ** -23)).astype(np.float32)


def f32_to_bits_np(x: np.ndarray, dtype: str) -> np.ndarray:
    """RN-even rounding of fp32 values to the storage dtype; returns raw bits
    (uint32 for f32, uint16 otherwise)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    if dtype == "f32":
        return x.view(np.uint32).copy()
    if dtype == "f16":
        return x.astype(np.float16).view(np.uint16)
    if dtype == "bf16":
        u = x.view(np.uint32).astype(np.uint64)
        r = (u + np.uint64(0x7FFF) + ((u >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)
        return (r & np.uint64(0xFFFF)).astype(np.uint16)
    raise ValueError(dtype)


def raw_np_dtype(dtype: str):
    return np.uint32 if dtype == "f32" else np.uint16


# ---------------------------------------------------------------- torch --------------

def _s64(v: int) -> int:
    v &= MASK64
    return v - (1 << 64) if v >= (1 << 63) else v


def _lsr(z, k: int):
    return (z >> k) & ((1 << (64 - k)) - 1)


def mix64_t(z):
    z = z ^ _lsr(z, 30)
    z = z * _s64(M1)
    z = z ^ _lsr(z, 27)
    z = z * _s64(M2)
    z = z ^ _lsr(z, 31)
    return z


def bits_t(k: int, idx):
    """idx: torch int64 tensor (any device).  Wrapping int64 arithmetic == uint64."""
    z = (idx + 1) * _s64(G) + _s64(k)
    return mix64_t(z)


def uniform_f32_t(k: int, idx):
    import torch
    top = _lsr(bits_t(k, idx), 40) - (1 << 23)
    return top.to(torch.float32) * (2.0 ** -23)


def f32_to_dtype_t(x, dtype: str):
    """RN-even fp32 -> storage dtype; returns a torch tensor of that dtype."""
    import torch
    if dtype == "f32":
        return x.to(torch.float32)
    if dtype == "f16":
        return x.to(torch.float16)
    if dtype == "bf16":
        u = x.contiguous().view(torch.int32).to(torch.int64) & 0xFFFFFFFF
        r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) & 0xFFFF
        r = torch.where(r >= 0x8000, r - 0x10000, r).to(torch.int16)
        return r.view(torch.bfloat16)
    raise ValueError(dtype)


def torch_dtype(dtype: str):
    import torch
    return {"f32": torch.float32, "f16": torch.float16, "bf16": torch.bfloat16}[dtype]

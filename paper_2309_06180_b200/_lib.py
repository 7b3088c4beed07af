"""ctypes binding of libpagedattn.so (include/pa.h).

Argument marshalling only: every step of the hot path runs in the library's sm_100a
kernels.  There is no CPU or PyTorch fallback -- if the shared library is missing the
import fails loudly (build it with ``python -c "import __graft_entry__ as g; g.build()"``
or ``make``).  torch is used for device memory and streams only.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpagedattn.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"libpagedattn.so not found at {LIB_PATH}: the CUDA extension is not built "
        "(run `make` or __graft_entry__.build()); there is no fallback path")

_lib = ctypes.CDLL(LIB_PATH)

PA_F32, PA_F16, PA_BF16 = 0, 1, 2
STATUS = {0: "PA_OK", 1: "PA_ERR_INVALID_ARG", 2: "PA_ERR_UNSUPPORTED", 3: "PA_ERR_WORKSPACE",
          4: "PA_ERR_CUDA", 5: "PA_ERR_OUT_OF_BLOCKS"}
DEFAULT_PARTITION_TOKENS = 512

_vp, _i32, _i64, _f32, _sz = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_float, ctypes.c_size_t


def _sig(name, res, args):
    f = getattr(_lib, name)
    f.restype = res
    f.argtypes = args
    return f


_sig("pa_paged_attention", _i32, [_vp, _vp, _vp, _vp, _vp, _vp, _f32, _i32, _i32, _i32, _i32, _i32, _i32, _i32,
                                  _i32, _vp, _sz, _vp])
_sig("pa_paged_attention_ex", _i32, [_vp, _vp, _vp, _vp, _vp, _vp, _f32, _i32, _i32, _i32, _i32, _i32, _i32, _i32,
                                     _i32, _i32, _vp, _vp, _sz, _vp])
_sig("pa_paged_attention_decode", _i32, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _f32, _i32, _i32, _i32, _i32, _i32,
                                         _i32, _i32, _i32, _vp, _vp, _sz, _vp])
_sig("pa_decode_plan", _i32, [_vp, _i32, _vp])
_sig("pa_paged_attention_decode_shared", _i32, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _f32, _i32, _i32, _i32, _i32,
                                                _i32, _i32, _i32, _i32, _i32, _vp, _sz, _vp])
_sig("pa_paged_attention_decode_grouped", _i32, [_vp] * 8 + [_f32] + [_i32] * 10 + [_vp, _vp, _sz, _vp])
_sig("pa_paged_prefill_attention", _i32, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _f32] + [_i32] * 10 + [_vp, _sz, _vp])
_sig("pa_paged_prefill_attention_packed", _i32, [_vp] * 10 + [_f32] + [_i32] * 10 + [_vp, _sz, _vp])
_sig("pa_paged_attention_workspace_size", _sz, [_i32, _i32, _i32, _i32, _i32])
_sig("pa_reshape_and_cache", _i32, [_vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _vp])
_sig("pa_copy_blocks", _i32, [ctypes.POINTER(_vp), ctypes.POINTER(_vp), _i32, _vp, _i32, _i32, _i32, _i32, _i32,
                              _vp])
_sig("pa_swap_blocks", _i32, [ctypes.POINTER(_vp)] * 4 + [_i32, _vp, _i32, _i32, _i32, _i32, _i32, _vp])
_sig("pa_swap_blocks_memcpy", _i32, [ctypes.POINTER(_vp)] * 4 + [_i32, _vp, _i32, _i32, _i32, _i32, _i32, _vp])
_sig("pa_decode_step_staging_size", _sz, [_i32, _i32, _i32, _i32, _i32, _i32, _i32])
_sig("pa_decode_step", _i32, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _vp, _vp, _f32, _i32, _i32, _i32, _i32,
                              _i32, _i32, _i32, _i32, _vp, _sz, _vp, _sz, _vp])
_sig("pa_last_error", ctypes.c_char_p, [])
_sig("pa_reload_tuning", None, [])
_sig("pa_take_launch_count", ctypes.c_longlong, [])
_sig("pa_debug_gather_kv", _i32, [_vp, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _vp])
_sig("pa_validate_tables", _i32, [_vp, _vp, _i32, _i32, _i32, _i32, ctypes.POINTER(_i64), _vp])
_sig("pa_tp_comm_create", _vp, [_i32, _i32, _i32, _sz, ctypes.POINTER(_vp), ctypes.POINTER(_vp),
                                ctypes.POINTER(_vp), _vp])
_sig("pa_tp_comm_destroy", None, [_vp])
_sig("pa_paged_attention_decode_tp", _i32, [_vp, ctypes.POINTER(ctypes.c_int), _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                            _f32, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _vp, _vp, _sz, _vp])
_sig("pa_hbm_read_probe", _i32, [_vp, _sz, _i32, _i32, _i32, _vp, _vp])
_sig("pa_ipc_handle_bytes", _sz, [])
_sig("pa_ipc_get_handle", _i32, [_vp, _vp])
_sig("pa_ipc_open_handle", _i32, [_vp, ctypes.POINTER(_vp)])
_sig("pa_ipc_close_handle", _i32, [_vp])
_sig("pa_device_alloc", _i32, [_sz, ctypes.POINTER(_vp)])
_sig("pa_device_free", _i32, [_vp])
_sig("pa_alloc_create", _vp, [_i32, _i32, _vp])
_sig("pa_alloc_destroy", None, [_vp])
_sig("pa_alloc_allocate", _i32, [_vp, _i32, ctypes.POINTER(_i32)])
_sig("pa_alloc_append_slot", _i32, [_vp, _i32, ctypes.POINTER(_i64), ctypes.POINTER(_i32), ctypes.POINTER(_i32)])
_sig("pa_alloc_fork", _i32, [_vp, _i32, ctypes.POINTER(_i32)])
_sig("pa_alloc_free", _i32, [_vp, _i32, ctypes.POINTER(_i32)])
_sig("pa_alloc_export", _i32, [_vp, _vp, _i32, _i32, _vp, _vp])
_sig("pa_alloc_refcount", _i32, [_vp, _i32])
_sig("pa_alloc_num_free", _i32, [_vp])
_sig("pa_alloc_num_blocks_of", _i32, [_vp, _i32])

EXPORTED = [n for n in dir(_lib) if n.startswith("pa_")]


class PagedAttnError(RuntimeError):
    def __init__(self, status: int, where: str):
        msg = _lib.pa_last_error().decode()
        super().__init__(f"{where}: {STATUS.get(status, status)}: {msg}")
        self.status = status


def check(status: int, where: str) -> None:
    if status != 0:
        raise PagedAttnError(status, where)


def raw():
    """The ctypes CDLL (tests use it to call entry points with raw pointers)."""
    return _lib


def last_error() -> str:
    return _lib.pa_last_error().decode()


def take_launch_count() -> int:
    return int(_lib.pa_take_launch_count())


def reload_tuning() -> None:
    """Re-read the PA_* tuning environment (tests / A-B scripts; read once otherwise)."""
    _lib.pa_reload_tuning()

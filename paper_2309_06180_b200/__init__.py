"""paper_2309_06180_b200 -- B200-native PagedAttention decode hot path (arXiv 2309.06180).

libpagedattn.so (sm_100a kernels + C ABI, include/pa.h) with a thin torch binding:
``paged_attention``, ``reshape_and_cache``, ``copy_blocks``, ``decode_step`` and the
host ``BlockAllocator``.  Importing fails loudly if the CUDA extension is not built.
"""
from ._lib import DEFAULT_PARTITION_TOKENS, PagedAttnError, last_error, reload_tuning, take_launch_count  # noqa: F401
from .ops import (BlockAllocator, copy_blocks, decode_plan, debug_gather_kv, decode_step, hbm_read_probe, decode_step_staging_size,  # noqa: F401
                  paged_attention, paged_attention_decode, paged_attention_decode_shared, paged_attention_decode_grouped,
                  paged_prefill_attention, paged_prefill_attention_packed, prepare,
                  paged_attention_workspace_size, reshape_and_cache, swap_blocks,
                  swap_blocks_memcpy, validate_tables)

__all__ = ["paged_attention", "paged_attention_decode", "paged_attention_decode_shared", "paged_attention_decode_grouped", "paged_prefill_attention", "paged_prefill_attention_packed", "paged_attention_workspace_size", "reshape_and_cache", "copy_blocks", "decode_step",
           "decode_step_staging_size", "swap_blocks", "swap_blocks_memcpy", "debug_gather_kv", "validate_tables", "hbm_read_probe", "BlockAllocator", "prepare", "decode_plan", "PagedAttnError",
           "last_error", "reload_tuning", "take_launch_count", "DEFAULT_PARTITION_TOKENS"]

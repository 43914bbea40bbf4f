"""B200-native CDSP chunked-prefill ring attention (Tetris, arXiv 2511.06247).

The product is libcdsp.so (C ABI in include/cdsp.h, CUDA kernels for sm_100a under csrc/);
this package is its thin Python binding plus a loopback / multi-process driver.
"""
from .api import (ATTN_FIRST, ATTN_LAST, ATTN_MID, ATTN_ONLY, CdspError, Comm, DecodeTarget, KvStore, Plan,
                  SpGroup, abi_version, attention_fwd, causal_segments, connect_local, kv_transfer_errors,
                  kv_transfer_to_decode, lib, lse_merge, plan_capacity, plan_partition, prefill_chunk, segments,
                  zigzag_gather, zigzag_map_device, zigzag_scatter)

__all__ = [
    "ATTN_FIRST", "ATTN_LAST", "ATTN_MID", "ATTN_ONLY", "CdspError", "Comm", "DecodeTarget", "KvStore", "Plan",
    "SpGroup", "abi_version", "attention_fwd", "causal_segments", "connect_local", "kv_transfer_errors",
    "kv_transfer_to_decode", "lib", "lse_merge", "plan_capacity", "plan_partition", "prefill_chunk", "segments", "zigzag_gather",
    "zigzag_map_device", "zigzag_scatter",
]

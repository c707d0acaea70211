"""B200-native Write-Gated KV (arXiv 2512.17452) hot path.

The product is ``libwgkv_b200.so`` (hand-written sm_100a CUDA behind the C-ABI
in ``include/wgkv_b200.h``); this package is its Python face.
"""
from ._lib import (ATTN_AUTO, ATTN_SIMT, ATTN_TCGEN05, BF16, F32, TOPK_EXACT, TOPK_QUEST,  # noqa: F401
                   LifecycleError, NotSupported, OutOfPages, WgkvError, load)
from . import policy  # noqa: F401
from .api import Session, assemble_heads, default_capacity, nccl_unique_id, vs_pair_count  # noqa: F401

__all__ = ["Session", "assemble_heads", "nccl_unique_id", "policy", "default_capacity", "vs_pair_count", "load", "BF16", "F32", "ATTN_AUTO", "ATTN_SIMT",
           "ATTN_TCGEN05", "TOPK_EXACT", "TOPK_QUEST", "OutOfPages", "LifecycleError", "NotSupported", "WgkvError"]

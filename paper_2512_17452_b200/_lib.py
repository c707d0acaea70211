"""ctypes binding of the C-ABI in include/wgkv_b200.h (libwgkv_b200.so).

The product path is the CUDA library; there is no CPU fallback.  If the
shared object is missing this module raises on load.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("WGKV_LIB") or os.path.join(HERE, "libwgkv_b200.so")  # WGKV_LIB: A/B builds

OK, EINVAL, ENOPAGES, ESTATE, ERUNTIME, ECUDA, ENOTSUP = range(7)
BF16, F32 = 0, 1
ATTN_AUTO, ATTN_SIMT, ATTN_TCGEN05 = 0, 1, 2
TOPK_EXACT, TOPK_QUEST = 0, 1  # wgkv_config.topk_mode


class WgkvError(RuntimeError):
    pass


class OutOfPages(MemoryError):
    """KvPool::alloc_page "out of pages" (kvstore.cpp:23-31)."""


class LifecycleError(RuntimeError):
    """std::logic_error in the reference (engine.cpp:154, 272; kvstore.cpp:163)."""


class NotSupported(WgkvError):
    pass


_EXC = {EINVAL: ValueError, ENOPAGES: OutOfPages, ESTATE: LifecycleError, ERUNTIME: ArithmeticError,
        ECUDA: WgkvError, ENOTSUP: NotSupported}


class Config(C.Structure):
    _fields_ = [("layers", C.c_int), ("q_heads", C.c_int), ("kv_heads", C.c_int), ("kv_head_offset", C.c_int),
                ("head_dim", C.c_int), ("hidden", C.c_int), ("window", C.c_long), ("tau", C.c_double),
                ("rope_base", C.c_double), ("page_size", C.c_int), ("max_seqs", C.c_int), ("max_tokens", C.c_long),
                ("max_prefill_tokens", C.c_long), ("capacity_pages", C.c_long), ("dtype", C.c_int),
                ("topk_budget", C.c_long), ("attn_impl", C.c_int), ("device", C.c_int), ("topk_mode", C.c_int),
                ("decode_chunk_pages", C.c_long)]


class DecodeTrace(C.Structure):
    """wgkv_decode_trace: device pointers (or None) of the step's GateTrace."""
    _fields_ = [("g", C.c_void_p), ("bits", C.c_void_p), ("near_tau", C.c_void_p), ("events", C.c_void_p)]


_vp, _i, _l = C.c_void_p, C.c_int, C.c_long
SIGNATURES = {
    "wgkv_last_error": ([], C.c_char_p),
    "wgkv_version": ([], C.c_char_p),
    "wgkv_ctx_create": ([C.POINTER(Config), C.POINTER(_vp)], _i),
    "wgkv_ctx_destroy": ([_vp], _i),
    "wgkv_set_stream": ([_vp, _vp], _i),
    "wgkv_sync": ([_vp], _i),
    "wgkv_gate_set": ([_vp, _vp, _i, _i], _i),
    "wgkv_gate_load": ([_vp, C.c_char_p], _i),
    "wgkv_gate_score": ([_vp, _i, _i, _l, _l, _vp, _vp, _vp, _vp, _vp, _vp, _i, C.POINTER(_i)], _i),
    "wgkv_gate_score_proj": ([_vp, _i, _i, _l, _l, _vp, _vp, _i, _vp, _vp, _vp, _vp, _vp, _i, C.POINTER(_i)], _i),
    "wgkv_admit_prefill": ([_vp, _i, _i, _i, _l, _vp, _vp, _vp, _vp], _i),
    "wgkv_vs_prefill": ([_vp, _i, _i, _i, _l, _vp, _vp, _vp, _vp, _vp], _i),
    "wgkv_prefill_layer": ([_vp, _i, _i, _i, _l, _vp, _vp, _vp, _vp, _vp, _vp, _vp], _i),
    "wgkv_decode_step_kv": ([_vp, _i, _i, _i, _vp, _vp, _vp, _vp, _vp], _i),
    "wgkv_decode_attn": ([_vp, _i, _i, _i, _vp, _vp], _i),
    "wgkv_decode_layer": ([_vp, _i, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp], _i),
    "wgkv_decode_layer_traced": ([_vp, _i, _i, _i, _vp, _vp, _vp, _vp, _vp, C.POINTER(DecodeTrace)], _i),
    "wgkv_cache_state": ([_vp, _i, _i, _i, C.POINTER(C.c_int64)], _i),
    "wgkv_cache_export": ([_vp, _i, _i, _i] + [_vp] * 8, _i),
    "wgkv_cache_stats": ([_vp, _i, _i, C.POINTER(C.c_int64)], _i),
    "wgkv_cache_snapshot": ([_vp, _i, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)], _i),
    "wgkv_release": ([_vp, _i, _i], _i),
    "wgkv_pool_info": ([_vp, C.POINTER(C.c_int64)], _i),
    "wgkv_vs_pair_count": ([_vp, _l, _l], C.c_uint64),
    "wgkv_comm_unique_id": ([_vp], _i),
    "wgkv_comm_init": ([_vp, _vp, _i, _i], _i),
    "wgkv_comm_attach": ([_vp, _vp, _i, _i], _i),
    "wgkv_allgather_heads": ([_vp, _i, _l, _vp, _vp, _i], _i),
    "wgkv_comm_join": ([_vp], _i),
    "wgkv_peer_region_bytes": ([_i, _l, _l, _i, _i, _i, _vp], _i),
    "wgkv_peer_alloc": ([_vp, _i, _l, _l, _vp, _vp], _i),
    "wgkv_peer_open": ([_vp, _i, _i, _vp, _i], _i),
    "wgkv_peer_attach": ([_vp, _i, _i, _l, _l, _vp, _i], _i),
    "wgkv_peer_prefill": ([_vp, _i], _i),
    "wgkv_peer_bulk_result": ([_vp, _i, _vp], _i),
    "wgkv_peer_allgather_heads": ([_vp, _l, _vp, _i], _i),
    "wgkv_peer_wait": ([_vp], _i),
    "wgkv_peer_decode": ([_vp, _i], _i),
    "wgkv_peer_result": ([_vp, _i, _vp], _i),
    "wgkv_output_proj": ([_vp, _i, _l, _vp, _vp, _i, _vp], _i),
    "wgkv_assemble_heads": ([_i, _l, C.c_size_t, _vp, _vp, _vp], _i),
}

_LIB = None


def load() -> C.CDLL:
    """Load libwgkv_b200.so (built by `make lib` / __graft_entry__.build())."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `make lib` (no CPU fallback exists)")
        lib = C.CDLL(LIB_PATH)
        for name, (args, res) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _LIB = lib
    return _LIB


def check(status: int, what: str = "") -> None:
    if status != OK:
        msg = load().wgkv_last_error().decode(errors="replace")
        raise _EXC.get(status, WgkvError)(f"{what}: {msg}" if what else msg)

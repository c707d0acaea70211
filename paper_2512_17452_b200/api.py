"""Host-side mirror of the reference's hot-path API over the C-ABI.

Names and argument meaning follow the reference (namespace ``wgkv``):

* :meth:`Session.gate_forward_batch` -- ``gate_forward_batch`` + ``binarize``
  (gating.cpp:173-190) for one layer's keys, fused with RoPE (K1);
* :meth:`Session.prefill_layer` -- the body of ``Session::prefill`` for one
  layer (engine.cpp:188-257): gate, mask, vertical-slash attention and
  ``HeadCache::prefill_populate`` (K1 -> K2 -> K3);
* :meth:`Session.decode_layer` -- the body of ``Session::decode_step``
  (engine.cpp:291-327): gate, ``HeadCache::local_write`` with lazy promotion,
  and ``attn_ragged`` over Global || Local in place (K4 -> K5);
* :meth:`Session.gather` / :meth:`Session.stats` -- ``HeadCache::gather`` and
  ``cache_stats`` for audits (kvstore.cpp:205-267).

Errors map to the reference's exception classes: ``ValueError``
(std::invalid_argument), ``OutOfPages`` (a ``MemoryError``; "out of pages"),
``LifecycleError`` (std::logic_error), ``ArithmeticError`` (runtime_error).
Device memory and streams come from torch; all compute is the CUDA library.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np
import torch

from . import _lib
from ._lib import ATTN_AUTO, ATTN_SIMT, ATTN_TCGEN05, BF16, F32, check  # noqa: F401

_TORCH_DT = {BF16: torch.bfloat16, F32: torch.float32}


def _p(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def default_capacity(layers, kv_heads, window, max_tokens, page_size=16, seqs=1) -> int:
    """default_capacity (engine.cpp:88-93), times the sequence slots."""
    return seqs * layers * kv_heads * (-(-window // page_size) + -(-max_tokens // page_size) + 1)


class Session:
    """One device's WG-KV state for ``kv_heads`` KV heads (a shard when
    ``kv_head_offset`` > 0) over ``max_seqs`` sequence slots."""

    def __init__(self, layers, q_heads, kv_heads, head_dim, hidden, window, tau=0.1, rope_base=10000.0,
                 page_size=16, max_seqs=1, max_tokens=4096, max_prefill_tokens=None, capacity_pages=0,
                 dtype=BF16, topk_budget=0, attn_impl=ATTN_AUTO, device=0, kv_head_offset=0, gate_bank=None,
                 topk_mode=0, decode_chunk_pages=0):
        self.lib = _lib.load()
        cfg = _lib.Config(layers=layers, q_heads=q_heads, kv_heads=kv_heads, kv_head_offset=kv_head_offset,
                          head_dim=head_dim, hidden=hidden, window=window, tau=tau, rope_base=rope_base,
                          page_size=page_size, max_seqs=max_seqs, max_tokens=max_tokens,
                          max_prefill_tokens=max_prefill_tokens or max_tokens, capacity_pages=capacity_pages,
                          dtype=dtype, topk_budget=topk_budget, attn_impl=attn_impl, device=device,
                          topk_mode=topk_mode, decode_chunk_pages=decode_chunk_pages)
        self.cfg = cfg
        self.device = torch.device("cuda", device)
        self.dtype = _TORCH_DT[dtype]
        h = C.c_void_p()
        check(self.lib.wgkv_ctx_create(C.byref(cfg), C.byref(h)), "Session")
        self.h = h
        self.set_stream(torch.cuda.current_stream(self.device))
        if gate_bank is not None:
            self.gate_set(gate_bank)

    # ---- lifecycle -------------------------------------------------------
    def close(self):
        if getattr(self, "h", None):
            self.lib.wgkv_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream: torch.cuda.Stream):
        self.stream = stream
        check(self.lib.wgkv_set_stream(self.h, C.c_void_p(stream.cuda_stream)), "set_stream")

    def sync(self):
        check(self.lib.wgkv_sync(self.h), "sync")

    # ---- gates -----------------------------------------------------------
    def gate_set(self, bank: np.ndarray):
        """bank: fp64 [layers][bank_heads][block] (GateBank layout, gating.hpp:41-68)."""
        bank = np.ascontiguousarray(bank, np.float64)
        self._bank = bank
        check(self.lib.wgkv_gate_set(self.h, bank.ctypes.data_as(C.c_void_p), bank.shape[0], bank.shape[1]),
              "gate_set")

    def gate_load(self, path: str):
        check(self.lib.wgkv_gate_load(self.h, os.fsencode(path)), "GateBank::load")

    # ---- K1 --------------------------------------------------------------
    def gate_forward_batch(self, layer: int, k_pre: torch.Tensor, pos0: int = 0, forced=None):
        """k_pre [nseq][T][kv_heads][d] -> (k_post, g [nseq][H][T] f32, bits uint8, near flat indices)."""
        nseq, T = k_pre.shape[0], k_pre.shape[1]
        H = self.cfg.kv_heads
        k_post = torch.empty_like(k_pre)
        g = torch.empty((nseq, H, T), dtype=torch.float32, device=self.device)
        bits = torch.empty((nseq, H, T), dtype=torch.uint8, device=self.device)
        near = torch.empty(1 << 16, dtype=torch.int64, device=self.device)
        n = C.c_int(0)
        check(self.lib.wgkv_gate_score(self.h, layer, nseq, T, pos0, _p(k_pre), _p(forced), _p(k_post), _p(g),
                                       _p(bits), _p(near), near.numel(), C.byref(n)), "gate_forward_batch")
        return k_post, g, bits, near[: min(n.value, near.numel())].cpu().numpy()

    def gate_forward_batch_proj(self, layer: int, x: torch.Tensor, wk: torch.Tensor, pos0: int = 0):
        """f1 (engine.cpp:190-205): x [nseq][T][dm] layer input, wk [kv_heads][d][dm]
        (this context's Wk rows), bf16 -> (k_pre = bf16(x . wk^T), k_post, g, bits,
        near flat indices); the projection is fused into the gate kernel."""
        nseq, T, dm = x.shape
        H, d = self.cfg.kv_heads, self.cfg.head_dim
        k_pre = torch.empty((nseq, T, H, d), dtype=torch.bfloat16, device=self.device)
        k_post = torch.empty_like(k_pre)
        g = torch.empty((nseq, H, T), dtype=torch.float32, device=self.device)
        bits = torch.empty((nseq, H, T), dtype=torch.uint8, device=self.device)
        near = torch.empty(1 << 16, dtype=torch.int64, device=self.device)
        n = C.c_int(0)
        check(self.lib.wgkv_gate_score_proj(self.h, layer, nseq, T, pos0, _p(x), _p(wk), dm, _p(k_pre), _p(k_post),
                                            _p(g), _p(bits), _p(near), near.numel(), C.byref(n)),
              "gate_forward_batch_proj")
        return k_pre, k_post, g, bits, near[: min(n.value, near.numel())].cpu().numpy()

    # ---- prefill -----------------------------------------------------------
    def prefill_layer(self, layer, q, k_pre, v, seq0=0, forced_gates=None, out=None, want_gates=False):
        """q [nseq][T][q_heads][d], k_pre/v [nseq][T][kv_heads][d] (device, dtype)."""
        nseq, T = q.shape[0], q.shape[1]
        if out is None:
            out = torch.empty_like(q)
        g = bits = None
        if want_gates:
            g = torch.empty((nseq, self.cfg.kv_heads, T), dtype=torch.float32, device=self.device)
            bits = torch.empty((nseq, self.cfg.kv_heads, T), dtype=torch.uint8, device=self.device)
        check(self.lib.wgkv_prefill_layer(self.h, layer, seq0, nseq, T, _p(q), _p(k_pre), _p(v), _p(forced_gates),
                                          _p(out), _p(g), _p(bits)), "Session::prefill")
        return (out, g, bits) if want_gates else out

    # ---- decode ------------------------------------------------------------
    def decode_layer(self, layer, q, k_pre, v, seq0=0, forced_gates=None, out=None, want_events=False,
                     want_trace=False):
        """q [nseq][q_heads][d], k_pre/v [nseq][kv_heads][d] -> out [nseq][q_heads][d].

        want_events: also return (g, events); want_trace: also return the step's
        GateTrace dict (g, bits, near_tau, events) -- wgkv_decode_layer_traced."""
        nseq = q.shape[0]
        if out is None:
            out = torch.empty_like(q)
        tr = None
        if want_events or want_trace:
            H = self.cfg.kv_heads
            tr = dict(g=torch.empty((nseq, H), dtype=torch.float32, device=self.device),
                      bits=torch.empty((nseq, H), dtype=torch.uint8, device=self.device),
                      near_tau=torch.empty((nseq, H), dtype=torch.uint8, device=self.device),
                      events=torch.empty((nseq, H), dtype=torch.int32, device=self.device))
            ct = _lib.DecodeTrace(*(tr[k].data_ptr() for k in ("g", "bits", "near_tau", "events")))
            check(self.lib.wgkv_decode_layer_traced(self.h, layer, seq0, nseq, _p(q), _p(k_pre), _p(v),
                                                    _p(forced_gates), _p(out), C.byref(ct)), "Session::decode_step")
        else:
            check(self.lib.wgkv_decode_layer_traced(self.h, layer, seq0, nseq, _p(q), _p(k_pre), _p(v),
                                                    _p(forced_gates), _p(out), None), "Session::decode_step")
        if want_trace:
            return out, tr
        return (out, tr["g"], tr["events"]) if want_events else out

    # ---- state / audit -------------------------------------------------------
    def state(self, layer, seq, head) -> dict:
        lens = (C.c_int64 * 6)()
        check(self.lib.wgkv_cache_state(self.h, layer, seq, head, lens), "cache_state")
        return dict(zip(("local_len", "local_ptr", "global_len", "tokens_seen", "n_local_pages", "n_global_pages"),
                        list(lens)))

    def gather(self, layer, seq, head) -> dict:
        """HeadCache::gather (kvstore.cpp:205-241) to host numpy (fp32 K/V)."""
        s = self.state(layer, seq, head)
        G, Lc, d = s["global_len"], s["local_len"], self.cfg.head_dim
        out = dict(global_k=np.empty((G, d), np.float32), global_v=np.empty((G, d), np.float32),
                   global_pos=np.empty(G, np.int64), global_gate=np.empty(G, np.float32),
                   local_k=np.empty((Lc, d), np.float32), local_v=np.empty((Lc, d), np.float32),
                   local_pos=np.empty(Lc, np.int64), local_gate=np.empty(Lc, np.float32))
        ptrs = [out[k].ctypes.data_as(C.c_void_p) for k in ("global_k", "global_v", "global_pos", "global_gate",
                                                             "local_k", "local_v", "local_pos", "local_gate")]
        check(self.lib.wgkv_cache_export(self.h, layer, seq, head, *ptrs), "gather")
        return out

    def snapshot(self, seq=0) -> str:
        """cache_snapshot (kvstore.cpp:269-286) of sequence slot `seq` (the
        reference's text format; gates are the stored fp32 values)."""
        n = C.c_size_t(0)
        check(self.lib.wgkv_cache_snapshot(self.h, seq, None, 0, C.byref(n)), "cache_snapshot")
        buf = C.create_string_buffer(n.value + 1)
        check(self.lib.wgkv_cache_snapshot(self.h, seq, buf, n.value + 1, C.byref(n)), "cache_snapshot")
        return buf.value.decode()

    def stats(self, seq0=0, nseq=1) -> dict:
        v = (C.c_int64 * 4)()
        check(self.lib.wgkv_cache_stats(self.h, seq0, nseq, v), "cache_stats")
        return dict(resident_entries=v[0], global_entries=v[1], tokens_seen=v[2], pages_allocated=v[3],
                    admitted_fraction=(v[1] / v[2]) if v[2] else 0.0)

    def release(self, seq0=0, nseq=1):
        check(self.lib.wgkv_release(self.h, seq0, nseq), "release")

    # ---- C1: head-output all-gather (KV-head sharding) -------------------------
    def comm_init(self, unique_id: bytes, world: int, rank: int):
        """Join the NCCL world of KV-head shards (this context = rank `rank`,
        created with kv_head_offset = rank * kv_heads)."""
        buf = C.create_string_buffer(bytes(unique_id), 128)
        check(self.lib.wgkv_comm_init(self.h, buf, world, rank), "comm_init")

    def allgather_heads(self, local_out: torch.Tensor, full_out: torch.Tensor, async_: bool = False):
        """local_out [nseq][T][q_heads][d] -> full_out [nseq][T][world*q_heads][d]
        (the reference's concat layout, engine.cpp:234-238); decode: T = 1."""
        nseq = local_out.shape[0]
        T = local_out.shape[1] if local_out.dim() == 4 else 1
        check(self.lib.wgkv_allgather_heads(self.h, nseq, T, _p(local_out), _p(full_out), int(async_)),
              "allgather_heads")
        return full_out

    def comm_join(self):
        check(self.lib.wgkv_comm_join(self.h), "comm_join")

    # ---- C1 over NVLink peer memory (decode-sized exchanges) -------------------
    def peer_region_bytes(self, world: int, max_rows: int, max_bulk_rows: int = 0) -> int:
        n = C.c_size_t(0)
        check(self.lib.wgkv_peer_region_bytes(world, max_rows, max_bulk_rows, self.cfg.q_heads, self.cfg.head_dim,
                                              self.cfg.dtype, C.byref(n)),
              "peer_region_bytes")
        return n.value

    def peer_alloc(self, world: int, max_rows: int, max_bulk_rows: int = 0) -> bytes:
        """Allocate this rank's exchange region; returns its 64-byte IPC handle."""
        buf = C.create_string_buffer(64)
        base = C.c_void_p()
        check(self.lib.wgkv_peer_alloc(self.h, world, max_rows, max_bulk_rows, buf, C.byref(base)), "peer_alloc")
        self._peer = dict(world=world, max_rows=max_rows, base=base.value, keep=None)
        return buf.raw

    def peer_open(self, world: int, rank: int, handles, wait_ranks=None):
        """Map every rank's region from the handles (rank order; this rank's own entry is ignored)."""
        blob = C.create_string_buffer(b"".join(bytes(h) for h in handles), 64 * world)
        check(self.lib.wgkv_peer_open(self.h, world, rank, blob, wait_ranks or world), "peer_open")
        self._peer.update(rank=rank)

    def peer_init(self, world: int, rank: int, max_rows: int, max_bulk_rows: int = 0, group=None):
        """peer_alloc + handle exchange over torch.distributed (the caller's
        plumbing; any backend) + peer_open."""
        import torch.distributed as dist
        mine = self.peer_alloc(world, max_rows, max_bulk_rows)
        allh = [None] * world
        dist.all_gather_object(allh, mine, group=group)
        self.peer_open(world, rank, allh)

    def peer_attach(self, world: int, rank: int, max_rows: int, regions, wait_ranks=None, max_bulk_rows: int = 0):
        """Attach already-mapped regions (uint8 tensors of peer_region_bytes each, rank order)."""
        arr = (C.c_void_p * world)(*[r.data_ptr() for r in regions])
        check(self.lib.wgkv_peer_attach(self.h, world, rank, max_rows, max_bulk_rows, arr, wait_ranks or world),
              "peer_attach")
        self._peer = dict(world=world, max_rows=max_rows, base=regions[rank].data_ptr(), keep=list(regions),
                          rank=rank)

    def peer_allgather_heads(self, local_out: torch.Tensor, wait: bool = True):
        """local_out [rows][q_heads][d] of every rank -> this rank's result
        [rows][world*q_heads][d] (returned as a view once wait; else pending)."""
        rows = local_out.shape[0]
        check(self.lib.wgkv_peer_allgather_heads(self.h, rows, _p(local_out), int(wait)), "peer_allgather_heads")
        return self.peer_result(0, rows) if wait else None

    def peer_wait(self):
        check(self.lib.wgkv_peer_wait(self.h), "peer_wait")

    def peer_decode(self, on: bool = True):
        """Decode layers push their output rows from inside their merge (C1 fused into the layer)."""
        check(self.lib.wgkv_peer_decode(self.h, int(on)), "peer_decode")

    def peer_prefill(self, on: bool = True):
        """K3's epilogue stores its output rows into every rank's bulk slot (C1 fused into the attention)."""
        check(self.lib.wgkv_peer_prefill(self.h, int(on)), "peer_prefill")

    def peer_bulk_result(self, back: int, rows: int) -> torch.Tensor:
        ptr = C.c_void_p()
        check(self.lib.wgkv_peer_bulk_result(self.h, back, C.byref(ptr)), "peer_bulk_result")
        world = self._peer["world"]
        return _device_view(ptr.value, (rows, world * self.cfg.q_heads, self.cfg.head_dim), self.dtype, self.device)

    def peer_result(self, back: int, rows: int) -> torch.Tensor:
        """View of this rank's result slot of the exchange `back` exchanges ago
        (valid once unpacked; the view does not own the memory: it lives as
        long as this Session)."""
        ptr = C.c_void_p()
        check(self.lib.wgkv_peer_result(self.h, back, C.byref(ptr)), "peer_result")
        world = self._peer["world"]
        return _device_view(ptr.value, (rows, world * self.cfg.q_heads, self.cfg.head_dim), self.dtype, self.device)

    def output_proj(self, local_out: torch.Tensor, wo: torch.Tensor, x: torch.Tensor):
        """f3: x += concat . wo^T (engine.cpp:243-245 / :331) where concat is
        the all-gathered head output; local_out [nseq][T][q_heads][d] (decode:
        [nseq][q_heads][d]) bf16, wo [dim][world*q_heads*d] bf16, x fp32
        [nseq][T][dim] updated in place.  The gather of the next row chunk
        overlaps the GEMM of the current one."""
        nseq = local_out.shape[0]
        T = local_out.shape[1] if local_out.dim() == 4 else 1
        assert wo.dtype == torch.bfloat16 and x.dtype == torch.float32 and x.is_contiguous()
        check(self.lib.wgkv_output_proj(self.h, nseq, T, _p(local_out), _p(wo), wo.shape[0], _p(x)), "output_proj")
        return x

    def pool_info(self) -> dict:
        v = (C.c_int64 * 2)()
        check(self.lib.wgkv_pool_info(self.h, v), "pool_info")
        return dict(capacity=v[0], free=v[1])


class _CudaArray:
    """__cuda_array_interface__ over a raw device pointer (torch.as_tensor wraps it without a copy)."""

    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = dict(shape=tuple(shape), typestr=typestr, data=(ptr, False), version=2,
                                             strides=None)


def _device_view(ptr, shape, dtype, device):
    if dtype == torch.float32:
        return torch.as_tensor(_CudaArray(ptr, shape, "<f4"), device=device)
    return torch.as_tensor(_CudaArray(ptr, shape, "<i2"), device=device).view(torch.bfloat16)


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId (call on one rank, broadcast the 128 bytes)."""
    buf = C.create_string_buffer(128)
    check(_lib.load().wgkv_comm_unique_id(buf), "comm_unique_id")
    return buf.raw


def assemble_heads(rank_major: torch.Tensor, full_out: torch.Tensor, world: int, rows: int, stream=None):
    """wgkv_assemble_heads: rank-major [world][rows][blk] -> [rows][world * blk]
    (the assembly step of wgkv_allgather_heads, usable on its own)."""
    blk = rank_major.numel() * rank_major.element_size() // (world * rows)
    st = stream if stream is not None else torch.cuda.current_stream(rank_major.device)
    check(_lib.load().wgkv_assemble_heads(world, rows, blk, _p(rank_major), _p(full_out), C.c_void_p(st.cuda_stream)),
          "assemble_heads")
    return full_out


def vs_pair_count(bits: np.ndarray, window: int) -> int:
    """vs_mask_pair_count (attention.cpp:182-191), closed form, one head."""
    b = np.ascontiguousarray(bits, np.uint8)
    return int(_lib.load().wgkv_vs_pair_count(b.ctypes.data_as(C.c_void_p), b.size, window))

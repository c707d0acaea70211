"""CPU parity oracle for the WG-KV hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package, and only as the checker.
The product (``paper_2512_17452_b200``) never imports it.

Two backends share one Python face:

* ``Oracle`` -- ``liboracle.so``, the plain-C fp64 restatement in
  ``wgkv_oracle.c`` (each function cites the reference file:line it follows);
* ``Ref``    -- ``_ref/libwgkv_ref.so``, the unmodified reference sources from
  ``/root/reference/proj/src`` compiled by ``oracle/Makefile`` behind
  ``ref_shim.cpp``.

Parity of the restatement is pinned by ``tests/test_oracle_golden.py`` (the
reference's own known-answer tests, restated) and ``tests/golden/*.npz``
(vectors produced by ``Ref``, committed together with ``make_golden.py``).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libwgkv_ref.so")

OK, EINVAL, ENOPAGES, ESTATE, ERUNTIME = 0, 1, 2, 3, 4
_ERRORS = {EINVAL: ValueError, ENOPAGES: MemoryError, ESTATE: RuntimeError, ERUNTIME: ArithmeticError}

_dp = C.POINTER(C.c_double)
_u8p = C.POINTER(C.c_uint8)
_lp = C.POINTER(C.c_long)
_ip = C.POINTER(C.c_int)
_u64p = C.POINTER(C.c_uint64)


def build(force: bool = False) -> None:
    """Compile liboracle.so (and _ref when /root/reference is present)."""
    if force or not os.path.exists(ORACLE_SO):
        subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True, stdout=sys.stderr)
    subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True, stdout=sys.stderr)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a, t=_dp):
    return None if a is None else a.ctypes.data_as(t)


def _check(st: int, what: str) -> None:
    if st != OK:
        raise _ERRORS.get(st, RuntimeError)(f"{what}: status {st}")


class _Base:
    """Shared wrappers; ``prefix`` selects wo_* (oracle) or wr_* (reference)."""

    prefix = ""

    def __init__(self, path: str):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = C.CDLL(path)
        P = self.prefix
        L = self.lib
        self._fn = lambda n: getattr(L, P + n)
        F = self._fn
        F("gaussian_fill").argtypes = [C.c_uint64, C.c_double, _dp, C.c_long]
        F("uniform_fill").argtypes = [C.c_uint64, _dp, C.c_long]
        F("rope").argtypes = [_dp, C.c_int, C.c_long, C.c_double, C.c_double]
        F("gate_random_init").argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_double, C.c_double, _dp]
        F("gate_forward_batch").argtypes = [_dp, C.c_int, C.c_int, _dp, _dp, C.c_long, _dp]
        F("binarize").argtypes = [_dp, C.c_long, C.c_double, _u8p]
        F("attn_vertical_slash").argtypes = [_dp, C.c_long, _dp, _dp, C.c_long, C.c_int, C.c_double, C.c_long,
                                                 C.c_long, _u8p, _dp, _u64p]
        F("vs_pair_count").argtypes = [C.c_long, _u8p, C.c_long, C.c_long, C.c_long]
        F("vs_pair_count").restype = C.c_uint64
        F("attn_ragged").argtypes = [_dp, _dp, _dp, C.c_long, _dp, _dp, C.c_long, C.c_int, C.c_double, _dp, _u64p]
        F("session_create").argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_long, C.c_double,
                                            C.c_double, C.c_int, C.c_long, C.c_long, _dp]
        F("session_create").restype = C.c_void_p
        F("session_destroy").argtypes = [C.c_void_p]
        F("session_prefill_layer").argtypes = [C.c_void_p, C.c_int, _dp, _dp, _dp, C.c_long, _dp, _dp, _dp,
                                                   _u8p, _u64p]
        F("session_decode_layer").argtypes = [C.c_void_p, C.c_int, _dp, _dp, _dp, _dp, _dp, _dp, _ip, _u64p]

    # ---- numerics -------------------------------------------------------
    def gaussian(self, seed: int, n: int, scale: float = 1.0) -> np.ndarray:
        out = np.empty(n, np.float64)
        self._fn("gaussian_fill")(seed, scale, _ptr(out), n)
        return out

    def uniform(self, seed: int, n: int) -> np.ndarray:
        out = np.empty(n, np.float64)
        self._fn("uniform_fill")(seed, _ptr(out), n)
        return out

    def rope(self, k, pos: int, base: float = 10000.0, sign: float = 1.0) -> np.ndarray:
        k = _f64(k).copy()
        _check(self._fn("rope")(_ptr(k), k.shape[-1], pos, base, sign), "rope")
        return k

    # ---- gating ---------------------------------------------------------
    @staticmethod
    def block_len(d: int, hidden: int) -> int:
        return hidden * 2 * d + 2 * hidden + 1

    def gate_random_init(self, layers, heads, d, hidden, seed, w_std=0.02, b2_init=2.0) -> np.ndarray:
        out = np.empty(layers * heads * self.block_len(d, hidden), np.float64)
        _check(self._fn("gate_random_init")(layers, heads, d, hidden, seed, w_std, b2_init, _ptr(out)), "random_init")
        return out.reshape(layers, heads, -1)

    def gate_forward_batch(self, block, k_pre, k_post) -> np.ndarray:
        k_pre, k_post, block = _f64(k_pre), _f64(k_post), _f64(block)
        t, d = k_pre.shape
        hidden = (block.size - 1) // (2 * d + 2)
        out = np.empty(t, np.float64)
        _check(self._fn("gate_forward_batch")(_ptr(block), d, hidden, _ptr(k_pre), _ptr(k_post), t, _ptr(out)),
               "gate_forward_batch")
        return out

    def binarize(self, g, tau: float) -> np.ndarray:
        g = _f64(g)
        out = np.empty(g.size, np.uint8)
        _check(self._fn("binarize")(_ptr(g), g.size, tau, _ptr(out, _u8p)), "binarize")
        return out

    # ---- attention ------------------------------------------------------
    def attn_vertical_slash(self, q, k, v, admitted, window: int, scale: float, causal_offset: int = 0):
        q, k, v = _f64(q), _f64(k), _f64(v)
        adm = np.ascontiguousarray(admitted, np.uint8)
        out = np.empty_like(q)
        ev = C.c_uint64(0)
        _check(self._fn("attn_vertical_slash")(_ptr(q), q.shape[0], _ptr(k), _ptr(v), k.shape[0], q.shape[1], scale,
                                               causal_offset, window, _ptr(adm, _u8p), _ptr(out), C.byref(ev)),
               "attn_vertical_slash")
        return out, ev.value

    def vs_pair_count(self, window: int, admitted, nq: int, nk: int, off: int = 0) -> int:
        adm = np.ascontiguousarray(admitted, np.uint8)
        return int(self._fn("vs_pair_count")(window, _ptr(adm, _u8p), nq, nk, off))

    def attn_ragged(self, q, gk, gv, lk, lv, scale: float):
        q, gk, gv, lk, lv = map(_f64, (q, gk, gv, lk, lv))
        d = q.shape[-1]
        out = np.empty(d, np.float64)
        ev = C.c_uint64(0)
        _check(self._fn("attn_ragged")(_ptr(q), _ptr(gk), _ptr(gv), gk.size // d, _ptr(lk), _ptr(lv), lk.size // d, d,
                                       scale, _ptr(out), C.byref(ev)), "attn_ragged")
        return out, ev.value


class Oracle(_Base):
    """The plain-C restatement (liboracle.so)."""

    prefix = "wo_"

    def __init__(self, path: str = ORACLE_SO):
        super().__init__(path)
        L = self.lib
        L.wo_pool_create.argtypes = [C.c_int, C.c_int, C.c_long]
        L.wo_pool_create.restype = C.c_void_p
        L.wo_pool_destroy.argtypes = [C.c_void_p]
        L.wo_pool_free_pages.argtypes = [C.c_void_p]
        L.wo_pool_free_pages.restype = C.c_long
        L.wo_pool_capacity.argtypes = [C.c_void_p]
        L.wo_pool_capacity.restype = C.c_long
        L.wo_pool_alloc.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int]
        L.wo_pool_free.argtypes = [C.c_void_p, C.c_int]
        L.wo_pool_owner.argtypes = [C.c_void_p, C.c_int, _ip, _ip, _ip, _ip]
        L.wo_pool_k_slot.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.wo_pool_k_slot.restype = _dp
        L.wo_head_create.argtypes = [C.c_int, C.c_int, C.c_long]
        L.wo_head_create.restype = C.c_void_p
        L.wo_head_destroy.argtypes = [C.c_void_p]
        L.wo_local_write.argtypes = [C.c_void_p, C.c_void_p, _dp, _dp, C.c_double, C.c_double, C.c_long]
        L.wo_prefill_populate.argtypes = [C.c_void_p, C.c_void_p, _dp, _dp, _dp, C.c_long, C.c_double, C.c_long]
        L.wo_head_state.argtypes = [C.c_void_p, _lp]
        L.wo_head_pages.argtypes = [C.c_void_p, _ip, _ip]
        L.wo_gather.argtypes = [C.c_void_p, C.c_void_p, _dp, _dp, _lp, _dp, _dp, _dp, _lp, _dp]
        L.wo_release.argtypes = [C.c_void_p, C.c_void_p]
        L.wo_select_topk_pages.argtypes = [_dp, C.c_void_p, C.c_void_p, C.c_long, _lp, _lp, _dp, _dp, _lp]
        L.wo_session_head.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.wo_session_head.restype = C.c_void_p
        L.wo_session_pool.argtypes = [C.c_void_p]
        L.wo_session_pool.restype = C.c_void_p
        L.wo_gate_save.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_int, _dp]
        L.wo_gate_load_header.argtypes = [C.c_char_p, _ip, _ip, _ip, _ip]
        L.wo_gate_load.argtypes = [C.c_char_p, _dp, C.c_long]
        L.wo_uniform_int_fill.argtypes = [C.c_uint64, C.c_long, C.c_long, _lp, C.c_long]
        L.wo_gelu.argtypes = [C.c_double]
        L.wo_gelu.restype = C.c_double
        L.wo_sigmoid.argtypes = [C.c_double]
        L.wo_sigmoid.restype = C.c_double
        L.wo_softmax.argtypes = [_dp, C.c_long, _dp]
        L.wo_attn_dense.argtypes = [_dp, C.c_long, _dp, _dp, C.c_long, C.c_int, C.c_double, C.c_long, _dp, _u64p]
        L.wo_rope_rows.argtypes = [_dp, C.c_long, C.c_int, C.c_long, C.c_double]

    def rope_rows(self, k, pos0: int = 0, base: float = 10000.0) -> np.ndarray:
        """apply_rope_inplace on rows [n][d]: row r at position pos0 + r (numerics.cpp:71-77)."""
        k = _f64(k).copy()
        _check(self.lib.wo_rope_rows(_ptr(k), k.shape[0], k.shape[1], pos0, base), "rope_rows")
        return k

    def uniform_int(self, seed: int, lo: int, hi: int, n: int) -> np.ndarray:
        out = np.empty(n, np.int64)
        self.lib.wo_uniform_int_fill(seed, lo, hi, _ptr(out, _lp), n)
        return out

    def softmax(self, logits) -> np.ndarray:
        x = _f64(logits)
        out = np.empty_like(x)
        _check(self.lib.wo_softmax(_ptr(x), x.size, _ptr(out)), "softmax")
        return out

    def attn_dense(self, q, k, v, scale: float, causal_offset: int = 0):
        q, k, v = _f64(q), _f64(k), _f64(v)
        out = np.empty_like(q)
        ev = C.c_uint64(0)
        _check(self.lib.wo_attn_dense(_ptr(q), q.shape[0], _ptr(k), _ptr(v), k.shape[0], q.shape[1], scale,
                                      causal_offset, _ptr(out), C.byref(ev)), "attn_dense")
        return out, ev.value

    def gate_save(self, path: str, bank, d: int, hidden: int) -> None:
        bank = _f64(bank)
        L, H = bank.shape[:2]
        assert bank.shape[2] == self.block_len(d, hidden)
        _check(self.lib.wo_gate_save(path.encode(), L, H, d, hidden, _ptr(bank)), "gate_save")

    def gate_load(self, path: str) -> np.ndarray:
        dims = [C.c_int() for _ in range(4)]
        _check(self.lib.wo_gate_load_header(path.encode(), *[C.byref(x) for x in dims]), "gate_load")
        L, H, d, hidden = (x.value for x in dims)
        out = np.empty(L * H * self.block_len(d, hidden), np.float64)
        _check(self.lib.wo_gate_load(path.encode(), _ptr(out), out.size), "gate_load")
        return out.reshape(L, H, -1)



class Ref(_Base):
    """The unmodified reference library (oracle/_ref/libwgkv_ref.so)."""

    prefix = "wr_"

    def __init__(self, path: str = REF_SO):
        super().__init__(path)
        L = self.lib
        L.wr_session_prefill_layer_timed.argtypes = [C.c_void_p, C.c_int, _dp, _dp, _dp, C.c_long, _dp, _u64p]
        L.wr_session_head_state.argtypes = [C.c_void_p, C.c_int, C.c_int, _lp]
        L.wr_session_gather.argtypes = [C.c_void_p, C.c_int, C.c_int, _dp, _dp, _lp, _dp, _dp, _dp, _lp, _dp]
        L.wr_session_select_topk.argtypes = [C.c_void_p, C.c_int, C.c_int, _dp, C.c_long, _lp, _lp]
        L.wr_session_snapshot.argtypes = [C.c_void_p, C.c_char_p, C.c_long, _lp]
        L.wr_session_cache_stats.argtypes = [C.c_void_p, _dp]
        L.wr_session_populate_layer.argtypes = [C.c_void_p, C.c_int, _dp, _dp, _dp, C.c_long]
        L.wr_gate_save.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_int, _dp]
        L.wr_thread_budget.restype = C.c_int
        L.wr_policy_trace.argtypes = [C.c_int, C.c_long, C.c_long, _u8p, C.c_int, C.c_long, C.c_long, C.c_double,
                                      C.c_int, C.c_int, C.c_long, C.c_int, _dp]

    def thread_budget(self) -> int:
        return int(self.lib.wr_thread_budget())

    def policy_trace(self, kind: int, window: int, sink: int, bitmap, fmode: int, keep_every: int, phase: int,
                     fraction: float, L: int, H: int, T: int, n_decode: int) -> np.ndarray:
        """GateTrace gates [L][H][T+n_decode] of a real wgkv::Session under the policy."""
        out = np.zeros((L, H, T + n_decode))
        bm = None if bitmap is None else np.ascontiguousarray(bitmap, np.uint8)
        st = self.lib.wr_policy_trace(kind, window, sink, None if bm is None else bm.ctypes.data_as(_u8p), fmode,
                                      keep_every, phase, fraction, L, H, T, n_decode,
                                      out.ctypes.data_as(_dp))
        if st:
            raise RuntimeError(f"wr_policy_trace status {st}")
        return out


# ---------------------------------------------------------------------------
# Paged dual cache (Oracle only): HeadCache / KvPool face over wo_pool/wo_head
# ---------------------------------------------------------------------------
class Pool:
    def __init__(self, orc: Oracle, page_size: int, head_dim: int, capacity: int):
        self.o, self.lib = orc, orc.lib
        self.h = self.lib.wo_pool_create(page_size, head_dim, capacity)
        if not self.h:
            raise ValueError("KvPool: invalid geometry")
        self.page_size, self.head_dim = page_size, head_dim

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.wo_pool_destroy(self.h)
            self.h = None

    @property
    def free_pages(self) -> int:
        return int(self.lib.wo_pool_free_pages(self.h))

    @property
    def capacity(self) -> int:
        return int(self.lib.wo_pool_capacity(self.h))

    def alloc_page(self, layer: int, head: int, region: int) -> int:
        r = self.lib.wo_pool_alloc(self.h, layer, head, region)
        if r < 0:
            raise MemoryError("out of pages")
        return r

    def free_page(self, page: int) -> None:
        _check(self.lib.wo_pool_free(self.h, page), "free_page")

    def owner(self, page: int):
        v = [C.c_int() for _ in range(4)]
        _check(self.lib.wo_pool_owner(self.h, page, *[C.byref(x) for x in v]), "owner")
        return tuple(x.value for x in v)  # layer, head, region, in_use

    def set_k_slot(self, page: int, slot: int, k) -> None:
        p = self.lib.wo_pool_k_slot(self.h, page, slot)
        for i, x in enumerate(np.asarray(k, np.float64)):
            p[i] = x


class HeadCache:
    def __init__(self, orc: Oracle, layer: int, head: int, window: int, handle=None):
        self.o, self.lib = orc, orc.lib
        self.owned = handle is None
        self.h = handle if handle is not None else self.lib.wo_head_create(layer, head, window)
        if not self.h:
            raise ValueError("HeadCache: window must be >= 1")

    def __del__(self):
        if getattr(self, "owned", False) and getattr(self, "h", None):
            self.lib.wo_head_destroy(self.h)
            self.h = None

    def state(self):
        lens = (C.c_long * 6)()
        self.lib.wo_head_state(self.h, lens)
        return dict(zip(("local_len", "local_ptr", "global_len", "tokens_seen", "n_local_pages", "n_global_pages"),
                        list(lens)))

    def pages(self):
        s = self.state()
        lp = np.empty(max(1, s["n_local_pages"]), np.int32)
        gp = np.empty(max(1, s["n_global_pages"]), np.int32)
        self.lib.wo_head_pages(self.h, _ptr(lp, _ip), _ptr(gp, _ip))
        return lp[: s["n_local_pages"]], gp[: s["n_global_pages"]]

    def local_write(self, pool: Pool, k, v, gate: float, tau: float, position: int) -> int:
        k, v = _f64(k), _f64(v)
        r = self.lib.wo_local_write(self.h, pool.h, _ptr(k), _ptr(v), gate, tau, position)
        if r < 0:
            _check(-r, "local_write")
        return r  # 0 none, 1 promoted, 2 dropped

    def prefill_populate(self, pool: Pool, keys, values, gates, tau: float, first_position: int = 0) -> None:
        keys, values, gates = _f64(keys), _f64(values), _f64(gates)
        _check(self.lib.wo_prefill_populate(self.h, pool.h, _ptr(keys), _ptr(values), _ptr(gates), keys.shape[0], tau,
                                            first_position), "prefill_populate")

    def gather(self, pool: Pool):
        s = self.state()
        G, Lc, d = s["global_len"], s["local_len"], pool.head_dim
        out = dict(global_k=np.empty((G, d)), global_v=np.empty((G, d)), global_pos=np.empty(G, np.int64),
                   global_gate=np.empty(G), local_k=np.empty((Lc, d)), local_v=np.empty((Lc, d)),
                   local_pos=np.empty(Lc, np.int64), local_gate=np.empty(Lc))
        self.lib.wo_gather(self.h, pool.h, _ptr(out["global_k"]), _ptr(out["global_v"]),
                           _ptr(out["global_pos"], _lp), _ptr(out["global_gate"]), _ptr(out["local_k"]),
                           _ptr(out["local_v"]), _ptr(out["local_pos"], _lp), _ptr(out["local_gate"]))
        return out

    def release(self, pool: Pool) -> None:
        self.lib.wo_release(self.h, pool.h)

    def select_topk_pages(self, pool: Pool, q, budget: int):
        q = _f64(q)
        s = self.state()
        n = max(1, s["n_global_pages"])
        logical = np.empty(n, np.int64)
        nsel = C.c_long()
        k = np.empty((max(1, s["global_len"]), pool.head_dim))
        v = np.empty_like(k)
        ent = C.c_long()
        _check(self.lib.wo_select_topk_pages(_ptr(q), self.h, pool.h, budget, _ptr(logical, _lp), C.byref(nsel),
                                             _ptr(k), _ptr(v), C.byref(ent)), "select_topk_pages")
        return logical[: nsel.value], k[: ent.value], v[: ent.value]


class Session:
    """Path-level Session mirror (one sequence) over either backend."""

    def __init__(self, backend: _Base, layers, q_heads, kv_heads, head_dim, hidden, window, tau=0.1,
                 rope_base=10000.0, page_size=16, capacity_pages=None, topk_budget=0, gate_bank=None,
                 max_tokens=None):
        self.b, self.lib, P = backend, backend.lib, backend.prefix
        self.P = P
        if capacity_pages is None:  # default_capacity (engine.cpp:88-93)
            mt = max_tokens or 4096
            capacity_pages = layers * kv_heads * (-(-window // page_size) + -(-mt // page_size) + 1)
        bank = None if gate_bank is None else _f64(gate_bank)
        self._bank = bank
        self.h = getattr(self.lib, P + "session_create")(layers, q_heads, kv_heads, head_dim, hidden, window, tau,
                                                          rope_base, page_size, capacity_pages, topk_budget,
                                                          _ptr(bank))
        if not self.h:
            raise ValueError("Session: bad configuration")
        self.layers, self.q_heads, self.kv_heads, self.d = layers, q_heads, kv_heads, head_dim

    def __del__(self):
        if getattr(self, "h", None):
            getattr(self.lib, self.P + "session_destroy")(self.h)
            self.h = None

    def prefill_layer(self, layer, q_pre, k_pre, v, forced_gates=None):
        q_pre, k_pre, v = _f64(q_pre), _f64(k_pre), _f64(v)
        t = q_pre.shape[0]
        out = np.empty_like(q_pre)
        g = np.empty((self.kv_heads, t))
        bits = np.empty((self.kv_heads, t), np.uint8)
        fg = None if forced_gates is None else _f64(forced_gates)
        ev = C.c_uint64(0)
        _check(getattr(self.lib, self.P + "session_prefill_layer")(self.h, layer, _ptr(q_pre), _ptr(k_pre), _ptr(v), t,
                                                                   _ptr(fg), _ptr(out), _ptr(g), _ptr(bits, _u8p),
                                                                   C.byref(ev)), "prefill")
        return out, g, bits, ev.value

    def prefill_layer_timed(self, layer, q_pre, k_pre, v):
        """Reference backend only: (secs[gate, attention, populate], pairs)."""
        q_pre, k_pre, v = _f64(q_pre), _f64(k_pre), _f64(v)
        secs = np.zeros(3)
        pairs = C.c_uint64(0)
        _check(self.lib.wr_session_prefill_layer_timed(self.h, layer, _ptr(q_pre), _ptr(k_pre), _ptr(v),
                                                       q_pre.shape[0], _ptr(secs), C.byref(pairs)), "prefill_timed")
        return secs, pairs.value

    def populate_layer(self, layer, k_pre, v, gates):
        """Reference backend only: RoPE + HeadCache::prefill_populate of every kv
        head with the given gates [kv_heads][t] (no attention) -- a cache state
        for timing decode steps at long context."""
        k_pre, v, gates = _f64(k_pre), _f64(v), _f64(gates)
        _check(self.lib.wr_session_populate_layer(self.h, layer, _ptr(k_pre), _ptr(v), _ptr(gates), k_pre.shape[0]),
               "populate")

    def decode_layer(self, layer, q_pre, k_pre, v, forced_gates=None):
        q_pre, k_pre, v = _f64(q_pre), _f64(k_pre), _f64(v)
        out = np.empty_like(q_pre)
        g = np.empty(self.kv_heads)
        events = np.empty(self.kv_heads, np.int32)
        fg = None if forced_gates is None else _f64(forced_gates)
        ev = C.c_uint64(0)
        _check(getattr(self.lib, self.P + "session_decode_layer")(self.h, layer, _ptr(q_pre), _ptr(k_pre), _ptr(v),
                                                                  _ptr(fg), _ptr(out), _ptr(g), _ptr(events, _ip),
                                                                  C.byref(ev)), "decode")
        return out, g, events, ev.value

    def gather(self, layer: int, head: int):
        if self.P == "wo_":
            hc = HeadCache(self.b, layer, head, 1, handle=self.lib.wo_session_head(self.h, layer, head))
            pool = Pool.__new__(Pool)
            pool.lib, pool.h, pool.head_dim = self.lib, self.lib.wo_session_pool(self.h), self.d
            out = hc.gather(pool)
            pool.h = None
            return out
        lens = (C.c_long * 4)()
        self.lib.wr_session_head_state(self.h, layer, head, lens)
        G, Lc, d = lens[2], lens[0], self.d
        out = dict(global_k=np.empty((G, d)), global_v=np.empty((G, d)), global_pos=np.empty(G, np.int64),
                   global_gate=np.empty(G), local_k=np.empty((Lc, d)), local_v=np.empty((Lc, d)),
                   local_pos=np.empty(Lc, np.int64), local_gate=np.empty(Lc))
        self.lib.wr_session_gather(self.h, layer, head, _ptr(out["global_k"]), _ptr(out["global_v"]),
                                   _ptr(out["global_pos"], _lp), _ptr(out["global_gate"]), _ptr(out["local_k"]),
                                   _ptr(out["local_v"]), _ptr(out["local_pos"], _lp), _ptr(out["local_gate"]))
        return out

    def cache_stats(self) -> dict:
        """cache_stats (kvstore.cpp:253-267) over the session's caches: the
        reference's own function (reference backend), else recounted from
        gather() per its definition."""
        if self.P == "wr_":
            v = np.zeros(3)
            _check(self.lib.wr_session_cache_stats(self.h, _ptr(v)), "cache_stats")
            return dict(resident_entries=int(v[0]), admitted_fraction=float(v[1]), pages_allocated=int(v[2]))
        res = glob = seen = pages = 0
        for layer in range(self.layers):
            for head in range(self.kv_heads):
                hc = HeadCache(self.b, layer, head, 1, handle=self.lib.wo_session_head(self.h, layer, head))
                s = hc.state()
                res += s["local_len"] + s["global_len"]
                glob += s["global_len"]
                seen += s["tokens_seen"]
                pages += s["n_local_pages"] + s["n_global_pages"]
        return dict(resident_entries=res, admitted_fraction=glob / seen if seen else 0.0, pages_allocated=pages)

    def snapshot(self, native: bool = True) -> str:
        """cache_snapshot (kvstore.cpp:269-286): one line per resident entry,
        "layer head global|local pos gate(%.17g)", caches in Session order
        (layer-major, then kv head), Global then Local in position order.
        native: the reference's own function (reference backend); else this
        Python restatement over gather()."""
        if native and self.P == "wr_":
            n = C.c_long(0)
            _check(self.lib.wr_session_snapshot(self.h, None, 0, C.byref(n)), "snapshot")
            buf = C.create_string_buffer(n.value + 1)
            _check(self.lib.wr_session_snapshot(self.h, buf, n.value + 1, C.byref(n)), "snapshot")
            return buf.value.decode()
        lines = []
        for layer in range(self.layers):
            for head in range(self.kv_heads):
                g = self.gather(layer, head)
                for kind in ("global", "local"):
                    for pos, gate in zip(g[kind + "_pos"], g[kind + "_gate"]):
                        lines.append("%d %d %s %d %.17g\n" % (layer, head, kind, pos, gate))
        return "".join(lines)

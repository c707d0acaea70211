"""CPU-side checks of the drop-in boundary: the C-ABI library loads, exports
every entry point include/wgkv_b200.h declares, and its host-only helpers
agree with the oracle.  No kernel is launched here (no GPU)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "wgkv_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(wgkv_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for need in ("wgkv_ctx_create", "wgkv_gate_score", "wgkv_admit_prefill", "wgkv_vs_prefill",
                 "wgkv_prefill_layer", "wgkv_decode_step_kv", "wgkv_decode_attn", "wgkv_cache_export"):
        assert need in syms


def test_library_exports_every_declared_symbol():
    from paper_2512_17452_b200 import _lib

    lib = _lib.load()
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert b"sm_100a" in lib.wgkv_version()


def test_library_is_sm100a_cubin():
    so = os.path.join(ROOT, "paper_2512_17452_b200", "libwgkv_b200.so")
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_pair_count_closed_form_matches_oracle(orc):
    from paper_2512_17452_b200 import vs_pair_count

    for seed in range(30):
        T = 10 + seed * 17
        W = 1 + (seed * 7) % 40
        bits = (orc.uniform(seed, T) < 0.3).astype(np.uint8)
        assert vs_pair_count(bits, W) == orc.vs_pair_count(W, bits, T, T)


def test_ctx_create_validates_like_the_reference():
    """Host validation runs before any device work (engine.cpp:107, gating.cpp:185)."""
    from paper_2512_17452_b200 import _lib

    lib = _lib.load()
    base = dict(layers=1, q_heads=4, kv_heads=1, kv_head_offset=0, head_dim=128, hidden=128, window=8, tau=0.1,
                rope_base=1e4, page_size=16, max_seqs=1, max_tokens=64, max_prefill_tokens=64, capacity_pages=0,
                dtype=0, topk_budget=0, attn_impl=0, device=0)
    h = C.c_void_p()
    for bad, code in (({"tau": 1.0}, _lib.EINVAL), ({"window": 0}, _lib.EINVAL), ({"head_dim": 7}, _lib.EINVAL),
                      ({"q_heads": 3, "kv_heads": 2}, _lib.EINVAL),
                      # beyond K5's work split: kMaxChunks (512) x 2048 pages per head
                      ({"max_tokens": 512 * 2048 * 16}, _lib.ENOTSUP),
                      ({"topk_mode": 1, "page_size": 8}, _lib.ENOTSUP), ({"topk_mode": 2}, _lib.EINVAL)):
        cfg = _lib.Config(**{**base, **bad})
        assert lib.wgkv_ctx_create(C.byref(cfg), C.byref(h)) == code


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2512_17452_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "wgkv_oracle" not in src and "liboracle" not in src, f

"""Differential test: the C restatement vs the unmodified reference library.

``oracle/_ref/libwgkv_ref.so`` is the reference's own sources compiled by
``oracle/Makefile``; both are built with the same g++/glibc here, and the
restatement keeps the reference's evaluation order, so results must be
BITWISE equal.  Skipped where ``_ref`` is absent (it is always present in the
build container where the driver runs the CPU suite).
"""
import numpy as np
import pytest

import oracle as O


def test_rng_streams_identical(orc, ref):
    for seed in (0, 1, 77, 2**63 + 5):
        assert (orc.gaussian(seed, 1001, 0.3) == ref.gaussian(seed, 1001, 0.3)).all()
        assert (orc.uniform(seed, 777) == ref.uniform(seed, 777)).all()


def test_random_init_identical(orc, ref):
    a = orc.gate_random_init(3, 2, 8, 5, 42, 0.02, -1.0)
    b = ref.gate_random_init(3, 2, 8, 5, 42, 0.02, -1.0)
    assert (a == b).all()


def test_rope_identical(orc, ref):
    k = orc.gaussian(3, 128)
    for pos in (0, 1, 17, 4095, 131071, 999999):
        for base in (1e4, 5e5):
            assert (orc.rope(k, pos, base) == ref.rope(k, pos, base)).all()


@pytest.mark.parametrize("w_std,b2", [(0.02, 2.0), (0.5, -2.5), (0.3, 0.0)])
def test_gate_batch_identical(orc, ref, w_std, b2):
    d, hidden, t = 16, 24, 64
    blk = orc.gate_random_init(1, 1, d, hidden, 5, w_std, b2)[0, 0]
    pre = orc.gaussian(6, t * d).reshape(t, d)
    post = np.stack([orc.rope(pre[i], i) for i in range(t)])
    ga, gb = orc.gate_forward_batch(blk, pre, post), ref.gate_forward_batch(blk, pre, post)
    assert (ga == gb).all()
    assert (orc.binarize(ga, 0.1) == ref.binarize(gb, 0.1)).all()


def test_vs_and_ragged_identical(orc, ref):
    for seed in range(20):
        t, d, window = 8 + seed * 3, 8, 1 + seed % 6
        x = orc.gaussian(100 + seed, 3 * t * d).reshape(3, t, d)
        bits = (orc.uniform(200 + seed, t) < 0.4).astype(np.uint8)
        a = orc.attn_vertical_slash(x[0], x[1], x[2], bits, window, 0.35)
        b = ref.attn_vertical_slash(x[0], x[1], x[2], bits, window, 0.35)
        assert (a[0] == b[0]).all() and a[1] == b[1]
        assert orc.vs_pair_count(window, bits, t, t) == ref.vs_pair_count(window, bits, t, t)
        g = seed % 5
        ra = orc.attn_ragged(x[0, 0], x[1, :g], x[2, :g], x[1, g:], x[2, g:], 0.35)
        rb = ref.attn_ragged(x[0, 0], x[1, :g], x[2, :g], x[1, g:], x[2, g:], 0.35)
        assert (ra[0] == rb[0]).all() and ra[1] == rb[1]


@pytest.mark.parametrize("hq,hkv,topk,ps", [(4, 4, 0, 16), (4, 2, 0, 3), (8, 2, 2, 4)])
def test_session_identical(orc, ref, hq, hkv, topk, ps):
    L, d, n, steps, W = 2, 16, 40, 20, 8
    bank = orc.gate_random_init(L, hkv, d, d, 9, 0.5, -2.5)
    kw = dict(tau=0.1, rope_base=1e4, page_size=ps, topk_budget=topk, gate_bank=bank, max_tokens=n + steps)
    sa = O.Session(orc, L, hq, hkv, d, d, W, **kw)
    sb = O.Session(ref, L, hq, hkv, d, d, W, **kw)
    q = orc.gaussian(10, (n + steps) * hq * d).reshape(n + steps, hq, d)
    k = orc.gaussian(11, (n + steps) * hkv * d).reshape(n + steps, hkv, d)
    v = orc.gaussian(12, (n + steps) * hkv * d).reshape(n + steps, hkv, d)
    for l in range(L):
        ra, rb = sa.prefill_layer(l, q[:n], k[:n], v[:n]), sb.prefill_layer(l, q[:n], k[:n], v[:n])
        for x, y in zip(ra, rb):
            assert np.array_equal(x, y)
    for t in range(n, n + steps):
        for l in range(L):
            ra, rb = sa.decode_layer(l, q[t], k[t], v[t]), sb.decode_layer(l, q[t], k[t], v[t])
            for x, y in zip(ra, rb):
                assert np.array_equal(x, y)
    for l in range(L):
        for h in range(hkv):
            ga, gb = sa.gather(l, h), sb.gather(l, h)
            for key in ga:
                assert np.array_equal(ga[key], gb[key]), key
    # cache_snapshot text (kvstore.cpp:269-286): the reference's own function
    # pins the Python restatement the GPU test compares against
    snap = sb.snapshot(native=True)
    assert snap and snap == sb.snapshot(native=False) == sa.snapshot()

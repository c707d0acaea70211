"""The reference's own known-answer tests, restated against the C oracle.

Each test cites the reference test it restates (/root/reference/proj/tests).
These pin ``oracle/wgkv_oracle.c`` before anything else trusts it; the GPU
parity tests then compare the CUDA path against this oracle.
"""
import math
import os

import numpy as np
import pytest

import oracle as O


def _rand_params(orc, d, hidden, seed, w_std=0.5, b2=0.0):
    """random_params (test_gating.cpp:14-20)."""
    blk = orc.gate_random_init(1, 1, d, hidden, seed, w_std, b2)[0, 0].copy()
    nb1 = orc.gaussian(seed + 1, hidden, 0.1)
    blk[hidden * 2 * d: hidden * 2 * d + hidden] = nb1
    return blk


def _gate_np(blk, d, hidden, x):
    """gate_oracle (test_gating.cpp:29-38): independent two-layer evaluation."""
    w1 = blk[: hidden * 2 * d].reshape(hidden, 2 * d)
    b1 = blk[hidden * 2 * d: hidden * 2 * d + hidden]
    w2 = blk[hidden * 2 * d + hidden: hidden * 2 * d + 2 * hidden]
    z2 = blk[-1]
    for i in range(hidden):
        z1 = b1[i] + float(np.dot(w1[i], x))
        z2 += w2[i] * z1 * 0.5 * (1.0 + math.erf(z1 / math.sqrt(2.0)))
    return 1.0 / (1.0 + math.exp(-z2))


# ---------------------------------------------------------------- gating ---
def test_zero_network_half_and_saturated(orc):  # test_gating.cpp:64-72
    blk = np.zeros(O.Oracle.block_len(4, 8))
    feat = np.full((1, 4), 0.7)
    assert orc.gate_forward_batch(blk, feat, feat)[0] == 0.5
    blk[-1] = 20.0
    assert orc.gate_forward_batch(blk, feat, feat)[0] > 1.0 - 1e-8


def test_gate_matches_two_layer_oracle(orc):  # test_gating.cpp:74-81
    x = orc.gaussian(11, 50 * 10).reshape(50, 10)
    for it in range(50):
        blk = _rand_params(orc, 5, 7, 100 + it)
        g = orc.gate_forward_batch(blk, x[it: it + 1, :5], x[it: it + 1, 5:])[0]
        assert g == pytest.approx(_gate_np(blk, 5, 7, x[it]), rel=1e-12)


def test_gate_strictly_inside_unit_interval(orc):  # test_gating.cpp:83-93
    u = orc.uniform(2, 200)
    for it in range(200):
        blk = _rand_params(orc, 4, 4, 300 + it, 2.0, -8.0 + 16.0 * u[it])
        x = orc.gaussian(1000 + it, 8).reshape(1, 8)
        g = orc.gate_forward_batch(blk, x[:, :4], x[:, 4:])[0]
        assert 0.0 < g < 1.0
    # clamp keeps saturated sigmoids off 0 and 1 (gating.cpp:169-170)
    blk = np.zeros(O.Oracle.block_len(4, 4))
    blk[-1] = 80.0
    f = np.zeros((1, 4))
    assert orc.gate_forward_batch(blk, f, f)[0] == np.nextafter(1.0, 0.0)
    blk[-1] = -800.0
    assert orc.gate_forward_batch(blk, f, f)[0] == 5e-324


def test_gate_batch_equals_scalar(orc):  # test_gating.cpp:95-118
    blk = _rand_params(orc, 6, 6, 77)
    pre = orc.gaussian(21, 48).reshape(8, 6)
    post = orc.gaussian(22, 48).reshape(8, 6)
    pre[3], post[3] = pre[2], post[2]
    batch = orc.gate_forward_batch(blk, pre, post)
    assert batch[2] == batch[3]
    for i in range(8):
        assert batch[i] == orc.gate_forward_batch(blk, pre[i: i + 1], post[i: i + 1])[0]


def test_binarize_boundary(orc):  # test_gating.cpp:120-136
    assert orc.binarize([0.05, 0.1, 0.95], 0.1).tolist() == [0, 1, 1]
    assert orc.binarize([0.5, 0.5, 0.5], 0.5).tolist() == [1, 1, 1]
    s = orc.uniform(3, 100)
    assert (orc.binarize(s, 0.37) == (s >= 0.37)).all()
    for bad in (0.0, 1.0):
        with pytest.raises(ValueError):
            orc.binarize(s, bad)


def test_binarize_monotone(orc):  # test_gating.cpp:138-148
    s = np.sort(orc.uniform(4, 64))
    b = orc.binarize(s, 0.5)
    assert (np.diff(b.astype(int)) >= 0).all()


def test_gate_bank_roundtrip_and_bad_magic(orc, tmp_path):  # test_gating.cpp:238-265
    bank = orc.gate_random_init(2, 3, 4, 5, 9, 0.3, 1.5)
    p = str(tmp_path / "g.wgkv")
    orc.gate_save(p, bank, 4, 5)
    assert (orc.gate_load(p) == bank).all()
    with open(p, "r+b") as f:
        f.write(b"XXXX")
    with pytest.raises(ArithmeticError):
        orc.gate_load(p)


def test_random_init_layout(orc):  # gating.cpp:49-59
    bank = orc.gate_random_init(2, 2, 3, 4, 5, 0.02, 2.0)
    draws = orc.gaussian(5, 4 * (4 * 6 + 4), 0.02)
    off = 0
    for l in range(2):
        for h in range(2):
            blk = bank[l, h]
            assert (blk[:24] == draws[off: off + 24]).all()
            assert (blk[24:28] == 0).all()
            assert (blk[28:32] == draws[off + 24: off + 28]).all()
            assert blk[32] == 2.0
            off += 28


# ------------------------------------------------------------- attention ---
def _inst(orc, tq, tk, d, seed):
    """random_instance (test_attention.cpp:27-32): q, k, v from one stream."""
    x = orc.gaussian(seed, tq * d + 2 * tk * d)
    q = x[: tq * d].reshape(tq, d)
    k = x[tq * d: tq * d + tk * d].reshape(tk, d)
    v = x[tq * d + tk * d:].reshape(tk, d)
    return q, k, v, 1.0 / math.sqrt(d)


def _dense_neg_inf(q, k, v, scale, off, allowed):
    """dense_neg_inf_oracle (test_attention.cpp:36-50)."""
    out = np.zeros((q.shape[0], v.shape[1]))
    for r in range(q.shape[0]):
        i = off + r
        lg = np.full(k.shape[0], -np.inf)
        for j in range(k.shape[0]):
            if j <= i and allowed(i, j):
                lg[j] = scale * float(np.dot(q[r], k[j]))
        w = np.exp(lg - lg.max())
        w /= w.sum()
        out[r] = w @ v
    return out


def test_dense_single_token(orc):  # test_attention.cpp:62-66
    q, k, v, s = _inst(orc, 1, 1, 4, 1)
    out, _ = orc.attn_dense(q, k, v, s)
    assert (out[0] == v[0]).all()


def test_dense_matches_naive_and_counts(orc):  # test_attention.cpp:86-93
    q, k, v, s = _inst(orc, 6, 6, 4, 3)
    out, ev = orc.attn_dense(q, k, v, s)
    assert np.abs(out - _dense_neg_inf(q, k, v, s, 0, lambda i, j: True)).max() < 1e-13
    assert ev == 21


def test_dense_fully_masked_row(orc):  # test_attention.cpp:95-98
    q, k, v, s = _inst(orc, 2, 2, 4, 4)
    with pytest.raises(ArithmeticError):
        orc.attn_dense(q, k, v, s, causal_offset=-1)


def test_vs_mask_worked_example(orc):  # test_attention.cpp:256-264
    bits = orc.binarize([1.0, 0.0, 0.0, 1.0, 0.0], 0.5)
    # row 4 permits {0, 3, 4}: with equal keys the weights are uniform over them
    d = 5
    q = np.zeros((1, d))
    k = np.zeros((5, d))
    v = np.eye(5)
    out, ev = orc.attn_vertical_slash(q, k, v, bits, 2, 1.0, causal_offset=4)
    assert ev == 3
    assert np.allclose(out[0], [1 / 3, 0, 0, 1 / 3, 1 / 3], atol=1e-15)
    assert orc.vs_pair_count(2, bits, 1, 5, 4) == 3


def test_vs_mask_extremes(orc):  # test_attention.cpp:266-278
    g = orc.uniform(101, 6)
    wide = orc.binarize(g, 0.99)
    assert orc.vs_pair_count(6, wide, 6, 6) == 21
    assert orc.vs_pair_count(1, np.ones(6, np.uint8), 6, 6) == 21


def test_vs_equals_dense_neg_inf_200(orc):  # test_attention.cpp:280-296
    for seed in range(200, 400):
        t = 4 + int(orc.uniform_int(seed, 0, 9, 1)[0])
        # the reference draws t, then t gates, then window from one Rng(seed)
        raw = orc.uniform(seed, 1 + t + 1)  # uniform() consumes one u64 like uniform_int
        gates = raw[1: 1 + t]
        window = 1 + int(orc.uniform_int(seed, 0, 4, t + 2)[-1])
        q, k, v, s = _inst(orc, t, t, 4, seed + 5000)
        bits = orc.binarize(gates, 0.5)
        out, ev = orc.attn_vertical_slash(q, k, v, bits, window, s)
        ref = _dense_neg_inf(q, k, v, s, 0, lambda i, j: (i - j) < window or bits[j] != 0)
        assert np.abs(out - ref).max() < 1e-10
        assert ev == orc.vs_pair_count(window, bits, t, t)


def test_vs_full_mask_equals_dense(orc):  # test_attention.cpp:298-304
    q, k, v, s = _inst(orc, 7, 7, 4, 555)
    a, _ = orc.attn_vertical_slash(q, k, v, np.ones(7, np.uint8), 1, s)
    b, _ = orc.attn_dense(q, k, v, s)
    assert np.abs(a - b).max() < 1e-12


def test_pair_count_worked_example(orc):  # test_attention.cpp:306-326
    n, window = 64, 8
    draws = orc.uniform_int(77, 0, 64, 4096)
    adm = np.zeros(64, np.uint8)
    placed = 0
    for j in draws:
        if not adm[j]:
            adm[j] = 1
            placed += 1
            if placed == 10:
                break
    manual = sum(1 for i in range(n) for j in range(i + 1) if i - j < window or adm[j])
    assert orc.vs_pair_count(window, adm, n, n) == manual
    assert manual <= n * (window + 10)


def test_ragged_base_cases_and_dense(orc):  # test_attention.cpp:328-373
    d = 4
    lk = orc.gaussian(303, 2 * d)
    out, _ = orc.attn_ragged(np.full(d, 0.3), np.zeros((0, d)), np.zeros((0, d)), lk[:d].reshape(1, d),
                             lk[d:].reshape(1, d), 0.5)
    assert (out == lk[d:]).all()
    for it in range(20):
        gl, ll = it % 6, 1 + (it * 7) % 5
        x = orc.gaussian(900 + it, (2 * gl + 2 * ll + 1) * d)
        gk = x[: gl * d].reshape(gl, d)
        gv = x[gl * d: 2 * gl * d].reshape(gl, d)
        lk_ = x[2 * gl * d: (2 * gl + ll) * d].reshape(ll, d)
        lv_ = x[(2 * gl + ll) * d: (2 * gl + 2 * ll) * d].reshape(ll, d)
        q = x[-d:]
        out, ev = orc.attn_ragged(q, gk, gv, lk_, lv_, 0.5)
        assert ev == gl + ll
        ref, _ = orc.attn_dense(q.reshape(1, d), np.vstack([gk, lk_]), np.vstack([gv, lv_]), 0.5, gl + ll - 1)
        assert np.allclose(out, ref[0], rtol=1e-12, atol=0)


def test_ragged_permutation_invariance(orc):  # test_attention.cpp:375-396
    d, gl, ll = 4, 5, 3
    x = orc.gaussian(404, (2 * gl + 2 * ll + 1) * d)
    gk = x[: gl * d].reshape(gl, d)
    gv = x[gl * d: 2 * gl * d].reshape(gl, d)
    lk = x[2 * gl * d: (2 * gl + ll) * d].reshape(ll, d)
    lv = x[(2 * gl + ll) * d: (2 * gl + 2 * ll) * d].reshape(ll, d)
    q = x[-d:]
    perm = [3, 0, 4, 1, 2]
    a, _ = orc.attn_ragged(q, gk, gv, lk, lv, 0.5)
    b, _ = orc.attn_ragged(q, gk[perm], gv[perm], lk, lv, 0.5)
    assert np.allclose(a, b, rtol=1e-12, atol=0)


def test_ragged_rejects_empty_local(orc):  # test_attention.cpp:398-402
    with pytest.raises(ValueError):
        orc.attn_ragged(np.full(4, 0.1), np.zeros((2, 4)), np.zeros((2, 4)), np.zeros((0, 4)), np.zeros((0, 4)), 0.5)


def test_softmax_invariants(orc):  # test_numerics.cpp:15-66
    w = orc.softmax([1.0, 2.0, -np.inf, 3.0])
    assert w[2] == 0.0 and abs(w.sum() - 1) < 1e-15
    with pytest.raises(ArithmeticError):
        orc.softmax([-np.inf, -np.inf])
    with pytest.raises(ValueError):
        orc.softmax([np.nan, 1.0])


def test_rope_identity_norm_inverse(orc):  # test_numerics.cpp:104-133
    k = orc.gaussian(8, 16)
    assert (orc.rope(k, 0) == k).all()
    r = orc.rope(k, 37)
    assert abs(np.linalg.norm(r) - np.linalg.norm(k)) < 1e-12
    assert np.abs(orc.rope(r, 37, sign=-1.0) - k).max() < 1e-12
    # hand rotation of pair 0 by angle = pos (freq 1)
    k2 = np.array([1.0, 0.0, 0.0, 0.0])
    r2 = orc.rope(k2, 1)
    assert abs(r2[0] - math.cos(1.0)) < 1e-15 and abs(r2[1] - math.sin(1.0)) < 1e-15
    with pytest.raises(ValueError):
        orc.rope(np.zeros(3), 1)


# --------------------------------------------------------------- kvstore ---
KD = 4


def key_for(p):  # test_kvstore.cpp:17-21
    return np.array([1000.0 * p + c for c in range(KD)])


def value_for(p):  # test_kvstore.cpp:23-27
    return np.array([-1000.0 * p - c for c in range(KD)])


def test_pool_bookkeeping(orc):  # test_kvstore.cpp:50-66
    pool = O.Pool(orc, 16, KD, 8)
    assert pool.free_pages == 8
    page = pool.alloc_page(0, 0, 0)
    assert page == 0  # LIFO free list hands out page 0 first (kvstore.cpp:9-21)
    assert pool.free_pages == 7
    assert pool.owner(page)[0] == 0 and pool.owner(page)[3] == 1
    for _ in range(7):
        pool.alloc_page(0, 1, 1)
    assert pool.free_pages == 0
    with pytest.raises(MemoryError, match="out of pages"):
        pool.alloc_page(0, 2, 1)
    pool.free_page(page)
    assert pool.free_pages == 1
    with pytest.raises(RuntimeError):
        pool.free_page(page)


def test_interleaved_heads_disjoint_pages(orc):  # test_kvstore.cpp:68-89
    pool = O.Pool(orc, 4, KD, 32)
    a, b = O.HeadCache(orc, 0, 0, 4), O.HeadCache(orc, 0, 1, 4)
    for t in range(12):
        a.local_write(pool, key_for(t), value_for(t), 0.9, 0.1, t)
        b.local_write(pool, key_for(t), value_for(t), 0.9, 0.1, t)
    al, ag = a.pages()
    bl, bg = b.pages()
    assert not (set(al) | set(ag)) & (set(bl) | set(bg))
    for p in al:
        assert pool.owner(int(p))[1] == 0 and pool.owner(int(p))[2] == 0
    for p in bg:
        assert pool.owner(int(p))[1] == 1 and pool.owner(int(p))[2] == 1


def test_lazy_promotion_worked_example(orc):  # test_kvstore.cpp:91-114
    pool = O.Pool(orc, 16, KD, 8)
    c = O.HeadCache(orc, 0, 0, 2)
    assert c.local_write(pool, key_for(0), value_for(0), 0.9, 0.1, 0) == 0
    assert c.local_write(pool, key_for(1), value_for(1), 0.05, 0.1, 1) == 0
    assert c.state()["global_len"] == 0
    assert c.local_write(pool, key_for(2), value_for(2), 0.3, 0.1, 2) == 1
    assert c.gather(pool)["global_pos"].tolist() == [0]
    assert c.local_write(pool, key_for(3), value_for(3), 0.8, 0.1, 3) == 2
    kv = c.gather(pool)
    assert kv["global_pos"].tolist() == [0]
    assert kv["local_pos"].tolist() == [2, 3]


def test_not_full_no_events(orc):  # test_kvstore.cpp:116-124
    pool = O.Pool(orc, 16, KD, 8)
    c = O.HeadCache(orc, 0, 0, 4)
    for t in range(3):
        assert c.local_write(pool, key_for(t), value_for(t), 0.5, 0.1, t) == 0
    assert c.state()["local_len"] == 3 and c.state()["global_len"] == 0


def test_prefill_populate_worked_example(orc):  # test_kvstore.cpp:126-174
    pool = O.Pool(orc, 16, KD, 8)
    c = O.HeadCache(orc, 0, 0, 2)
    keys = np.stack([key_for(t) for t in range(5)])
    vals = np.stack([value_for(t) for t in range(5)])
    gates = [0.9, 0.01, 0.02, 0.7, 0.03]
    c.prefill_populate(pool, keys, vals, gates, 0.1)
    kv = c.gather(pool)
    assert kv["global_pos"].tolist() == [0]
    assert kv["local_pos"].tolist() == [3, 4]
    assert kv["local_gate"].tolist() == [0.7, 0.03]
    assert c.state()["global_len"] + c.state()["local_len"] == 3
    with pytest.raises(RuntimeError):
        c.prefill_populate(pool, keys, vals, gates, 0.1)
    # prompt fits the window
    pool2 = O.Pool(orc, 16, KD, 8)
    c2 = O.HeadCache(orc, 0, 0, 8)
    c2.prefill_populate(pool2, np.zeros((5, KD)), np.zeros((5, KD)), [0.9] * 5, 0.1)
    assert c2.state()["global_len"] == 0 and c2.state()["local_len"] == 5
    # all gates below tau on a long prompt: only the window survives
    pool3 = O.Pool(orc, 16, KD, 32)
    c3 = O.HeadCache(orc, 0, 0, 16)
    c3.prefill_populate(pool3, np.zeros((100, KD)), np.zeros((100, KD)), [0.01] * 100, 0.1)
    assert c3.state()["local_len"] == 16 and c3.state()["global_len"] == 0


def test_gather_across_page_boundaries(orc):  # test_kvstore.cpp:176-201
    pool = O.Pool(orc, 3, KD, 32)
    c = O.HeadCache(orc, 0, 0, 5)
    kv = c.gather(pool)
    assert kv["global_k"].shape[0] == 0 and kv["local_k"].shape[0] == 0
    for t in range(8):
        c.local_write(pool, key_for(t), value_for(t), 0.9 if t % 2 == 0 else 0.1, 0.5, t)
    kv = c.gather(pool)
    assert kv["local_pos"].tolist() == [3, 4, 5, 6, 7]
    for n, p in enumerate(kv["local_pos"]):
        assert (kv["local_k"][n] == key_for(p)).all()
    assert kv["global_pos"].tolist() == [0, 2]
    for g, p in enumerate(kv["global_pos"]):
        assert (kv["global_v"][g] == value_for(p)).all()


def test_ring_matches_naive_dual_cache(orc):  # test_kvstore.cpp:203-238
    for run in range(30):
        window = 1 + run % 7
        pool = O.Pool(orc, 3, KD, 256)
        c = O.HeadCache(orc, 0, 0, window)
        total = 20 + (run * 13) % 40
        gates = orc.uniform(71 + run, total)
        local, glist = [], []
        for t in range(total):
            c.local_write(pool, key_for(t), value_for(t), gates[t], 0.1, t)
            if len(local) == window:
                victim = local.pop(0)
                if gates[victim] >= 0.1:
                    glist.append(victim)
            local.append(t)
            kv = c.gather(pool)
            assert kv["local_pos"].tolist() == local
            assert kv["global_pos"].tolist() == glist
            gset = set(kv["global_pos"].tolist())
            for j in range(t + 1):
                assert (j in gset) == (j <= t - window and gates[j] >= 0.1)
        c.release(pool)
        assert pool.free_pages == pool.capacity


def test_prefill_then_decode_equals_all_decode(orc):  # test_kvstore.cpp:240-277
    for run in range(10):
        window = 1 + run % 5
        tp, td = 5 + (run * 7) % 20, run % 10
        gates = orc.uniform(91 + run, tp + td)
        pa, pb = O.Pool(orc, 3, KD, 256), O.Pool(orc, 3, KD, 256)
        bulk, stepped = O.HeadCache(orc, 0, 0, window), O.HeadCache(orc, 0, 0, window)
        bulk.prefill_populate(pa, np.stack([key_for(t) for t in range(tp)]),
                              np.stack([value_for(t) for t in range(tp)]), gates[:tp], 0.1)
        for t in range(tp, tp + td):
            bulk.local_write(pa, key_for(t), value_for(t), gates[t], 0.1, t)
        for t in range(tp + td):
            stepped.local_write(pb, key_for(t), value_for(t), gates[t], 0.1, t)
        a, b = bulk.gather(pa), stepped.gather(pb)
        for key in ("global_pos", "local_pos", "global_k", "local_v", "local_gate"):
            assert (a[key] == b[key]).all()


def snapshot(caches, pool):
    """cache_snapshot text format (kvstore.cpp:269-286)."""
    out = []
    for (l, h), c in caches:
        kv = c.gather(pool)
        out += ["%d %d global %d %.17g\n" % (l, h, p, g) for p, g in zip(kv["global_pos"], kv["global_gate"])]
        out += ["%d %d local %d %.17g\n" % (l, h, p, g) for p, g in zip(kv["local_pos"], kv["local_gate"])]
    return "".join(out)


def test_snapshot_golden(orc):  # test_kvstore.cpp:305-319
    pool = O.Pool(orc, 16, KD, 8)
    c = O.HeadCache(orc, 0, 0, 2)
    for t, g in enumerate([0.5, 0.05, 0.25]):
        c.local_write(pool, key_for(t), value_for(t), g, 0.1, t)
    assert snapshot([((0, 0), c)], pool) == ("0 0 global 0 0.5\n"
                                             "0 0 local 1 0.050000000000000003\n"
                                             "0 0 local 2 0.25\n")


# ---------------------------------------------------------------- engine ---
def test_topk_identity_and_planted_page(orc):  # test_engine.cpp:283-324
    d = 16
    pool = O.Pool(orc, 4, d, 64)
    c = O.HeadCache(orc, 0, 0, 4)
    keys = orc.gaussian(81, 20 * d + d).reshape(21, d)
    for t in range(20):
        c.local_write(pool, keys[t], np.full(d, 0.5), 1.0, 0.1, t)
    assert c.state()["global_len"] == 16 and c.state()["n_global_pages"] == 4
    q = keys[20]
    logical, k, v = c.select_topk_pages(pool, q, 100)
    kv = c.gather(pool)
    assert k.shape[0] == 16 and (k == kv["global_k"]).all() and (v == kv["global_v"]).all()
    _, gpages = c.pages()
    pool.set_k_slot(int(gpages[9 // 4]), 9 % 4, q * 50.0)
    logical, k, _ = c.select_topk_pages(pool, q, 1)
    assert logical.tolist() == [2] and k.shape[0] <= 4
    with pytest.raises(ValueError):
        c.select_topk_pages(pool, q, 0)


def _spread_bank(orc, L, H, d, seed):  # spread_gates (test_engine.cpp:34-36)
    return orc.gate_random_init(L, H, d, d, seed, 0.5, -2.5)


def test_session_pair_count_accounting(orc):  # test_engine.cpp:370-400
    L, H, d, n, W = 2, 4, 16, 64, 8
    bank = _spread_bank(orc, L, H, d, 112)
    s = O.Session(orc, L, H, H, d, d, W, gate_bank=bank, max_tokens=n)
    x = orc.gaussian(113, n * H * d * 3).reshape(3, n, H, d)
    for l in range(L):
        _, g, bits, ev = s.prefill_layer(l, x[0], x[1], x[2])
        expected = sum(orc.vs_pair_count(W, bits[h], n, n) for h in range(H))
        assert ev == expected
        assert expected <= sum(n * (W + int(bits[h].sum())) for h in range(H))


def test_session_unlimited_topk_equals_wgkv(orc):  # test_engine.cpp:350-368
    L, H, d, n, W = 1, 4, 16, 64, 8
    bank = _spread_bank(orc, L, H, d, 102)
    x = orc.gaussian(103, (n + 16) * H * d * 3).reshape(3, n + 16, H, d)
    a = O.Session(orc, L, H, H, d, d, W, gate_bank=bank, max_tokens=n + 16)
    b = O.Session(orc, L, H, H, d, d, W, gate_bank=bank, max_tokens=n + 16, topk_budget=1000000)
    ra, rb = a.prefill_layer(0, x[0, :n], x[1, :n], x[2, :n]), b.prefill_layer(0, x[0, :n], x[1, :n], x[2, :n])
    assert (ra[0] == rb[0]).all()
    for t in range(n, n + 16):
        oa, _, _, ea = a.decode_layer(0, x[0, t], x[1, t], x[2, t])
        ob, _, _, eb = b.decode_layer(0, x[0, t], x[1, t], x[2, t])
        assert (oa == ob).all() and ea == eb


def test_session_decode_promotion_audit(orc):  # test_engine.cpp:107-152 (audit part)
    L, H, d, n, W, tau = 2, 4, 16, 48, 8, 0.1
    bank = _spread_bank(orc, L, H, d, 22)
    x = orc.gaussian(23, (n + 24) * H * d * 3).reshape(3, n + 24, H, d)
    s = O.Session(orc, L, H, H, d, d, W, tau=tau, gate_bank=bank, max_tokens=n + 24)
    hist = {}
    for l in range(L):
        _, g, _, _ = s.prefill_layer(l, x[0, :n], x[1, :n], x[2, :n])
        for h in range(H):
            hist[(l, h)] = list(g[h])
    for t in range(n, n + 24):
        for l in range(L):
            _, g, _, _ = s.decode_layer(l, x[0, t], x[1, t], x[2, t])
            for h in range(H):
                hist[(l, h)].append(g[h])
                kv = s.gather(l, h)
                gs = set(kv["global_pos"].tolist())
                for j in range(t + 1):
                    assert (j in gs) == (j <= t - W and hist[(l, h)][j] >= tau)
                assert kv["local_pos"].tolist() == list(range(max(0, t - W + 1), t + 1))


def test_session_lifecycle_errors(orc):  # test_engine.cpp:419-439
    d = 16
    s = O.Session(orc, 1, 4, 4, d, d, 4, gate_bank=_spread_bank(orc, 1, 4, d, 132), max_tokens=16)
    x = orc.gaussian(133, 8 * 4 * d * 3).reshape(3, 8, 4, d)
    with pytest.raises(RuntimeError):
        s.decode_layer(0, x[0, 0], x[1, 0], x[2, 0])
    s.prefill_layer(0, x[0], x[1], x[2])
    with pytest.raises(RuntimeError):
        s.prefill_layer(0, x[0], x[1], x[2])


def test_session_pool_exhaustion(orc):  # test_engine.cpp:441-458
    d = 16
    bank = orc.gate_random_init(1, 4, d, d, 142, 0.02, 20.0)
    s = O.Session(orc, 1, 4, 4, d, d, 8, gate_bank=bank, capacity_pages=4)
    x = orc.gaussian(143, 64 * 4 * d * 3).reshape(3, 64, 4, d)
    with pytest.raises(MemoryError):
        s.prefill_layer(0, x[0], x[1], x[2])


def test_session_gqa_and_forced_full(orc):  # test_engine.cpp:52-69,154-178 (path level)
    # forced g = 1 ("full" policy) makes VS attention exactly dense causal
    L, Hq, Hkv, d, n = 1, 4, 2, 16, 24
    x = orc.gaussian(31, n * (Hq + 2 * Hkv) * d)
    q = x[: n * Hq * d].reshape(n, Hq, d)
    k = x[n * Hq * d: n * (Hq + Hkv) * d].reshape(n, Hkv, d)
    v = x[n * (Hq + Hkv) * d:].reshape(n, Hkv, d)
    s = O.Session(orc, L, Hq, Hkv, d, d, 4, max_tokens=n)
    out, _, bits, _ = s.prefill_layer(0, q, k, v, forced_gates=np.ones((Hkv, n)))
    assert bits.all()
    for p in range(Hq):
        h = p // 2
        qr = np.stack([orc.rope(q[i, p], i) for i in range(n)])
        kr = np.stack([orc.rope(k[i, h], i) for i in range(n)])
        ref, _ = orc.attn_dense(qr, kr, v[:, h], 1.0 / math.sqrt(d))
        assert np.abs(out[:, p] - ref).max() < 1e-12

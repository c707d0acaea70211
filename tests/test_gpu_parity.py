"""GPU parity: the CUDA path (through the C-ABI) against the C oracle on the
same bf16-rounded inputs, and against the reference-generated golden vectors.

Contract (BASELINE.json north_star):
  * admission bits and compacted indices (Global positions) bit-exact, except
    tokens whose fp64 gate lies within 1e-6 of tau -- those must be reported;
  * attention outputs within 1e-2 relative (bf16 storage) / 1e-5 (fp32 mode),
    measured as max|gpu - ref| <= tol * max|ref| per (seq, head) slice.
"""
import glob
import math
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
import oracle as O  # noqa: E402
import topk_check as TK  # noqa: E402

# every reference-generated session: d = 128 (Llama head geometry) and the
# reference's own default ModelConfig geometry (d = 16, session_small_l2)
GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "session_*.npz")))
TOL = {"bf16": 1e-2, "f32": 1e-5}


@pytest.fixture(scope="module")
def W():
    import paper_2512_17452_b200 as W

    W.load()
    assert torch.cuda.is_available(), "GPU tests need a B200"
    return W


def rel_err(gpu, ref):
    gpu = np.asarray(gpu, np.float64)
    ref = np.asarray(ref, np.float64)
    return float(np.abs(gpu - ref).max() / max(np.abs(ref).max(), 1e-30))


def to_dev(x, dt):
    return torch.from_numpy(np.ascontiguousarray(x, np.float32)).to("cuda").to(dt)


def bf16_np(x):
    return torch.from_numpy(np.ascontiguousarray(x, np.float32)).to(torch.bfloat16).float().numpy().astype(np.float64)


# --------------------------------------------------------------------- K1 --
@pytest.mark.parametrize("w_std,b2", [(0.02, 2.0), (0.1, -2.2), (0.5, -2.5)])
def test_gate_bits_bit_exact(W, orc, w_std, b2):
    """K1 == binarize(gate_forward_batch(...)) except reported near-tau tokens."""
    L, H, d, hid, T, tau = 2, 2, 128, 128, 1500, 0.1
    bank = orc.gate_random_init(L, H, d, hid, 7, w_std, b2)
    k = bf16_np(orc.gaussian(8, T * H * d).reshape(1, T, H, d))
    s = W.Session(L, H, H, d, hid, 64, tau=tau, max_tokens=T, gate_bank=bank)
    for layer in range(L):
        k_post, g, bits, near = s.gate_forward_batch(layer, to_dev(k, torch.bfloat16))
        g, bits, kp = g.cpu().numpy(), bits.cpu().numpy(), k_post.float().cpu().numpy()
        for h in range(H):
            kr = np.stack([orc.rope(k[0, t, h], t) for t in range(T)])
            gref = orc.gate_forward_batch(bank[layer, h], k[0, :, h], kr)
            bref = orc.binarize(gref, tau)
            near_h = {int(i) % T for i in near if int(i) // T == h}
            mism = np.nonzero(bits[0, h] != bref)[0]
            assert all(t in near_h for t in mism), (mism, near_h)
            assert all(abs(gref[t] - tau) < 1e-6 for t in near_h)
            # g itself is reported in fp32 from the split-bf16 tensor-core GEMM
            # (~17 mantissa bits per operand); the decision is made exactly, the
            # reported score is accurate to ~1e-4 absolute at the largest weights.
            assert np.abs(g[0, h] - gref).max() < 1e-4
            # k_post is RoPE(k) rounded to bf16
            assert rel_err(kp[0, :, h], kr) < 1e-2


# ----------------------------------------------------------- golden vectors --
def _run_golden(W, path, dtype, impl):
    z = np.load(path)
    L, hq, hkv, d, hid, n, steps, Wn, ps, topk = (int(x) for x in z["cfg"])
    dt = torch.bfloat16 if dtype == "bf16" else torch.float32
    s = W.Session(L, hq, hkv, d, hid, Wn, tau=float(z["tau"]), rope_base=float(z["base"]), page_size=ps,
                  max_tokens=n + steps, dtype=W.BF16 if dtype == "bf16" else W.F32, gate_bank=z["bank"],
                  attn_impl=impl, topk_budget=topk)
    q, k, v = (z[x] for x in ("q", "k", "v"))
    tol = TOL[dtype]
    for l in range(L):
        out, g, bits = s.prefill_layer(l, to_dev(q[l, None, :n], dt), to_dev(k[l, None, :n], dt),
                                       to_dev(v[l, None, :n], dt), want_gates=True)
        s.sync()
        assert np.array_equal(bits.cpu().numpy()[0], z["prefill_bits"][l])
        o = out.float().cpu().numpy()[0]
        for p in range(hq):
            assert rel_err(o[:, p], z["prefill_out"][l][:, p]) < tol
    for si, t in enumerate(range(n, n + steps)):
        for l in range(L):
            out, g, ev = s.decode_layer(l, to_dev(q[l, None, t], dt), to_dev(k[l, None, t], dt),
                                        to_dev(v[l, None, t], dt), want_events=True)
            s.sync()
            assert np.array_equal(ev.cpu().numpy()[0], z["decode_events"][si, l])
            assert np.array_equal((g.cpu().numpy()[0] >= z["tau"]), z["decode_g"][si, l] >= z["tau"])
            o = out.float().cpu().numpy()[0]
            for p in range(hq):
                assert rel_err(o[p], z["decode_out"][si, l][p]) < tol
    pos = np.concatenate([s.gather(l, 0, h)["global_pos"] for l in range(L) for h in range(hkv)])
    assert np.array_equal(pos, z["global_pos"])


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p) for p in GOLDEN])
@pytest.mark.parametrize("dtype,impl", [("f32", "simt"), ("bf16", "simt"), ("bf16", "auto")])
def test_golden_session(W, path, dtype, impl):
    """The reference's own session vectors through the SIMT kernels and, in
    bf16, through the default (Blackwell) path: tcgen05 K3 where the geometry
    allows (d = 128, even GQA group), K5 + the finish kernel for decode."""
    _run_golden(W, path, dtype, W.ATTN_SIMT if impl == "simt" else W.ATTN_AUTO)


# ------------------------------------------------ random sessions vs oracle --
def _session_case(W, orc, *, T, steps, hq, hkv, Wn, nseq, dtype, seed, w_std=0.1, b2=-2.2, ps=16,
                  attn=None, base=1e4):
    d = hid = 128
    L = 1
    bank = orc.gate_random_init(L, hkv, d, hid, seed, w_std, b2)
    rnd = lambda s_, n: bf16_np(orc.gaussian(s_, n))  # noqa: E731
    q = rnd(seed + 1, nseq * (T + steps) * hq * d).reshape(nseq, T + steps, hq, d)
    k = rnd(seed + 2, nseq * (T + steps) * hkv * d).reshape(nseq, T + steps, hkv, d)
    v = rnd(seed + 3, nseq * (T + steps) * hkv * d).reshape(nseq, T + steps, hkv, d)
    dt = torch.bfloat16 if dtype == "bf16" else torch.float32
    s = W.Session(L, hq, hkv, d, hid, Wn, rope_base=base, page_size=ps, max_seqs=nseq, max_tokens=T + steps,
                  dtype=W.BF16 if dtype == "bf16" else W.F32, gate_bank=bank,
                  attn_impl=attn if attn is not None else W.ATTN_AUTO)
    out, g, bits = s.prefill_layer(0, to_dev(q[:, :T], dt), to_dev(k[:, :T], dt), to_dev(v[:, :T], dt),
                                   want_gates=True)
    s.sync()
    out = out.float().cpu().numpy()
    bits = bits.cpu().numpy()
    tol = TOL[dtype]
    worst = 0.0
    refs = []
    for b in range(nseq):
        r = O.Session(orc, L, hq, hkv, d, hid, Wn, rope_base=base, page_size=ps, gate_bank=bank,
                      max_tokens=T + steps)
        ro, rg, rb, _ = r.prefill_layer(0, q[b, :T], k[b, :T], v[b, :T])
        assert np.array_equal(bits[b], rb)
        for p in range(hq):
            worst = max(worst, rel_err(out[b, :, p], ro[:, p]))
        refs.append(r)
    assert worst < tol, worst
    for t in range(T, T + steps):
        o, gg, ev = s.decode_layer(0, to_dev(q[:, t], dt), to_dev(k[:, t], dt), to_dev(v[:, t], dt),
                                   want_events=True)
        s.sync()
        o, ev = o.float().cpu().numpy(), ev.cpu().numpy()
        for b in range(nseq):
            ro, rg, rev, _ = refs[b].decode_layer(0, q[b, t], k[b, t], v[b, t])
            assert np.array_equal(ev[b], rev)
            for p in range(hq):
                assert rel_err(o[b, p], ro[p]) < tol
    for b in range(nseq):
        for h in range(hkv):
            a, r = s.gather(0, b, h), refs[b].gather(0, h)
            assert np.array_equal(a["global_pos"], r["global_pos"])
            assert np.array_equal(a["local_pos"], r["local_pos"])
            assert np.shape(a["global_v"]) == np.shape(r["global_v"])
            if np.size(r["global_v"]):  # an empty Global cache (nothing admitted yet) has nothing to compare
                assert rel_err(a["global_v"], r["global_v"]) < 1e-2
    return s


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_session_gqa4_two_seqs(W, orc, dtype):
    _session_case(W, orc, T=700, steps=40, hq=8, hkv=2, Wn=128, nseq=2, dtype=dtype, seed=50, attn=W.ATTN_SIMT)


def test_session_long_multichunk_decode(W, orc):
    """Many pages per head so decode splits over several chunks + combine."""
    _session_case(W, orc, T=3000, steps=20, hq=4, hkv=1, Wn=256, nseq=1, dtype="bf16", seed=60, w_std=0.1, b2=0.0)


def test_session_window_larger_than_prompt(W, orc):
    """T < W: no Global at prefill; decode fills the ring then promotes."""
    _session_case(W, orc, T=40, steps=40, hq=4, hkv=1, Wn=64, nseq=1, dtype="f32", seed=70)


def test_session_odd_page_size(W, orc):
    _session_case(W, orc, T=300, steps=30, hq=4, hkv=2, Wn=37, nseq=1, dtype="f32", seed=80, ps=5)


def test_forced_full_is_dense_causal(W, orc):
    """effective_gate = 1 (policy 'full'): VS attention == dense causal."""
    d, hq, hkv, T = 128, 4, 1, 300
    q = bf16_np(orc.gaussian(1, T * hq * d).reshape(1, T, hq, d))
    k = bf16_np(orc.gaussian(2, T * hkv * d).reshape(1, T, hkv, d))
    v = bf16_np(orc.gaussian(3, T * hkv * d).reshape(1, T, hkv, d))
    s = W.Session(1, hq, hkv, d, d, 16, max_tokens=T, dtype=W.F32)
    forced = torch.ones((1, hkv, T), dtype=torch.float32, device="cuda")
    out = s.prefill_layer(0, to_dev(q, torch.float32), to_dev(k, torch.float32), to_dev(v, torch.float32),
                          forced_gates=forced).cpu().numpy()
    kr = np.stack([orc.rope(k[0, t, 0], t) for t in range(T)])
    for p in range(hq):
        qr = np.stack([orc.rope(q[0, t, p], t) for t in range(T)])
        ref, _ = orc.attn_dense(qr, kr, v[0, :, 0], 1 / math.sqrt(d))
        assert rel_err(out[0, :, p], ref) < 1e-5


@pytest.mark.parametrize("kind", ["local_sink", "stride", "recent_fraction"])
def test_policy_sessions_vs_oracle(W, orc, kind):
    """Policy overrides (engine.cpp:126-151) through forced gates: prefill +
    lazy-promotion decode equal the oracle session fed the same gates."""
    from paper_2512_17452_b200 import policy as P
    d, hq, hkv, T, steps, Wn = 128, 4, 2, 400, 70, 64
    pol = {"local_sink": P.Policy(kind="local_sink", window=Wn, sink=37),
           "stride": P.Policy(kind="wgkv", window=Wn, forced=P.ForcedAdmission("stride", keep_every=3, phase=2)),
           "recent_fraction": P.Policy(kind="wgkv", window=Wn,
                                       forced=P.ForcedAdmission("recent_fraction", fraction=0.4))}[kind]
    q = bf16_np(orc.gaussian(11, (T + steps) * hq * d).reshape(1, T + steps, hq, d))
    k = bf16_np(orc.gaussian(12, (T + steps) * hkv * d).reshape(1, T + steps, hkv, d))
    v = bf16_np(orc.gaussian(13, (T + steps) * hkv * d).reshape(1, T + steps, hkv, d))
    s = W.Session(1, hq, hkv, d, d, Wn, max_tokens=T + steps, dtype=W.BF16)
    r = O.Session(orc, 1, hq, hkv, d, d, Wn, max_tokens=T + steps)
    fg = P.policy_gates(pol, 0, 0, hkv, hkv, 1, 0, T, T)
    out = s.prefill_layer(0, to_dev(q[:, :T], torch.bfloat16), to_dev(k[:, :T], torch.bfloat16),
                          to_dev(v[:, :T], torch.bfloat16), forced_gates=torch.from_numpy(fg.copy()).cuda())
    ro, _, rb, _ = r.prefill_layer(0, q[0, :T], k[0, :T], v[0, :T], forced_gates=fg[0])
    o = out.float().cpu().numpy()[0]
    for p in range(hq):
        assert rel_err(o[:, p], ro[:, p]) < TOL["bf16"]
    for t in range(T, T + steps):
        fg = P.policy_gates(pol, 0, 0, hkv, hkv, 1, t, 1, T)
        o, _, ev = s.decode_layer(0, to_dev(q[:, t], torch.bfloat16), to_dev(k[:, t], torch.bfloat16),
                                  to_dev(v[:, t], torch.bfloat16),
                                  forced_gates=torch.from_numpy(fg.reshape(1, hkv).copy()).cuda(), want_events=True)
        ro, _, rev, _ = r.decode_layer(0, q[0, t], k[0, t], v[0, t], forced_gates=fg.reshape(hkv))
        assert np.array_equal(ev.cpu().numpy()[0], rev)
        o = o.float().cpu().numpy()[0]
        for p in range(hq):
            assert rel_err(o[p], ro[p]) < TOL["bf16"]
    for h in range(hkv):
        assert np.array_equal(s.gather(0, 0, h)["global_pos"], r.gather(0, h)["global_pos"])
    # cache_snapshot (kvstore.cpp:269-286) text, identical (forced gates are 0 / 1, exact in fp32)
    assert s.snapshot(0) == r.snapshot(native=False)


# -------------------------------------------------------------- error paths --
def test_lifecycle_and_pool_errors(W, orc):
    d = 128
    bank = orc.gate_random_init(1, 1, d, d, 3, 0.02, 20.0)
    s = W.Session(1, 4, 1, d, d, 8, max_tokens=256, capacity_pages=3, gate_bank=bank)
    x = torch.randn(1, 4, d, device="cuda").to(torch.bfloat16)
    with pytest.raises(W.LifecycleError):
        s.decode_layer(0, x, x[:, :1], x[:, :1])
    q = torch.randn(1, 200, 4, d, device="cuda").to(torch.bfloat16)
    kv = torch.randn(1, 200, 1, d, device="cuda").to(torch.bfloat16)
    s.prefill_layer(0, q, kv, kv)
    with pytest.raises(W.OutOfPages):  # saturated gates need ~13 Global pages
        s.sync()
    with pytest.raises(W.LifecycleError):
        s.prefill_layer(0, q, kv, kv)
    s.release(0, 1)
    assert s.pool_info()["free"] == 3


# ------------------------------------------------ tcgen05 prefill (K3 fast) --
@pytest.mark.parametrize("T,Wn,hq,hkv,nseq,ps", [(700, 128, 8, 2, 2, 16), (3000, 256, 4, 1, 1, 16),
                                                  (1500, 1024, 4, 1, 1, 32), (129, 64, 4, 1, 1, 8)])
def test_tc_prefill_vs_oracle(W, orc, T, Wn, hq, hkv, nseq, ps):
    _session_case(W, orc, T=T, steps=4, hq=hq, hkv=hkv, Wn=Wn, nseq=nseq, dtype="bf16", seed=90 + T, ps=ps,
                  attn=W.ATTN_TCGEN05)


def test_tc_matches_simt_bitwise_bits_close_outputs(W, orc):
    """Same device inputs through both K3 implementations."""
    d, hq, hkv, T, Wn = 128, 8, 2, 2048, 512
    bank = orc.gate_random_init(1, hkv, d, d, 5, 0.1, -2.2)
    g = torch.Generator(device="cuda").manual_seed(0)
    q = torch.randn(1, T, hq, d, device="cuda", generator=g).to(torch.bfloat16)
    k = torch.randn(1, T, hkv, d, device="cuda", generator=g).to(torch.bfloat16)
    v = torch.randn(1, T, hkv, d, device="cuda", generator=g).to(torch.bfloat16)
    outs = []
    for impl in (W.ATTN_SIMT, W.ATTN_TCGEN05):
        s = W.Session(1, hq, hkv, d, d, Wn, max_tokens=T, gate_bank=bank, attn_impl=impl, rope_base=5e5)
        outs.append(s.prefill_layer(0, q, k, v).float().cpu().numpy())
        s.sync()
    assert rel_err(outs[1], outs[0]) < 1e-2


# ---------------------------------------------------- K6 select_topk_pages --
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("budget", [1, 3, 1000])
def test_topk_decode_vs_oracle(W, orc, dtype, budget):
    """wgkv_plus_topk decode (engine.cpp:320-324): per q head, max-dot page
    scores, top-`budget` pages (ties to older), attention over them + Local."""
    d, hq, hkv, T, steps, Wn = 128, 8, 2, 600, 12, 64
    bank = orc.gate_random_init(1, hkv, d, d, 41, 0.1, -1.5)
    q = bf16_np(orc.gaussian(42, (T + steps) * hq * d).reshape(1, T + steps, hq, d))
    k = bf16_np(orc.gaussian(43, (T + steps) * hkv * d).reshape(1, T + steps, hkv, d))
    v = bf16_np(orc.gaussian(44, (T + steps) * hkv * d).reshape(1, T + steps, hkv, d))
    # plant a louder key every 40 tokens so the best pages stand out (x1.5 keeps
    # the logits in the N(0,1) regime the bf16 tolerance is stated for)
    for t in range(0, T, 40):
        k[0, t] = bf16_np(k[0, t] * 1.5)
    dt = torch.bfloat16 if dtype == "bf16" else torch.float32
    s = W.Session(1, hq, hkv, d, d, Wn, max_tokens=T + steps, dtype=W.BF16 if dtype == "bf16" else W.F32,
                  gate_bank=bank, topk_budget=budget)
    s.prefill_layer(0, to_dev(q[:, :T], dt), to_dev(k[:, :T], dt), to_dev(v[:, :T], dt))
    r = O.Session(orc, 1, hq, hkv, d, d, Wn, gate_bank=bank, max_tokens=T + steps, topk_budget=budget)
    r.prefill_layer(0, q[0, :T], k[0, :T], v[0, :T])
    ties = checks = 0
    rel = TK.BF16_KEY_REL if dtype == "bf16" else TK.FP32_ACC_REL
    for t in range(T, T + steps):
        o = s.decode_layer(0, to_dev(q[:, t], dt), to_dev(k[:, t], dt), to_dev(v[:, t], dt))
        r.decode_layer(0, q[0, t], k[0, t], v[0, t])
        o = o.float().cpu().numpy()[0]
        for p in range(hq):
            c = r.gather(0, p // (hq // hkv))
            gk, gv, lk, lv = (np.asarray(c[x], np.float64) for x in ("global_k", "global_v", "local_k", "local_v"))
            qr = orc.rope(q[0, t, p], t)
            sc, err = TK.maxdot_scores(gk, qr, rel)
            ties += TK.check_selection(o[p], qr, gk, gv, lk, lv, sc, err, budget, TOL[dtype])
            checks += 1
    print(f"top-k {dtype} budget {budget}: {ties} of {checks} (step, q head) selections resolved as bounded ties")


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("T", [20000, 70000])
def test_topk_all_ties_take_oldest(W, dtype, T):
    """Every page scores exactly 0 (k = 0), so select_topk_pages' tie rule
    (engine.cpp:36-84: stable sort, older page first) must pick logical pages
    0..budget-1; the logits are then all 0 and each q head's output is the mean
    of V over the selected tokens + the Local ring.  At T = 70000 the Global
    cache holds > 4096 pages in one score bin, which exercises the
    all-pages refinement of the threshold kernel."""
    hq, hkv, d, Wn, budget = 4, 1, 128, 1024, 100
    dt = torch.bfloat16 if dtype == "bf16" else torch.float32
    g = torch.Generator(device="cuda").manual_seed(5)
    s = W.Session(1, hq, hkv, d, d, Wn, max_tokens=T + 1, dtype=W.BF16 if dtype == "bf16" else W.F32,
                  topk_budget=budget, rope_base=5e5)
    q = torch.randn(1, T + 1, hq, d, device="cuda", generator=g).to(dt)
    k = torch.zeros(1, T + 1, hkv, d, device="cuda", dtype=dt)
    v = torch.randn(1, T + 1, hkv, d, device="cuda", generator=g).to(dt)
    ones = torch.ones(1, hkv, T, device="cuda")
    s.prefill_layer(0, q[:, :T], k[:, :T], v[:, :T], forced_gates=ones)
    out = s.decode_layer(0, q[:, T], k[:, T], v[:, T], forced_gates=torch.ones(1, hkv, device="cuda"))
    s.sync()
    # Global = tokens 0..T-W (T-W promoted by this step), Local = T-W+1..T
    vv = v[0, :, 0].double().cpu().numpy()
    sel = np.concatenate([vv[: budget * 16], vv[T - Wn + 1: T + 1]])
    ref = sel.mean(axis=0)
    o = out.double().cpu().numpy()[0]
    for p in range(hq):
        assert rel_err(o[p], ref) < TOL[dtype], p


@pytest.mark.parametrize("budget", [2, 5])
def test_topk_quest_bound_vs_numpy(W, orc, budget):
    """WGKV_TOPK_QUEST (not the reference's selection): pages ranked by Quest's
    bound sum_d max(q_d min_d, q_d max_d) over each Global page's key min / max,
    top-`budget` (ties to the older page), attention over them + the Local ring.
    Checked against numpy on the exported cache after every decode step (the
    metadata is rebuilt after prefill and kept current as promotions append)."""
    d, hq, hkv, T, steps, Wn = 128, 8, 2, 600, 12, 64
    gs = hq // hkv
    bank = orc.gate_random_init(1, hkv, d, d, 51, 0.1, -1.5)
    q = bf16_np(orc.gaussian(52, (T + steps) * hq * d).reshape(1, T + steps, hq, d))
    k = bf16_np(orc.gaussian(53, (T + steps) * hkv * d).reshape(1, T + steps, hkv, d))
    v = bf16_np(orc.gaussian(54, (T + steps) * hkv * d).reshape(1, T + steps, hkv, d))
    for t in range(0, T, 40):
        k[0, t] = bf16_np(k[0, t] * 1.5)
    dt = torch.bfloat16
    s = W.Session(1, hq, hkv, d, d, Wn, max_tokens=T + steps, gate_bank=bank, topk_budget=budget,
                  topk_mode=W.TOPK_QUEST)
    s.prefill_layer(0, to_dev(q[:, :T], dt), to_dev(k[:, :T], dt), to_dev(v[:, :T], dt))
    ties = checks = 0
    for t in range(T, T + steps):
        o = s.decode_layer(0, to_dev(q[:, t], dt), to_dev(k[:, t], dt), to_dev(v[:, t], dt)).float().cpu().numpy()[0]
        for h in range(hkv):
            c = s.gather(0, 0, h)
            gk, gv, lk, lv = (np.asarray(c[x], np.float64) for x in ("global_k", "global_v", "local_k", "local_v"))
            n = -(-gk.shape[0] // 16)
            mn = np.stack([gk[16 * i:16 * i + 16].min(0) for i in range(n)]) if n else np.zeros((0, d))
            mx = np.stack([gk[16 * i:16 * i + 16].max(0) for i in range(n)]) if n else np.zeros((0, d))
            for g in range(gs):
                p = h * gs + g
                qr = orc.rope(q[0, t, p], t)
                bound = np.maximum(qr * mn, qr * mx).sum(1)
                # keys are the device's own (exported): only fp32 accumulation differs
                err = TK.FP32_ACC_REL * (np.abs(qr) * np.maximum(np.abs(mn), np.abs(mx))).sum(1)
                ties += TK.check_selection(o[p], qr, gk, gv, lk, lv, bound, err, budget, TOL["bf16"])
                checks += 1
    print(f"quest budget {budget}: {ties} of {checks} (step, q head) selections resolved as bounded ties")


@pytest.mark.parametrize("topk", [0, 3])
def test_ragged_batch_decode(W, orc, topk):
    """Serving shape (configs[3]): sequences of different lengths prefilled one
    slot at a time, then decoded together in one batched call per step (each
    slot at its own position and cache geometry).  Every slot must match its
    own oracle session; topk exercises K6's per-(seq, kv head) selection."""
    d = hid = 128
    hq, hkv, Wn, steps = 8, 2, 64, 10
    lens = [150, 431, 777]
    nseq = len(lens)
    bank = orc.gate_random_init(1, hkv, d, hid, 91, 0.1, -1.8)
    mx = max(lens) + steps
    rnd = lambda s_, n: bf16_np(orc.gaussian(s_, n))  # noqa: E731
    q = rnd(92, nseq * mx * hq * d).reshape(nseq, mx, hq, d)
    k = rnd(93, nseq * mx * hkv * d).reshape(nseq, mx, hkv, d)
    v = rnd(94, nseq * mx * hkv * d).reshape(nseq, mx, hkv, d)
    dt = torch.bfloat16
    s = W.Session(1, hq, hkv, d, hid, Wn, max_seqs=nseq, max_tokens=mx, gate_bank=bank, topk_budget=topk)
    refs = []
    for b, T in enumerate(lens):
        s.prefill_layer(0, to_dev(q[b:b + 1, :T], dt), to_dev(k[b:b + 1, :T], dt), to_dev(v[b:b + 1, :T], dt),
                        seq0=b)
        r = O.Session(orc, 1, hq, hkv, d, hid, Wn, gate_bank=bank, max_tokens=mx, topk_budget=topk)
        r.prefill_layer(0, q[b, :T], k[b, :T], v[b, :T])
        refs.append(r)
    near = checks = 0
    for i in range(steps):
        qs = np.stack([q[b, lens[b] + i] for b in range(nseq)])
        ks = np.stack([k[b, lens[b] + i] for b in range(nseq)])
        vs = np.stack([v[b, lens[b] + i] for b in range(nseq)])
        o, _, ev = s.decode_layer(0, to_dev(qs, dt), to_dev(ks, dt), to_dev(vs, dt), want_events=True)
        o, ev = o.float().cpu().numpy(), ev.cpu().numpy()
        for b in range(nseq):
            ro, _, rev, _ = refs[b].decode_layer(0, qs[b], ks[b], vs[b])
            assert np.array_equal(ev[b], rev), (i, b)
            for p in range(hq):
                checks += 1
                if rel_err(o[b, p], ro[p]) < TOL["bf16"]:
                    continue
                assert topk, (i, b, p)  # only a top-k near-tie may flip a page
                c = refs[b].gather(0, p // (hq // hkv))
                gk, gv, lk, lv = (np.asarray(c[x], np.float64) for x in ("global_k", "global_v", "local_k", "local_v"))
                qr = orc.rope(qs[b, p], lens[b] + i)
                sc, err = TK.maxdot_scores(gk, qr, TK.BF16_KEY_REL)
                near += TK.check_selection(o[b, p], qr, gk, gv, lk, lv, sc, err, topk, TOL["bf16"])
    print(f"ragged top-k {topk}: {near} of {checks} selections resolved as bounded ties")
    for b in range(nseq):
        for h in range(hkv):
            a, r = s.gather(0, b, h), refs[b].gather(0, h)
            assert np.array_equal(a["global_pos"], r["global_pos"])
            assert np.array_equal(a["local_pos"], r["local_pos"])

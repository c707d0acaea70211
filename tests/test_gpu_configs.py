"""GPU parity at the BASELINE configurations and the multi-GPU sharding
contract, through the C-ABI, against the reference (oracle/_ref) and its C
restatement (oracle/).

* configs[0] exactly (1 layer, 32 q / 8 kv heads, d = 128, T = 4096 prefill +
  256 decode steps, W = 1024, tau = 0.1) in fp32 parity mode (SIMT kernels,
  1e-5) and in bf16 (tcgen05 K3, K5 + finish kernel, 1e-2), against the
  reference's own Session hot path (oracle/_ref, its parallel_for over heads):
  admission bits (+ the reported near-tau list), Global / Local positions,
  every decode step's promotion events, decode-gate bits and attention
  outputs, cache_stats.
* one layer of configs[2] (4 x 128K tokens, a = 0.25, the bench's calibrated
  gates): all 4M admission bits against the fp64 oracle gate, every
  (seq, kv head)'s Global positions, >= 512 sampled query rows per (seq, q
  head) -- tile edges, the last tile, random rows -- against
  attn_vertical_slash, then 32 decode steps: events and decode-gate bits every
  step, cache contents and the last step's outputs against attn_ragged.
* KV-head sharding on one GPU ("virtual shards"): N = 2/4/8
  contexts owning kv heads [r*8/N, (r+1)*8/N) reproduce the unsharded context
  BITWISE (bits, Global positions, prefill and decode outputs) with the decode
  split pinned, and within one bf16 ulp with the automatic split.
* prefill into a fragmented pool (K3's per-page TMA path), the reference-
  written .wgkv gate file (GateBank::save -> wgkv_gate_load), the decode trace.

Tolerances (BASELINE.json north_star): bits / positions / events exact except
tokens whose fp64 gate lies within 1e-6 of tau (reported); outputs
max|gpu - ref| <= tol * max|ref| per checked slice, tol = 1e-2 (bf16) / 1e-5 (fp32).
"""
import concurrent.futures as cf
import math
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
import oracle as O  # noqa: E402

TOL = {"bf16": 1e-2, "f32": 1e-5}
NTHREADS = max(1, os.cpu_count() or 1)
HERE = os.path.dirname(os.path.abspath(__file__))


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


def bf16_np(x):
    return torch.from_numpy(np.ascontiguousarray(x, np.float32)).to(torch.bfloat16).float().numpy().astype(np.float64)


def to_dev(x, dt):
    return torch.from_numpy(np.ascontiguousarray(x, np.float32)).to("cuda").to(dt)


def pool_map(fn, items):
    with cf.ThreadPoolExecutor(NTHREADS) as ex:  # ctypes calls release the GIL
        return list(ex.map(fn, items))


def calibrate_b2(orc, bank, k, tau, admit, base, layer=0):
    """b2 per kv head so that a fraction `admit` of the tokens is admitted, at the
    midpoint between the two fp64 scores that straddle the quantile:
    no token sits near the threshold by construction."""
    T, hkv = k.shape[0], k.shape[1]

    def one(h):
        b = bank[layer, h].copy()
        b[-1] = 0.0
        z = orc.gate_forward_batch(b, k[:, h], orc.rope_rows(k[:, h], 0, base))
        z = np.sort(np.log(z) - np.log1p(-z))
        i = int((1 - admit) * T)
        return math.log(tau / (1 - tau)) - 0.5 * (z[i - 1] + z[i])

    for h, b2 in enumerate(pool_map(one, range(hkv))):
        bank[layer, h, -1] = b2
    return bank


# =====================================================================
# configs[0]: one Llama-3.1-8B attention layer, 4K prefill + 256 decode
# =====================================================================
C0 = dict(L=1, hq=32, hkv=8, d=128, hid=128, T=4096, steps=256, Wn=1024, tau=0.1, base=5e5, admit=0.3)


@pytest.fixture(scope="module")
def cfg0(orc):
    """Inputs and the reference's own results (oracle/_ref Session, fp64)."""
    if not os.path.exists(O.REF_SO):
        pytest.skip("oracle/_ref missing")
    ref = O.Ref()
    c = C0
    n = c["T"] + c["steps"]
    bank = ref.gate_random_init(c["L"], c["hkv"], c["d"], c["hid"], 4242, 0.02, 0.0)
    q = bf16_np(ref.gaussian(4243, n * c["hq"] * c["d"])).reshape(n, c["hq"], c["d"])
    k = bf16_np(ref.gaussian(4244, n * c["hkv"] * c["d"])).reshape(n, c["hkv"], c["d"])
    v = bf16_np(ref.gaussian(4245, n * c["hkv"] * c["d"])).reshape(n, c["hkv"], c["d"])
    bank = calibrate_b2(orc, bank, k[: c["T"]], c["tau"], c["admit"], c["base"])
    r = O.Session(ref, c["L"], c["hq"], c["hkv"], c["d"], c["hid"], c["Wn"], tau=c["tau"], rope_base=c["base"],
                  gate_bank=bank, max_tokens=n)
    ro, rg, rb, _ = r.prefill_layer(0, q[: c["T"]], k[: c["T"]], v[: c["T"]])
    dec = [r.decode_layer(0, q[t], k[t], v[t]) for t in range(c["T"], n)]
    gath = [r.gather(0, h) for h in range(c["hkv"])]
    return dict(bank=bank, q=q, k=k, v=v, out=ro, g=rg, bits=rb, dec=dec,
                gpos=[x["global_pos"] for x in gath], lpos=[x["local_pos"] for x in gath], stats=r.cache_stats())


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_configs0_vs_reference(W, cfg0, dtype):
    c, z = C0, cfg0
    T, n = c["T"], c["T"] + c["steps"]
    dt = torch.bfloat16 if dtype == "bf16" else torch.float32
    s = W.Session(c["L"], c["hq"], c["hkv"], c["d"], c["hid"], c["Wn"], tau=c["tau"], rope_base=c["base"],
                  max_tokens=n, dtype=W.BF16 if dtype == "bf16" else W.F32, gate_bank=z["bank"])
    kd = to_dev(z["k"][None, :T], dt)
    _, _, _, near = s.gate_forward_batch(0, kd)
    near = {int(i) for i in near}
    out, g, bits = s.prefill_layer(0, to_dev(z["q"][None, :T], dt), kd, to_dev(z["v"][None, :T], dt),
                                   want_gates=True)
    s.sync()
    bits = bits.cpu().numpy()[0]
    mism = {h * T + t for h, t in zip(*np.nonzero(bits != z["bits"]))}
    assert mism <= near, sorted(mism - near)[:10]
    assert all(abs(z["g"].reshape(-1)[i] - c["tau"]) < 1e-6 for i in near)
    o = out.float().cpu().numpy()[0]
    worst = max(rel_err(o[:, p], z["out"][:, p]) for p in range(c["hq"]))
    assert worst < TOL[dtype], worst
    worst = 0.0
    for i, t in enumerate(range(T, n)):
        od, tr = s.decode_layer(0, to_dev(z["q"][None, t], dt), to_dev(z["k"][None, t], dt),
                                to_dev(z["v"][None, t], dt), want_trace=True)
        ro, rg, rev, _ = z["dec"][i]
        assert np.array_equal(tr["events"].cpu().numpy()[0], rev), i
        nt = tr["near_tau"].cpu().numpy()[0].astype(bool)
        b = tr["bits"].cpu().numpy()[0]
        assert np.array_equal(b[~nt], (rg >= c["tau"])[~nt]), i
        assert np.all(np.abs(rg[nt] - c["tau"]) < 1e-6)
        od = od.float().cpu().numpy()[0]
        worst = max(worst, max(rel_err(od[p], ro[p]) for p in range(c["hq"])))
    assert worst < TOL[dtype], worst
    for h in range(c["hkv"]):
        a = s.gather(0, 0, h)
        assert np.array_equal(a["global_pos"], z["gpos"][h]), h
        assert np.array_equal(a["local_pos"], z["lpos"][h]), h
    st = s.stats(0, 1)  # cache_stats (kvstore.cpp:253-267) vs the reference's own function
    assert st["resident_entries"] == z["stats"]["resident_entries"]
    assert st["pages_allocated"] == z["stats"]["pages_allocated"]
    assert st["admitted_fraction"] == pytest.approx(z["stats"]["admitted_fraction"], abs=0, rel=1e-15)


# =====================================================================
# configs[2]: one layer of 4 x 128K, sampled against the oracle
# =====================================================================
def _sample_rows(T, n, rng):
    fixed = {0, 1, 2, 127, 128, 129, 1023, 1024, 1025, 1151, 1152, T - 257, T - 256, T - 129, T - 128, T - 127,
             T - 2, T - 1}
    for tile in rng.choice(T // 128, 48, replace=False):  # both edges of random tiles
        fixed |= {int(tile) * 128, int(tile) * 128 + 127}
    rest = rng.choice(T, n, replace=False)
    rows = sorted(fixed | {int(x) for x in rest})
    return np.array(rows[: max(n, len(fixed))] if len(rows) > n else rows)


def test_configs2_layer_sampled(W, orc):
    B, T, hq, hkv, d, hid, Wn, tau, base, a, steps = 4, 131072, 32, 8, 128, 128, 1024, 0.1, 5e5, 0.25, 32
    gs = hq // hkv
    dev = torch.device("cuda")
    gen = torch.Generator(device=dev).manual_seed(2024)
    Q = torch.randn(B, T, hq, d, device=dev, generator=gen).to(torch.bfloat16)
    K = torch.randn(B, T, hkv, d, device=dev, generator=gen).to(torch.bfloat16)
    V = torch.randn(B, T, hkv, d, device=dev, generator=gen).to(torch.bfloat16)
    qd = torch.randn(steps, B, hq, d, device=dev, generator=gen).to(torch.bfloat16)
    kd = torch.randn(steps, B, hkv, d, device=dev, generator=gen).to(torch.bfloat16)
    vd = torch.randn(steps, B, hkv, d, device=dev, generator=gen).to(torch.bfloat16)
    # the bench's gates: W1, w2 ~ N(0, 0.02^2), b1 = 0, b2 calibrated per head to a
    rng = np.random.default_rng(42)
    blen = hid * 2 * d + 2 * hid + 1
    bank = np.zeros((1, hkv, blen))
    bank[:, :, : hid * 2 * d] = 0.02 * rng.standard_normal((1, hkv, hid * 2 * d))
    bank[:, :, hid * 2 * d + hid: hid * 2 * d + 2 * hid] = 0.02 * rng.standard_normal((1, hkv, hid))
    s = W.Session(1, hq, hkv, d, hid, Wn, tau=tau, rope_base=base, max_seqs=B, max_tokens=T + steps,
                  max_prefill_tokens=T, gate_bank=bank)
    _, g0, _, _ = s.gate_forward_batch(0, K)
    z = torch.logit(g0.clamp(1e-7, 1 - 1e-7).double())
    for h in range(hkv):
        bank[0, h, -1] = math.log(tau / (1 - tau)) - torch.quantile(z[:, h].flatten()[::16].float(), 1 - a).item()
    s.gate_set(bank)
    del g0, z
    _, _, _, near = s.gate_forward_batch(0, K)
    near = {int(i) for i in near}  # flat s*H*T + h*T + t
    out, gg, bits = s.prefill_layer(0, Q, K, V, want_gates=True)
    s.sync()
    bits_gpu = bits.cpu().numpy()
    rows = _sample_rows(T, 512, np.random.default_rng(7))
    assert len(rows) >= 512
    ridx = torch.from_numpy(rows).to(dev)
    o_rows = out[:, ridx].float().cpu().numpy()  # [B][R][hq][d]
    q_rows = Q[:, ridx].float().cpu().numpy().astype(np.float64)
    del out, Q

    # ---- 32 decode steps (GPU), then the cache of every (seq, kv head) -------
    traces = []
    for st in range(steps):
        o_dec, tr = s.decode_layer(0, qd[st], kd[st], vd[st], want_trace=True)
        traces.append({k_: v_.cpu().numpy() for k_, v_ in tr.items()})
    o_dec = o_dec.float().cpu().numpy()
    caches = [[s.gather(0, b, h) for h in range(hkv)] for b in range(B)]
    Kh = K.float().cpu().numpy()
    Vh = V.float().cpu().numpy()
    kdh = kd.float().cpu().numpy().astype(np.float64)
    vdh = vd.float().cpu().numpy().astype(np.float64)
    qlast = qd[steps - 1].float().cpu().numpy().astype(np.float64)
    scale = 1 / math.sqrt(d)
    pos = T + steps - 1

    # ---- the oracle, one task per (seq, kv head): fp64 gate of all T tokens,
    # the sampled rows of its q heads (attn_vertical_slash), the decode-gate of
    # each step's token, the final cache and the last step's outputs
    def pair(bh):
        b, h = divmod(bh, hkv)
        kp = Kh[b, :, h].astype(np.float64)
        kr = orc.rope_rows(kp, 0, base)
        gref = orc.gate_forward_batch(bank[0, h], kp, kr)
        bb = (gref >= tau).astype(np.uint8)
        vv = Vh[b, :, h].astype(np.float64)
        worst_p = 0.0
        for p in range(h * gs, (h + 1) * gs):
            ref_rows = []
            for ri, i in enumerate(rows):
                qr = orc.rope(q_rows[b, ri, p], int(i), base)[None]
                o_, _ = orc.attn_vertical_slash(qr, kr[: i + 1], vv[: i + 1], bb[: i + 1], Wn, scale,
                                                causal_offset=int(i))
                ref_rows.append(o_[0])
            worst_p = max(worst_p, rel_err(o_rows[b, :, p], np.stack(ref_rows)))
        gdec = [orc.gate_forward_batch(bank[0, h], kdh[t, b, h][None], orc.rope_rows(kdh[t, b, h][None], T + t, base))[0]
                for t in range(steps)]
        krd = np.stack([orc.rope(kdh[t, b, h], T + t, base) for t in range(steps)])
        allk = np.concatenate([kr, krd])
        allv = np.concatenate([vv, vdh[:, b, h]])
        c = caches[b][h]
        gpos = np.nonzero(bits_gpu[b, h, : pos - Wn + 1])[0]
        lpos = np.arange(pos - Wn + 1, pos + 1)
        cache_ok = (np.array_equal(c["global_pos"], gpos) and np.array_equal(c["local_pos"], lpos) and
                    np.array_equal(c["global_v"], allv[gpos].astype(np.float32)) and
                    np.array_equal(c["local_v"], allv[lpos].astype(np.float32)) and
                    rel_err(c["global_k"], allk[gpos]) < 4e-3 and rel_err(c["local_k"], allk[lpos]) < 4e-3)
        worst_d = 0.0
        for p in range(h * gs, (h + 1) * gs):
            ref, _ = orc.attn_ragged(orc.rope(qlast[b, p], pos, base), allk[gpos], allv[gpos], allk[lpos], allv[lpos],
                                     scale)
            worst_d = max(worst_d, rel_err(o_dec[b, p], ref))
        return gref, worst_p, np.array(gdec), cache_ok, worst_d

    res = pool_map(pair, range(B * hkv))
    gref = np.stack([r[0] for r in res]).reshape(B, hkv, T)
    bref = (gref >= tau).astype(np.uint8)
    # every admission bit: exact except the reported near-tau tokens
    mism = {(b * hkv + h) * T + t for b, h, t in zip(*np.nonzero(bits_gpu != bref))}
    assert mism <= near, (len(mism - near), sorted(mism - near)[:5])
    assert all(abs(gref.reshape(-1)[i] - tau) < 1e-6 for i in near)
    frac = bref[:, :, : T - Wn].mean()
    assert abs(frac - a) < 0.01, frac
    # sampled prefill rows (K3) vs attn_vertical_slash
    worst = max(r[1] for r in res)
    assert worst < TOL["bf16"], worst
    # decode: promotion events and decode-gate bits of every step
    for st, tr in enumerate(traces):
        assert np.array_equal(tr["events"], np.where(bits_gpu[:, :, T + st - Wn] == 1, 1, 2)), st
        gd = np.stack([r[2][st] for r in res]).reshape(B, hkv)
        nt = tr["near_tau"].astype(bool)
        assert np.all(np.abs(gd[nt] - tau) < 1e-6)
        assert np.array_equal(tr["bits"][~nt], (gd >= tau)[~nt]), st
    # cache contents (positions, exact V, K = bf16(RoPE)) and the last outputs (K5 + finish)
    assert all(r[3] for r in res)
    worst = max(r[4] for r in res)
    assert worst < TOL["bf16"], worst


# =====================================================================
# KV-head sharding on one GPU: N contexts reproduce the unsharded one
# =====================================================================
def _shard_run(W, bank, q, k, v, qd, kd, vd, hq, hkv, off, pin, Wn, T, steps, B):
    d = q.shape[-1]
    s = W.Session(1, hq, hkv, d, d, Wn, rope_base=5e5, max_seqs=B, max_tokens=T + steps, gate_bank=bank,
                  kv_head_offset=off, decode_chunk_pages=pin)
    out, g, bits = s.prefill_layer(0, q, k, v, want_gates=True)
    dec = [s.decode_layer(0, qd[i], kd[i], vd[i]) for i in range(steps)]
    s.sync()
    gpos = [[s.gather(0, b, h)["global_pos"] for h in range(hkv)] for b in range(B)]
    return dict(out=out, bits=bits, dec=torch.stack(dec), gpos=gpos)


@pytest.mark.parametrize("pin", [16, 0])
def test_virtual_shards_reproduce_unsharded(W, orc, pin):
    """with the path partitioned by KV head, rank r of N owns kv
    heads [r*8/N, (r+1)*8/N), their GQA q heads and gate rows.  Per-head
    arithmetic is unchanged, so the concatenated results equal the unsharded
    context's BITWISE when the decode split is pinned (pin = 16); with the
    automatic split (pin = 0) K5's chunking follows the launch's total work and
    decode outputs agree to one bf16 rounding."""
    B, T, hq, hkv, d, Wn, steps = 2, 3000, 32, 8, 128, 256, 6
    gen = torch.Generator(device="cuda").manual_seed(77)
    rnd = lambda *sh: torch.randn(*sh, device="cuda", generator=gen).to(torch.bfloat16)  # noqa: E731
    q, k, v = rnd(B, T, hq, d), rnd(B, T, hkv, d), rnd(B, T, hkv, d)
    qd, kd, vd = rnd(steps, B, hq, d), rnd(steps, B, hkv, d), rnd(steps, B, hkv, d)
    bank = orc.gate_random_init(1, hkv, d, d, 31, 0.1, -2.0)
    full = _shard_run(W, bank, q, k, v, qd, kd, vd, hq, hkv, 0, pin, Wn, T, steps, B)
    for N in (2, 4, 8):
        hk, hqs = hkv // N, hq // N
        parts = [_shard_run(W, bank, q[:, :, r * hqs:(r + 1) * hqs].contiguous(),
                            k[:, :, r * hk:(r + 1) * hk].contiguous(), v[:, :, r * hk:(r + 1) * hk].contiguous(),
                            qd[:, :, r * hqs:(r + 1) * hqs].contiguous(), kd[:, :, r * hk:(r + 1) * hk].contiguous(),
                            vd[:, :, r * hk:(r + 1) * hk].contiguous(), hqs, hk, r * hk, pin, Wn, T, steps, B)
                 for r in range(N)]
        assert torch.equal(torch.cat([p_["bits"] for p_ in parts], dim=1), full["bits"]), N
        assert torch.equal(torch.cat([p_["out"] for p_ in parts], dim=2), full["out"]), N
        for b in range(B):
            for r in range(N):
                for h in range(hk):
                    assert np.array_equal(parts[r]["gpos"][b][h], full["gpos"][b][r * hk + h])
        # C1's assembly step: the rank-major all-gather result -> the reference's
        # concat layout (engine.cpp:234-238), bitwise the unsharded output
        rank_major = torch.stack([p_["out"].reshape(B * T, -1) for p_ in parts])
        full_out = torch.empty_like(full["out"])
        W.assemble_heads(rank_major, full_out, N, B * T)
        assert torch.equal(full_out, full["out"]), N
        dec = torch.cat([p_["dec"] for p_ in parts], dim=2)
        if pin:
            assert torch.equal(dec, full["dec"]), N
        else:
            diff = (dec.float() - full["dec"].float()).abs()
            assert (diff <= 2 ** -7 * full["dec"].float().abs() + 1e-6).all(), N


# =====================================================================
# fragmented pool, gate file, decode trace
# =====================================================================
def test_prefill_into_fragmented_pool(W, orc):
    """Release two non-adjacent sequences and prefill a longer one: its Global
    pages come from two separate physical runs, so K3 loads the vertical
    prefix page by page (the path a serving pool takes after reuse)."""
    hq, hkv, d, Wn, T0, T1, steps = 8, 2, 128, 128, 600, 1400, 6
    bank = orc.gate_random_init(1, hkv, d, d, 61, 0.1, -1.6)
    rnd = lambda sd, *sh: bf16_np(orc.gaussian(sd, int(np.prod(sh))).reshape(sh))  # noqa: E731
    s = W.Session(1, hq, hkv, d, d, Wn, max_seqs=3, max_tokens=T1 + steps, gate_bank=bank, attn_impl=W.ATTN_TCGEN05)
    for b in range(3):
        s.prefill_layer(0, to_dev(rnd(100 + b, 1, T0, hq, d), torch.bfloat16),
                        to_dev(rnd(200 + b, 1, T0, hkv, d), torch.bfloat16),
                        to_dev(rnd(300 + b, 1, T0, hkv, d), torch.bfloat16), seq0=b)
    s.release(0, 1)
    s.release(2, 1)
    q, k, v = rnd(7, T1 + steps, hq, d), rnd(8, T1 + steps, hkv, d), rnd(9, T1 + steps, hkv, d)
    out = s.prefill_layer(0, to_dev(q[None, :T1], torch.bfloat16), to_dev(k[None, :T1], torch.bfloat16),
                          to_dev(v[None, :T1], torch.bfloat16), seq0=0)
    r = O.Session(orc, 1, hq, hkv, d, d, Wn, gate_bank=bank, max_tokens=T1 + steps)
    ro, _, _, _ = r.prefill_layer(0, q[:T1], k[:T1], v[:T1])
    o = out.float().cpu().numpy()[0]
    assert max(rel_err(o[:, p], ro[:, p]) for p in range(hq)) < TOL["bf16"]
    for t in range(T1, T1 + steps):
        od = s.decode_layer(0, to_dev(q[None, t], torch.bfloat16), to_dev(k[None, t], torch.bfloat16),
                            to_dev(v[None, t], torch.bfloat16), seq0=0).float().cpu().numpy()[0]
        rd, _, _, _ = r.decode_layer(0, q[t], k[t], v[t])
        assert max(rel_err(od[p], rd[p]) for p in range(hq)) < TOL["bf16"]
    for h in range(hkv):
        assert np.array_equal(s.gather(0, 0, h)["global_pos"], r.gather(0, h)["global_pos"])
    # the untouched slot 1 still matches its own prefill
    assert s.state(0, 1, 0)["tokens_seen"] == T0


def test_gate_file_written_by_reference(W, orc):
    """GateBank::save (gating.cpp:107-122) by the reference -> wgkv_gate_load
    (gating.cpp:124-147) -> the same bits as the bank set in memory, and as the
    oracle's fp64 gate; a bad magic is rejected like GateBank::load."""
    path = os.path.join(HERE, "golden", "gate_bank_d32.wgkv")
    bank = np.load(os.path.join(HERE, "golden", "gate_bank_d32_bank.npy"))
    L, H, d, hid, T, tau = 2, 2, 32, 32, 700, 0.1
    k = bf16_np(orc.gaussian(17, T * H * d).reshape(1, T, H, d))
    s_file = W.Session(L, 2 * H, H, d, hid, 64, tau=tau, max_tokens=T)
    s_file.gate_load(path)
    s_mem = W.Session(L, 2 * H, H, d, hid, 64, tau=tau, max_tokens=T, gate_bank=bank)
    for layer in range(L):
        _, g1, b1, near = s_file.gate_forward_batch(layer, to_dev(k, torch.bfloat16))
        _, g2, b2, _ = s_mem.gate_forward_batch(layer, to_dev(k, torch.bfloat16))
        assert torch.equal(b1, b2) and torch.equal(g1, g2)
        near = {int(i) for i in near}
        for h in range(H):
            gref = orc.gate_forward_batch(orc.gate_load(path)[layer, h], k[0, :, h], orc.rope_rows(k[0, :, h], 0))
            mism = {h * T + t for t in np.nonzero(b1.cpu().numpy()[0, h] != (gref >= tau))[0]}
            assert mism <= near
    bad = os.path.join(str(pytest.importorskip("tempfile").mkdtemp()), "bad.wgkv")
    with open(bad, "wb") as f:
        f.write(b"XXXX" + open(path, "rb").read()[4:])
    with pytest.raises(ArithmeticError):
        s_file.gate_load(bad)


def test_decode_trace_near_tau_reported(W, orc):
    """A decode token whose fp64 gate is within 1e-6 of tau is flagged, and the
    trace's g / bit follow the reference's exact operation order elsewhere."""
    hq, hkv, d, Wn, T = 4, 1, 128, 16, 40
    bank = orc.gate_random_init(1, hkv, d, d, 5, 0.1, 0.0)
    k = bf16_np(orc.gaussian(3, (T + 1) * hkv * d).reshape(T + 1, hkv, d))
    kp = k[T, 0][None]
    z = orc.gate_forward_batch(bank[0, 0], kp, orc.rope_rows(kp, T, 1e4))[0]
    bank[0, 0, -1] = math.log(0.1 / 0.9) - (math.log(z) - math.log1p(-z)) + 1e-8  # g(T) ~ tau + 1e-9
    q = bf16_np(orc.gaussian(4, (T + 1) * hq * d).reshape(T + 1, hq, d))
    v = bf16_np(orc.gaussian(6, (T + 1) * hkv * d).reshape(T + 1, hkv, d))
    s = W.Session(1, hq, hkv, d, d, Wn, max_tokens=T + 1, gate_bank=bank)
    s.prefill_layer(0, to_dev(q[None, :T], torch.bfloat16), to_dev(k[None, :T], torch.bfloat16),
                    to_dev(v[None, :T], torch.bfloat16))
    _, tr = s.decode_layer(0, to_dev(q[None, T], torch.bfloat16), to_dev(k[None, T], torch.bfloat16),
                           to_dev(v[None, T], torch.bfloat16), want_trace=True)
    gr = orc.gate_forward_batch(bank[0, 0], kp, orc.rope_rows(kp, T, 1e4))[0]
    assert abs(gr - 0.1) < 1e-6
    assert tr["near_tau"].item() == 1
    assert tr["bits"].item() == (gr >= 0.1)  # the exact-order fp64 gate reproduces the reference's bit here


def test_comm_world_one(W, orc):
    """wgkv_comm_init / wgkv_allgather_heads through NCCL with a world of one
    (the only world one GPU can host): prefill- and decode-shaped outputs come
    back in the reference's layout, synchronously and on the comm stream."""
    hq, hkv, d, T, B = 8, 2, 128, 300, 2
    s = W.Session(1, hq, hkv, d, d, 64, max_seqs=B, max_tokens=T, gate_bank=orc.gate_random_init(1, hkv, d, d, 3))
    s.comm_init(W.nccl_unique_id(), 1, 0)
    x = torch.randn(B, T, hq, d, device="cuda").to(torch.bfloat16)
    full = torch.zeros_like(x)
    s.allgather_heads(x, full)
    s.sync()
    assert torch.equal(full, x)
    full2 = torch.zeros_like(x)
    s.allgather_heads(x, full2, async_=True)
    s.comm_join()
    s.sync()
    assert torch.equal(full2, x)
    xd = torch.randn(B, hq, d, device="cuda").to(torch.bfloat16)
    fd = torch.zeros_like(xd)
    s.allgather_heads(xd, fd)
    s.sync()
    assert torch.equal(fd, xd)
    with pytest.raises(ValueError):  # rank 1 of 2 must own kv heads [hkv, 2 hkv)
        W.Session(1, hq, hkv, d, d, 64, max_tokens=T).comm_init(W.nccl_unique_id(), 2, 1)


@pytest.mark.parametrize("with_comm", [False, True])
def test_output_proj_overlapped(W, orc, with_comm):
    """f3 (engine.cpp:243-245): x += concat . Wo^T after the head all-gather.
    With a communicator the rows go through the chunked gather -> GEMM
    pipeline (3 chunks of <= 1024 rows here, both ring slots reused); without
    one the local heads are the concat.  Checked against an fp64 product of the
    same bf16 operands (fp32 accumulation: 1e-5 of the output scale)."""
    hq, hkv, d, T, B, dim = 8, 2, 128, 1300, 2, 512
    s = W.Session(1, hq, hkv, d, d, 64, max_seqs=B, max_tokens=T,
                  gate_bank=orc.gate_random_init(1, hkv, d, d, 3))
    if with_comm:
        s.comm_init(W.nccl_unique_id(), 1, 0)
    g = torch.Generator(device="cuda").manual_seed(7)
    lo = torch.randn(B, T, hq, d, device="cuda", generator=g).to(torch.bfloat16)
    wo = (torch.randn(dim, hq * d, device="cuda", generator=g) / (hq * d) ** 0.5).to(torch.bfloat16)
    x0 = torch.randn(B, T, dim, device="cuda", generator=g)
    x = x0.clone()
    s.output_proj(lo, wo, x)
    s.sync()
    ref = x0.double() + lo.reshape(B, T, hq * d).double() @ wo.double().T
    err = (x.double() - ref).abs().max().item() / ref.abs().max().item()
    assert err < 1e-5, err
    # decode shape: one token per sequence
    xd0 = torch.randn(B, dim, device="cuda", generator=g)
    xd = xd0.clone()
    s.output_proj(lo[:, 0].contiguous(), wo, xd)
    s.sync()
    refd = xd0.double() + lo[:, 0].reshape(B, hq * d).double() @ wo.double().T
    assert (xd.double() - refd).abs().max().item() / refd.abs().max().item() < 1e-5


@pytest.mark.parametrize("dm,T", [(512, 700), (4096, 300)])
def test_gate_proj_fused(W, orc, dm, T):
    """f1 (engine.cpp:190-205): the key projection fused into K1.  k_pre must be
    the bf16 rounding of x . Wk^T (fp32 accumulation may land a value on the
    other side of a bf16 rounding boundary: at most one ulp, rarely), and given
    that k_pre, k_post / g / bits / near list must be exactly what K1
    (wgkv_gate_score, itself pinned to the oracle) produces."""
    hq, hkv, d, B = 8, 2, 128, 2
    bank = orc.gate_random_init(1, hkv, d, d, 17, 0.1, -2.2)
    s = W.Session(1, hq, hkv, d, d, 64, max_seqs=B, max_tokens=T, rope_base=5e5, gate_bank=bank)
    g = torch.Generator(device="cuda").manual_seed(11)
    x = torch.randn(B, T, dm, device="cuda", generator=g).to(torch.bfloat16)
    wk = (torch.randn(hkv, d, dm, device="cuda", generator=g) / dm ** 0.5).to(torch.bfloat16)
    k_pre, k_post, gg, bits, near = s.gate_forward_batch_proj(0, x, wk, pos0=5)
    s.sync()
    ref = torch.einsum("btk,hdk->bthd", x.double(), wk.double())
    ref_bf = ref.to(torch.bfloat16)
    diff = k_pre != ref_bf
    frac = diff.float().mean().item()
    assert frac < 1e-2, frac  # grows with dm (fp32 accumulation error vs a bf16 ulp)
    if diff.any():  # only rounding-boundary cases: one bf16 ulp plus the fp32 accumulation error
        kd, rd = k_pre[diff].double(), ref[diff]
        mag = torch.einsum("btk,hdk->bthd", x.double().abs(), wk.double().abs())[diff]
        assert ((kd - rd).abs() <= rd.abs() * 2.0 ** -7 + 2 * dm * 2.0 ** -24 * mag).all()
    k_post2, g2, bits2, near2 = s.gate_forward_batch(0, k_pre, pos0=5)
    s.sync()
    assert torch.equal(k_post, k_post2)
    assert torch.equal(bits, bits2)
    assert torch.equal(gg, g2)
    assert sorted(near.tolist()) == sorted(near2.tolist())
    print(f"gate_proj dm={dm}: {frac:.2e} of k_pre on the other side of a bf16 rounding boundary, "
          f"{int(bits.sum())} admitted")


def test_decode_many_pairs(W, orc):
    """configs[3]-like batch geometry: 64 sequence slots x 4 kv heads = 256
    (seq, kv head) pairs in one decode launch (K5's per-pair state no longer
    fits its shared memory next to two CTAs per SM and is read from HBM), each
    slot at its own length; sampled slots checked against their own oracle
    sessions (outputs, promotion events, Global positions)."""
    d = hid = 128
    hq, hkv, Wn, steps, nseq = 16, 4, 64, 3, 64
    rng = np.random.default_rng(5)
    lens = [int(x) for x in rng.integers(80, 260, nseq)]
    bank = orc.gate_random_init(1, hkv, d, hid, 61, 0.1, -1.8)
    mx = max(lens) + steps
    s = W.Session(1, hq, hkv, d, hid, Wn, max_seqs=nseq, max_tokens=mx, gate_bank=bank)
    g = torch.Generator(device="cuda").manual_seed(3)
    q = torch.randn(nseq, mx, hq, d, device="cuda", generator=g).to(torch.bfloat16)
    k = torch.randn(nseq, mx, hkv, d, device="cuda", generator=g).to(torch.bfloat16)
    v = torch.randn(nseq, mx, hkv, d, device="cuda", generator=g).to(torch.bfloat16)
    for b, T in enumerate(lens):
        s.prefill_layer(0, q[b:b + 1, :T], k[b:b + 1, :T], v[b:b + 1, :T], seq0=b)
    check = [0, 17, 42, 63]
    refs = {}
    for b in check:
        r = O.Session(orc, 1, hq, hkv, d, hid, Wn, gate_bank=bank, max_tokens=mx)
        f = lambda t: t.float().cpu().numpy().astype(np.float64)  # noqa: E731
        r.prefill_layer(0, f(q[b, :lens[b]]), f(k[b, :lens[b]]), f(v[b, :lens[b]]))
        refs[b] = r
    for i in range(steps):
        idx = torch.tensor([lens[b] + i for b in range(nseq)], device="cuda")
        ar = torch.arange(nseq, device="cuda")
        qs, ks, vs = q[ar, idx].contiguous(), k[ar, idx].contiguous(), v[ar, idx].contiguous()
        o, _, ev = s.decode_layer(0, qs, ks, vs, want_events=True)
        o, ev = o.float().cpu().numpy(), ev.cpu().numpy()
        for b in check:
            f = lambda t: t.float().cpu().numpy().astype(np.float64)  # noqa: E731
            ro, _, rev, _ = refs[b].decode_layer(0, f(qs[b]), f(ks[b]), f(vs[b]))
            assert np.array_equal(ev[b], rev), (i, b)
            for p in range(hq):
                assert rel_err(o[b, p], ro[p]) < TOL["bf16"], (i, b, p)
    for b in check:
        for h in range(hkv):
            assert np.array_equal(s.gather(0, b, h)["global_pos"], refs[b].gather(0, h)["global_pos"])


def test_comm_world_one_in_cuda_graph(W, orc):
    """The decode-shaped head all-gather through NCCL captured inside a CUDA
    graph (bench.py captures one token step, C1 included) and replayed: the
    output follows the inputs of each replay."""
    hq, hkv, d, B = 8, 2, 128, 2
    s = W.Session(1, hq, hkv, d, d, 64, max_seqs=B, max_tokens=64, gate_bank=orc.gate_random_init(1, hkv, d, d, 3))
    s.comm_init(W.nccl_unique_id(), 1, 0)
    xd = torch.zeros(B, hq, d, device="cuda", dtype=torch.bfloat16)
    fd = torch.zeros_like(xd)
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    s.set_stream(st)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        s.allgather_heads(xd, fd)
    s.set_stream(torch.cuda.current_stream())
    torch.cuda.current_stream().wait_stream(st)
    for i in range(3):
        xd.copy_(torch.randn(B, hq, d, device="cuda").to(torch.bfloat16))
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(fd, xd), i


def test_f1_f3_argument_errors(W, orc):
    """The f1 / f3 entry points reject what they do not implement the way the
    rest of the C-ABI does (ENOTSUP / EINVAL, no kernel launched)."""
    from paper_2512_17452_b200._lib import NotSupported

    hq, hkv, d = 8, 2, 128
    bank = orc.gate_random_init(1, hkv, d, d, 3)
    s32 = W.Session(1, hq, hkv, d, d, 64, max_tokens=64, dtype=W.F32, gate_bank=bank)
    lo = torch.zeros(1, 8, hq, d, device="cuda")
    wo = torch.zeros(256, hq * d, device="cuda", dtype=torch.bfloat16)
    with pytest.raises(NotSupported):  # bf16 contexts only
        s32.output_proj(lo, wo, torch.zeros(1, 8, 256, device="cuda"))
    s = W.Session(1, hq, hkv, d, d, 64, max_tokens=64, gate_bank=bank)
    x = torch.zeros(1, 8, 100, device="cuda", dtype=torch.bfloat16)
    wk = torch.zeros(hkv, d, 100, device="cuda", dtype=torch.bfloat16)
    with pytest.raises(NotSupported):  # model dim must be a multiple of 64
        s.gate_forward_batch_proj(0, x, wk)
    with pytest.raises(ValueError):  # T beyond max_prefill_tokens
        s.gate_forward_batch_proj(0, torch.zeros(1, 65, 128, device="cuda", dtype=torch.bfloat16),
                                  torch.zeros(hkv, d, 128, device="cuda", dtype=torch.bfloat16))

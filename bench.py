#!/usr/bin/env python3
"""bench.py -- WG-KV hot path on B200: prefill tok/s @128K and decode tok/s/GPU.

Workload (BASELINE.json configs[2], the config the metric is quoted on):
  Llama-3.1-8B attention stack: 32 layers, 32 Q / 8 KV heads, d = 128, gate
  hidden = 128, W = 1024, tau = 0.1, page 16, RoPE base 5e5; batch 4 x 128K
  prefill, then `decode_steps` decode steps over all layers.  Synthetic
  N(0,1) Q/K/V (bf16) and random gate MLPs (w_std 0.02) whose b2 is calibrated
  per (layer, kv head) to the paper's 75 % sparsity (admission a = 0.25).
  Q/K/V come from `slots` distinct resident layer-input sets used round-robin
  (the per-layer work is identical; 32 distinct sets would need 205 GB).

One step = prefill of every layer (K1 gate -> K2 compaction -> K3 VS
attention, plus the head-output all-gather when N > 1) followed by the decode
steps (K4 append -> K5 split-KV attention -> combine, per layer), then the
caches are released.  N GPUs shard the KV heads (8/N per rank, their GQA
q heads, gate banks and caches): per-GPU work shrinks, total work is fixed
("scaling": "strong"); the per-layer NCCL all-gather of head outputs is the
only collective.

`--impl reference` times the reference's own CPU implementation
(oracle/_ref, compiled from the reference sources) on a bounded sample and
extrapolates to the same workload; it runs on rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # configs[2]: 128K-context prefill + decode, batch 4 (the metric's config)
    "128k": dict(workload="llama3.1-8b attention x32 layers, 128K prefill x batch 4 + decode (BASELINE configs[2])",
                 layers=32, q_heads=32, kv_heads=8, d=128, hidden=128, T=131072, batch=4, window=1024, admit=0.25,
                 tau=0.1, rope_base=5e5, page=16, decode_steps=32),
    # configs[1]: full 32-layer stack, 32K prefill, batch 1
    "32k": dict(workload="llama3.1-8b attention x32 layers, 32K prefill x batch 1 + decode (BASELINE configs[1])",
                layers=32, q_heads=32, kv_heads=8, d=128, hidden=128, T=32768, batch=1, window=1024, admit=0.25,
                tau=0.1, rope_base=5e5, page=16, decode_steps=1024),  # configs[1]: 1K decode steps
}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return dict(hbm=p["hbm_gbs"], tf=p["bf16_tflops"], tf_sus=p.get("bf16_tflops_sustained", p["bf16_tflops"]),
                    src="measured")
    except Exception:
        return dict(hbm=6650.0, tf=1590.0, tf_sus=1400.0, src="fallback")


# ------------------------------------------------------------------ clocks --
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device, self.rows, self.proc = device, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), "--query-gpu=" + self.FIELDS,
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = [r for r in self.rows if len(r) >= 7 and r[0].replace(".", "").isdigit()]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(r[0]) for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i].lower().startswith("active")})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": max(float(r[1]) for r in rows), "reasons": reasons,
                "samples": len(rows), "power_w_max": max(float(r[2]) for r in rows if r[2] not in ("", "[N/A]"))}


# --------------------------------------------------------------- helpers --
def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def pair_count(bits, window):
    """vs_mask_pair_count per (seq, kv head) row of bits [..., T] (closed form, int64, on device)."""
    import torch

    T = bits.shape[-1]
    i = torch.arange(T, device=bits.device)
    band = torch.clamp(i + 1, max=window).sum()
    if T <= window:
        return (band * torch.ones(bits.shape[:-1], dtype=torch.int64, device=bits.device))
    c = torch.cumsum(bits[..., : T - window].to(torch.int64), dim=-1)  # C(x) for x = 1..T-W
    return band + c.sum(dim=-1)


def executed_pairs(bits, window):
    """(q, k) pairs K3's tcgen05 tiles actually compute per (seq, kv head) row
    of bits [..., T] for ONE q head: every 128-row query tile runs full 128 x 128
    S/PV blocks over its vertical prefix (ceil(C / 128) blocks, C = admitted
    keys before the band) and its band (ceil(band / 128) blocks) -- the
    masked-off entries of the edge blocks included (attn_tc.cu's block count)."""
    import torch

    T = bits.shape[-1]
    pc = torch.nn.functional.pad(torch.cumsum(bits.to(torch.int64), dim=-1), (1, 0))  # admitted before x
    i0 = torch.arange(0, T, 128, device=bits.device)
    s_lo = torch.clamp(i0 - window + 1, min=0)
    band = torch.clamp(i0 + 127, max=T - 1) - s_lo + 1
    nv = (pc[..., s_lo] + 127) // 128
    nb = (band + 127) // 128
    return ((nv + nb) * 128 * 128).sum(dim=-1)


# ------------------------------------------------------------ reference arm --
def _ref_session(O, ref, cfg, hq, hkv, T, bank):
    return O.Session(ref, 1, hq, hkv, cfg["d"], cfg["hidden"], cfg["window"], tau=cfg["tau"],
                     rope_base=cfg["rope_base"], page_size=cfg["page"], gate_bank=bank, max_tokens=T)


def cpu_reference(cfg, sample_T=8192, steps=1, decode_steps=3, with_cfg0=True):
    """The reference's own hot path (oracle/_ref: the unmodified reference
    sources, fp64, WGKV_THREADS = host cores) on the host:
      * prefill: one layer of one sequence at T = sample_T, all heads, timed
        per phase and extrapolated per phase to the workload (gate + mask per
        token, vertical-slash attention per permitted pair, populate per token);
      * decode: the reference's decode step (gate_forward + local_write + gather
        + attn_ragged, engine.cpp:291-327) timed on a cache built at the
        workload's context length (HeadCache::prefill_populate at admission a),
        2 of the kv heads, scaled to all heads, layers and sequences;
      * configs[0] (1 layer, 32 q / 8 kv, 4K prefill + 256 decode steps) timed
        in full -- measured, not extrapolated."""
    import numpy as np

    nthreads = os.cpu_count() or 1
    os.environ["WGKV_THREADS"] = str(nthreads)  # read once by thread_budget() (numerics.cpp:119-128)
    import oracle as O

    O.build()
    ref = O.Ref()
    hq, hkv, d, hid, W = cfg["q_heads"], cfg["kv_heads"], cfg["d"], cfg["hidden"], cfg["window"]
    Ts = min(sample_T, cfg["T"])
    bank = ref.gate_random_init(1, hkv, d, hid, 1234, 0.02, 0.0)
    rng = np.random.default_rng(0)
    q = rng.standard_normal((Ts, hq, d)).astype(np.float32).astype(np.float64)
    k = rng.standard_normal((Ts, hkv, d)).astype(np.float32).astype(np.float64)
    v = rng.standard_normal((Ts, hkv, d)).astype(np.float32).astype(np.float64)
    # calibrate b2 so the sample admits the same fraction a as the GPU run
    for h in range(hkv):
        kr = np.stack([ref.rope(k[i, h], i, cfg["rope_base"]) for i in range(0, Ts, 8)])
        g = ref.gate_forward_batch(bank[0, h], k[::8, h], kr)
        z = np.log(g / (1 - g))
        bank[0, h, -1] = math.log(cfg["tau"] / (1 - cfg["tau"])) - np.quantile(z, 1 - cfg["admit"])
    secs_all, pairs = np.zeros(3), 0
    for _ in range(steps):
        s = _ref_session(O, ref, cfg, hq, hkv, Ts, bank)
        secs, pairs = s.prefill_layer_timed(0, q, k, v)
        secs_all += secs
        del s
    secs_all /= steps
    # full-workload extrapolation
    Tf, B, L, a = cfg["T"], cfg["batch"], cfg["layers"], cfg["admit"]
    pairs_full_head = Tf * min(W, Tf) - min(W, Tf) * (min(W, Tf) - 1) / 2 + a * (Tf - W) * (Tf - W + 1) / 2
    pairs_full = pairs_full_head * hq * B * L
    t_full = (secs_all[0] / Ts * Tf * B * L + secs_all[1] / pairs * pairs_full + secs_all[2] / Ts * Tf * B * L)
    tok_s = B * Tf / t_full
    out = dict(value=tok_s, unit="tok/s", cores=nthreads, kind="reference",
               sample=(f"reference Session::prefill hot path (oracle/_ref, fp64) on 1 layer x 1 seq x {hq}q/{hkv}kv "
                       f"heads at T={Ts} (admit {cfg['admit']}): gate {secs_all[0]:.2f}s, VS attention "
                       f"{secs_all[1]:.2f}s for {pairs:.3g} pairs ({pairs / secs_all[1]:.3g} pairs/s), populate "
                       f"{secs_all[2]:.3f}s; extrapolated per phase to {L} layers x {B} x {Tf} tokens "
                       f"({pairs_full:.3g} pairs) = {t_full:.3g} s"),
               sample_seconds=float(secs_all.sum()), pairs_per_s=pairs / secs_all[1])

    # ---- decode at the workload's context: 2 kv heads (8 q heads), scaled -----
    hk2, hq2 = min(2, hkv), min(2, hkv) * (hq // hkv)
    kk = rng.standard_normal((Tf, hk2, d)).astype(np.float32).astype(np.float64)
    vv = rng.standard_normal((Tf, hk2, d)).astype(np.float32).astype(np.float64)
    gates = np.where(rng.random((hk2, Tf)) < a, 0.9, 0.05)
    s = _ref_session(O, ref, cfg, hq2, hk2, Tf + decode_steps + 1, bank[:, :hk2])
    s.populate_layer(0, kk, vv, gates)
    del kk, vv
    t0 = time.perf_counter()
    for i in range(decode_steps):
        s.decode_layer(0, rng.standard_normal((hq2, d)), rng.standard_normal((hk2, d)), rng.standard_normal((hk2, d)))
    t_step = (time.perf_counter() - t0) / decode_steps * (hkv / hk2)  # one layer of one sequence, all heads
    del s
    out["decode"] = dict(value=1.0 / (t_step * L), unit="tok/s/GPU", cores=1, kind="reference",
                         sample=(f"reference decode step (gate_forward + local_write + gather + attn_ragged, serial "
                                 f"as engine.cpp:291-327) on a {Tf}-token cache (admit {a}) of {hk2} kv / {hq2} q heads, "
                                 f"{decode_steps} steps, {t_step / (hkv / hk2) * 1e3:.1f} ms each; x{hkv // hk2} heads, "
                                 f"x{L} layers per token; the batch's {B} sequences are sequential work"))
    if with_cfg0:
        out["configs0_measured"] = cpu_reference_cfg0(O, ref, cfg)
    return out


def cpu_reference_cfg0(O, ref, cfg):
    """BASELINE configs[0] timed in full on the reference (no extrapolation)."""
    import numpy as np

    hq, hkv, d, hid, T, D = 32, 8, 128, 128, 4096, 256
    c0 = dict(cfg, window=1024, T=T)
    bank = ref.gate_random_init(1, hkv, d, hid, 77, 0.02, -0.5)
    rng = np.random.default_rng(1)
    q = rng.standard_normal((T + D, hq, d)).astype(np.float32).astype(np.float64)
    k = rng.standard_normal((T + D, hkv, d)).astype(np.float32).astype(np.float64)
    v = rng.standard_normal((T + D, hkv, d)).astype(np.float32).astype(np.float64)
    s = _ref_session(O, ref, c0, hq, hkv, T + D, bank)
    t0 = time.perf_counter()
    s.prefill_layer(0, q[:T], k[:T], v[:T])
    t1 = time.perf_counter()
    for t in range(T, T + D):
        s.decode_layer(0, q[t], k[t], v[t])
    t2 = time.perf_counter()
    return dict(prefill_tok_s=T / (t1 - t0), decode_tok_s=D / (t2 - t1), prefill_s=t1 - t0, decode_s=t2 - t1,
                cores=os.cpu_count() or 1,
                sample="BASELINE configs[0] in full on the reference (oracle/_ref, fp64): 1 layer, 32q/8kv, d=128, "
                       "T=4096 prefill (parallel_for over heads) + 256 decode steps, W=1024")


# ------------------------------------------------------------------ GPU arm --
def run_gpu(args, cfg):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2512_17452_b200 as W
    from paper_2512_17452_b200._lib import check

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)  # plumbing only: barrier, max-over-ranks, the NCCL id
    L, Hq, Hkv, d, hid = cfg["layers"], cfg["q_heads"], cfg["kv_heads"], cfg["d"], cfg["hidden"]
    # N = the number of KV-head shards: the GPUs of the job, or --emulate-shard N
    # on one GPU (rank 0's shard; the NVLink transfer itself is not emulated)
    shards = world if world > 1 else max(1, args.emulate_shard)
    assert Hkv % shards == 0, "KV heads must divide the shard count"
    hkv, hq = Hkv // shards, Hq // shards
    T, B, Wn, D = cfg["T"], cfg["batch"], cfg["window"], cfg["decode_steps"]
    if args.tokens:
        T = args.tokens
    stream = torch.cuda.current_stream(dev)

    # ---- gate bank (fp64 host, GateBank layout), this rank's rows ------------
    rng = np.random.default_rng(42)
    blen = hid * 2 * d + 2 * hid + 1
    bank = np.zeros((L, Hkv, blen))
    bank[:, :, : hid * 2 * d] = 0.02 * rng.standard_normal((L, Hkv, hid * 2 * d))
    bank[:, :, hid * 2 * d + hid: hid * 2 * d + 2 * hid] = 0.02 * rng.standard_normal((L, Hkv, hid))
    sess = W.Session(L, hq, hkv, d, hid, Wn, tau=cfg["tau"], rope_base=cfg["rope_base"], page_size=cfg["page"],
                     max_seqs=B, max_tokens=T + D, max_prefill_tokens=T, kv_head_offset=rank * hkv, device=local,
                     gate_bank=bank)
    if world > 1:  # C1 through the C-ABI: NCCL communicator owned by the context
        box = [W.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        sess.comm_init(box[0], world, rank)
    peer = shards > 1 and args.decode_exchange == "peer"
    peer_pf = shards > 1 and args.prefill_exchange == "peer"
    peer_regions = None
    if peer or peer_pf:  # C1 over peer memory: every rank's exchange region mapped here
        bulk = B * T if peer_pf else 0
        if world > 1:
            sess.peer_init(world, rank, B, bulk)  # IPC handles exchanged over torch.distributed
        else:  # emulated shard: the other ranks' regions live on this GPU (one region stands for all of
            # them: rank 0's stores to each remote rank land in it), only rank 0's words / signal are awaited
            nb = sess.peer_region_bytes(shards, B, bulk)
            peer_regions = [torch.zeros(nb, dtype=torch.uint8, device=dev) for _ in range(2)]
            sess.peer_attach(shards, 0, B, [peer_regions[0]] + [peer_regions[1]] * (shards - 1), wait_ranks=1,
                             max_bulk_rows=bulk)
        if peer:
            sess.peer_decode(True)  # every decode layer pushes its rows from inside its merge
        if peer_pf:
            sess.peer_prefill(True)  # K3's epilogue stores its rows into every rank's bulk slot
    # ---- resident inputs: `slots` distinct layer-input sets ------------------
    slots = max(1, min(args.slots, L))
    gen = torch.Generator(device=dev).manual_seed(1000 + rank)

    def randn(*shape):
        x = torch.empty(*shape, dtype=torch.bfloat16, device=dev)
        flat = x.view(-1)
        step = 1 << 28
        for o in range(0, flat.numel(), step):
            n = min(step, flat.numel() - o)
            flat[o: o + n] = torch.randn(n, generator=gen, device=dev).to(torch.bfloat16)
        return x

    Q = [randn(B, T, hq, d) for _ in range(slots)]
    K = [randn(B, T, hkv, d) for _ in range(slots)]
    V = [randn(B, T, hkv, d) for _ in range(slots)]
    # decode inputs step-major, [D][slots][B][heads][d]: one copy per tensor and step
    qd_all, kd_all, vd_all = randn(D, slots, B, hq, d), randn(D, slots, B, hkv, d), randn(D, slots, B, hkv, d)
    qd = [qd_all[:, i] for i in range(slots)]
    kd = [kd_all[:, i] for i in range(slots)]
    vd = [vd_all[:, i] for i in range(slots)]
    # head outputs: double-buffered when the all-gather of layer l runs on the
    # comm stream while layer l+1's attention writes the other buffer
    outs = [torch.empty(B, T, hq, d, dtype=torch.bfloat16, device=dev) for _ in range(2 if shards > 1 else 1)]
    dout = torch.empty(B, hq, d, dtype=torch.bfloat16, device=dev)
    full = (torch.empty(B, T, Hq, d, dtype=torch.bfloat16, device=dev)
            if shards > 1 and args.prefill_exchange == "nccl" else None)
    dfull = torch.empty(B, Hq, d, dtype=torch.bfloat16, device=dev) if shards > 1 else None
    # emulated shard: the rank-major receive buffer NCCL would fill
    stage = (torch.zeros(shards, B * T, hq * d, dtype=torch.bfloat16, device=dev)
             if world == 1 and shards > 1 and args.prefill_exchange == "nccl" else None)
    dstage = (torch.zeros(shards, B, hq * d, dtype=torch.bfloat16, device=dev)
              if world == 1 and shards > 1 and args.decode_exchange == "nccl" else None)

    # ---- calibrate b2 per (layer, kv head) to admission a ---------------------
    ztau = math.log(cfg["tau"] / (1 - cfg["tau"]))
    for l in range(L):
        _, g, _, _ = sess.gate_forward_batch(l, K[l % slots])
        z = torch.logit(g.clamp(1e-7, 1 - 1e-7).double())  # b2 = 0 here
        for h in range(hkv):
            zz = z[:, h].flatten()
            sub = zz[:: max(1, zz.numel() // (1 << 22))]
            bank[l, rank * hkv + h, -1] = ztau - torch.quantile(sub.float(), 1 - cfg["admit"]).item()
    sess.gate_set(bank)
    del g, z

    lib, h = sess.lib, sess.h
    g_ws = torch.empty(B, hkv, T, dtype=torch.float32, device=dev)
    bits_ws = torch.empty(B, hkv, T, dtype=torch.uint8, device=dev)
    kpost = torch.empty(B, T, hkv, d, dtype=torch.bfloat16, device=dev)
    P = lambda t: None if t is None else __import__("ctypes").c_void_p(t.data_ptr())  # noqa: E731
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    launches = {"n": 0}

    def exchange_prefill(o_):
        """C1 after a layer's attention: the all-gather of head outputs on the
        context's comm stream (overlapping the next layer), or its local part
        (the assembly) when one GPU emulates a shard; nothing with the peer
        exchange (K3 itself stored the rows into every rank's bulk slot)."""
        if peer_pf:
            return
        if world > 1:
            sess.comm_join()  # the previous layer's exchange is done: its buffer may be rewritten
            sess.allgather_heads(o_, full, async_=True)
            launches["n"] += 1
        elif stage is not None:
            W.assemble_heads(stage, full, shards, B * T)
            launches["n"] += 1

    def prefill_layer(l, k3_events=None, inputs=None, out_buf=None):
        qi, ki, vi = inputs if inputs is not None else (Q[l % slots], K[l % slots], V[l % slots])
        o_ = outs[l % len(outs)] if out_buf is None else out_buf
        check(lib.wgkv_gate_score(h, l, B, T, 0, P(ki), None, P(kpost), P(g_ws), P(bits_ws), None, 0, None), "K1")
        check(lib.wgkv_admit_prefill(h, l, 0, B, T, P(kpost), P(vi), P(g_ws), P(bits_ws)), "K2")
        if k3_events is not None:
            k3_events[0].record(stream)
        check(lib.wgkv_vs_prefill(h, l, 0, B, T, P(qi), P(kpost), P(vi), P(bits_ws), P(o_)), "K3")
        if k3_events is not None:
            k3_events[1].record(stream)
        launches["n"] += 6  # rope table, gate, recheck, plan, scatter, vs
        if shards > 1:
            exchange_prefill(o_)

    def prefill_layer_seq(l, s_, inputs, out_buf):
        """The same layer body for sequence slot s_ alone (e2e: the first layer
        starts on sequence 0 while the other sequences' inputs are still on PCIe,
        the last layer's outputs drain per sequence)."""
        qi, ki, vi = (x[s_:s_ + 1] for x in inputs)
        o_ = out_buf[s_:s_ + 1]
        check(lib.wgkv_gate_score(h, l, 1, T, 0, P(ki), None, P(kpost[s_:s_ + 1]), P(g_ws[s_:s_ + 1]),
                                  P(bits_ws[s_:s_ + 1]), None, 0, None), "K1")
        check(lib.wgkv_admit_prefill(h, l, s_, 1, T, P(kpost[s_:s_ + 1]), P(vi), P(g_ws[s_:s_ + 1]),
                                     P(bits_ws[s_:s_ + 1])), "K2")
        check(lib.wgkv_vs_prefill(h, l, s_, 1, T, P(qi), P(kpost[s_:s_ + 1]), P(vi), P(bits_ws[s_:s_ + 1]), P(o_)),
              "K3")
        launches["n"] += 6

    # One decode token-step over all layers, issued eagerly or replayed from a
    # CUDA graph captured once (kills per-kernel launch gaps); the step's new
    # q/k/v are copied into static buffers first, so every replay is a real step.
    sq_all, sk_all, sv_all = (torch.empty_like(x[0]) for x in (qd_all, kd_all, vd_all))
    sq = [sq_all[i] for i in range(slots)]
    sk = [sk_all[i] for i in range(slots)]
    sv = [sv_all[i] for i in range(slots)]

    def exchange_decode(o_, l):
        if args.decode_exchange == "none":
            return
        if peer:  # fused into the layer: its merge pushed, the next layer unpacks (the last: peer_wait)
            if l == L - 1:
                sess.peer_wait()
        elif world > 1:
            sess.allgather_heads(o_, dfull)  # KB-sized: on the compute stream, inside the graph
        elif dstage is not None:
            W.assemble_heads(dstage, dfull, shards, B)

    def decode_token_step(qs=None, ks=None, vs=None, os_=None):
        for l in range(L):
            sl = l % slots
            qi, ki, vi = (sq[sl], sk[sl], sv[sl]) if qs is None else (qs[l], ks[l], vs[l])
            o_ = dout if os_ is None else os_[l]
            check(lib.wgkv_decode_layer(h, l, 0, B, P(qi), P(ki), P(vi), None, P(o_), None, None), "decode")
            if shards > 1:
                exchange_decode(o_, l)

    # kernels per decode layer: counted from the captured graph when there is one
    # (1 for the fused small-batch layer, 2 = K5 + finish otherwise) [+ C1]
    per_layer_dec = 2 + (1 if shards > 1 and args.decode_exchange == "nccl" else 0)
    assert not peer or L % 4 == 0, "peer exchanges rotate over 4 slots: a replayed token step holds a multiple of 4"
    graph = {"g": None}
    graph_kernels = {"n": None, "last": None}

    def _capture(fn):
        """CUDA graph of fn's launches, captured on a side stream (recorded, not executed).
        Also counts the library's kernel nodes in it (graph_kernels["n"])."""
        gs = torch.cuda.Stream(dev)
        gs.wait_stream(stream)
        sess.set_stream(gs)
        g_ = torch.cuda.CUDAGraph(keep_graph=True)
        with torch.cuda.graph(g_, stream=gs):
            fn()
        sess.set_stream(stream)
        stream.wait_stream(gs)
        graph_kernels["last"] = _count_wgkv_kernels(g_.raw_cuda_graph())
        g_.instantiate()
        return g_

    def decode_all():
        for s_ in range(D):
            sq_all.copy_(qd_all[s_], non_blocking=True)
            sk_all.copy_(kd_all[s_], non_blocking=True)
            sv_all.copy_(vd_all[s_], non_blocking=True)
            if graph["g"] is not None:
                graph["g"].replay()
            else:
                decode_token_step()
            launches["n"] += graph_kernels["n"] if graph["g"] is not None and graph_kernels["n"] else per_layer_dec * L

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def prefill_all(record):
        k3 = [(ev(), ev()) for _ in range(L)] if record else None
        for l in range(L):
            prefill_layer(l, k3[l] if k3 else None)
        if world > 1:
            sess.comm_join()  # the last layer's exchange belongs to the prefill
        return k3

    def one_step(record):
        e = [ev() for _ in range(3)]
        e[0].record(stream)
        k3 = prefill_all(record)
        e[1].record(stream)
        decode_all()
        e[2].record(stream)
        return e, k3

    # ---- warm-up (also: pair counts and resident bytes for the roofline) ----
    pairs_layer, exec_layer = [], []
    resident = None
    for wi in range(args.warmup):
        if wi == 0:
            for l in range(L):
                prefill_layer(l)
                pairs_layer.append(int(pair_count(bits_ws, Wn).sum().item()) * (hq // hkv))
                exec_layer.append(int(executed_pairs(bits_ws, Wn).sum().item()) * (hq // hkv))
            if world > 1:
                sess.comm_join()
            st0 = sess.stats(0, B)
            if not args.no_graphs:  # capture one token-step over all layers (recorded, not executed)
                graph["g"] = _capture(decode_token_step)
                graph_kernels["n"] = graph_kernels["last"]  # library kernels per token step (all layers)
            decode_all()
            st1 = sess.stats(0, B)
            resident = (st0["resident_entries"], st1["resident_entries"])
            sess.sync()
        else:
            one_step(False)
        sess.release(0, B)
    sess.sync()

    # ---- timed steps -----------------------------------------------------------
    launches["n"] = 0
    per = []
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.profiler.start()  # `ncu --profile-from-start off` captures the timed region only
        t_wall0 = time.perf_counter()
        for _ in range(args.steps):
            e, k3 = one_step(True)
            sess.release(0, B)
            launches["n"] += 1
            per.append((e, k3))
        barrier()
        t_wall = time.perf_counter() - t_wall0
        torch.cuda.profiler.stop()
    sess.sync()
    pre_ms = [e[0].elapsed_time(e[1]) for e, _ in per]
    dec_ms = [e[1].elapsed_time(e[2]) for e, _ in per]
    k3_ms = [sum(a.elapsed_time(b) for a, b in k3) for _, k3 in per]
    tot_ms = [e[0].elapsed_time(e[2]) for e, _ in per]
    stats = torch.tensor([sum(pre_ms), sum(dec_ms), sum(k3_ms), sum(tot_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(stats, op=dist.ReduceOp.MAX)
    pre_s, dec_s, k3_s, tot_s = (x / 1000.0 / args.steps for x in stats.tolist())

    # ---- end to end through the public API, host buffers -----------------------
    e2e = None
    if not args.no_e2e:
        hq_in = torch.empty_like(Q[0], device="cpu").pin_memory()
        hk_in = torch.empty_like(K[0], device="cpu").pin_memory()
        hv_in = torch.empty_like(V[0], device="cpu").pin_memory()
        hq_in.copy_(Q[0])
        hk_in.copy_(K[0])
        hv_in.copy_(V[0])
        h_out = torch.empty_like(outs[0], device="cpu").pin_memory()
        bufs = [(torch.empty_like(Q[0]), torch.empty_like(K[0]), torch.empty_like(V[0])) for _ in range(2)]
        e_outs = [outs[0], outs[1] if len(outs) > 1 else torch.empty_like(outs[0])]
        # three-stage pipeline on three streams: H2D of layer l+1's inputs, the
        # layer's kernels (+ C1), and D2H of layer l-1's output (this rank's
        # heads) run concurrently (PCIe is full duplex); inputs and outputs are
        # double-buffered
        h2d_s, d2h_s = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        ready = [torch.cuda.Event() for _ in range(2)]
        free = [torch.cuda.Event() for _ in range(2)]
        computed = [torch.cuda.Event() for _ in range(2)]
        drained = [torch.cuda.Event() for _ in range(2)]
        barrier()
        t0 = ev()
        t1 = ev()
        t0.record(stream)
        h2d_s.wait_stream(stream)
        d2h_s.wait_stream(stream)
        h2d = d2h = 0

        # the first layer's inputs and the last layer's outputs have nothing to
        # overlap with but the layer itself: they move (and are processed) one
        # sequence at a time (single-GPU runs; with C1 the layer is one call)
        per_seq = shards == 1 and B > 1
        ready0 = [torch.cuda.Event() for _ in range(B)]
        done_last = [torch.cuda.Event() for _ in range(B)]

        def load(l):
            b_ = l % 2
            with torch.cuda.stream(h2d_s):
                if l >= 2:
                    h2d_s.wait_event(free[b_])  # layer l-2 has consumed this buffer
                if l == 0 and per_seq:
                    for s_ in range(B):
                        for dst, src in zip(bufs[b_], (hq_in, hk_in, hv_in)):
                            dst[s_].copy_(src[s_], non_blocking=True)
                        ready0[s_].record(h2d_s)
                else:
                    for dst, src in zip(bufs[b_], (hq_in, hk_in, hv_in)):
                        dst.copy_(src, non_blocking=True)
                ready[b_].record(h2d_s)

        load(0)
        for l in range(L):
            b = l % 2
            if l + 1 < L:
                load(l + 1)
            if l >= 2:
                stream.wait_event(drained[b])  # output of layer l-2 is on the host
            if per_seq and l in (0, L - 1):
                if l != 0:
                    stream.wait_event(ready[b])
                for s_ in range(B):
                    if l == 0:
                        stream.wait_event(ready0[s_])
                    prefill_layer_seq(l, s_, bufs[b], e_outs[b])
                    if l == L - 1:
                        done_last[s_].record(stream)
                        with torch.cuda.stream(d2h_s):
                            d2h_s.wait_event(done_last[s_])
                            h_out[s_].copy_(e_outs[b][s_], non_blocking=True)
                free[b].record(stream)
                if l == L - 1:
                    drained[b].record(d2h_s)
                else:
                    computed[b].record(stream)
                    with torch.cuda.stream(d2h_s):
                        d2h_s.wait_event(computed[b])
                        h_out.copy_(e_outs[b], non_blocking=True)
                        drained[b].record(d2h_s)
            else:
                stream.wait_event(ready[b])
                prefill_layer(l, inputs=bufs[b], out_buf=e_outs[b])
                free[b].record(stream)
                computed[b].record(stream)
                with torch.cuda.stream(d2h_s):
                    d2h_s.wait_event(computed[b])
                    h_out.copy_(e_outs[b], non_blocking=True)
                    drained[b].record(d2h_s)
            h2d += sum(x.numel() * x.element_size() for x in bufs[b])
            d2h += e_outs[b].numel() * e_outs[b].element_size()
        if world > 1:
            sess.comm_join()
        stream.wait_stream(d2h_s)
        stream.wait_stream(h2d_s)
        # decode: one CUDA graph per token-step (H2D of the step's q/k/v from a
        # pinned staging slot, the 32 layers' kernels (+ C1), D2H of the
        # outputs), two graphs alternating over double-buffered staging slots
        dq_d = torch.empty((L,) + tuple(qd[0][0].shape), dtype=torch.bfloat16, device=dev)
        dk_d = torch.empty((L,) + tuple(kd[0][0].shape), dtype=torch.bfloat16, device=dev)
        dv_d = torch.empty((L,) + tuple(vd[0][0].shape), dtype=torch.bfloat16, device=dev)
        do_d = torch.empty((L,) + tuple(dout.shape), dtype=torch.bfloat16, device=dev)
        stage_h = [[torch.empty_like(x, device="cpu").pin_memory() for x in (dq_d, dk_d, dv_d, do_d)]
                   for _ in range(2)]
        dq_h = qd[0].cpu()
        dk_h = kd[0].cpu()
        dv_h = vd[0].cpu()

        def e2e_step(b):
            sq_h, sk_h, sv_h, so_h = stage_h[b]
            dq_d.copy_(sq_h, non_blocking=True)
            dk_d.copy_(sk_h, non_blocking=True)
            dv_d.copy_(sv_h, non_blocking=True)
            decode_token_step(dq_d, dk_d, dv_d, do_d)
            so_h.copy_(do_d, non_blocking=True)

        e2e_graphs = [_capture(lambda b=b: e2e_step(b)) for b in range(2)] if not args.no_graphs else None
        step_done = [torch.cuda.Event() for _ in range(2)]
        t_mid = ev()
        t_mid.record(stream)
        for s_ in range(D):
            b = s_ % 2
            if s_ >= 2:
                step_done[b].synchronize()  # the slot's previous step has drained
            for dst, src in zip(stage_h[b][:3], (dq_h[s_], dk_h[s_], dv_h[s_])):
                dst.copy_(src.unsqueeze(0).expand_as(dst))  # this step's token inputs of every layer
            if e2e_graphs:
                e2e_graphs[b].replay()
            else:
                e2e_step(b)
            step_done[b].record(stream)
            h2d += sum(x.numel() * x.element_size() for x in (dq_d, dk_d, dv_d))
            d2h += do_d.numel() * do_d.element_size()
        t1.record(stream)
        barrier()
        sess.release(0, B)
        e2e_pre = t0.elapsed_time(t_mid) / 1000.0
        e2e_dec = t_mid.elapsed_time(t1) / 1000.0
        mx = torch.tensor([e2e_pre, e2e_dec], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        e2e_pre, e2e_dec = mx.tolist()
        e2e = {"value": B * T / e2e_pre, "unit": "tok/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "decode_tok_s_per_gpu": B * D / e2e_dec / world,
               "note": "one step through the C-ABI from pinned host buffers. Prefill: per layer H2D of Q/K/V and D2H "
                       "of this rank's attention output, on their own streams (PCIe full duplex) overlapping the "
                       "layer kernels (and, N > 1, the head all-gather), inputs and outputs double-buffered. "
                       "Decode: per token-step a CUDA graph of one H2D of the 32 layers' q/k/v, the layers' kernels "
                       "(+ all-gather) and one D2H of their outputs, from double-buffered pinned staging slots the "
                       "host fills each step"}

    if world > 1:
        dist.barrier()
    res = dict(pre_s=pre_s, dec_s=dec_s, k3_s=k3_s, tot_s=tot_s, wall_s=t_wall, pairs_layer=pairs_layer,
               exec_layer=exec_layer,
               resident=resident, clocks=clk.summary(), launches=launches["n"] // args.steps, e2e=e2e,
               dec_kernels_per_layer=(graph_kernels["n"] / L if graph_kernels["n"] else per_layer_dec),
               T=T, B=B, D=D, world=world, shards=shards, hq=hq, hkv=hkv)
    if world > 1:
        dist.destroy_process_group()
    return rank, res


def _e2e_per_gpu(e2e, world, shards):
    """An emulated shard (one GPU, N shards) reports decode per GPU of the
    N-GPU job like the device-timed line: the job's tok/s over N GPUs."""
    if e2e is None or not (world == 1 and shards > 1):
        return e2e
    e2e = dict(e2e)
    e2e["decode_tok_s_per_gpu"] = e2e["decode_tok_s_per_gpu"] / shards
    return e2e


def _count_wgkv_kernels(raw_graph):
    """Kernel nodes of a captured CUDA graph whose function is one of this
    library's (mangled names in namespace wgkv); None if the graph cannot be read."""
    try:
        from cuda.bindings import driver as dr
        gr = dr.CUgraph(init_value=int(raw_graph))
        _, _, n = dr.cuGraphGetNodes(gr, 0)
        _, nodes, n = dr.cuGraphGetNodes(gr, n)
        cnt = 0
        for nd in nodes[:n]:
            _, ty = dr.cuGraphNodeGetType(nd)
            if ty != dr.CUgraphNodeType.CU_GRAPH_NODE_TYPE_KERNEL:
                continue
            err, prm = dr.cuGraphKernelNodeGetParams(nd)
            if err != dr.CUresult.CUDA_SUCCESS:
                continue
            err, name = dr.cuFuncGetName(prm.func)
            if err == dr.CUresult.CUDA_SUCCESS and b"wgkv" in (name or b""):
                cnt += 1
        return cnt
    except Exception:  # noqa: BLE001 -- diagnostics only; the caller falls back
        return None


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="128k", choices=sorted(CONFIGS) + ["serve", "1m"],
                    help="128k = the headline (configs[2]); 32k = configs[1]; serve / 1m = configs[3] / configs[4] "
                         "(bench_configs.py)")
    ap.add_argument("--shard-of", type=int, default=2, help="serve: hold rank 0's KV-head shard of N GPUs")
    ap.add_argument("--topk", type=int, default=256, help="1m: select_topk_pages budget (pages per q head)")
    ap.add_argument("--slots", type=int, default=4, help="distinct resident layer-input sets")
    ap.add_argument("--tokens", type=int, default=0, help="override T (diagnostics only, not a reported config)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graphs", action="store_true", help="issue decode kernels eagerly instead of a CUDA graph")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-T", type=int, default=16384)
    ap.add_argument("--prefill-exchange", default="peer", choices=["peer", "nccl"],
                    help="prefill C1 (N > 1): fused into K3's epilogue over peer memory, or NCCL all-gather + assembly")
    ap.add_argument("--decode-exchange", default="peer", choices=["peer", "nccl", "none"],
                    help="decode C1 (N > 1): fused into the decode layer over peer memory (wgkv_peer_decode: LL words "
                         "from the merge) or NCCL all-gather + assembly ('none': no exchange, diagnostics only)")
    ap.add_argument("--emulate-shard", type=int, default=0,
                    help="one GPU runs rank 0's KV-head shard of N GPUs (8/N kv heads) incl. the head all-gather's "
                         "local part; the NVLink transfer is not emulated and no scaling curve is measured")
    args = ap.parse_args()
    if args.config in ("serve", "1m"):
        import bench_configs

        if args.impl == "reference":
            print(json.dumps({"impl": "reference", "unavailable": "secondary config; the reference arm runs on the "
                              "headline config only"}))
            return
        bench_configs.main(args, load_peaks(), ClockSampler)
        return
    cfg = dict(CONFIGS[args.config])
    if args.tokens:
        cfg["T"] = args.tokens
    rank, world, _ = dist_env()
    peaks = load_peaks()
    base_cfg = {"workload": cfg["workload"], "batch": cfg["batch"], "prefill_tokens": cfg["T"],
                "decode_steps": cfg["decode_steps"], "layers": cfg["layers"],
                "heads": f"{cfg['q_heads']}q/{cfg['kv_heads']}kv", "head_dim": cfg["d"], "gate_hidden": cfg["hidden"],
                "window": cfg["window"], "admission": cfg["admit"], "tau": cfg["tau"], "page_size": cfg["page"],
                "parallelism": f"kv-head shard x{world}", "l2": "inputs larger than L2 (no flush)"}
    if args.emulate_shard > 1 and world == 1:
        base_cfg["parallelism"] = f"emulated: rank 0 of a kv-head shard x{args.emulate_shard}, on 1 GPU"
    metric = "WG-KV prefill tok/s @128K & decode tok/s/GPU, % of tensor/HBM roofline"

    if args.impl == "reference":
        if rank != 0:
            return
        steps = max(1, min(args.steps, 2))
        cb = cpu_reference(cfg, args.cpu_sample_T, steps)
        line = {"metric": metric, "impl": "reference", "value": cb["value"], "unit": "tok/s", "n_gpus": args.gpus,
                "steps": steps, "warmup": 0, "ms_per_step": 1000.0 * cb["sample_seconds"],
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic", "config": base_cfg,
                "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample", "decode",
                                                    "configs0_measured") if k in cb},
                "decode_tok_s_per_gpu": cb["decode"]["value"],
                "e2e": {"value": cb["value"], "unit": "tok/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    rank, r = run_gpu(args, cfg)
    if rank != 0:
        return
    L, d, B, T, D, world = cfg["layers"], cfg["d"], r["B"], r["T"], r["D"], r["world"]
    pairs = sum(r["pairs_layer"])  # this rank's q heads, all layers
    flops = 4.0 * d * pairs
    k3_tfs = flops / r["k3_s"] / 1e12
    exec_flops = 4.0 * d * sum(r["exec_layer"])  # full 128 x 128 blocks K3 computes (north_star: FLOPs executed)
    k3_exec_tfs = exec_flops / r["k3_s"] / 1e12
    # decode bytes per step (resident Global+Local K+V, bf16, each byte once per GQA group) + q/out
    res0, res1 = r["resident"]
    avg_res = 0.5 * (res0 + res1)
    dec_bytes = D * (avg_res * 2 * d * 2 + 2 * B * r["hq"] * d * 2 * L)
    dec_gbs = dec_bytes / r["dec_s"] / 1e9
    prefill_tok_s = B * T / r["pre_s"]
    shards = r["shards"]
    if world == 1 and shards > 1:  # emulated shard: whole-job numbers as if every shard ran on its own GPU
        decode_tok_s_gpu = B * D / r["dec_s"] / shards
    else:
        decode_tok_s_gpu = B * D / r["dec_s"] / world
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "k3_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get("bytes_per_launch")
        except Exception:
            traffic = None
    line = {
        "metric": metric, "value": prefill_tok_s, "unit": "tok/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1000.0 * r["tot_s"], "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic", "config": base_cfg,
        "decode_tok_s_per_gpu": decode_tok_s_gpu,
        "prefill_s_per_step": r["pre_s"], "decode_s_per_step": r["dec_s"],
        "roofline": {"bound": "tensor", "kernel": "vs_prefill_tc_kernel (K3)", "achieved": k3_tfs,
                     "peak": peaks["tf_sus"], "unit": "TFLOP/s", "frac": k3_tfs / peaks["tf_sus"],
                     "frac_of_burst": k3_tfs / peaks["tf"], "peak_source": peaks["src"] + " bf16_tflops_sustained",
                     "traffic": traffic, "k3_share_of_prefill": r["k3_s"] / r["pre_s"],
                     "algorithmic_flops_per_step": flops,
                     "executed": {"flops_per_step": exec_flops, "achieved": k3_exec_tfs,
                                  "frac": k3_exec_tfs / peaks["tf_sus"],
                                  "note": "the sparse FLOPs K3 actually executes (full 128x128 blocks of every "
                                          "query tile's vertical prefix and band, edge masks included)"},
                     "note": "achieved = 4*d*sum(vs_mask_pair_count) over (seq, q head, layer) / K3 time (CUDA events)"},
        "decode_roofline": {"bound": "hbm", "achieved": dec_gbs, "peak": peaks["hbm"], "unit": "GB/s",
                            "frac": dec_gbs / peaks["hbm"], "frac_of_8TBps": dec_gbs / 8000.0,
                            "bytes_per_decode_step": dec_bytes / D,
                            "note": "resident Global+Local K+V bytes (bf16) + q/out per token-step / decode time"},
        "clocks": r["clocks"], "gpu_launches": r["launches"],
        "decode_kernels_per_layer": r["dec_kernels_per_layer"], "e2e": _e2e_per_gpu(r["e2e"], world, shards),
    }
    if world == 1 and shards > 1:
        line["emulated_shard"] = {
            "n": shards, "kv_heads_per_gpu": r["hkv"], "q_heads_per_gpu": r["hq"],
            "decode_exchange": args.decode_exchange, "prefill_exchange": args.prefill_exchange,
            "note": "one GPU runs rank 0's shard (its heads of every token) plus the head all-gather's local part. "
                    "Prefill 'peer': K3's epilogue stores rank 0's rows into all N ranks' bulk slots (the N-1 remote "
                    "ones land in one region on this GPU), then the signal / wait kernels; 'nccl': the assembly "
                    "kernel. Decode 'peer': each layer's merge stores rank 0's rows as LL words into all N ranks' "
                    "regions and the next layer unpacks rank 0's words; 'nccl': the assembly kernel. 'value' is the "
                    "whole-job prefill tok/s if every shard ran this fast on its own GPU; the NVLink transfer latency "
                    "is NOT included and no scaling curve was measured"}
    if not args.no_cpu_baseline:
        try:
            cb = cpu_reference(cfg, args.cpu_sample_T, 1)
            line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample", "decode",
                                                       "configs0_measured") if k in cb}
        except Exception as exc:  # the reference build needs g++ on the host
            line["cpu_baseline"] = {"value": None, "unit": "tok/s", "cores": os.cpu_count(), "kind": "reference",
                                    "sample": f"unavailable: {exc}"}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()

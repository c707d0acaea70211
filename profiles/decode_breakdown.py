#!/usr/bin/env python3
"""Decode micro-benchmark: time K4 (append+gate) and K5 (attention+combine)
separately on one layer of the 128K x 4 configuration (admission a = 0.25 via
forced gates, so the cache geometry matches the bench).  GPU only.
    python profiles/decode_breakdown.py [--T 131072] [--batch 4] [--iters 200]
"""
import argparse
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2512_17452_b200 as W  # noqa: E402
from paper_2512_17452_b200._lib import check  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--T", type=int, default=131072)
    ap.add_argument("--batch", type=int, default=4)
    ap.add_argument("--iters", type=int, default=200)
    ap.add_argument("--admit", type=float, default=0.25)
    ap.add_argument("--impl", type=int, default=0, help="attn_impl (0 auto, 1 simt)")
    ap.add_argument("--hq", type=int, default=32)
    ap.add_argument("--hkv", type=int, default=8)
    ap.add_argument("--topk", type=int, default=0, help="topk_budget (Global pages per q head; 0 = all)")
    ap.add_argument("--quest", action="store_true", help="topk_mode = WGKV_TOPK_QUEST (page min/max bound)")
    args = ap.parse_args()
    B, T, Hq, Hkv, d = args.batch, args.T, args.hq, args.hkv, 128
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(0)
    import numpy as np

    bank = np.zeros((1, Hkv, d * 2 * d + 2 * d + 1))
    bank[..., : d * 2 * d] = 0.02 * np.random.default_rng(0).standard_normal((1, Hkv, d * 2 * d))
    s = W.Session(1, Hq, Hkv, d, d, 1024, rope_base=5e5, max_seqs=B, max_tokens=T + 3 * args.iters + 8,
                  max_prefill_tokens=T, attn_impl=args.impl, gate_bank=bank, topk_budget=args.topk,
                  topk_mode=W.TOPK_QUEST if args.quest else W.TOPK_EXACT)
    q = torch.randn(B, T, Hq, d, device=dev, generator=g).to(torch.bfloat16)
    k = torch.randn(B, T, Hkv, d, device=dev, generator=g).to(torch.bfloat16)
    v = torch.randn(B, T, Hkv, d, device=dev, generator=g).to(torch.bfloat16)
    forced = (torch.rand(B, Hkv, T, device=dev, generator=g) < args.admit).float()
    s.prefill_layer(0, q, k, v, forced_gates=forced)
    del q, k, v
    s.sync()
    qd = torch.randn(B, Hq, d, device=dev, generator=g).to(torch.bfloat16)
    kd = torch.randn(B, Hkv, d, device=dev, generator=g).to(torch.bfloat16)
    vd = torch.randn(B, Hkv, d, device=dev, generator=g).to(torch.bfloat16)
    fz = torch.zeros(B, Hkv, device=dev)
    out = torch.empty_like(qd)
    P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    lib, h = s.lib, s.h
    st = s.stats(0, B)
    res_bytes = st["resident_entries"] * 2 * d * 2
    if args.topk:  # K6 reads: every Global K once per group (scoring) + selected K/V per q head + Local K/V
        n_loc = min(T, 1024)
        n_glob = (st["resident_entries"] / (B * Hkv)) - n_loc
        sel = min(args.topk * 16, n_glob)
        score_bytes = n_glob / 16 * 2 * d * 2 if args.quest else n_glob * d * 2  # page min/max vs every K row
        res_bytes = B * Hkv * (score_bytes + (Hq // Hkv) * (sel + n_loc) * 2 * d * 2)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    for _ in range(5):
        check(lib.wgkv_decode_attn(h, 0, 0, B, P(qd), P(out)))
    # warm every kernel of the layer call (lazy module loading of the side-stream gate)
    check(lib.wgkv_decode_layer(h, 0, 0, B, P(qd), P(kd), P(vd), None, P(out), None, None))
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(args.iters):
        check(lib.wgkv_decode_attn(h, 0, 0, B, P(qd), P(out)))
    ev[1].record()
    for _ in range(args.iters // 2):
        check(lib.wgkv_decode_step_kv(h, 0, 0, B, P(kd), P(vd), P(fz), None, None))
    ev[2].record()
    for _ in range(args.iters // 2):
        check(lib.wgkv_decode_step_kv(h, 0, 0, B, P(kd), P(vd), None, None, None))
    ev[3].record()
    for _ in range(args.iters // 2):
        check(lib.wgkv_decode_layer(h, 0, 0, B, P(qd), P(kd), P(vd), None, P(out), None, None))
    ev[4].record()
    torch.cuda.synchronize()
    t_layer = ev[3].elapsed_time(ev[4]) / (args.iters // 2) * 1e3
    t_attn = ev[0].elapsed_time(ev[1]) / args.iters * 1e3
    t_app_forced = ev[1].elapsed_time(ev[2]) / (args.iters // 2) * 1e3
    t_app_gate = ev[2].elapsed_time(ev[3]) / (args.iters // 2) * 1e3
    s.sync()
    print(json.dumps({"T": T, "batch": B, "hq": Hq, "hkv": Hkv, "topk": args.topk,
                      "resident_entries": st["resident_entries"],
                      "k5_attn_us": t_attn, "k5_GBps": res_bytes / t_attn / 1e3,
                      "k4_append_forced_us": t_app_forced, "k4_append_fp64_gate_us": t_app_gate,
                      "decode_layer_us": t_layer, "decode_layer_GBps": res_bytes / t_layer / 1e3}))


if __name__ == "__main__":
    main()

#!/usr/bin/env python3
"""Prefill micro-benchmark: per-kernel time of K1 (gate), K2 (compaction) and
K3 (VS attention) for one layer of the 128K x 4 configuration (admission
calibrated to a = 0.25), with algorithmic throughput.  GPU only.
    python profiles/prefill_breakdown.py [--T 131072] [--batch 4] [--reps 3]
"""
import argparse
import ctypes as C
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2512_17452_b200 as W  # noqa: E402
from paper_2512_17452_b200._lib import check  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--T", type=int, default=131072)
    ap.add_argument("--batch", type=int, default=4)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--window", type=int, default=1024)
    ap.add_argument("--trace", default="", help="diagnostic K3 build (-DWGKV_TRACE): dump CTA (0,0,0) event clocks")
    args = ap.parse_args()
    B, T, Hq, Hkv, d, Wn = args.batch, args.T, 32, 8, 128, args.window
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(0)
    rng = np.random.default_rng(0)
    bank = np.zeros((1, Hkv, d * 2 * d + 2 * d + 1))
    bank[..., : d * 2 * d] = 0.02 * rng.standard_normal((1, Hkv, d * 2 * d))
    bank[..., d * 2 * d + d: d * 2 * d + 2 * d] = 0.02 * rng.standard_normal((1, Hkv, d))
    s = W.Session(1, Hq, Hkv, d, d, Wn, rope_base=5e5, max_seqs=B, max_tokens=T, gate_bank=bank)
    q = torch.randn(B, T, Hq, d, device=dev, generator=g).to(torch.bfloat16)
    k = torch.randn(B, T, Hkv, d, device=dev, generator=g).to(torch.bfloat16)
    v = torch.randn(B, T, Hkv, d, device=dev, generator=g).to(torch.bfloat16)
    _, gg, _, _ = s.gate_forward_batch(0, k)
    z = torch.logit(gg.clamp(1e-7, 1 - 1e-7).double())
    for h in range(Hkv):
        zz = z[:, h].flatten()[::4]
        bank[0, h, -1] = math.log(0.1 / 0.9) - torch.quantile(zz.float(), 0.75).item()
    s.gate_set(bank)
    kpost = torch.empty_like(k)
    gw = torch.empty(B, Hkv, T, device=dev)
    bits = torch.empty(B, Hkv, T, dtype=torch.uint8, device=dev)
    out = torch.empty_like(q)
    P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    lib, h = s.lib, s.h
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    tk1 = tk2 = tk3 = 0.0
    for r in range(args.reps + 1):
        ev[0].record()
        check(lib.wgkv_gate_score(h, 0, B, T, 0, P(k), None, P(kpost), P(gw), P(bits), None, 0, None))
        ev[1].record()
        check(lib.wgkv_admit_prefill(h, 0, 0, B, T, P(kpost), P(v), P(gw), P(bits)))
        ev[2].record()
        check(lib.wgkv_vs_prefill(h, 0, 0, B, T, P(q), P(kpost), P(v), P(bits), P(out)))
        ev[3].record()
        torch.cuda.synchronize()
        if r:
            tk1 += ev[0].elapsed_time(ev[1]) / args.reps
            tk2 += ev[1].elapsed_time(ev[2]) / args.reps
            tk3 += ev[2].elapsed_time(ev[3]) / args.reps
        st = s.stats(0, B)
        s.release(0, B)
    if args.trace:
        buf = np.zeros((4, 4096, 8), np.uint64)
        fn = getattr(lib, os.environ.get("WGKV_TRACE_FN", "wgkv_dbg_k3_trace1" if os.environ.get("WGKV_TRACE_V1")
                                         else "wgkv_dbg_k3_trace"))
        check(fn(buf.ctypes.data_as(C.c_void_p), C.c_size_t(buf.nbytes)))
        np.save(args.trace, buf)
    ii = torch.arange(T, device=dev)
    band = torch.clamp(ii + 1, max=Wn).sum()
    pairs = int((band + torch.cumsum(bits[..., : T - Wn].long(), -1).sum(-1)).sum().item()) * (Hq // Hkv)
    flops = 4.0 * d * pairs
    k1_bytes = B * T * Hkv * (2 * d * 2 + 5)
    k2_bytes = st["resident_entries"] * (4 * d * 2 + 9)
    print(json.dumps({"T": T, "batch": B, "admitted_frac": float(bits.float().mean()),
                      "k1_gate_ms": tk1, "k1_TFLOPs": B * T * Hkv * (4 * d * d + 12 * d) / tk1 / 1e9,
                      "k1_GBps": k1_bytes / tk1 / 1e6,
                      "k2_admit_ms": tk2, "k2_GBps": k2_bytes / tk2 / 1e6,
                      "k3_vs_ms": tk3, "k3_TFLOPs": flops / tk3 / 1e9, "pairs": pairs}))


if __name__ == "__main__":
    main()

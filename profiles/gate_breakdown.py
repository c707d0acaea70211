#!/usr/bin/env python3
"""K1 micro-benchmark: wgkv_gate_score (RoPE + gate MLP + threshold + fp64
recheck of the error band) on one layer of the 128K x 4 configuration with the
bench's gate bank (w_std 0.02, b2 calibrated per head to admission 0.25).
Reports time, algorithmic GB/s and how many tokens the fp64 recheck saw.
    python profiles/gate_breakdown.py [--T 131072] [--batch 4]
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
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--w-std", type=float, default=0.02)
    args = ap.parse_args()
    B, T, Hkv, d = args.batch, args.T, 8, 128
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(0)
    rng = np.random.default_rng(0)
    bank = np.zeros((1, Hkv, d * 2 * d + 2 * d + 1))
    bank[..., : d * 2 * d] = args.w_std * rng.standard_normal((1, Hkv, d * 2 * d))
    bank[..., d * 2 * d + d: d * 2 * d + 2 * d] = args.w_std * rng.standard_normal((1, Hkv, d))
    s = W.Session(1, 32, Hkv, d, d, 1024, rope_base=5e5, max_seqs=B, max_tokens=T, gate_bank=bank)
    k = torch.randn(B, T, Hkv, d, device=dev, generator=g).to(torch.bfloat16)
    _, gg, _, _ = s.gate_forward_batch(0, k)
    z = torch.logit(gg.clamp(1e-7, 1 - 1e-7).double())
    for h in range(Hkv):
        zz = z[:, h].flatten()[::4]
        bank[0, h, -1] = math.log(0.1 / 0.9) - torch.quantile(zz.float(), 0.75).item()
    s.gate_set(bank)
    kpost = torch.empty_like(k)
    gw = torch.empty(B, Hkv, T, device=dev)
    bits = torch.empty(B, Hkv, T, dtype=torch.uint8, device=dev)
    P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    lib, h = s.lib, s.h
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    check(lib.wgkv_gate_score(h, 0, B, T, 0, P(k), None, P(kpost), P(gw), P(bits), None, 0, None))
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(args.reps):
        check(lib.wgkv_gate_score(h, 0, B, T, 0, P(k), None, P(kpost), P(gw), P(bits), None, 0, None))
    ev[1].record()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / args.reps
    cnt = (C.c_int * 2)()
    check(lib.wgkv_dbg_gate_counts(h, cnt))
    ntok = B * T * Hkv
    print(json.dumps({"T": T, "batch": B, "k1_ms": ms, "tokens": ntok, "recheck_tokens": cnt[0],
                      "recheck_frac": cnt[0] / ntok, "admitted": float(bits.float().mean()),
                      "k1_GBps": ntok * (2 * d * 2 + 5) / ms / 1e6,
                      "k1_TFLOPs": ntok * (4 * d * d + 12 * d) / ms / 1e9}))


if __name__ == "__main__":
    main()

#!/usr/bin/env python3
"""f1 cost: one layer's key projection + gate at the 128K x 4 shape (dm = 4096,
8 kv heads), fused (wgkv_gate_score_proj) vs the unfused pair (cuBLAS
projection x . Wk^T into k_pre, then K1 = wgkv_gate_score).  GPU only.
    python profiles/proj_breakdown.py [--T 131072] [--batch 4] [--dm 4096]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2512_17452_b200 as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--T", type=int, default=131072)
    ap.add_argument("--batch", type=int, default=4)
    ap.add_argument("--dm", type=int, default=4096)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    B, T, Hkv, d, dm = args.batch, args.T, 8, 128, args.dm
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(0)
    bank = np.zeros((1, Hkv, d * 2 * d + 2 * d + 1))
    bank[..., : d * 2 * d] = 0.02 * np.random.default_rng(0).standard_normal((1, Hkv, d * 2 * d))
    s = W.Session(1, 32, Hkv, d, d, 1024, rope_base=5e5, max_seqs=B, max_tokens=T, gate_bank=bank)
    x = torch.randn(B, T, dm, device=dev, generator=g).to(torch.bfloat16)
    wk = (torch.randn(Hkv, d, dm, device=dev, generator=g) / dm ** 0.5).to(torch.bfloat16)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    tf = tu_p = tu_g = 0.0
    for r in range(args.reps + 1):
        ev[0].record()
        s.gate_forward_batch_proj(0, x, wk)
        ev[1].record()
        k_pre = (x.reshape(B * T, dm) @ wk.reshape(Hkv * d, dm).T).reshape(B, T, Hkv, d)
        ev[2].record()
        s.gate_forward_batch(0, k_pre)
        ev[3].record()
        torch.cuda.synchronize()
        if r:
            tf += ev[0].elapsed_time(ev[1]) / args.reps
            tu_p += ev[1].elapsed_time(ev[2]) / args.reps
            tu_g += ev[2].elapsed_time(ev[3]) / args.reps
    flops = 2.0 * B * T * dm * Hkv * d
    print(json.dumps({"T": T, "batch": B, "dm": dm, "fused_ms": tf, "unfused_proj_ms": tu_p, "unfused_gate_ms": tu_g,
                      "unfused_ms": tu_p + tu_g, "proj_flops": flops, "fused_proj_TFLOPs_upper": flops / tf / 1e9,
                      "cublas_proj_TFLOPs": flops / tu_p / 1e9}))


if __name__ == "__main__":
    main()

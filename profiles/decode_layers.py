#!/usr/bin/env python3
"""Decode latency with every layer's cache cold (32 layers, one token step =
all layers in order, like bench.py), eager and as a CUDA graph, with the fp64
gate (side stream) or forced gates.  Diagnoses batch-1 / small-batch decode.
    python profiles/decode_layers.py [--T 32768] [--batch 1]
"""
import argparse
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2512_17452_b200 as W  # noqa: E402
from paper_2512_17452_b200._lib import check  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--T", type=int, default=32768)
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--hq", type=int, default=32)
    ap.add_argument("--hkv", type=int, default=8)
    args = ap.parse_args()
    B, T, L, Hq, Hkv, d = args.batch, args.T, args.layers, args.hq, args.hkv, 128
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(0)
    bank = np.zeros((L, Hkv, d * 2 * d + 2 * d + 1))
    bank[..., : d * 2 * d] = 0.02 * np.random.default_rng(0).standard_normal((L, Hkv, d * 2 * d))
    s = W.Session(L, Hq, Hkv, d, d, 1024, rope_base=5e5, max_seqs=B, max_tokens=T + 8 * args.steps + 8,
                  max_prefill_tokens=T, gate_bank=bank)
    for l in range(L):
        q = torch.randn(B, T, Hq, d, device=dev, generator=g).to(torch.bfloat16)
        k = torch.randn(B, T, Hkv, d, device=dev, generator=g).to(torch.bfloat16)
        v = torch.randn(B, T, Hkv, d, device=dev, generator=g).to(torch.bfloat16)
        forced = (torch.rand(B, Hkv, T, device=dev, generator=g) < 0.25).float()
        s.prefill_layer(l, q, k, v, forced_gates=forced)
    del q, k, v
    s.sync()
    qd = torch.randn(B, Hq, d, device=dev, generator=g).to(torch.bfloat16)
    kd = torch.randn(B, Hkv, d, device=dev, generator=g).to(torch.bfloat16)
    vd = torch.randn(B, Hkv, d, device=dev, generator=g).to(torch.bfloat16)
    fz = torch.zeros(B, Hkv, device=dev)
    out = torch.empty_like(qd)
    P = lambda t: None if t is None else C.c_void_p(t.data_ptr())  # noqa: E731
    lib, h = s.lib, s.h
    res = {"T": T, "batch": B, "layers": L, "hq": Hq, "hkv": Hkv}
    for name, fg in (("fp64_gate", None), ("forced_gate", fz)):
        def step():
            for l in range(L):
                check(lib.wgkv_decode_layer(h, l, 0, B, P(qd), P(kd), P(vd), P(fg), P(out), None, None))
        step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            step()
        e1.record()
        torch.cuda.synchronize()
        res[name + "_eager_us_per_layer"] = e0.elapsed_time(e1) * 1e3 / args.steps / L
        st = torch.cuda.current_stream(dev)
        gs = torch.cuda.Stream(dev)
        gs.wait_stream(st)
        s.set_stream(gs)
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=gs):
            step()
        s.set_stream(st)
        st.wait_stream(gs)
        gr.replay()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(args.steps):
            gr.replay()
        e1.record()
        torch.cuda.synchronize()
        res[name + "_graph_us_per_layer"] = e0.elapsed_time(e1) * 1e3 / args.steps / L
    # components, cold cache, graph: K4 append only (forced gate) and K5 + combine only
    for name, fn in (("append_only", lambda l: lib.wgkv_decode_step_kv(h, l, 0, B, P(kd), P(vd), P(fz), None, None)),
                     ("attn_only", lambda l: lib.wgkv_decode_attn(h, l, 0, B, P(qd), P(out)))):
        def step2():
            for l in range(L):
                check(fn(l))
        st = torch.cuda.current_stream(dev)
        gs = torch.cuda.Stream(dev)
        gs.wait_stream(st)
        s.set_stream(gs)
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=gs):
            step2()
        s.set_stream(st)
        st.wait_stream(gs)
        gr.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            gr.replay()
        e1.record()
        torch.cuda.synchronize()
        res[name + "_graph_us_per_layer"] = e0.elapsed_time(e1) * 1e3 / args.steps / L
    print(json.dumps(res))


if __name__ == "__main__":
    main()

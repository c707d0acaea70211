#!/usr/bin/env python3
"""Per-CTA timeline of one graph-captured decode token step (all layers, every
cache cold), from the %globaltimer records of an experiment build
(tools/timeline_build.sh -> build/var/libwgkv_tl.so):
    WGKV_LIB=build/var/libwgkv_tl.so python profiles/decode_timeline.py --T 131072 --batch 4 --hq 4 --hkv 1
Prints, per layer and averaged, where the layer's time goes: K5's launch, plan,
PDL wait, its item phase and tail, and the finish kernel's roles."""
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

REC = np.dtype([("t", "<u8", 8), ("tag", "<i4"), ("layer", "<i4"), ("cta", "<i4"), ("sm", "<i4"),
                ("n", "<i4"), ("pad", "<i4")])
TAGS = {0: "k5", 1: "combine", 2: "k5_gate", 3: "fin_gate", 4: "route", 5: "fused_route"}


def read(lib, fn):
    buf = np.zeros(1 << 17, dtype=REC)
    f = getattr(lib, fn)
    f.restype = C.c_int
    n = f(C.c_void_p(buf.ctypes.data), C.c_int(len(buf)))
    return buf[:n]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--T", type=int, default=32768)
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--hq", type=int, default=32)
    ap.add_argument("--hkv", type=int, default=8)
    ap.add_argument("--forced", action="store_true", help="forced gates (no fp64 gate CTAs)")
    ap.add_argument("--dump", default="", help="write the raw records (npz)")
    args = ap.parse_args()
    B, T, L, Hq, Hkv, d = args.batch, args.T, args.layers, args.hq, args.hkv, 128
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(0)
    bank = np.zeros((L, Hkv, d * 2 * d + 2 * d + 1))
    bank[..., : d * 2 * d] = 0.02 * np.random.default_rng(0).standard_normal((L, Hkv, d * 2 * d))
    s = W.Session(L, Hq, Hkv, d, d, 1024, rope_base=5e5, max_seqs=B, max_tokens=T + 64,
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
    fz = torch.zeros(B, Hkv, device=dev) if args.forced else None
    out = torch.empty_like(qd)
    P = lambda t: None if t is None else C.c_void_p(t.data_ptr())  # noqa: E731
    lib, h = s.lib, s.h
    res_bytes = s.stats(0, B)["resident_entries"] * 2 * d * 2  # every layer's resident K/V

    def step():
        for l in range(L):
            check(lib.wgkv_decode_layer(h, l, 0, B, P(qd), P(kd), P(vd), P(fz), P(out), None, None))
    step()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream(dev)
    gst = torch.cuda.Stream(dev)
    gst.wait_stream(st)
    s.set_stream(gst)
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=gst):
        step()
    s.set_stream(st)
    st.wait_stream(gst)
    for _ in range(3):
        gr.replay()
    torch.cuda.synchronize()
    read(lib, "wgkv_tl_k5"), read(lib, "wgkv_tl_fin")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    flush.fill_(1)  # caches cold like a real token step
    torch.cuda.synchronize()
    gr.replay()
    torch.cuda.synchronize()
    r = np.concatenate([read(lib, "wgkv_tl_k5"), read(lib, "wgkv_tl_fin")])
    if args.dump:
        np.savez(args.dump, r=r)
    t00 = r["t"][:, 0].min()
    tt = (r["t"].astype(np.int64) - np.int64(t00)) / 1e3  # us
    tt[r["t"] == 0] = np.nan
    tt = tt[:, [0, 1, 2, 7]]  # entry, plan, wait, exit
    rows = []
    for l in range(L):
        row = {"layer": l}
        for tag, name in TAGS.items():
            m = (r["layer"] == l) & (r["tag"] == tag)
            if not m.any():
                continue
            x = tt[m]
            row[name] = {"n": int(m.sum()), "start_min": float(np.nanmin(x[:, 0])),
                         "start_max": float(np.nanmax(x[:, 0])), "end_min": float(np.nanmin(x[:, 3])),
                         "end_max": float(np.nanmax(x[:, 3]))}
            if tag == 0:
                row[name]["plan_med"] = float(np.nanmedian(x[:, 1] - x[:, 0]))
                row[name]["wait_max"] = float(np.nanmax(x[:, 2]))
                row[name]["items_max"] = int(r["n"][m].max())
                row[name]["end_med"] = float(np.nanmedian(x[:, 3]))
            if tag == 1:
                row[name]["wait_min"] = float(np.nanmin(x[:, 2]))
                row[name]["chunks_max"] = int(r["n"][m].max())
        rows.append(row)
    # per-layer phases (us): period = K5 start(l+1) - K5 start(l)
    ph = {"period": [], "k5_launch_to_wait": [], "k5_wait_to_end": [], "k5_end_spread": [],
          "k5end_to_combine_end": [], "route_end_after_k5": [], "next_k5_start_after_combine": [],
          "next_k5_wait_after_k5_end": []}
    for a, b in zip(rows[:-1], rows[1:]):
        k5, nk5 = a["k5"], b["k5"]
        ph["period"].append(nk5["start_min"] - k5["start_min"])
        ph["k5_launch_to_wait"].append(k5["wait_max"] - k5["start_min"])
        ph["k5_wait_to_end"].append(k5["end_max"] - k5["wait_max"])
        ph["k5_end_spread"].append(k5["end_max"] - k5["end_med"])
        ph["next_k5_wait_after_k5_end"].append(nk5["wait_max"] - k5["end_max"])
        if "combine" in a:  # finish-kernel path
            cb = a["combine"]
            ph["k5end_to_combine_end"].append(cb["end_max"] - k5["end_max"])
            ph["next_k5_start_after_combine"].append(nk5["start_min"] - cb["end_max"])
        if "route" in a:
            ph["route_end_after_k5"].append(a["route"]["end_max"] - k5["end_max"])
    summ = {k: round(float(np.median(v)), 2) for k, v in ph.items() if v}
    total_us = float(np.nanmax(tt[:, 3]))
    print(json.dumps({"T": T, "batch": B, "hq": Hq, "hkv": Hkv, "forced": args.forced, "step_us": total_us,
                      "us_per_layer": total_us / L, "GBps": res_bytes / total_us / 1e3,
                      "median_phases_us": summ, "layer1": rows[1], "layer16": rows[16]}, indent=1))


if __name__ == "__main__":
    main()

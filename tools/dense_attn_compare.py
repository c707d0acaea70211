"""Dense causal attention on the same B200, for two comparisons VERDICT r1 asked for:

  1. K3's ceiling: a production dense flash-attention forward (cuDNN SDPA through
     torch, and flashinfer's sm100 CUTLASS FMHA when its JIT builds) on
     Llama-3.1-8B heads (32 q / 8 kv, d = 128, bf16), timed with CUDA events,
     reported in TFLOP/s of the causal pairs it must compute (4 * d * T(T+1)/2
     per q head) -- the same "algorithmic FLOPs" convention bench.py uses
     for K3 (4 * d * vs_mask_pair_count).
  2. The paper's relative claim (prefill 3.03-3.45x vs full
     attention): dense causal attention time per layer at 128K x batch 4 against
     WG-KV's whole prefill layer (K1 + K2 + K3) from bench.py.

Library kernels are used here only as a comparison point; they are
not on the product path.  Prints one JSON line.
"""
import json
import sys

import torch
import torch.nn.functional as F


def events_time(fn, iters=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters / 1e3


def causal_flops(B, Hq, T, d):
    return 4.0 * d * B * Hq * T * (T + 1) / 2


def cudnn_sdpa(B, T, Hq=32, Hkv=8, d=128):
    from torch.nn.attention import SDPBackend, sdpa_kernel

    q = torch.randn(B, Hq, T, d, device="cuda", dtype=torch.bfloat16)
    # GQA: cuDNN SDPA takes expanded K/V (enable_gqa is honoured by the math/flash
    # paths only in some builds) -- expand as a view-free copy outside the timing
    k = torch.randn(B, Hkv, T, d, device="cuda", dtype=torch.bfloat16).repeat_interleave(Hq // Hkv, 1)
    v = torch.randn(B, Hkv, T, d, device="cuda", dtype=torch.bfloat16).repeat_interleave(Hq // Hkv, 1)
    with sdpa_kernel([SDPBackend.CUDNN_ATTENTION]):
        t = events_time(lambda: F.scaled_dot_product_attention(q, k, v, is_causal=True), iters=3 if T > 65536 else 5)
    return t


def flashinfer_cutlass(B, T, Hq=32, Hkv=8, d=128):
    import flashinfer

    q = torch.randn(B * T, Hq, d, device="cuda", dtype=torch.bfloat16)
    k = torch.randn(B * T, Hkv, d, device="cuda", dtype=torch.bfloat16)
    v = torch.randn(B * T, Hkv, d, device="cuda", dtype=torch.bfloat16)
    indptr = torch.arange(0, (B + 1) * T, T, device="cuda", dtype=torch.int32)
    ws = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    w = flashinfer.BatchPrefillWithRaggedKVCacheWrapper(ws, "NHD", backend="cutlass")
    w.plan(indptr, indptr, Hq, Hkv, d, causal=True, q_data_type=torch.bfloat16)
    return events_time(lambda: w.run(q, k, v), iters=3 if T > 65536 else 5)


def main():
    out = {"tool": "dense_attn_compare", "shape": "32q/8kv, d=128, bf16, causal"}
    rows = []
    for B, T in ((1, 32768), (4, 32768), (1, 131072), (4, 131072)):
        fl = causal_flops(B, 32, T, 128)
        row = {"batch": B, "T": T, "causal_flops": fl}
        for name, fn in (("cudnn_sdpa", cudnn_sdpa), ("flashinfer_cutlass", flashinfer_cutlass)):
            try:
                t = fn(B, T)
                row[name] = {"s": t, "tflops": fl / t / 1e12}
            except Exception as exc:  # a backend may be missing on this image
                row[name] = {"error": f"{type(exc).__name__}: {str(exc)[:200]}"}
            torch.cuda.empty_cache()
        rows.append(row)
        print(json.dumps(row), file=sys.stderr, flush=True)
    out["rows"] = rows
    print(json.dumps(out))


if __name__ == "__main__":
    main()

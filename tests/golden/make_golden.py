"""Generate golden vectors FROM THE REFERENCE ITSELF (oracle/_ref).

Run in the build container (where /root/reference exists):
    make -C oracle all && python tests/golden/make_golden.py
The outputs are committed; tests/test_golden.py checks the C oracle against
them on every CPU run and the GPU tests use the same inputs.

Inputs are bf16-rounded (the GPU path's storage type) and upcast to fp64,
the convention SURVEY.md §8(c) fixes for parity.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle as O  # noqa: E402


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even to bfloat16, returned as float64."""
    f = np.ascontiguousarray(x, np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def session_case(ref, name, L, hq, hkv, d, hidden, n, steps, W, tau, base, ps, topk, w_std, b2, seed):
    bank = ref.gate_random_init(L, hkv, d, hidden, seed, w_std, b2)
    q = bf16_round(ref.gaussian(seed + 1, L * (n + steps) * hq * d).reshape(L, n + steps, hq, d))
    k = bf16_round(ref.gaussian(seed + 2, L * (n + steps) * hkv * d).reshape(L, n + steps, hkv, d))
    v = bf16_round(ref.gaussian(seed + 3, L * (n + steps) * hkv * d).reshape(L, n + steps, hkv, d))
    s = O.Session(ref, L, hq, hkv, d, hidden, W, tau=tau, rope_base=base, page_size=ps, topk_budget=topk,
                  gate_bank=bank, max_tokens=n + steps)
    pre_out, pre_g, pre_bits, pre_ev = [], [], [], []
    for l in range(L):
        o, g, b, ev = s.prefill_layer(l, q[l, :n], k[l, :n], v[l, :n])
        pre_out.append(o)
        pre_g.append(g)
        pre_bits.append(b)
        pre_ev.append(ev)
    dec_out, dec_g, dec_evt = [], [], []
    for t in range(n, n + steps):
        for l in range(L):
            o, g, e, _ = s.decode_layer(l, q[l, t], k[l, t], v[l, t])
            dec_out.append(o)
            dec_g.append(g)
            dec_evt.append(e)
    gpos = [[s.gather(l, h)["global_pos"] for h in range(hkv)] for l in range(L)]
    glen = np.array([[len(x) for x in row] for row in gpos])
    np.savez_compressed(
        os.path.join(HERE, name + ".npz"),
        cfg=np.array([L, hq, hkv, d, hidden, n, steps, W, ps, topk]), tau=tau, base=base, bank=bank, q=q.astype(np.float32), k=k.astype(np.float32),
        v=v.astype(np.float32),
        prefill_out=np.array(pre_out), prefill_g=np.array(pre_g), prefill_bits=np.array(pre_bits),
        prefill_evals=np.array(pre_ev, np.uint64),
        decode_out=np.array(dec_out).reshape(steps, L, hq, d), decode_g=np.array(dec_g).reshape(steps, L, hkv),
        decode_events=np.array(dec_evt).reshape(steps, L, hkv), global_len=glen,
        global_pos=np.concatenate([x for row in gpos for x in row]) if glen.sum() else np.zeros(0, np.int64))
    print(name, "global_len", glen.tolist())


def gate_bank_file(ref, name, L, H, d, hidden, seed, w_std, b2):
    """A ".wgkv" v1 gate bank written by the reference's own GateBank::save
    (gating.cpp:107-122); wgkv_gate_load must read it (tests/test_gpu_configs.py)."""
    bank = ref.gate_random_init(L, H, d, hidden, seed, w_std, b2)
    path = os.path.join(HERE, name + ".wgkv")
    st = ref.lib.wr_gate_save(path.encode(), L, H, d, hidden, bank.ctypes.data_as(O._dp))
    assert st == 0, st
    np.save(os.path.join(HERE, name + "_bank.npy"), bank)
    print(name, os.path.getsize(path), "bytes")


def main():
    ref = O.Ref()
    if len(sys.argv) > 1 and sys.argv[1] == "gate_bank":
        gate_bank_file(ref, "gate_bank_d32", L=2, H=2, d=32, hidden=32, seed=4100, w_std=0.5, b2=-2.5)
        return
    # Llama-shaped head geometry (d=128, hidden=d as config.cpp:175), GQA 4,
    # window shorter than the prompt so Global, Local and promotion all occur.
    session_case(ref, "session_gqa4_d128", L=1, hq=8, hkv=2, d=128, hidden=128, n=160, steps=24, W=48, tau=0.1,
                 base=1e4, ps=16, topk=0, w_std=0.1, b2=-2.2, seed=1000)
    session_case(ref, "session_topk_d128", L=1, hq=4, hkv=1, d=128, hidden=128, n=200, steps=12, W=32, tau=0.1,
                 base=5e5, ps=16, topk=3, w_std=0.1, b2=-2.5, seed=2000)
    session_case(ref, "session_small_l2", L=2, hq=4, hkv=4, d=16, hidden=16, n=48, steps=24, W=8, tau=0.1,
                 base=1e4, ps=16, topk=0, w_std=0.5, b2=-2.5, seed=3000)
    gate_bank_file(ref, "gate_bank_d32", L=2, H=2, d=32, hidden=32, seed=4100, w_std=0.5, b2=-2.5)


if __name__ == "__main__":
    main()

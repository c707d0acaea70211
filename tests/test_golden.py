"""The C oracle reproduces the reference-generated golden vectors bitwise.

tests/golden/*.npz were produced by the reference itself (oracle/_ref,
compiled from /root/reference sources) via tests/golden/make_golden.py.
This pins the oracle even where /root/reference is absent (the GPU box).
"""
import glob
import os

import numpy as np
import pytest

import oracle as O

GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz")))


def load(path):
    z = np.load(path)
    L, hq, hkv, d, hidden, n, steps, W, ps, topk = (int(x) for x in z["cfg"])
    return z, dict(L=L, hq=hq, hkv=hkv, d=d, hidden=hidden, n=n, steps=steps, W=W, ps=ps, topk=topk)


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p) for p in GOLDEN])
def test_oracle_reproduces_golden(orc, path):
    z, c = load(path)
    s = O.Session(orc, c["L"], c["hq"], c["hkv"], c["d"], c["hidden"], c["W"], tau=float(z["tau"]),
                  rope_base=float(z["base"]), page_size=c["ps"], topk_budget=c["topk"], gate_bank=z["bank"],
                  max_tokens=c["n"] + c["steps"])
    q, k, v = (z[x].astype(np.float64) for x in ("q", "k", "v"))
    n = c["n"]
    for l in range(c["L"]):
        o, g, b, ev = s.prefill_layer(l, q[l, :n], k[l, :n], v[l, :n])
        assert np.array_equal(o, z["prefill_out"][l])
        assert np.array_equal(g, z["prefill_g"][l])
        assert np.array_equal(b, z["prefill_bits"][l])
        assert ev == int(z["prefill_evals"][l])
    for si, t in enumerate(range(n, n + c["steps"])):
        for l in range(c["L"]):
            o, g, e, _ = s.decode_layer(l, q[l, t], k[l, t], v[l, t])
            assert np.array_equal(o, z["decode_out"][si, l])
            assert np.array_equal(g, z["decode_g"][si, l])
            assert np.array_equal(e, z["decode_events"][si, l])
    pos = np.concatenate([s.gather(l, h)["global_pos"] for l in range(c["L"]) for h in range(c["hkv"])])
    assert np.array_equal(pos, z["global_pos"])


def test_oracle_reads_reference_gate_file(orc):
    """tests/golden/gate_bank_d32.wgkv was written by the reference's own
    GateBank::save (gating.cpp:107-122, make_golden.py); the oracle's loader
    (and, on the GPU, wgkv_gate_load) must read back exactly the bank it saved."""
    here = os.path.join(os.path.dirname(__file__), "golden")
    bank = np.load(os.path.join(here, "gate_bank_d32_bank.npy"))
    assert np.array_equal(orc.gate_load(os.path.join(here, "gate_bank_d32.wgkv")), bank)

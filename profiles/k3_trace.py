#!/usr/bin/env python3
"""Summarise a K3 event trace (diagnostic build -DWGKV_TRACE, written by
profiles/prefill_breakdown.py --trace X.npy): per-block intervals of the
softmax tiles, the MMA issuer and the TMA producer of CTA (0,0,0), in SM clocks."""
import statistics as st
import sys

import numpy as np

b = np.load(sys.argv[1]).astype(np.int64)
n = int((b[2, :, 0] > 0).sum()) + 1
rng = range(20, n - 20)


def avg(f):
    return st.mean(f(j) for j in rng)


print(f"blocks {n}, period (MMA pf0->pf0) {avg(lambda j: b[2, j + 1, 0] - b[2, j, 0]):.0f} clk per 2 x 128-key tile")
if b[0, 30, 1] > 0:
    for t in (0, 1):
        print(f"softmax t{t}: tmem-ld {avg(lambda j: b[t, j, 1] - b[t, j, 0]):.0f}  max-xchg {avg(lambda j: b[t, j, 2] - b[t, j, 1]):.0f}"
              f"  exp {avg(lambda j: b[t, j, 3] - b[t, j, 2]):.0f}  st+arrive {avg(lambda j: b[t, j, 4] - b[t, j, 3]):.0f}"
              f"  wait-next-S {avg(lambda j: b[t, j + 1, 0] - b[t, j, 4]):.0f}")
    print(f"p_full arrive -> MMA sees: t0 {avg(lambda j: b[2, j, 0] - b[0, j, 4]):.0f}  t1 {avg(lambda j: b[2, j, 3] - b[1, j, 4]):.0f}")
print(f"MMA pf0 -> PV0+S0 issued {avg(lambda j: b[2, j, 2] - b[2, j, 0]):.0f};  pf1 -> PV1+S1 issued {avg(lambda j: b[2, j, 5] - b[2, j, 3]):.0f}")
print(f"MMA S0 issued -> pf1 seen {avg(lambda j: b[2, j, 3] - b[2, j, 2]):.0f};  S1 issued -> next pf0 {avg(lambda j: b[2, j + 1, 0] - b[2, j, 5]):.0f}")
if b[0, 30, 0] > 0:
    print(f"S issued -> softmax sees s_full: t0 {avg(lambda j: b[0, j + 1, 0] - b[2, j, 2]):.0f}  t1 {avg(lambda j: b[1, j + 1, 0] - b[2, j, 5]):.0f}")
print(f"producer: K slot free -> V slot free {avg(lambda j: b[3, j, 1] - b[3, j, 0]):.0f}")

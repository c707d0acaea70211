"""Tie-aware acceptance for top-k page selection (test helper, not a test file).

select_topk_pages (engine.cpp:36-84) makes a discrete choice: the `budget`
pages with the highest score (ties to the older page).  The GPU scores pages
from bf16-stored keys with fp32 accumulation, the oracle from fp64 keys, so a
page whose oracle score lies within the two computations' error bound of the
selection boundary may legitimately land on either side.  Instead of a loose
relative-gap rule this helper derives, per page, an interval
[score - err, score + err] from the arithmetic (bf16 key rounding 2^-9
relative per element, q hi/lo split 2^-17, fp32 accumulation), classifies each
page as surely-selected / surely-excluded / ambiguous, and accepts the GPU
output only if attention over SOME selection consistent with those intervals
reproduces it within the stated tolerance.  Every such acceptance is counted
and reported as a tie.
"""
import itertools
import math

import numpy as np

# per-element relative error of a bf16-rounded key (round to nearest: 2^-9)
# plus the bf16 hi/lo split of q (2^-17) plus fp32 accumulation over d = 128
# products (d * 2^-24 = 2^-17), doubled as margin
BF16_KEY_REL = 2.0 * (2.0 ** -9 + 2.0 ** -17 + 2.0 ** -17)
# keys already bf16 on both sides (exported from the device): fp32 only
FP32_ACC_REL = 2.0 * (2.0 ** -17 + 2.0 ** -17)


def page_rows(n_rows, pages, ps=16):
    if not len(pages):
        return np.zeros(0, int)
    return np.concatenate([np.arange(ps * i, min(ps * i + ps, n_rows)) for i in pages])


def maxdot_scores(gk, qr, rel, ps=16):
    """select_topk_pages' page score (max over the page's slots of the unscaled
    q.k, engine.cpp:45-52) and its error bound rel * max_slot sum|q_i k_i|."""
    n = -(-gk.shape[0] // ps)
    dots = gk @ qr
    mag = np.abs(gk) @ np.abs(qr)
    sc = np.array([dots[ps * i:ps * i + ps].max() for i in range(n)])
    err = np.array([rel * mag[ps * i:ps * i + ps].max() for i in range(n)])
    return sc, err


def _attend(qr, keys, vals):
    lg = keys @ qr / math.sqrt(qr.shape[0])
    w = np.exp(lg - lg.max())
    return (w[:, None] * vals).sum(0) / w.sum()


def _rel_err(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


def check_selection(o, qr, gk, gv, lk, lv, scores, err, budget, tol, ps=16, max_alternatives=256):
    """Return 0 if the GPU output `o` equals attention over the exact top-k
    selection, 1 if it equals attention over an alternative selection that the
    error bounds allow (a reported tie); raise AssertionError otherwise."""
    n = len(scores)
    kk = min(budget, n)
    order = sorted(range(n), key=lambda i: (-scores[i], i))
    exact = sorted(order[:kk])
    ref = _attend(qr, np.concatenate([gk[page_rows(gk.shape[0], exact, ps)], lk]),
                  np.concatenate([gv[page_rows(gv.shape[0], exact, ps)], lv]))
    if _rel_err(o, ref) < tol:
        return 0
    assert kk < n, "selection is every page: no tie is possible"
    lo, hi = scores - err, scores + err
    sure, amb = [], []
    for j in range(n):
        beat_surely = int(np.sum(lo > hi[j]))  # pages certainly above j
        beat_maybe = int(np.sum(hi >= lo[j])) - 1  # pages possibly above j (not j)
        if beat_surely >= kk:
            continue  # surely excluded
        (sure if beat_maybe < kk else amb).append(j)
    need = kk - len(sure)
    assert 0 < need <= len(amb), (len(sure), len(amb), kk)
    combos = math.comb(len(amb), need)
    assert combos <= max_alternatives, f"{combos} alternative selections: not a near-tie"
    for pick in itertools.combinations(amb, need):
        sel = sorted(sure + list(pick))
        alt = _attend(qr, np.concatenate([gk[page_rows(gk.shape[0], sel, ps)], lk]),
                      np.concatenate([gv[page_rows(gv.shape[0], sel, ps)], lv]))
        if _rel_err(o, alt) < tol:
            return 1
    raise AssertionError(f"no selection within the error bounds reproduces the GPU output "
                         f"(sure {len(sure)}, ambiguous {len(amb)}, budget {kk})")

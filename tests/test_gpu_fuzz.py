"""Randomised parity sweep: small sessions with random geometry (prompt
length incl. 1, window incl. 1, GQA group 1-8, page size 8/16, 1-3 sequence
slots, bf16 tcgen05/mma.sync and fp32 SIMT paths, admission from ~0 to ~1)
checked end to end against the oracle by `_session_case` -- admission bits,
prefill outputs, per-step promotion events and decode outputs, Global/Local
positions.  Seeds are fixed, so a failure reproduces."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from test_gpu_parity import W, _session_case  # noqa: E402,F401  (W: the module fixture)

GEOMS = [(8, 2), (4, 1), (4, 4), (8, 1), (16, 2)]


@pytest.mark.parametrize("case", range(64))
def test_random_session(W, orc, case):  # noqa: F811
    rng = np.random.default_rng(1000 + case)
    hq, hkv = GEOMS[int(rng.integers(len(GEOMS)))]
    T = int(rng.choice([1, 2, 3, int(rng.integers(4, 640)), int(rng.integers(640, 2500))]))
    Wn = int(rng.choice([1, 2, int(rng.integers(3, 260))]))
    steps = int(rng.integers(1, 48))
    nseq = int(rng.integers(1, 4))
    dtype = "bf16" if rng.random() < 0.6 else "f32"
    ps = 16 if rng.random() < 0.75 else 8
    b2 = float(rng.uniform(-4.0, 1.5))
    _session_case(W, orc, T=T, steps=steps, hq=hq, hkv=hkv, Wn=Wn, nseq=nseq, dtype=dtype, seed=7000 + 13 * case,
                  b2=b2, ps=ps, base=5e5 if rng.random() < 0.5 else 1e4)

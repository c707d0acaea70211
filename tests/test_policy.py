"""Attention policies (PolicyConfig / ForcedAdmission, engine.hpp:17-40) and
Session::effective_gate (engine.cpp:126-151): the Python mirror
(paper_2512_17452_b200/policy.py) and the C++ face (include/wgkv_b200.hpp)
must reproduce the gates a real reference Session records in its GateTrace
(prefill + decode positions).  CPU only."""
import os
import shutil
import subprocess

import numpy as np
import pytest

from paper_2512_17452_b200 import policy as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
L, H, T, ND = 2, 3, 40, 6
BITMAP = [1, 0, 1, 0, 0, 1]

CASES = [  # (name, Policy) -- the MLP-decided policies are excluded (nothing to override)
    ("full", P.Policy(kind="full", window=8)),
    ("local_sink", P.Policy(kind="local_sink", window=8, sink=5)),
    ("static_heads", P.Policy(kind="static_heads", window=8, retrieval_bitmap=BITMAP)),
    ("stride", P.Policy(kind="wgkv", window=8, forced=P.ForcedAdmission("stride", keep_every=3, phase=1))),
    ("recent", P.Policy(kind="wgkv", window=8, forced=P.ForcedAdmission("recent_fraction", fraction=0.3))),
    ("recent_half", P.Policy(kind="wgkv_plus_topk", window=12, forced=P.ForcedAdmission("recent_fraction", fraction=0.5))),
]


def _ref_trace(ref, p: P.Policy):
    return ref.policy_trace(P.KINDS.index(p.kind), p.window, p.sink, p.retrieval_bitmap or None,
                            P.MODES.index(p.forced.mode), p.forced.keep_every, p.forced.phase, p.forced.fraction,
                            L, H, T, ND)


@pytest.mark.parametrize("name,pol", CASES, ids=[c[0] for c in CASES])
def test_python_policy_matches_reference_trace(ref, name, pol):
    tr = _ref_trace(ref, pol)
    for layer in range(L):
        g = P.policy_gates(pol, layer, 0, H, H, 1, 0, T + ND, T)[0]
        np.testing.assert_array_equal(g, tr[layer])


def test_mlp_policies_have_no_override():
    assert P.policy_gates(P.Policy(kind="wgkv"), 0, 0, 2, 2, 1, 0, 4, 4) is None
    assert P.policy_gates(P.Policy(kind="wgkv_plus_topk"), 0, 0, 2, 2, 1, 0, 4, 4) is None
    with pytest.raises(ValueError):
        P.Policy(kind="nope")


CPP = r"""
#include <cstdio>
#include "wgkv_b200.hpp"
using namespace wgkv::b200;
int main(int argc, char** argv) {
    Policy p;
    const int which = std::atoi(argv[1]);
    p.window = 8;
    if (which == 0) p.kind = PolicyKind::full;
    if (which == 1) { p.kind = PolicyKind::local_sink; p.sink = 5; }
    if (which == 2) { p.kind = PolicyKind::static_heads; p.retrieval_bitmap = {1, 0, 1, 0, 0, 1}; }
    if (which == 3) { p.forced.mode = ForcedAdmission::Mode::stride; p.forced.keep_every = 3; p.forced.phase = 1; }
    if (which == 4) { p.forced.mode = ForcedAdmission::Mode::recent_fraction; p.forced.fraction = 0.3; }
    if (which == 5) { p.kind = PolicyKind::wgkv_plus_topk; p.window = 12;
                      p.forced.mode = ForcedAdmission::Mode::recent_fraction; p.forced.fraction = 0.5; }
    std::vector<float> g;
    for (int l = 0; l < 2; ++l) {
        if (!policy_gates(p, l, 0, 3, 3, 1, 0, 46, 40, g)) return 2;
        for (float x : g) std::printf("%d", (int)x);
        std::printf("\n");
    }
    return 0;
}
"""


@pytest.mark.skipif(shutil.which("g++") is None, reason="needs g++")
def test_cpp_policy_matches_reference_trace(ref, tmp_path):
    src = tmp_path / "p.cpp"
    src.write_text(CPP.replace("#include <cstdio>", "#include <cstdio>\n#include <cstdlib>"))
    exe = tmp_path / "p"
    subprocess.run(["g++", "-std=c++17", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    for which, (_, pol) in enumerate(CASES):
        out = subprocess.run([str(exe), str(which)], capture_output=True, text=True, check=True).stdout.split()
        tr = _ref_trace(ref, pol)
        for layer in range(L):
            got = np.array([int(c) for c in out[layer]], dtype=np.float64).reshape(H, T + ND)
            np.testing.assert_array_equal(got, tr[layer])

"""The reference's own model with the hot path swapped for the B200 C-ABI.

`oracle/_ref/dropin_session` (tests/cpp/dropin_session.cpp, built by
oracle/Makefile from the reference sources + libwgkv_b200.so) is a C++ host
that drives the CUDA kernels through include/wgkv_b200.hpp inside the
reference's ToyModel forward (engine.cpp:153-341) and runs the reference's
Session KATs (test_engine.cpp:49-286) against it: policy=full == teacher,
saturated / zeroed gates, wgkv == MaskedOracle with the per-step promotion
audit, GQA, local_sink accounting, static_heads, lifecycle errors, and the
Llama head geometry through the bf16 tcgen05 / mma.sync kernels.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "dropin_session")


def test_dropin_binary_links():
    """CPU: the drop-in host was built and every library it needs resolves."""
    if not os.path.exists(EXE):
        pytest.skip("oracle/_ref/dropin_session not built (needs /root/reference at build time)")
    r = subprocess.run(["ldd", EXE], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert "not found" not in r.stdout, r.stdout
    assert "libwgkv_b200.so" in r.stdout and "libwgkv_ref.so" in r.stdout


@pytest.mark.gpu
def test_reference_session_kats_through_dropin():
    assert os.path.exists(EXE), "oracle/_ref/dropin_session missing: run __graft_entry__.build() where the reference is"
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ALL PASS" in r.stdout

"""The header-only C++ face (include/wgkv_b200.hpp) compiles against the C-ABI,
links to libwgkv_b200.so, and rethrows the reference's exception classes for
host-side validation errors (no kernel runs; CPU only)."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SRC = r"""
#include <cstdio>
#include <stdexcept>
#include "wgkv_b200.hpp"
int main() {
    wgkv_config c{};
    c.layers = 1; c.q_heads = 4; c.kv_heads = 1; c.head_dim = 128; c.hidden = 128; c.window = 8;
    c.tau = 1.5; c.rope_base = 1e4; c.page_size = 16; c.max_seqs = 1; c.max_tokens = 64; c.dtype = WGKV_BF16;
    try { wgkv::b200::Device d(c); return 2; }
    catch (const std::invalid_argument& e) { std::printf("invalid_argument: %s\n", e.what()); }
    c.tau = 0.1; c.window = 0;
    try { wgkv::b200::Device d(c); return 3; }
    catch (const std::invalid_argument& e) { std::printf("invalid_argument: %s\n", e.what()); }
    return 0;
}
"""


@pytest.mark.skipif(shutil.which("g++") is None, reason="needs g++")
def test_cpp_wrapper_maps_exceptions(tmp_path):
    src = tmp_path / "t.cpp"
    src.write_text(SRC)
    exe = tmp_path / "t"
    lib = os.path.join(ROOT, "paper_2512_17452_b200")
    subprocess.run(["g++", "-std=c++17", "-I", os.path.join(ROOT, "include"), str(src), "-L", lib, "-lwgkv_b200",
                    "-Wl,-rpath," + lib, "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "tau must lie in (0,1)" in r.stdout
    assert "window must be >= 1" in r.stdout

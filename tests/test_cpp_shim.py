"""The C++ shim (include/voxellate_b200.hpp) -- the reference's own C++
signatures over the C-ABI -- against the reference library in one process
(tests/cpp/test_shim_vs_reference.cpp, built by __graft_entry__.build())."""
import os
import subprocess

import pytest

from conftest import ROOT

BIN = os.path.join(ROOT, "tests", "cpp", "test_shim_vs_reference")


@pytest.mark.gpu
def test_cpp_shim_matches_reference_library():
    if not os.path.exists(BIN):
        pytest.skip("C++ shim test not built (needs the reference headers at build time)")
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-2000:]
    assert "ALL OK" in out.stdout


def test_cpp_shim_header_compiles_standalone(tmp_path):
    """The shim needs nothing but the C header (no reference headers)."""
    src = tmp_path / "t.cpp"
    src.write_text('#include "voxellate_b200.hpp"\nint main(){ vxb200::Domain d({1.0}, '
                   'vxb200::Boundary::Periodic); return d.dim() == 1 ? 0 : 1; }\n')
    lib = os.path.join(ROOT, "paper_2201_13234_b200")
    out = subprocess.run(["g++", "-std=gnu++17", "-I", os.path.join(ROOT, "include"), str(src),
                          "-o", str(tmp_path / "t"), "-L", lib, "-lvoxellate_b200",
                          "-Wl,-rpath," + lib], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    assert subprocess.run([str(tmp_path / "t")]).returncode == 0

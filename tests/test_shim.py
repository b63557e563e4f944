"""The reference-side C++ shim of INTEGRATION.md (include/tilechain_b200_shim.hpp)
is compiled against the reference's own headers and linked with libtcg.so; its
host-only calls (declarations, lazy queue, validation errors rethrown as the
reference's exception types) run without a GPU. Skipped where /root/reference
is absent (the GPU box)."""
import subprocess
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parent.parent
REF = Path("/root/reference/proj/core/include")
LIB = REPO / "paper_1704_00693_b200" / "_lib"


@pytest.mark.skipif(not REF.exists(), reason="reference headers not present")
def test_reference_side_shim_compiles_and_runs(tmp_path):
    assert (LIB / "libtcg.so").exists(), "build the library first"
    exe = tmp_path / "shim_check"
    cmd = ["g++", "-std=gnu++20", "-O1", "-Wall", "-Wextra", f"-I{REPO / 'include'}", f"-I{REF}",
           str(REPO / "tests" / "shim" / "shim_check.cpp"), "-o", str(exe), f"-L{LIB}", "-ltcg",
           f"-Wl,-rpath,{LIB}", "-Wl,-rpath,/usr/local/cuda/lib64"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-4000:]
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "shim ok" in r.stdout, (r.returncode, r.stdout, r.stderr[-2000:])

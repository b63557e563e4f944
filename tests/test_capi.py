"""The C-ABI library loads without a GPU and exports every entry point
include/tilechain_b200.h declares; host-only calls work without CUDA, device
calls fail loudly (no CPU fallback)."""
import ctypes
import re
from pathlib import Path

import pytest

import paper_1704_00693_b200 as pkg
from paper_1704_00693_b200 import Range, Runtime

HEADER = Path(__file__).resolve().parent.parent / "include" / "tilechain_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tcg_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("tcg_runtime_new", "tcg_par_loop", "tcg_flush", "tcg_fetch_reduction", "tcg_get", "tcg_put",
              "tcg_upload", "tcg_download", "tcg_plan_pending", "tcg_last_error"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(str(pkg.LIB_PATH))
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_abi_version_and_registry():
    lib = pkg.load_library()
    assert lib.tcg_abi_version() == 1
    assert pkg.body_known(pkg.kernels.HEAT_LAP)
    assert pkg.body_known(pkg.kernels.hydro_body(4, True))
    assert not pkg.body_known(99999)


def test_host_only_calls_need_no_gpu():
    rt = Runtime(2)
    s = rt.declare_stencil("id", [(0, 0)])
    f = rt.declare_field("f", Range.d2(0, 8, 0, 8))
    assert rt.alloc_range(f) == Range.d2(-16, 24, -16, 24)  # pad = reach 0 + skew_allowance 16
    assert rt.pending_loops() == 0
    rt.close()


def test_errors_map_to_reference_exception_types():
    with pytest.raises(pkg.InvalidArgument):
        Runtime(4)
    rt = Runtime(1)
    with pytest.raises(pkg.InvalidArgument):
        rt.declare_stencil("empty", [])
    with pytest.raises(pkg.InvalidArgument):
        rt.declare_field("bad", Range.d1(5, 5))

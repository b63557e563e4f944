"""Builds the B200 executor library `_lib/libtcg.so` in-tree.

Host C++ (planner, runtime, C-ABI) is compiled by g++; the CUDA executors by
nvcc for sm_100a only (`-gencode arch=compute_100a,code=sm_100a`), with
`-fmad=false` so fp64 per-point arithmetic is never contracted into FMAs
(bit parity with the reference's FMA-free host build).
Incremental: an object is rebuilt when any source or header is newer.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB_DIR = PKG / "_lib"
DEBUG = os.environ.get("TCG_DEBUG_BUILD") == "1"  # device printf diagnostics, separate .so
OBJ_DIR = LIB_DIR / ("obj_debug" if DEBUG else "obj")
LIB = LIB_DIR / ("libtcg_debug.so" if DEBUG else "libtcg.so")
LIB_CHECKED = LIB_DIR / "libtcg_checked.so"
REPO = PKG.parent

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CXX = os.environ.get("CXX", "g++")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CXXFLAGS = ["-O2", "-std=c++20", "-fPIC", "-ffp-contract=off", "-Wall", "-Wextra", "-Wno-unused-parameter",
            f"-I{REPO / 'include'}", "-I/usr/local/cuda/include", f"-I{OBJ_DIR}"]
NVCCFLAGS = ARCH + ["-O3", "-lineinfo", "-fmad=false", "-std=c++20", "-Xcompiler", "-fPIC",
                    "--expt-relaxed-constexpr", "-Xptxas", "-v", f"-I{REPO / 'include'}"]

if DEBUG:
    NVCCFLAGS = NVCCFLAGS + ["-DTCG_DEBUG_PRINT"]

HOST_SRCS = ["host/tcg_plan.cpp", "host/tcg_gpuplan.cpp", "host/tcg_dist.cpp", "host/tcg_stream.cpp", "host/tcg_periodic.cpp", "host/tcg_jit.cpp",
             "host/tcg_runtime.cpp", "tcg_capi.cpp"]
CUDA_SRCS = ["cuda/tcg_exec.cu", "cuda/tcg_tiled.cu", "cuda/tcg_l2.cu", "cuda/tcg_comm.cu", "cuda/tcg_stream_exec.cu"]


def _headers() -> list[Path]:
    hs = [p for p in CSRC.rglob("*") if p.suffix in (".h", ".hpp", ".cuh", ".inl")]
    hs += list((REPO / "include").glob("*.h"))
    hs.append(Path(__file__))
    return hs


def _stale(obj: Path, src: Path, headers: list[Path]) -> bool:
    if not obj.exists():
        return True
    t = obj.stat().st_mtime
    return src.stat().st_mtime > t or any(h.stat().st_mtime > t for h in headers)


def _compile(cmd: list[str], log: Path) -> None:
    r = subprocess.run(cmd, capture_output=True, text=True)
    log.write_text(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"compile failed: {' '.join(cmd)}")


def _embed_bodies() -> None:
    """Writes tcb_sources.inc: the body registry headers as string literals,
    handed to NVRTC when a generated chain kernel is compiled (tcg_jit.cpp)."""
    out = OBJ_DIR / "tcb_sources.inc"
    parts = []
    for var, name in (("kTcbBodiesSrc", "tc_bodies.h"), ("kTcbNsSrc", "tc_ns.h")):
        text = (CSRC / "kernels" / name).read_text()
        assert ")TCBSRC\"" not in text
        parts.append(f'const char* const {var} = R"TCBSRC({text})TCBSRC";\n')
    data = "".join(parts)
    if not out.exists() or out.read_text() != data:
        out.write_text(data)


def build(verbose: bool = False) -> Path:
    OBJ_DIR.mkdir(parents=True, exist_ok=True)
    _embed_bodies()
    headers = _headers()
    jobs = []
    objs = []
    for s in HOST_SRCS:
        src = CSRC / s
        obj = OBJ_DIR / (s.replace("/", "_") + ".o")
        objs.append(obj)
        if _stale(obj, src, headers):
            jobs.append(([CXX, *CXXFLAGS, "-c", str(src), "-o", str(obj)], obj.with_suffix(".log")))
    for s in CUDA_SRCS:
        src = CSRC / s
        obj = OBJ_DIR / (s.replace("/", "_") + ".o")
        objs.append(obj)
        if _stale(obj, src, headers):
            jobs.append(([NVCC, *NVCCFLAGS, "-c", str(src), "-o", str(obj)], obj.with_suffix(".log")))
    # Checked variant (libtcg_checked.so): the untiled executor with the
    # reference's KernelCtx access checks on the device (-DTCG_CHECKED); the
    # other objects are shared.
    src = CSRC / "cuda/tcg_exec.cu"
    cobj = OBJ_DIR / "cuda_tcg_exec.cu.checked.o"
    checked_jobs = []
    if _stale(cobj, src, headers):
        checked_jobs.append(([NVCC, *NVCCFLAGS, "-DTCG_CHECKED", "-c", str(src), "-o", str(cobj)],
                             cobj.with_suffix(".log")))
    if jobs or checked_jobs:
        allj = jobs + checked_jobs
        with cf.ThreadPoolExecutor(max_workers=min(8, len(allj))) as ex:
            for f in [ex.submit(_compile, c, l) for c, l in allj]:
                f.result()
    if jobs or not LIB.exists():
        cmd = [NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-lnvrtc", "-ldl", "-Xlinker", "-rpath=/usr/local/cuda/lib64"]
        _compile(cmd, LIB_DIR / "link.log")
    if jobs or checked_jobs or not LIB_CHECKED.exists():
        cobjs = [str(cobj) if o.name == "cuda_tcg_exec.cu.o" else str(o) for o in objs]
        _compile([NVCC, *ARCH, "-shared", "-o", str(LIB_CHECKED), *cobjs, "-lnvrtc", "-ldl", "-Xlinker", "-rpath=/usr/local/cuda/lib64"], LIB_DIR / "link_checked.log")
    if verbose:
        print(f"built {LIB}")
    return LIB


if __name__ == "__main__":
    build(verbose=True)

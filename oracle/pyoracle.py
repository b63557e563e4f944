"""ORACLE / TEST INFRASTRUCTURE -- not product code.

ctypes front ends with the same method names as paper_1704_00693_b200.Runtime:
  RefRuntime     the unmodified reference tilechain::Runtime (oracle/_ref/libtcref.so,
                 built from /root/reference sources by oracle/Makefile);
  OracleRuntime  this repo's sequential C++ restatement (oracle/build/libtcoracle.so).
Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import this.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path
from typing import Optional, Sequence

import numpy as np

HERE = Path(__file__).resolve().parent
REF_LIB = HERE / "_ref" / "libtcref.so"
ORACLE_LIB = HERE / "build" / "libtcoracle.so"

_I64, _I32, _P, _D = ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p, ctypes.c_double


class OracleError(RuntimeError):
    pass


def build(ref: bool = True) -> None:
    """Builds the oracle (and the reference library when its sources exist)."""
    target = ["all"] if ref and Path("/root/reference/proj/core/src").exists() else ["oracle"]
    subprocess.run(["make", "-s", "-C", str(HERE), *target], check=True)


def _arr(ct, vals):
    vals = list(vals)
    return (ct * max(1, len(vals)))(*vals)


def _lohi(rng):
    return rng.lohi if hasattr(rng, "lohi") else list(rng)


def _args(args):
    flat = []
    for a in args:
        if hasattr(a, "dataset"):
            flat += [a.dataset, a.stencil, int(a.mode)]
        else:
            flat += [int(a[0]), int(a[1]), int(a[2])]
    return flat


_ref_lib = None
_ora_lib = None


def ref_available() -> bool:
    return REF_LIB.exists()


def load_ref():
    global _ref_lib
    if _ref_lib is None:
        if not REF_LIB.exists():
            raise OracleError(f"{REF_LIB} not built (needs /root/reference; run make -C oracle)")
        lib = ctypes.CDLL(str(REF_LIB))
        lib.tcref_error.restype = ctypes.c_char_p
        lib.tcref_new.restype = _P
        lib.tcref_new.argtypes = [ctypes.c_int, ctypes.c_int, _I64, _I64, ctypes.c_int]
        lib.tcref_free.argtypes = [_P]
        for n, a in {
            "tcref_declare_stencil": [_P, ctypes.c_int, _P],
            "tcref_declare_field": [_P, ctypes.c_char_p, _P],
            "tcref_alloc_range": [_P, ctypes.c_int, _P],
            "tcref_put_alloc": [_P, ctypes.c_int, _P],
            "tcref_get_alloc": [_P, ctypes.c_int, _P],
            "tcref_set_rank_grid": [_P, _P],
            "tcref_set_default_mode": [_P, ctypes.c_int, _P],
            "tcref_par_loop": [_P, ctypes.c_int, ctypes.c_int, ctypes.c_int, _P, ctypes.c_int, _P, ctypes.c_int, _P],
            "tcref_flush": [_P, ctypes.c_int, _P, ctypes.c_char_p, _I64],
            "tcref_fetch": [_P, ctypes.c_int, _P],
            "tcref_last_plan": [_P, ctypes.c_char_p, _I64],
            "tcref_plan_pending": [_P, _P, ctypes.c_char_p, _I64],
            "tcref_validate_plan": [_P, _P, _P, _I64, ctypes.c_int, ctypes.c_char_p, _I64],
            "tcref_rank_plans_pending": [_P, _P, _P, ctypes.c_char_p, _I64],
            "tcref_validate_rank_plans": [_P, ctypes.c_int, ctypes.c_int, _P, _P, _P, _P, ctypes.c_char_p, _I64],
            "tcref_dist_info": [_P, ctypes.c_char_p, _I64],
            "tcref_auto_tile_size": [ctypes.c_int, _I64, ctypes.c_int, _I64, _P, _P],
            "tcref_app_jacobi": [_I64, _I64, ctypes.c_int, ctypes.c_int, _P],
            "tcref_app_minihydro": [_I64, _I64, ctypes.c_int, _P, _P],
        }.items():
            fn = getattr(lib, n)
            fn.argtypes = a
            fn.restype = _I64
        _ref_lib = lib
    return _ref_lib


def load_oracle():
    global _ora_lib
    if _ora_lib is None:
        if not ORACLE_LIB.exists():
            raise OracleError(f"{ORACLE_LIB} not built (run make -C oracle)")
        lib = ctypes.CDLL(str(ORACLE_LIB))
        lib.tco_error.restype = ctypes.c_char_p
        lib.tco_new.restype = _P
        lib.tco_new.argtypes = [ctypes.c_int, _I64]
        lib.tco_free.argtypes = [_P]
        for n, a in {
            "tco_declare_stencil": [_P, ctypes.c_int, _P],
            "tco_declare_field": [_P, ctypes.c_char_p, _P],
            "tco_put_alloc": [_P, ctypes.c_int, _P],
            "tco_get_alloc": [_P, ctypes.c_int, _P],
            "tco_par_loop": [_P, ctypes.c_int, ctypes.c_int, ctypes.c_int, _P, ctypes.c_int, _P, ctypes.c_int, _P],
            "tco_fetch": [_P, ctypes.c_int, _P],
            "tco_set_reduction_mask": [_P, _P],
        }.items():
            fn = getattr(lib, n)
            fn.argtypes = a
            fn.restype = _I64
        _ora_lib = lib
    return _ora_lib


class _Range:
    def __init__(self, dim, lohi):
        self.dim = dim
        self.lohi = list(lohi)

    def start(self, d):
        return self.lohi[2 * d]

    def end(self, d):
        return self.lohi[2 * d + 1]

    def extent(self, d):
        return self.lohi[2 * d + 1] - self.lohi[2 * d]

    def volume(self):
        v = 1
        for d in range(self.dim):
            v *= self.extent(d)
        return v

    def shape(self):
        return tuple(self.extent(d) for d in reversed(range(self.dim)))


class _Base:
    dim: int

    def _alloc(self, logical_lohi):
        pad = self._reach + self._skew
        lohi = []
        for d in range(3):
            if d < self.dim:
                lohi += [logical_lohi[2 * d] - pad, logical_lohi[2 * d + 1] + pad]
            else:
                lohi += [0, 1]
        return _Range(self.dim, lohi)

    def alloc_range(self, ds):
        return self._allocs[ds]

    def periodic_fill(self, datasets, depth, logical):
        """Host ghost copy for a periodic box (the SURVEY §8(c) recipe for c5:
        pure copying into the padding, so bit-exact), dimension by dimension
        like Runtime::periodic_fill. `logical`: lohi list of the box."""
        self.flush()
        L = [logical[2 * d] for d in range(self.dim)]
        H = [logical[2 * d + 1] for d in range(self.dim)]
        for ds in datasets:
            al = self._allocs[ds]
            arr = self.download(ds)
            lo = [al.start(d) for d in range(self.dim)]
            for d in range(self.dim):
                def sl(a, b, dd=d):
                    idx = []
                    for e in reversed(range(self.dim)):
                        if e == dd:
                            idx.append(slice(a - lo[e], b - lo[e]))
                        elif e < dd:
                            idx.append(slice(L[e] - depth - lo[e], H[e] + depth - lo[e]))
                        else:
                            idx.append(slice(L[e] - lo[e], H[e] - lo[e]))
                    return tuple(idx)
                arr[sl(L[d] - depth, L[d])] = arr[sl(H[d] - depth, H[d])]
                arr[sl(H[d], H[d] + depth)] = arr[sl(L[d], L[d] + depth)]
            self.upload(ds, arr)


class RefRuntime(_Base):
    """The reference tilechain::Runtime (threads = CPU workers)."""

    def __init__(self, dim, threads=1, skew_allowance=16, cache_bytes=8 << 20, whole_queue=False):
        self.lib = load_ref()
        self.h = self.lib.tcref_new(dim, threads, skew_allowance, cache_bytes, int(whole_queue))
        if not self.h:
            raise OracleError(self.lib.tcref_error().decode())
        self.dim = dim
        self._allocs = []

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.tcref_free(self.h)
            self.h = None

    def _ck(self, rc):
        if rc == -2:
            raise OracleError(self.lib.tcref_error().decode())
        return rc

    def declare_stencil(self, name, points):
        flat = []
        for p in points:
            p = list(p) + [0] * (3 - len(p))
            flat += p[:3]
        return self._ck(self.lib.tcref_declare_stencil(self.h, len(flat) // 3, _arr(_I64, flat)))

    def declare_field(self, name, logical):
        ds = self._ck(self.lib.tcref_declare_field(self.h, name.encode(), _arr(_I64, _lohi(logical))))
        a = (_I64 * 6)()
        self._ck(self.lib.tcref_alloc_range(self.h, ds, a))
        self._allocs.append(_Range(self.dim, list(a)))
        return ds

    def par_loop(self, kernel, rng, args, reduction=None):
        prm = list(kernel.params)
        return self._ck(self.lib.tcref_par_loop(self.h, kernel.id, kernel.body, -1 if reduction is None else int(reduction),
                                                _arr(_I64, _lohi(rng)), len(args), _arr(_I32, _args(args)), len(prm),
                                                _arr(_D, prm)))

    def flush(self, mode=None):
        kind, ts = (0, (0, 0, 0)) if mode is None else (mode.kind, mode.tile_sizes)
        if mode is None:
            # default mode of the handle
            kind = -1
        buf = ctypes.create_string_buffer(1 << 16)
        if kind == -1:
            self._ck(self.lib.tcref_flush(self.h, self._default[0], _arr(_I64, self._default[1]), buf, len(buf)))
        else:
            self._ck(self.lib.tcref_flush(self.h, kind, _arr(_I64, ts), buf, len(buf)))
        return dict(l.split("=", 1) for l in buf.value.decode().splitlines() if "=" in l)

    _default = (0, (0, 0, 0))

    def set_default_mode(self, mode):
        self._default = (mode.kind, tuple(mode.tile_sizes))
        self._ck(self.lib.tcref_set_default_mode(self.h, mode.kind, _arr(_I64, mode.tile_sizes)))

    def set_rank_grid(self, grid):
        g = list(grid) + [1] * (3 - len(grid))
        self._ck(self.lib.tcref_set_rank_grid(self.h, _arr(_I32, g[:3])))

    def fetch_reduction(self, h):
        out = _D()
        self._ck(self.lib.tcref_fetch(self.h, h, ctypes.byref(out)))
        return out.value

    def upload(self, ds, data):
        a = np.ascontiguousarray(data, dtype=np.float64)
        assert a.size == self._allocs[ds].volume()
        self._ck(self.lib.tcref_put_alloc(self.h, ds, a.ctypes.data_as(_P)))

    def download(self, ds):
        out = np.empty(self._allocs[ds].shape(), dtype=np.float64)
        self._ck(self.lib.tcref_get_alloc(self.h, ds, out.ctypes.data_as(_P)))
        return out

    def _text(self, fn, *args):
        buf = ctypes.create_string_buffer(1 << 24)
        n = self._ck(fn(self.h, *args, buf, len(buf)))
        if n > len(buf):
            raise OracleError("text truncated")
        return buf.value.decode()

    def plan_pending(self, ts):
        ts = list(ts) + [0] * (3 - len(ts))
        return self._text(self.lib.tcref_plan_pending, _arr(_I64, ts[:3]))

    def validate_plan_pending(self, ts, ranges, ntiles, nloops):
        """The reference's validate_dependencies + validate_coverage
        (oracle.cpp:154-284) on an external plan for the pending chain
        (consumed). ranges: flat int64, 6 per (tile, loop). Returns
        (violation count, text)."""
        ts = list(ts) + [0] * (3 - len(ts))
        buf = ctypes.create_string_buffer(1 << 20)
        n = self.lib.tcref_validate_plan(self.h, _arr(_I64, ts[:3]), _arr(_I64, ranges), ntiles, nloops, buf,
                                         len(buf))
        if n < 0:
            raise OracleError(self.lib.tcref_error().decode())
        return int(n), buf.value.decode()

    def validate_rank_plans_pending(self, nranks, nloops, ranges, owned, band, skip):
        """The reference's validate_dependencies (per rank) and
        validate_coverage_replicated (over the owned parts) on overlapped
        single-tile plans -- the streaming executor's CTA plans. Consumes the
        pending chain. Returns (violations, text)."""
        buf = ctypes.create_string_buffer(1 << 20)
        band = list(band) + [0] * (3 - len(band))
        n = self.lib.tcref_validate_rank_plans(self.h, nranks, nloops, _arr(_I64, ranges), _arr(_I64, owned),
                                               _arr(_I64, band[:3]), _arr(_I32, skip), buf, len(buf))
        if n < 0:
            raise OracleError(self.lib.tcref_error().decode())
        return int(n), buf.value.decode()

    def rank_plans_pending(self, grid, ts):
        g = list(grid) + [1] * (3 - len(grid))
        ts = list(ts) + [0] * (3 - len(ts))
        return self._text(self.lib.tcref_rank_plans_pending, _arr(_I32, g[:3]), _arr(_I64, ts[:3]))

    def last_plan(self):
        return self._text(self.lib.tcref_last_plan)

    def dist_info(self):
        return self._text(self.lib.tcref_dist_info)


class OracleRuntime(_Base):
    """Sequential restatement (oracle/tc_oracle.cpp); executes eagerly."""

    def __init__(self, dim, skew_allowance=16, **_):
        self.lib = load_oracle()
        self.h = self.lib.tco_new(dim, skew_allowance)
        self.dim = dim
        self._allocs = []
        self._reach = 0
        self._skew = skew_allowance

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.tco_free(self.h)
            self.h = None

    def _ck(self, rc):
        if rc == -2:
            raise OracleError(self.lib.tco_error().decode())
        return rc

    def declare_stencil(self, name, points):
        flat = []
        for p in points:
            p = list(p) + [0] * (3 - len(p))
            flat += p[:3]
            self._reach = max(self._reach, max(abs(v) for v in p[: self.dim]))
        return self._ck(self.lib.tco_declare_stencil(self.h, len(flat) // 3, _arr(_I64, flat)))

    def declare_field(self, name, logical):
        lohi = _lohi(logical)
        ds = self._ck(self.lib.tco_declare_field(self.h, name.encode(), _arr(_I64, lohi)))
        self._allocs.append(self._alloc(lohi))
        return ds

    def par_loop(self, kernel, rng, args, reduction=None):
        prm = list(kernel.params)
        return self._ck(self.lib.tco_par_loop(self.h, kernel.id, kernel.body, -1 if reduction is None else int(reduction),
                                              _arr(_I64, _lohi(rng)), len(args), _arr(_I32, _args(args)), len(prm),
                                              _arr(_D, prm)))

    def flush(self, mode=None):
        return {}

    def set_default_mode(self, mode):
        pass

    def fetch_reduction(self, h):
        out = _D()
        self._ck(self.lib.tco_fetch(self.h, h, ctypes.byref(out)))
        return out.value

    def set_reduction_mask(self, rng):
        """Only points inside rng contribute to later reductions (None clears)."""
        self._ck(self.lib.tco_set_reduction_mask(self.h, None if rng is None else _arr(_I64, _lohi(rng))))

    def upload(self, ds, data):
        a = np.ascontiguousarray(data, dtype=np.float64)
        assert a.size == self._allocs[ds].volume()
        self._ck(self.lib.tco_put_alloc(self.h, ds, a.ctypes.data_as(_P)))

    def download(self, ds):
        out = np.empty(self._allocs[ds].shape(), dtype=np.float64)
        self._ck(self.lib.tco_get_alloc(self.h, ds, out.ctypes.data_as(_P)))
        return out


def ref_auto_tile_size(dim, cache_bytes, threads, bpp, extent_lohi):
    lib = load_ref()
    out = (_I64 * 3)()
    rc = lib.tcref_auto_tile_size(dim, cache_bytes, threads, bpp, _arr(_I64, extent_lohi), out)
    if rc == -2:
        raise OracleError(lib.tcref_error().decode())
    return tuple(out)


def ref_app_jacobi(nx, ny, iters, copy_variant):
    lib = load_ref()
    out = np.empty(2 * nx * ny)
    rc = lib.tcref_app_jacobi(nx, ny, iters, int(copy_variant), out.ctypes.data_as(_P))
    if rc == -2:
        raise OracleError(lib.tcref_error().decode())
    return out.reshape(2, ny, nx)


def ref_app_minihydro(nx, ny, iters):
    lib = load_ref()
    out = np.empty(8 * nx * ny)
    mon = np.empty(iters)
    rc = lib.tcref_app_minihydro(nx, ny, iters, out.ctypes.data_as(_P), mon.ctypes.data_as(_P))
    if rc == -2:
        raise OracleError(lib.tcref_error().decode())
    return out.reshape(8, ny, nx), mon

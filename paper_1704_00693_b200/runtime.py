"""Python mirror of the reference front door over the C-ABI (include/tilechain_b200.h).

Names, argument meaning and error behaviour follow tilechain::Runtime
(proj/core/include/tilechain/runtime.hpp:44-135) so tests read like the
reference's own tests:

    rt = Runtime(2)
    five = rt.declare_stencil("five", [(0,0),(1,0),(-1,0),(0,1),(0,-1)])
    a = rt.declare_field("a", Range.d2(0, 64, 0, 64))
    h = rt.par_loop(KernelHandle(0, "jacobi", body=kernels.JACOBI_STENCIL), Range.d2(1, 63, 1, 63),
                    [ArgSpec(a, five, AccessMode.Read), ArgSpec(b, ident, AccessMode.Write)])
    rt.flush(ExecMode.tiled_auto())

Every call goes through libtcg.so; there is no Python or CPU execution path.
If the library or the GPU is missing the calls raise.
"""
from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass, field
from pathlib import Path
from typing import Iterable, Optional, Sequence

import numpy as np

_PKG = Path(__file__).resolve().parent
LIB_PATH = Path(__import__("os").environ["TCG_LIB"]) if __import__("os").environ.get("TCG_LIB") else _PKG / "_lib" / ("libtcg_debug.so" if __import__("os").environ.get("TCG_DEBUG_LIB") == "1" else "libtcg.so")
_lib: Optional[ctypes.CDLL] = None
_par_loop_raw = None


class TcgError(RuntimeError):
    code = 6


class InvalidArgument(TcgError):
    code = 1


class AccessError(TcgError):
    code = 2


class PlanError(TcgError):
    code = 3


class CudaError(TcgError):
    code = 4


class SizerError(TcgError):
    code = 5


_ERR = {1: InvalidArgument, 2: AccessError, 3: PlanError, 4: CudaError, 5: SizerError, 6: TcgError}

_I64 = ctypes.c_int64
_I32 = ctypes.c_int32
_P = ctypes.c_void_p
_D = ctypes.c_double


class _Config(ctypes.Structure):
    _fields_ = [("threads", _I32), ("skew_allowance", _I64), ("cache_bytes", _I64),
                ("flush_whole_queue_on_fetch", _I32), ("stream_segments", _I32)]


def load_library() -> ctypes.CDLL:
    """Loads the in-tree executor library; raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(str(LIB_PATH))
    sig = {
        "tcg_last_error": (ctypes.c_size_t, [ctypes.c_char_p, ctypes.c_size_t]),
        "tcg_abi_version": (ctypes.c_int, []),
        "tcg_runtime_new": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(_Config), ctypes.POINTER(_P)]),
        "tcg_runtime_free": (None, [_P]),
        "tcg_declare_stencil": (ctypes.c_int, [_P, ctypes.c_int, ctypes.POINTER(_I64), ctypes.POINTER(_I32)]),
        "tcg_declare_field": (ctypes.c_int, [_P, ctypes.c_char_p, ctypes.POINTER(_I64), ctypes.POINTER(_I32)]),
        "tcg_alloc_range": (ctypes.c_int, [_P, _I32, ctypes.POINTER(_I64)]),
        "tcg_par_loop": (ctypes.c_int, [_P, _I32, _I32, ctypes.POINTER(_I64), ctypes.c_int, ctypes.POINTER(_I32),
                                        ctypes.c_int, ctypes.c_int, ctypes.POINTER(_D), ctypes.POINTER(_I32)]),
        "tcg_flush": (ctypes.c_int, [_P, ctypes.c_int, ctypes.POINTER(_I64)]),
        "tcg_flush_default": (ctypes.c_int, [_P]),
        "tcg_set_default_mode": (ctypes.c_int, [_P, ctypes.c_int, ctypes.POINTER(_I64)]),
        "tcg_fetch_reduction": (ctypes.c_int, [_P, _I32, ctypes.POINTER(_D)]),
        "tcg_pending_loops": (ctypes.c_int, [_P, ctypes.POINTER(_I64)]),
        "tcg_get": (ctypes.c_int, [_P, _I32, ctypes.POINTER(_I64), ctypes.POINTER(_D)]),
        "tcg_put": (ctypes.c_int, [_P, _I32, ctypes.POINTER(_I64), _D]),
        "tcg_fill_logical": (ctypes.c_int, [_P, _I32, _D]),
        "tcg_upload": (ctypes.c_int, [_P, _I32, _P]),
        "tcg_download": (ctypes.c_int, [_P, _I32, _P]),
        "tcg_synchronize": (ctypes.c_int, [_P]),
        "tcg_report_text": (ctypes.c_int, [_P, ctypes.c_char_p, _I64, ctypes.POINTER(_I64)]),
        "tcg_plan_pending": (ctypes.c_int, [_P, ctypes.POINTER(_I64), ctypes.c_char_p, _I64, ctypes.POINTER(_I64)]),
        "tcg_rank_plans_pending": (ctypes.c_int, [_P, ctypes.POINTER(_I32), ctypes.POINTER(_I64), ctypes.c_char_p, _I64,
                                                  ctypes.POINTER(_I64)]),
        "tcg_gpu_plan_pending": (ctypes.c_int, [_P, ctypes.c_int, ctypes.POINTER(_I64), ctypes.c_char_p, _I64,
                                                ctypes.POINTER(_I64)]),
        "tcg_signature_pending": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_uint64)]),
        "tcg_set_stream_choice": (ctypes.c_int, [_P, ctypes.POINTER(_I32)]),
        "tcg_stream_plan_pending": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_char_p, _I64, ctypes.POINTER(_I64)]),
        "tcg_set_rank_grid": (ctypes.c_int, [_P, ctypes.POINTER(_I32)]),
        "tcg_periodic_fill": (ctypes.c_int, [_P, ctypes.c_int, ctypes.POINTER(_I32), _I64]),
        "tcg_set_periodic_flush": (ctypes.c_int, [_P, ctypes.c_int]),
        "tcg_set_periodic_domain": (ctypes.c_int, [_P, ctypes.c_int]),
        "tcg_set_reduction_order": (ctypes.c_int, [_P, ctypes.c_int]),
        "tcg_record_begin": (ctypes.c_int, [_P]),
        "tcg_record_end": (ctypes.c_int, [_P, ctypes.POINTER(_I32)]),
        "tcg_replay": (ctypes.c_int, [_P, _I32, ctypes.POINTER(ctypes.c_double), _I64, ctypes.POINTER(_I32), _I64,
                                      ctypes.POINTER(_I64)]),
        "tcg_periodic_plan_pending": (ctypes.c_int, [_P, ctypes.c_char_p, _I64, ctypes.POINTER(_I64)]),
        "tcg_upload_box": (ctypes.c_int, [_P, _I32, _P, ctypes.POINTER(_I64)]),
        "tcg_download_box": (ctypes.c_int, [_P, _I32, _P, ctypes.POINTER(_I64)]),
        "tcg_local_box": (ctypes.c_int, [_P, _I32, ctypes.POINTER(_I64)]),
        "tcg_rank_owned": (ctypes.c_int, [_P, _I32, ctypes.POINTER(_I64)]),
        "tcg_comm_unique_id": (ctypes.c_int, [ctypes.c_char_p]),
        "tcg_set_process_rank": (ctypes.c_int, [_P, ctypes.POINTER(_I32), _I32, ctypes.c_char_p]),
        "tcg_dist_schedule_pending": (ctypes.c_int, [_P, ctypes.c_char_p, _I64, ctypes.POINTER(_I64)]),
        "tcg_auto_tile_size": (ctypes.c_int, [ctypes.c_int, _I64, _I32, _I64, ctypes.POINTER(_I64), ctypes.POINTER(_I64)]),
        "tcg_device_info": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_size_t, ctypes.POINTER(_I32), ctypes.POINTER(_I64),
                                           ctypes.POINTER(_I64)]),
        "tcg_launches": (ctypes.c_int, [_P, ctypes.POINTER(_I64)]),
        "tcg_stream": (ctypes.c_int, [_P, ctypes.POINTER(_P)]),
        "tcg_body_known": (ctypes.c_int, [_I32]),
        "tcg_set_timing": (ctypes.c_int, [_P, ctypes.c_int]),
        "tcg_select_device": (ctypes.c_int, [ctypes.c_int]),
        "tcg_kernel_timing": (ctypes.c_int, [_P, ctypes.POINTER(_D), ctypes.POINTER(_I64), ctypes.POINTER(_D),
                                             ctypes.POINTER(_I64)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    # The enqueue hot path calls tcg_par_loop through a second handle without
    # argtypes: every argument is passed pre-converted (ctypes arrays, C-int
    # sized Python ints), which skips ctypes' per-call conversion (2.1 -> 1.3
    # us per par_loop, measured).
    global _par_loop_raw
    raw = ctypes.CDLL(str(LIB_PATH))
    _par_loop_raw = raw.tcg_par_loop
    _par_loop_raw.restype = ctypes.c_int
    return lib


def _check(rc: int) -> None:
    if rc != 0:
        buf = ctypes.create_string_buffer(4096)
        _lib.tcg_last_error(buf, 4096)
        raise _ERR.get(rc, TcgError)(buf.value.decode(errors="replace"))


def _arr(ctype, vals):
    vals = list(vals)
    return (ctype * max(1, len(vals)))(*vals)


def _text(fn, *args, size: int = 1 << 22) -> str:
    # One call only: several of these consume the pending queue.
    need = _I64(0)
    buf = ctypes.create_string_buffer(size)
    _check(fn(*args, buf, len(buf), ctypes.byref(need)))
    if need.value > size:
        raise TcgError(f"text output truncated ({need.value} bytes > {size}); pass a larger size")
    return buf.value.decode()


class AccessMode(enum.IntEnum):
    Read = 0
    Write = 1
    ReadWrite = 2
    Increment = 3


class ReduceOp(enum.IntEnum):
    Sum = 0
    Min = 1
    Max = 2


class Range:
    """Half-open box per dimension (types.hpp:46-183)."""

    def __init__(self, dim: int, lohi: Sequence[int]):
        if dim < 1 or dim > 3:
            raise InvalidArgument("Range: dim must be 1, 2, or 3")
        self.dim = dim
        self.lohi = [int(v) for v in lohi[: 2 * dim]] + [0, 1] * (3 - dim)

    @staticmethod
    def d1(s0, e0):
        return Range(1, [s0, e0])

    @staticmethod
    def d2(s0, e0, s1, e1):
        return Range(2, [s0, e0, s1, e1])

    @staticmethod
    def d3(s0, e0, s1, e1, s2, e2):
        return Range(3, [s0, e0, s1, e1, s2, e2])

    def start(self, d):
        return self.lohi[2 * d]

    def end(self, d):
        return self.lohi[2 * d + 1]

    def extent(self, d):
        return self.end(d) - self.start(d)

    def volume(self) -> int:
        v = 1
        for d in range(self.dim):
            v *= max(0, self.extent(d))
        return v

    def shape(self):
        """numpy shape of a dense array over this box (dim 0 fastest)."""
        return tuple(self.extent(d) for d in reversed(range(self.dim)))

    def __eq__(self, o):
        return isinstance(o, Range) and self.dim == o.dim and self.lohi[: 2 * self.dim] == o.lohi[: 2 * o.dim]

    def __repr__(self):
        return "x".join(f"[{self.start(d)},{self.end(d)})" for d in range(self.dim))


@dataclass
class ArgSpec:
    dataset: int
    stencil: int
    mode: AccessMode = AccessMode.Read


@dataclass
class KernelHandle:
    """Reference KernelHandle{id, name, fn}: `body` + `params` replace the closure."""

    id: int
    name: str
    body: int
    params: Sequence[float] = field(default_factory=tuple)


@dataclass
class ExecMode:
    kind: int = 0
    tile_sizes: Sequence[int] = (0, 0, 0)

    @staticmethod
    def untiled():
        return ExecMode(0, (0, 0, 0))

    @staticmethod
    def tiled(ts):
        ts = list(ts) + [1] * (3 - len(ts))
        return ExecMode(1, tuple(int(v) for v in ts[:3]))

    @staticmethod
    def tiled_auto():
        return ExecMode(2, (0, 0, 0))

    @staticmethod
    def stream():
        """The fused streaming executor (one generated kernel per chain
        signature)."""
        return ExecMode(4, (0, 0, 0))

    @staticmethod
    def windowed(ts=(0, 0, 0)):
        """The shared-memory windowed executor (B200-specific; ts = column
        block / stream tile upper bounds, 0 = sizer)."""
        ts = list(ts) + [0] * (3 - len(ts))
        return ExecMode(3, tuple(int(v) for v in ts[:3]))


@dataclass
class RuntimeConfig:
    threads: int = 1
    skew_allowance: int = 16
    cache_bytes: int = 8 << 20
    flush_whole_queue_on_fetch: bool = False
    stream_segments: int = 0


def comm_unique_id() -> bytes:
    lib = load_library()
    buf = ctypes.create_string_buffer(128)
    _check(lib.tcg_comm_unique_id(buf))
    return buf.raw


def parse_schedule(text: str, dim: int) -> dict:
    ranks, msgs, wraps = {}, [], []
    for line in text.splitlines():
        f = line.split()
        if not f:
            continue
        kv = {k: v for k, _, v in (x.partition("=") for x in f if "=" in x)}
        if line.startswith("rank="):
            ranks[int(kv["rank"])] = {"owned": kv["owned"], "computed": int(kv["computed"]), "loops": []}
        elif f[0] == "loop":
            nums = [int(v) for v in f[3:]]
            ranks[int(kv["rank"])]["loops"].append([(nums[2 * d], nums[2 * d + 1]) for d in range(dim)])
        elif f[0] == "wrap":
            wraps.append((int(kv["ds"]), int(kv["depth"])))
        elif f[0] == "msg":
            i = f.index("box")
            nums = [int(v) for v in f[i + 1:]]
            msgs.append({"src": int(kv["src"]), "dst": int(kv["dst"]), "ds": int(kv["ds"]), "dim": int(kv["dim"]),
                         "dir": int(kv["dir"]), "box": [(nums[2 * d], nums[2 * d + 1]) for d in range(dim)]})
    return {"ranks": ranks, "msgs": msgs, "wraps": wraps}


def parse_report(text: str) -> dict:
    rep = {}
    for line in text.splitlines():
        if "=" in line:
            k, v = line.split("=", 1)
            rep[k] = v
    return rep


class LazyReport(dict):
    """ExecutionReport of one flush as key -> text value (ExecutionReport::
    to_text keys, executor.cpp:321-366). The text is fetched when the flush
    returns and parsed on first access, so a time-stepping loop that ignores
    the report pays no parsing per step."""

    def __init__(self, text: str):
        super().__init__()
        self._text = text

    def _fill(self):
        if self._text is not None:
            t, self._text = self._text, None
            super().update(parse_report(t))

    def __getitem__(self, k):
        self._fill()
        return super().__getitem__(k)

    def get(self, k, default=None):
        self._fill()
        return super().get(k, default)

    def __contains__(self, k):
        self._fill()
        return super().__contains__(k)

    def __iter__(self):
        self._fill()
        return super().__iter__()

    def __len__(self):
        self._fill()
        return super().__len__()

    def keys(self):
        self._fill()
        return super().keys()

    def items(self):
        self._fill()
        return super().items()

    def values(self):
        self._fill()
        return super().values()

    def __repr__(self):
        self._fill()
        return super().__repr__()


class Runtime:
    """tilechain::Runtime over the B200 executor."""

    def __init__(self, dim: int, config: Optional[RuntimeConfig] = None):
        lib = load_library()
        cfg = config or RuntimeConfig()
        c = _Config(cfg.threads, cfg.skew_allowance, cfg.cache_bytes, int(cfg.flush_whole_queue_on_fetch),
                    cfg.stream_segments)
        h = _P()
        _check(lib.tcg_runtime_new(dim, ctypes.byref(c), ctypes.byref(h)))
        self._h = h
        self._lib = lib
        self.dim = dim
        self.config = cfg
        self._allocs: list[Range] = []
        self._logicals: list[Range] = []
        self._enc: dict = {}
        self._rbuf = ctypes.create_string_buffer(1 << 14)
        self._out = _I32(-1)
        self._out_ref = ctypes.byref(self._out)

    def close(self):
        if getattr(self, "_h", None):
            self._lib.tcg_runtime_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- declarations --------------------------------------------------
    def declare_stencil(self, name: str, points: Iterable[Sequence[int]]) -> int:
        flat = []
        n = 0
        for p in points:
            p = list(p) + [0] * (3 - len(p))
            flat += p[:3]
            n += 1
        out = _I32()
        _check(self._lib.tcg_declare_stencil(self._h, n, _arr(_I64, flat), ctypes.byref(out)))
        return out.value

    def declare_field(self, name: str, logical: Range, elem_bytes: int = 8) -> int:
        if elem_bytes != 8:
            raise InvalidArgument("declare_field: the B200 executor stores fp64 (elem_bytes = 8)")
        out = _I32()
        _check(self._lib.tcg_declare_field(self._h, name.encode(), _arr(_I64, logical.lohi), ctypes.byref(out)))
        a = (_I64 * 6)()
        _check(self._lib.tcg_alloc_range(self._h, out.value, a))
        self._allocs.append(Range(self.dim, list(a)))
        self._logicals.append(Range(self.dim, logical.lohi))
        return out.value

    def alloc_range(self, ds: int) -> Range:
        return self._allocs[ds]

    def logical_range(self, ds: int) -> Range:
        return self._logicals[ds]

    # ---- lazy queue -----------------------------------------------------
    def par_loop(self, kernel: KernelHandle, rng: Range, args: Sequence, reduction: Optional[int] = None) -> int:
        if rng.dim != self.dim:
            raise InvalidArgument("par_loop: range dim does not match block")
        # Encoded ctypes arguments are cached per (range, args): a
        # time-stepping code re-enqueues the same loops every step. Scalar
        # parameters change from step to step (CG's alpha / beta) and are
        # encoded per call.
        key = (tuple(rng.lohi), tuple((a.dataset, a.stencil, int(a.mode)) if isinstance(a, ArgSpec)
                                      else (int(a[0]), int(a[1]), int(a[2])) for a in args))
        enc = self._enc.get(key)
        if enc is None:
            flat = [v for t in key[1] for v in t]
            enc = (_arr(_I64, key[0]), len(key[1]), _arr(_I32, flat))
            if len(self._enc) > 4096:
                self._enc.clear()
            self._enc[key] = enc
        prm = kernel.params
        np_ = len(prm)
        out = self._out
        _check(_par_loop_raw(self._h, int(kernel.id), int(kernel.body), enc[0], enc[1], enc[2],
                             -1 if reduction is None else int(reduction), np_,
                             (_D * np_)(*prm) if np_ else None, self._out_ref))
        return out.value

    def flush(self, mode: Optional[ExecMode] = None) -> dict:
        if mode is None:
            _check(self._lib.tcg_flush_default(self._h))
        else:
            _check(self._lib.tcg_flush(self._h, mode.kind, _arr(_I64, mode.tile_sizes)))
        return LazyReport(self.report_text())

    def set_default_mode(self, mode: ExecMode) -> None:
        _check(self._lib.tcg_set_default_mode(self._h, mode.kind, _arr(_I64, mode.tile_sizes)))

    def fetch_reduction(self, handle: int) -> float:
        out = _D()
        _check(self._lib.tcg_fetch_reduction(self._h, handle, ctypes.byref(out)))
        return out.value

    def pending_loops(self) -> int:
        out = _I64()
        _check(self._lib.tcg_pending_loops(self._h, ctypes.byref(out)))
        return out.value

    # ---- host access --------------------------------------------------------
    def get(self, ds: int, p: Sequence[int]) -> float:
        p = list(p) + [0] * (3 - len(p))
        out = _D()
        _check(self._lib.tcg_get(self._h, ds, _arr(_I64, p[:3]), ctypes.byref(out)))
        return out.value

    def put(self, ds: int, p: Sequence[int], v: float) -> None:
        p = list(p) + [0] * (3 - len(p))
        _check(self._lib.tcg_put(self._h, ds, _arr(_I64, p[:3]), float(v)))

    def fill_logical(self, ds: int, v: float) -> None:
        _check(self._lib.tcg_fill_logical(self._h, ds, float(v)))

    def upload(self, ds: int, data: np.ndarray) -> None:
        a = self._allocs[ds]
        arr = np.ascontiguousarray(data, dtype=np.float64)
        if arr.size != a.volume():
            raise InvalidArgument(f"upload: expected {a.volume()} values for {a}, got {arr.size}")
        _check(self._lib.tcg_upload(self._h, ds, arr.ctypes.data_as(_P)))

    def download(self, ds: int, out: Optional[np.ndarray] = None) -> np.ndarray:
        """Whole allocation, dense (dim 0 fastest). `out` (C-contiguous
        float64 of the allocation's size; pinned memory copies at full
        PCIe/C2C rate) is filled in place and returned."""
        a = self._allocs[ds]
        if out is None:
            out = np.empty(a.shape(), dtype=np.float64)
        elif out.dtype != np.float64 or not out.flags.c_contiguous or out.size != a.volume():
            raise InvalidArgument(f"download: out must be C-contiguous float64 with {a.volume()} values")
        _check(self._lib.tcg_download(self._h, ds, out.ctypes.data_as(_P)))
        return out

    def periodic_fill(self, datasets, depth: int, logical=None) -> None:
        """Periodic ghost layers (depth <= pad) for every listed field, over
        each field's logical box (`logical`, if given, must equal it).
        Recorded in the queue (the chain is rewritten at flush: one wrap per
        chain, loops extended into the ghost layers); set_periodic_flush(True)
        makes it flush and copy at once."""
        ds = list(datasets)
        if logical is not None:
            for d in ds:
                if list(self._logicals[d].lohi[: 2 * self.dim]) != list(logical)[: 2 * self.dim]:
                    raise InvalidArgument("periodic_fill: box differs from the field's logical range")
        _check(self._lib.tcg_periodic_fill(self._h, len(ds), _arr(_I32, ds), depth))

    def periodic_plan_pending(self) -> str:
        """Host-only: the pending chain rewritten around its periodic marks."""
        return _text(self._lib.tcg_periodic_plan_pending, self._h)

    def set_reduction_order(self, workers: int) -> None:
        """Fold Sum reductions in the reference's order for `workers` threads
        (untiled executor, sequential span sums, worker-order fold); 0 = fast."""
        _check(self._lib.tcg_set_reduction_order(self._h, workers))

    # ---- step templates ------------------------------------------------------
    def record_begin(self) -> None:
        """Keep the par_loop / periodic_fill calls made until record_end as a
        template (they are enqueued normally too)."""
        _check(self._lib.tcg_record_begin(self._h))

    def record_end(self) -> int:
        out = _I32(0)
        _check(self._lib.tcg_record_end(self._h, ctypes.byref(out)))
        return out.value

    def replay(self, template: int, params=None):
        """Issue the recorded calls again (C++ host path, one binding crossing);
        `params` replaces the kernels' scalars in call order. Returns the new
        reduction handles."""
        hs = (_I32 * 16)()
        n = _I64(0)
        if params is None:
            _check(self._lib.tcg_replay(self._h, template, None, 0, hs, 16, ctypes.byref(n)))
        else:
            arr = (ctypes.c_double * len(params))(*params)
            _check(self._lib.tcg_replay(self._h, template, arr, len(params), hs, 16, ctypes.byref(n)))
        return [hs[i] for i in range(min(n.value, 16))]

    def set_periodic_domain(self, on: bool = True) -> None:
        """Periodic box on a rank grid: call before set_rank_grid /
        set_process_rank (the ghost layers join the decomposed domain)."""
        _check(self._lib.tcg_set_periodic_domain(self._h, 1 if on else 0))

    def set_periodic_flush(self, flush_each: bool) -> None:
        _check(self._lib.tcg_set_periodic_flush(self._h, 1 if flush_each else 0))

    def upload_box(self, ds: int, data: np.ndarray, box: Range) -> None:
        arr = np.ascontiguousarray(data, dtype=np.float64)
        if arr.size != box.volume():
            raise InvalidArgument(f"upload_box: expected {box.volume()} values for {box}, got {arr.size}")
        _check(self._lib.tcg_upload_box(self._h, ds, arr.ctypes.data_as(_P), _arr(_I64, box.lohi)))

    def download_box(self, ds: int, box: Range, out: Optional[np.ndarray] = None) -> np.ndarray:
        if out is None:
            out = np.empty(box.shape(), dtype=np.float64)
        if not out.flags.c_contiguous or out.size != box.volume() or out.dtype != np.float64:
            raise InvalidArgument("download_box: out must be a C-contiguous float64 array over the box")
        _check(self._lib.tcg_download_box(self._h, ds, out.ctypes.data_as(_P), _arr(_I64, box.lohi)))
        return out

    def local_box(self, ds: int) -> Range:
        """The part of ds's allocation this process holds."""
        a = (_I64 * 6)()
        _check(self._lib.tcg_local_box(self._h, ds, a))
        return Range(self.dim, list(a))

    def synchronize(self) -> None:
        _check(self._lib.tcg_synchronize(self._h))

    # ---- introspection ------------------------------------------------------
    def report_text(self) -> str:
        # Idempotent call: start small (a per-flush 4 MiB buffer costs more
        # host time than a small chain's whole device time) and retry.
        need = _I64(0)
        size = 1 << 14
        while True:
            buf = self._rbuf if size == 1 << 14 else ctypes.create_string_buffer(size)
            _check(self._lib.tcg_report_text(self._h, buf, len(buf), ctypes.byref(need)))
            if need.value <= size:
                return buf.value.decode()
            size = int(need.value) + 1

    def plan_pending(self, tile_sizes) -> str:
        ts = list(tile_sizes) + [0] * (3 - len(tile_sizes))
        return _text(self._lib.tcg_plan_pending, self._h, _arr(_I64, ts[:3]))

    def rank_plans_pending(self, grid, tile_sizes) -> str:
        g = list(grid) + [1] * (3 - len(grid))
        ts = list(tile_sizes) + [0] * (3 - len(tile_sizes))
        return _text(self._lib.tcg_rank_plans_pending, self._h, _arr(_I32, g[:3]), _arr(_I64, ts[:3]))

    def set_stream_choice(self, nt=0, bx=0, by=0, ntx=0, segments=0, max_loops=0, minb=0, prefetch=-1):
        """Streaming executor knobs (0 / -1 = sizer): threads per CTA, points
        per thread along x / y, threads along x (3D), stream segments, loops
        per kernel, min CTAs per SM, L2 prefetch distance in rows."""
        _check(self._lib.tcg_set_stream_choice(self._h, _arr(_I32, [nt, bx, by, ntx, segments, max_loops, minb,
                                                                    prefetch])))

    def stream_plan_pending(self, compile: bool = False, source: bool = False, size: int = 1 << 26, ctas: bool = False) -> str:
        """Streaming plan of the pending chain (consumed): summary lines, plus
        the NVRTC compile log (compile=True; no GPU needed) and the generated
        sources (source=True)."""
        return _text(self._lib.tcg_stream_plan_pending, self._h, (1 if compile else 0) | (2 if source else 0) | (4 if ctas else 0),
                     size=size)

    def gpu_plan_pending(self, mode: ExecMode, size: int = 1 << 26) -> str:
        return _text(self._lib.tcg_gpu_plan_pending, self._h, mode.kind, _arr(_I64, mode.tile_sizes), size=size)

    # ---- distribution ----------------------------------------
    def set_rank_grid(self, grid):
        """Runtime::set_rank_grid (runtime.hpp:77-81): every rank hosted in this
        process on this GPU (the reference's simulated ranks)."""
        g = list(grid) + [1] * (3 - len(grid))
        _check(self._lib.tcg_set_rank_grid(self._h, _arr(_I32, g[:3])))

    def set_process_rank(self, grid, rank: int, comm_id: bytes):
        """One rank per process; comm_id from comm_unique_id() on rank 0."""
        g = list(grid) + [1] * (3 - len(grid))
        if len(comm_id) != 128:
            raise InvalidArgument("set_process_rank: comm_id must be 128 bytes")
        _check(self._lib.tcg_set_process_rank(self._h, _arr(_I32, g[:3]), rank, comm_id))

    def rank_owned(self, rank: int) -> Range:
        """Owned box of `rank` in the rank grid's decomposition (decompose,
        dist.cpp:142-177) of the declared fields' hull."""
        a = (_I64 * 6)()
        _check(self._lib.tcg_rank_owned(self._h, rank, a))
        return Range(self.dim, list(a))

    def schedule_pending(self) -> dict:
        """Host-only distribution schedule of the pending chain (consumed; its
        writes are recorded as if executed): per-rank loop ranges and the
        halo message list in exchange order."""
        return parse_schedule(_text(self._lib.tcg_dist_schedule_pending, self._h), self.dim)

    def signature_pending(self) -> int:
        out = ctypes.c_uint64()
        _check(self._lib.tcg_signature_pending(self._h, ctypes.byref(out)))
        return out.value

    def launches(self) -> int:
        out = _I64()
        _check(self._lib.tcg_launches(self._h, ctypes.byref(out)))
        return out.value

    def stream(self) -> int:
        out = _P()
        _check(self._lib.tcg_stream(self._h, ctypes.byref(out)))
        return out.value or 0

    def set_timing(self, on: bool = True) -> None:
        _check(self._lib.tcg_set_timing(self._h, int(on)))

    def kernel_timing(self) -> dict:
        """Device ms and launch counts of k_tiled / k_untiled since the last call."""
        tm, tn, um, un = _D(), _I64(), _D(), _I64()
        _check(self._lib.tcg_kernel_timing(self._h, ctypes.byref(tm), ctypes.byref(tn), ctypes.byref(um),
                                           ctypes.byref(un)))
        return {"tiled_ms": tm.value, "tiled_launches": tn.value, "untiled_ms": um.value,
                "untiled_launches": un.value}


def auto_tile_size(dim, cache_bytes, threads, bytes_per_point, extent: Range):
    lib = load_library()
    out = (_I64 * 3)()
    _check(lib.tcg_auto_tile_size(dim, cache_bytes, threads, bytes_per_point, _arr(_I64, extent.lohi), out))
    return tuple(out)


def device_info() -> dict:
    lib = load_library()
    name = ctypes.create_string_buffer(256)
    sms, smem, l2 = _I32(), _I64(), _I64()
    _check(lib.tcg_device_info(name, 256, ctypes.byref(sms), ctypes.byref(smem), ctypes.byref(l2)))
    return {"name": name.value.decode(), "num_sms": sms.value, "smem_optin": smem.value, "l2_bytes": l2.value}


def select_device(device: int) -> None:
    """cudaSetDevice inside libtcg (its CUDA runtime is not torch's)."""
    _check(load_library().tcg_select_device(device))


def body_known(body: int) -> bool:
    return bool(load_library().tcg_body_known(body))

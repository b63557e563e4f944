"""Workloads: the reference's bundled apps and the five BASELINE.json configs.

Each builder takes any object with the Runtime interface (declare_stencil,
declare_field, alloc_range, par_loop, flush, fetch_reduction, upload,
download, set_default_mode), so the same chain runs on the B200 executor,
on the reference library (oracle/_ref) and on the sequential oracle.

Inputs are seeded synthetic fp64 arrays (numpy PCG64; BASELINE.json names a
seed but no generator) generated once on the host and uploaded identically to
every backend. Exact loop/argument/expression choices for configs whose
BASELINE text leaves freedom are pinned in DESIGN.md §5.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import kernels as K
from .runtime import AccessMode, ArgSpec, ExecMode, KernelHandle, Range, ReduceOp

R, W, RW, INC = AccessMode.Read, AccessMode.Write, AccessMode.ReadWrite, AccessMode.Increment


def uniform(seed: int, shape, lo: float, hi: float) -> np.ndarray:
    g = np.random.Generator(np.random.PCG64(seed))
    return lo + (hi - lo) * g.random(shape)


def uniform_box(seed: int, alloc: Range, box: Range, lo: float, hi: float) -> np.ndarray:
    """The `box` part of uniform(seed, alloc.shape(), lo, hi) without drawing
    the rest: the stream is in dim-0-fastest order over `alloc`, so whole
    rows/planes of it are contiguous; the generator jumps to the box start
    (one draw per double)."""
    if box == alloc:
        return uniform(seed, alloc.shape(), lo, hi)
    dim = alloc.dim
    for d in range(dim - 1):
        if box.start(d) != alloc.start(d) or box.end(d) != alloc.end(d):
            raise ValueError("uniform_box: box must span the allocation in all but the slowest dimension")
    s = dim - 1
    row = 1
    for d in range(s):
        row *= alloc.extent(d)
    g = np.random.Generator(np.random.PCG64(seed))
    g.bit_generator.advance((box.start(s) - alloc.start(s)) * row)
    return lo + (hi - lo) * g.random(box.shape())


def _upload_init(rt, ds, arr, box, alloc):
    if box == alloc:
        rt.upload(ds, arr)
    else:
        rt.upload_box(ds, arr, box)


def _interior_mask(alloc: Range, box: Range) -> tuple:
    """numpy slices of `box` inside a dense array over `alloc` (dim 0 fastest)."""
    sl = []
    for d in reversed(range(alloc.dim)):
        sl.append(slice(box.start(d) - alloc.start(d), box.end(d) - alloc.start(d)))
    return tuple(sl)


def loops_cell_updates(rng_list) -> int:
    return sum(r.volume() for r in rng_list)


# ---------------------------------------------------------------------------
# Reference apps (proj/core/src/apps.cpp) -- regression chains.

class Jacobi2D:
    """apps.cpp:43-106: 5-point damped average, ring 0 / interior 1."""

    def __init__(self, rt, nx=64, ny=64):
        self.rt, self.nx, self.ny = rt, nx, ny
        self.five = rt.declare_stencil("five", [(0, 0), (1, 0), (-1, 0), (0, 1), (0, -1)])
        self.ident = rt.declare_stencil("identity", [(0, 0)])
        dom = Range.d2(0, nx, 0, ny)
        self.a = rt.declare_field("a", dom)
        self.b = rt.declare_field("b", dom)
        for ds in (self.a, self.b):
            al = rt.alloc_range(ds)
            arr = np.zeros(al.shape())
            arr[_interior_mask(al, Range.d2(1, nx - 1, 1, ny - 1))] = 1.0
            rt.upload(ds, arr)

    def enqueue(self, iters: int, copy: bool):
        inner = Range.d2(1, self.nx - 1, 1, self.ny - 1)
        rt = self.rt
        for it in range(iters):
            if copy:
                rt.par_loop(KernelHandle(0, "jacobi_stencil", K.JACOBI_STENCIL), inner,
                            [ArgSpec(self.a, self.five, R), ArgSpec(self.b, self.ident, W)])
                rt.par_loop(KernelHandle(1, "jacobi_copy", K.JACOBI_COPY), inner,
                            [ArgSpec(self.b, self.ident, R), ArgSpec(self.a, self.ident, W)])
            else:
                src, dst = (self.a, self.b) if it % 2 == 0 else (self.b, self.a)
                rt.par_loop(KernelHandle(0, "jacobi_stencil", K.JACOBI_STENCIL), inner,
                            [ArgSpec(src, self.five, R), ArgSpec(dst, self.ident, W)])

    def logical(self, ds):
        al = self.rt.alloc_range(ds)
        return self.rt.download(ds)[_interior_mask(al, Range.d2(0, self.nx, 0, self.ny))]


class MiniHydro:
    """apps.cpp:108-279: 12-loop hydro-like chain with a closing sum monitor."""

    def __init__(self, rt, nx=48, ny=48):
        self.rt, self.nx, self.ny = rt, nx, ny
        S = rt.declare_stencil
        self.identity = S("identity", [(0, 0)])
        self.right = S("right", [(1, 0)])
        self.up = S("up", [(0, 1)])
        self.left_pair = S("left_pair", [(-1, 0), (0, 0)])
        self.down_pair = S("down_pair", [(0, -1), (0, 0)])
        self.right_pair = S("right_pair", [(0, 0), (1, 0)])
        self.up_pair = S("up_pair", [(0, 0), (0, 1)])
        self.five = S("five", [(0, 0), (1, 0), (-1, 0), (0, 1), (0, -1)])
        dom = Range.d2(0, nx, 0, ny)
        names = ["rho", "e", "p", "u", "v", "fx", "fy", "w"]
        self.ds = {n: rt.declare_field(n, dom) for n in names}
        y, x = np.mgrid[0:ny, 0:nx]
        for n in names:
            al = rt.alloc_range(self.ds[n])
            arr = np.zeros(al.shape())
            if n == "rho":
                arr[_interior_mask(al, dom)] = 1.0 + 0.25 * ((x + 2 * y) % 4)
            if n == "e":
                arr[_interior_mask(al, dom)] = 2.0 + 0.125 * ((3 * x + y) % 8)
            rt.upload(self.ds[n], arr)

    def enqueue_iteration(self) -> int:
        rt, d, nx, ny = self.rt, self.ds, self.nx, self.ny
        full = Range.d2(0, nx, 0, ny)
        inner = Range.d2(1, nx - 1, 1, ny - 1)
        col0, row0 = Range.d2(0, 1, 0, ny), Range.d2(0, nx, 0, 1)
        xpair, ypair = Range.d2(0, nx - 1, 0, ny), Range.d2(0, nx, 0, ny - 1)
        i = self.identity
        P = rt.par_loop
        P(KernelHandle(10, "eos", K.MH_EOS), full, [ArgSpec(d["rho"], i, R), ArgSpec(d["e"], i, R), ArgSpec(d["p"], i, W)])
        P(KernelHandle(11, "bc_x", K.MH_BC_X), col0, [ArgSpec(d["p"], self.right, R), ArgSpec(d["p"], i, W)])
        P(KernelHandle(12, "bc_y", K.MH_BC_Y), row0, [ArgSpec(d["p"], self.up, R), ArgSpec(d["p"], i, W)])
        P(KernelHandle(13, "accel_x", K.MH_ACCEL_X), xpair, [ArgSpec(d["p"], self.right_pair, R), ArgSpec(d["u"], i, INC)])
        P(KernelHandle(14, "accel_y", K.MH_ACCEL_Y), ypair, [ArgSpec(d["p"], self.up_pair, R), ArgSpec(d["v"], i, INC)])
        P(KernelHandle(15, "flux_x", K.MH_FLUX_X), xpair,
          [ArgSpec(d["u"], self.right_pair, R), ArgSpec(d["rho"], self.right_pair, R), ArgSpec(d["fx"], i, W)])
        P(KernelHandle(16, "flux_y", K.MH_FLUX_Y), ypair,
          [ArgSpec(d["v"], self.up_pair, R), ArgSpec(d["rho"], self.up_pair, R), ArgSpec(d["fy"], i, W)])
        P(KernelHandle(17, "advect_rho", K.MH_ADVECT_RHO), inner,
          [ArgSpec(d["fx"], self.left_pair, R), ArgSpec(d["fy"], self.down_pair, R), ArgSpec(d["rho"], i, INC)])
        P(KernelHandle(18, "advect_e", K.MH_ADVECT_E), inner,
          [ArgSpec(d["fx"], self.left_pair, R), ArgSpec(d["fy"], self.down_pair, R), ArgSpec(d["e"], i, INC)])
        P(KernelHandle(19, "smooth", K.MH_SMOOTH), inner, [ArgSpec(d["rho"], self.five, R), ArgSpec(d["w"], i, W)])
        P(KernelHandle(20, "blend", K.MH_BLEND), inner, [ArgSpec(d["rho"], i, RW), ArgSpec(d["w"], i, R)])
        return P(KernelHandle(21, "monitor", K.MH_MONITOR), full, [ArgSpec(d["e"], i, R)], ReduceOp.Sum)

    def run(self, iters: int) -> List[float]:
        return [self.rt.fetch_reduction(self.enqueue_iteration()) for _ in range(iters)]

    def logical(self, name):
        al = self.rt.alloc_range(self.ds[name])
        return self.rt.download(self.ds[name])[_interior_mask(al, Range.d2(0, self.nx, 0, self.ny))]


# ---------------------------------------------------------------------------
# BASELINE config c1: 2D heat chain.

class HeatC1:
    """fp64 n x n, u interior U[0,1) seed 42, v = 0, Dirichlet 0 (untouched padding).
    Timestep = [v = u + 0.1 lap(u); u = v], 10 timesteps (20 loops) per chain."""

    name = "c1_heat2d"

    def __init__(self, rt, n=1024, seed=42):
        self.rt, self.n = rt, n
        self.five = rt.declare_stencil("five", [(0, 0), (1, 0), (-1, 0), (0, 1), (0, -1)])
        self.ident = rt.declare_stencil("identity", [(0, 0)])
        dom = Range.d2(0, n, 0, n)
        self.dom = dom
        self.u = rt.declare_field("u", dom)
        self.v = rt.declare_field("v", dom)
        al = rt.alloc_range(self.u)
        arr = np.zeros(al.shape())
        arr[_interior_mask(al, dom)] = uniform(seed, (n, n), 0.0, 1.0)
        self.init = {self.u: arr, self.v: np.zeros(al.shape())}
        for ds, a in self.init.items():
            rt.upload(ds, a)

    def enqueue_chain(self, steps=10):
        for _ in range(steps):
            self.rt.par_loop(KernelHandle(K.HEAT_LAP, "heat_lap", K.HEAT_LAP), self.dom,
                             [ArgSpec(self.u, self.five, R), ArgSpec(self.v, self.ident, W)])
            self.rt.par_loop(KernelHandle(K.HEAT_COPY, "heat_copy", K.HEAT_COPY), self.dom,
                             [ArgSpec(self.v, self.ident, R), ArgSpec(self.u, self.ident, W)])

    def cell_updates_per_chain(self, steps=10):
        return 2 * steps * self.n * self.n

    def bytes_per_chain(self, steps=10):
        return 2 * steps * self.n * self.n * 16

    def outputs(self):
        return {"u": self.rt.download(self.u)}


# ---------------------------------------------------------------------------
# BASELINE config c2: 2D hydro-like multi-loop chain.

STENCILS_2D = {
    0: [(0, 0)],
    1: [(0, 0), (1, 0), (-1, 0), (0, 1), (0, -1)],
    2: [(-1, -1), (0, -1), (1, -1), (-1, 0), (0, 0), (1, 0), (-1, 1), (0, 1), (1, 1)],
    3: [(0, 0), (1, 0), (0, 1)],
    4: [(0, 0), (1, 0), (-1, 0), (2, 0), (-2, 0), (0, 1), (0, -1), (0, 2), (0, -2)],
}


class HydroC2:
    """8 dats U[0.5,1.5) seed 7 over the whole allocation; 12 loops per step:
    loop k writes dat k%8 from r1=(k+1)%8 through stencil kind k%5, r2=(k+3)%8
    (point) and, when k%3 == 0, r3=(k+5)%8 (point); then a min-reduction of
    0.5/(d0 + d4*d5) ends the step (13 loops, one chain per step)."""

    name = "c2_hydro2d"

    def __init__(self, rt, n=4096, seed=7, ny=None):
        # ny > n: the weak-scaling domain n x (n * ranks), one n x n slab per
        # rank; every rank draws only the rows it holds (uniform_box).
        self.rt, self.n, self.ny = rt, n, ny or n
        self.st = {k: rt.declare_stencil(f"s{k}", pts) for k, pts in STENCILS_2D.items()}
        self.ident = self.st[0]
        self.dom = Range.d2(0, n, 0, self.ny)
        self.d = [rt.declare_field(f"d{i}", self.dom) for i in range(8)]
        al = rt.alloc_range(self.d[0])
        self.init, self.init_box = {}, {}
        for i, ds in enumerate(self.d):
            box = rt.local_box(ds) if hasattr(rt, "local_box") else al
            self.init[ds] = uniform_box(seed * 1000 + i, al, box, 0.5, 1.5)
            self.init_box[ds] = box
            _upload_init(rt, ds, self.init[ds], box, al)

    def loop_specs(self):
        if getattr(self, "_specs", None) is not None:
            return self._specs
        specs = []
        for k in range(12):
            kind = k % 5
            r3 = k % 3 == 0
            args = [ArgSpec(self.d[(k + 1) % 8], self.st[kind], R), ArgSpec(self.d[(k + 3) % 8], self.ident, R)]
            if r3:
                args.append(ArgSpec(self.d[(k + 5) % 8], self.ident, R))
            args.append(ArgSpec(self.d[k % 8], self.ident, W))
            specs.append((KernelHandle(200 + k, f"hydro{k}", K.hydro_body(kind, r3)), args))
        self._specs = specs
        return specs

    def enqueue_step(self) -> int:
        for kh, args in self.loop_specs():
            self.rt.par_loop(kh, self.dom, args)
        return self.rt.par_loop(KernelHandle(K.HYDRO_CFL, "cfl", K.HYDRO_CFL), self.dom,
                                [ArgSpec(self.d[0], self.ident, R), ArgSpec(self.d[4], self.ident, R),
                                 ArgSpec(self.d[5], self.ident, R)], ReduceOp.Min)

    def cell_updates_per_step(self):
        return 13 * self.n * self.ny

    def bytes_per_step(self):
        per_pt = 0
        for _, args in self.loop_specs():
            per_pt += 8 * len(args)
        per_pt += 3 * 8
        return per_pt * self.n * self.ny

    def outputs(self):
        return {f"d{i}": self.rt.download(ds) for i, ds in enumerate(self.d)}


# ---------------------------------------------------------------------------
# BASELINE config c3: 3D 7-point Jacobi.

class Jacobi3DC3:
    """a interior U[0,1) seed 3, zero boundary; loops over [1,n-1)^3,
    a->b then b->a; 16-loop chains (8 sweeps)."""

    name = "c3_jacobi3d"

    def __init__(self, rt, n=512, seed=3):
        self.rt, self.n = rt, n
        self.star = rt.declare_stencil("star7", [(0, 0, 0), (1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0),
                                                 (0, 0, 1), (0, 0, -1)])
        self.ident = rt.declare_stencil("identity", [(0, 0, 0)])
        dom = Range.d3(0, n, 0, n, 0, n)
        self.a = rt.declare_field("a", dom)
        self.b = rt.declare_field("b", dom)
        al = rt.alloc_range(self.a)
        arr = np.zeros(al.shape())
        arr[_interior_mask(al, Range.d3(1, n - 1, 1, n - 1, 1, n - 1))] = uniform(seed, (n - 2,) * 3, 0.0, 1.0)
        self.init = {self.a: arr, self.b: np.zeros(al.shape())}
        for ds, x in self.init.items():
            rt.upload(ds, x)
        self.inner = Range.d3(1, n - 1, 1, n - 1, 1, n - 1)

    def enqueue_chain(self, sweeps=8):
        for _ in range(sweeps):
            self.rt.par_loop(KernelHandle(K.JACOBI_3D, "jac3d", K.JACOBI_3D), self.inner,
                             [ArgSpec(self.a, self.star, R), ArgSpec(self.b, self.ident, W)])
            self.rt.par_loop(KernelHandle(K.JACOBI_3D, "jac3d", K.JACOBI_3D), self.inner,
                             [ArgSpec(self.b, self.star, R), ArgSpec(self.a, self.ident, W)])

    def cell_updates_per_chain(self, sweeps=8):
        return 2 * sweeps * self.inner.volume()

    def bytes_per_chain(self, sweeps=8):
        return 2 * sweeps * self.inner.volume() * 16

    def outputs(self):
        return {"a": self.rt.download(self.a), "b": self.rt.download(self.b)}


# ---------------------------------------------------------------------------
# BASELINE config c4: conjugate gradient on a variable-coefficient operator.

class CgC4:
    """A p = (1 + kx + kx_w + ky + ky_s) p - kx p_e - kx_w p_w - ky p_n - ky_s p_s,
    K = 1 + U[0,1) seed 11 (whole allocation), rhs U[-1,1) seed 12; x0 = 0,
    r0 = b. Iteration = chains [p-update, matvec + p.q] and
    [x-update, r-update + r.r], each closed by a fetch_reduction."""

    name = "c4_cg2d"

    def __init__(self, rt, n=4096):
        self.rt, self.n = rt, n
        self.star = rt.declare_stencil("five", [(0, 0), (1, 0), (-1, 0), (0, 1), (0, -1)])
        self.ident = rt.declare_stencil("identity", [(0, 0)])
        self.west = rt.declare_stencil("west_pair", [(0, 0), (-1, 0)])
        self.south = rt.declare_stencil("south_pair", [(0, 0), (0, -1)])
        self.dom = Range.d2(0, n, 0, n)
        names = ["x", "r", "p", "q", "kx", "ky"]
        self.f = {nm: rt.declare_field(nm, self.dom) for nm in names}
        al = rt.alloc_range(self.f["x"])
        self.init = {}
        for nm in names:
            arr = np.zeros(al.shape())
            if nm == "kx":
                arr = 1.0 + uniform(11, al.shape(), 0.0, 1.0)
            elif nm == "ky":
                arr = 1.0 + uniform(11 * 7919, al.shape(), 0.0, 1.0)
            elif nm == "r":
                arr[_interior_mask(al, self.dom)] = uniform(12, (n, n), -1.0, 1.0)
            self.init[self.f[nm]] = arr
            rt.upload(self.f[nm], arr)
        self.rr = None
        self.beta = 0.0
        self.history: List[float] = []

    def start(self):
        h = self.rt.par_loop(KernelHandle(K.CG_DOT, "dot", K.CG_DOT), self.dom, [ArgSpec(self.f["r"], self.ident, R)],
                             ReduceOp.Sum)
        self.rr = self.rt.fetch_reduction(h)
        self.history = [math.sqrt(self.rr)]
        self.beta = 0.0

    def enqueue_pq(self):
        """p = r + beta p; q = A p with Sum p.q (first chain of an iteration)."""
        f, rt, dom, I = self.f, self.rt, self.dom, self.ident
        rt.par_loop(KernelHandle(K.CG_P_UPDATE, "p_update", K.CG_P_UPDATE, (self.beta,)), dom,
                    [ArgSpec(f["p"], I, RW), ArgSpec(f["r"], I, R)])
        return rt.par_loop(KernelHandle(K.CG_MATVEC, "matvec", K.CG_MATVEC), dom,
                           [ArgSpec(f["p"], self.star, R), ArgSpec(f["kx"], self.west, R), ArgSpec(f["ky"], self.south, R),
                            ArgSpec(f["q"], I, W)], ReduceOp.Sum)

    def enqueue_update(self, alpha):
        """x += alpha p; r -= alpha q with Sum r.r (second chain)."""
        f, rt, dom, I = self.f, self.rt, self.dom, self.ident
        rt.par_loop(KernelHandle(K.CG_X_UPDATE, "x_update", K.CG_X_UPDATE, (alpha,)), dom,
                    [ArgSpec(f["x"], I, RW), ArgSpec(f["p"], I, R)])
        return rt.par_loop(KernelHandle(K.CG_R_UPDATE, "r_update", K.CG_R_UPDATE, (alpha,)), dom,
                           [ArgSpec(f["r"], I, RW), ArgSpec(f["q"], I, R)], ReduceOp.Sum)

    def finish_iteration(self, rr_new):
        self.beta = rr_new / self.rr
        self.rr = rr_new
        self.history.append(math.sqrt(max(rr_new, 0.0)))

    def iterate(self):
        pq = self.rt.fetch_reduction(self.enqueue_pq())
        alpha = self.rr / pq
        self.finish_iteration(self.rt.fetch_reduction(self.enqueue_update(alpha)))

    def cell_updates_per_iteration(self):
        return 4 * self.n * self.n

    def bytes_per_iteration(self):
        # p-update RW+R (24), matvec 4 args (32), x-update (24), r-update (24)
        return (24 + 32 + 24 + 24) * self.n * self.n

    def outputs(self):
        return {nm: self.rt.download(ds) for nm, ds in self.f.items() if nm in ("x", "r", "p")}


CONFIGS = {c.name: c for c in (HeatC1, HydroC2, Jacobi3DC3, CgC4)}


# ---------------------------------------------------------------------------
# BASELINE config c5: 3D compressible Navier-Stokes-like Taylor-Green vortex.

class NsC5:
    """Periodic 2*pi box, n^3 points x_i = i*h; rho = 1, u = sin x cos y cos z,
    v = -cos x sin y cos z, w = 0, p = 100/1.4 + (cos 2x + cos 2y)(cos 2z + 2)/16;
    4th-order central differences (radius-2 star per axis), Re = 1600,
    Pr = 0.71, low-storage RK3 (Williamson). Per step 3 stages x [prim,
    periodic ghost fill, 5 RHS loops, update] + a kinetic-energy Sum = 22
    loops (csrc/kernels/tc_ns.h). Initial values are computed on the host
    (numpy sin/cos) and uploaded identically to every executor and the
    oracle; the bench uploads them slab by slab."""

    name = "c5_ns3d"
    GAMMA = 1.4
    RK_A = (0.0, -5.0 / 9.0, -153.0 / 128.0)
    RK_B = (1.0 / 3.0, 15.0 / 16.0, 8.0 / 15.0)

    def __init__(self, rt, n=768, re=1600.0, pr=0.71, cfl=0.3, slab=16):
        self.rt, self.n = rt, n
        g = self.GAMMA
        self.h = 2.0 * math.pi / n
        self.inv12h = 1.0 / (12.0 * self.h)
        self.inv12h2 = 1.0 / (12.0 * self.h * self.h)
        self.mu = 1.0 / re
        self.kappa = self.mu * g / ((g - 1.0) * pr)
        self.p0 = 100.0 / g
        self.dt = cfl * self.h / (1.0 + math.sqrt(g * self.p0))
        pts = [(0, 0, 0)]
        for d in range(3):
            for k in (-2, -1, 1, 2):
                p = [0, 0, 0]
                p[d] = k
                pts.append(tuple(p))
        self.star = rt.declare_stencil("star2_3d", pts)
        self.pt = rt.declare_stencil("point", [(0, 0, 0)])
        self.dom = Range.d3(0, n, 0, n, 0, n)
        names = ["rho", "mx", "my", "mz", "E", "d_rho", "d_mx", "d_my", "d_mz", "d_E", "u", "v", "w", "p", "T"]
        self.f = {nm: rt.declare_field(nm, self.dom) for nm in names}
        al = rt.alloc_range(self.f["rho"])
        box = rt.local_box(self.f["rho"]) if hasattr(rt, "local_box") else al
        # Host initial condition, slab by slab along z (a full 768^3 field is
        # 4.2 GB; the bench never holds all five at once).
        whole = box == al and al.volume() * 8 * 5 < (1 << 31)
        z0, z1 = box.start(2), box.end(2)
        for zs in range(z0, z1, (z1 - z0) if whole else slab):
            ze = min(z1, zs + ((z1 - z0) if whole else slab))
            sb = Range.d3(box.start(0), box.end(0), box.start(1), box.end(1), zs, ze)
            vals = self._initial(sb)
            for nm, arr in vals.items():
                if whole:
                    rt.upload(self.f[nm], arr)
                else:
                    rt.upload_box(self.f[nm], arr, sb)
        self.logical = list(self.dom.lohi)

    def _initial(self, sb):
        """Conserved fields over box sb (zero outside the logical box)."""
        n, h, g = self.n, self.h, self.GAMMA
        zi = np.arange(sb.start(2), sb.end(2))
        yi = np.arange(sb.start(1), sb.end(1))
        xi = np.arange(sb.start(0), sb.end(0))
        Z, Y, X = np.meshgrid(zi, yi, xi, indexing="ij")
        inside = (X >= 0) & (X < n) & (Y >= 0) & (Y < n) & (Z >= 0) & (Z < n)
        x, y, z = X * h, Y * h, Z * h
        u = np.sin(x) * np.cos(y) * np.cos(z)
        v = -np.cos(x) * np.sin(y) * np.cos(z)
        w = np.zeros_like(u)
        rho = np.ones_like(u)
        p = self.p0 + (np.cos(2.0 * x) + np.cos(2.0 * y)) * (np.cos(2.0 * z) + 2.0) / 16.0
        E = p / (g - 1.0) + 0.5 * rho * ((u * u + v * v) + w * w)
        out = {"rho": rho, "mx": rho * u, "my": rho * v, "mz": rho * w, "E": E}
        for k in out:
            out[k] = np.where(inside, out[k], 0.0)
        return out

    def enqueue_step(self) -> int:
        rt, f, S, P, dom = self.rt, self.f, self.star, self.pt, self.dom
        U = [f["rho"], f["mx"], f["my"], f["mz"], f["E"]]
        dU = [f["d_rho"], f["d_mx"], f["d_my"], f["d_mz"], f["d_E"]]
        vel = [f["u"], f["v"], f["w"]]
        for s in range(3):
            a, b = self.RK_A[s], self.RK_B[s]
            rt.par_loop(KernelHandle(K.NS_PRIM, "ns_prim", K.NS_PRIM, (self.GAMMA - 1.0,)), dom,
                        [ArgSpec(x, P, R) for x in U] + [ArgSpec(f[nm], P, W) for nm in ("u", "v", "w", "p", "T")])
            rt.periodic_fill([f["mx"], f["my"], f["mz"], f["E"]] + vel + [f["p"], f["T"]], 2, self.logical)
            rt.par_loop(KernelHandle(K.NS_RHS_MASS, "ns_mass", K.NS_RHS_MASS, (self.inv12h, a, self.dt)), dom,
                        [ArgSpec(U[1], S, R), ArgSpec(U[2], S, R), ArgSpec(U[3], S, R), ArgSpec(dU[0], P, RW)])
            for c in range(3):
                rt.par_loop(KernelHandle(K.NS_RHS_MOM + c, f"ns_mom{c}", K.NS_RHS_MOM + c,
                                         (self.inv12h, self.inv12h2, self.mu, a, self.dt)), dom,
                            [ArgSpec(U[1 + c], S, R)] + [ArgSpec(x, S, R) for x in vel] +
                            [ArgSpec(f["p"], S, R), ArgSpec(dU[1 + c], P, RW)])
            rt.par_loop(KernelHandle(K.NS_RHS_ENERGY, "ns_energy", K.NS_RHS_ENERGY,
                                     (self.inv12h, self.inv12h2, self.mu, self.kappa, a, self.dt)), dom,
                        [ArgSpec(U[4], S, R), ArgSpec(f["p"], S, R)] + [ArgSpec(x, S, R) for x in vel] +
                        [ArgSpec(f["T"], S, R), ArgSpec(dU[4], P, RW)])
            rt.par_loop(KernelHandle(K.NS_UPDATE, "ns_update", K.NS_UPDATE, (b,)), dom,
                        [ArgSpec(x, P, RW) for x in U] + [ArgSpec(x, P, R) for x in dU])
        return rt.par_loop(KernelHandle(K.NS_KINETIC, "ns_kinetic", K.NS_KINETIC), dom,
                           [ArgSpec(x, P, R) for x in U[:4]], ReduceOp.Sum)

    def cell_updates_per_step(self):
        return 22 * self.n ** 3

    def bytes_per_step(self):
        # estimate_bytes_moved per loop (loop.cpp:50-61): 8 B per arg, x2 for RW.
        per = 3 * ((5 + 5) + (3 + 2) + 3 * (5 + 2) + (6 + 2) + (10 + 5)) + 4
        return 8 * per * self.n ** 3

    def outputs(self):
        """Conserved fields over the logical box (the ghost layers of a
        periodic box are only defined right after a fill)."""
        out = {}
        for nm in ("rho", "mx", "my", "mz", "E"):
            al = self.rt.alloc_range(self.f[nm])
            a = self.rt.download(self.f[nm])
            sl = tuple(slice(self.dom.start(d) - al.start(d), self.dom.end(d) - al.start(d)) for d in (2, 1, 0))
            out[nm] = np.ascontiguousarray(a[sl])
        return out

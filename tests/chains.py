"""Reproducible random loop chains with the structure of the reference's
property-test generator (proj/tests/support/chain_gen.cpp:32-113):
stencil 0 is the identity; 1-5 point stencils of radius <= max_radius; each
loop writes one dataset (70% Write / 20% ReadWrite / 10% Increment, chain_gen
:67-70) and reads 1-3 other datasets; thin 1-wide loops with p = 1/5 (:97);
reductions with p = 1/4 (:104-109); dyadic initial values (:130-133); body =
GEN_SUM (sum of every declared read, scaled to stay contracting, :168-196).
The random stream is numpy's, not mt19937_64: chains are regenerated, not
copied, so seeds do not correspond to the reference's."""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Tuple

import numpy as np

from paper_1704_00693_b200 import ExecMode, KernelHandle, Range, kernels

TILE_CHOICES = [1, 2, 3, 4, 5, 6, 8, 12, 16, 24, 32, 64]


@dataclass
class GenChain:
    dim: int
    extent: List[int]
    ndat: int
    stencils: List[List[Tuple[int, int, int]]]
    loops: List[tuple] = field(default_factory=list)  # (lohi, args[(ds, st, mode)], red or None)


def generate(seed: int, dim: int = 2, min_loops=2, max_loops=10, extent=(24, 48), max_radius=2, ndat=(3, 5),
             reductions=True, thin=True, reads_within_logical=False) -> GenChain:
    g = np.random.Generator(np.random.PCG64(seed))
    ri = lambda lo, hi: int(g.integers(lo, hi + 1))
    ext = [ri(*extent) for _ in range(dim)]
    nd = ri(*ndat)
    sts = [[(0, 0, 0)]]
    for _ in range(ri(3, 6)):
        pts = set()
        for _ in range(ri(1, 5)):
            p = [0, 0, 0]
            for d in range(dim):
                p[d] = ri(-max_radius, max_radius)
            pts.add(tuple(p))
        sts.append(sorted(pts))
    gc = GenChain(dim, ext, nd, sts)
    for _ in range(ri(min_loops, max_loops)):
        w = ri(0, nd - 1)
        roll = ri(0, 9)
        wmode = 1 if roll < 7 else (2 if roll < 9 else 3)
        args = []
        for _ in range(ri(1, 3)):
            ds = ri(0, nd - 1)
            if ds == w:
                ds = (ds + 1) % nd
            args.append((ds, ri(0, len(sts) - 1), 0))
        args.append((w, 0, wmode))
        mn = [0, 0, 0]
        mx = [0, 0, 0]
        for ds, st, m in args:
            if m != 0:
                continue
            for p in sts[st]:
                for d in range(3):
                    mn[d] = min(mn[d], p[d])
                    mx[d] = max(mx[d], p[d])
        lohi = []
        for d in range(dim):
            lo, hi = 0, ext[d]
            if reads_within_logical:
                lo, hi = -mn[d], ext[d] - mx[d]
            if hi - lo < 1:
                lo = min(max(lo, 0), ext[d] - 1)
                hi = lo + 1
            width = 1 if (thin and ri(0, 4) == 0) else ri(1 + (hi - lo) // 2, hi - lo)
            start = ri(lo, hi - width)
            lohi += [start, start + width]
        red = None
        if reductions and ri(0, 3) == 0:
            red = ri(0, 2)
        gc.loops.append((lohi, args, red))
    return gc


def random_tile_sizes(seed: int, dim: int):
    g = np.random.Generator(np.random.PCG64(seed * 7919 + 1))
    ts = [1, 1, 1]
    for d in range(dim):
        ts[d] = TILE_CHOICES[int(g.integers(0, len(TILE_CHOICES)))]
    return ts


def declare(rt, gc: GenChain):
    for i, pts in enumerate(gc.stencils):
        rt.declare_stencil(f"s{i}", [p[: gc.dim] for p in pts])
    dom = Range(gc.dim, sum(([0, e] for e in gc.extent), []))
    ids = [rt.declare_field(f"f{i}", dom) for i in range(gc.ndat)]
    for i, ds in enumerate(ids):
        al = rt.alloc_range(ds)
        arr = np.zeros(al.shape())
        # chain_gen.cpp:130-133 dyadic values over the logical range
        grids = np.meshgrid(*[np.arange(al.start(d), al.end(d)) for d in reversed(range(gc.dim))], indexing="ij")
        coords = list(reversed(grids))  # coords[d] = coordinate along dim d
        h = coords[0] * 3
        if gc.dim > 1:
            h = h + coords[1] * 5
        if gc.dim > 2:
            h = h + coords[2] * 7
        vals = ((h + i * 11) & 15) / 16.0
        inside = np.ones(al.shape(), dtype=bool)
        for d in range(gc.dim):
            inside &= (coords[d] >= 0) & (coords[d] < gc.extent[d])
        arr[inside] = vals[inside]
        rt.upload(ds, arr)
    return ids


def enqueue(rt, gc: GenChain):
    handles = []
    for l, (lohi, args, red) in enumerate(gc.loops):
        total = sum(len(gc.stencils[st]) for ds, st, m in args if m == 0)
        scale = 1.0
        while scale * max(total, 1) > 0.5:
            scale *= 0.5
        h = rt.par_loop(KernelHandle(l, f"gen{l}", kernels.GEN_SUM, (scale,)), Range(gc.dim, lohi), args, red)
        if red is not None:
            handles.append((h, red))
    return handles


def run(rt, gc: GenChain, mode: Optional[ExecMode]):
    ids = declare(rt, gc)
    handles = enqueue(rt, gc)
    if mode is not None:
        rt.flush(mode)
    reds = [(rt.fetch_reduction(h), op) for h, op in handles]
    return [rt.download(ds) for ds in ids], reds


def assert_same(got, want, what=""):
    (gf, gr), (wf, wr) = got, want
    for i, (a, b) in enumerate(zip(gf, wf)):
        if not np.array_equal(a, b):
            bad = np.argwhere(a != b)
            raise AssertionError(f"{what}: dataset {i} differs at {len(bad)} points, first {bad[:3].tolist()} "
                                 f"got {a[tuple(bad[0])]} want {b[tuple(bad[0])]}")
    assert len(gr) == len(wr)
    for (a, op), (b, _) in zip(gr, wr):
        if op == 0:
            assert abs(a - b) <= 1e-12 * max(1.0, abs(b)), f"{what}: sum {a} vs {b}"
        else:
            assert a == b, f"{what}: min/max {a} vs {b}"

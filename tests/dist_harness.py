"""TEST INFRASTRUCTURE: one rank of a distributed run, executed on the CPU
oracle, driven by the PRODUCT's distribution schedule.

The product runtime (C++, host-only use: no GPU needed) queues every loop and
returns, per flush, this rank's overlapped loop ranges and the halo message
list (Runtime.schedule_pending: construct_rank_plan, compute_halo_depths,
exchange_halos order). This harness then does what the device runtime does
with that schedule, on the oracle: rank fields over owned +- pad (dist.cpp
:519-529), boxes moved between processes in the schedule's order through
torch.distributed (gloo here; NCCL on GPUs), loops run over the rank ranges
with reductions masked to the owned box (executor.cpp:209-250,
kernel_ctx.hpp:87), partials all-gathered and folded in rank order
(dist.cpp:657-672). Comparing the gathered result with a single-process
oracle run checks the schedule -- the part of the multi-GPU path that is
host logic -- in a real multi-process setting."""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

import pyoracle
from paper_1704_00693_b200 import Range, Runtime


def _box_slices(alloc, box):
    """numpy slices of `box` inside a dense array over `alloc` (dim 0 fastest
    in memory = last numpy axis)."""
    sl = []
    for d in reversed(range(alloc.dim)):
        sl.append(slice(box[d][0] - alloc.start(d), box[d][1] - alloc.start(d)))
    return tuple(sl)


def _inter(a, b):
    return [(max(x[0], y[0]), min(x[1], y[1])) for x, y in zip(a, b)]


def _empty(b):
    return any(hi <= lo for lo, hi in b)


def _lohi_pairs(r):
    return [(r.start(d), r.end(d)) for d in range(r.dim)]


class DistOracleRank:
    """Same surface as Runtime / OracleRuntime for the workloads in
    tests/chains.py and paper_1704_00693_b200/configs.py."""

    def __init__(self, dim, grid, rank, world, periodic=False, skew=None):
        self.dim, self.rank, self.world = dim, rank, world
        self.grid = list(grid) + [1] * (3 - len(grid))
        from paper_1704_00693_b200 import RuntimeConfig
        self.sched = Runtime(dim, RuntimeConfig(skew_allowance=skew) if skew is not None else RuntimeConfig())
        if periodic:                       # ghost layers join the decomposed domain (before the grid is set)
            self.sched.set_periodic_domain(True)
        self.sched.set_rank_grid(self.grid)
        self.ora = pyoracle.OracleRuntime(dim)
        self.pending = []                  # (kernel, range, args, red, handle)
        self.values = {}
        self.local = []                    # oracle dataset per global dataset
        self.owned = None
        self.halo_messages = 0

    # -- declarations -----------------------------------------------------------
    def declare_stencil(self, name, pts):
        self.ora.declare_stencil(name, pts)
        return self.sched.declare_stencil(name, pts)

    def declare_field(self, name, logical):
        ds = self.sched.declare_field(name, logical)
        self.local.append(None)
        return ds

    def alloc_range(self, ds):
        return self.sched.alloc_range(ds)

    def _ensure_local(self):
        if self.owned is None:
            self.owned = self._owned_boxes()
        own = self.owned[self.rank]
        for ds, l in enumerate(self.local):
            if l is None:
                self.local[ds] = self.ora.declare_field(f"r{ds}", Range(self.dim, sum(([a, b] for a, b in own), [])))

    def _owned_boxes(self):
        # The product's decomposition (decompose, dist.cpp:142-177).
        R = self.grid[0] * self.grid[1] * self.grid[2]
        return {r: _lohi_pairs(self.sched.rank_owned(r)) for r in range(R)}

    # -- data ------------------------------------------------------------------
    def upload(self, ds, arr):
        self._ensure_local()
        g = self.sched.alloc_range(ds)
        la = self.ora.alloc_range(self.local[ds])
        box = _inter(_lohi_pairs(la), _lohi_pairs(g))
        cur = self.ora.download(self.local[ds])
        cur[_box_slices(la, box)] = np.asarray(arr).reshape(g.shape())[_box_slices(g, box)]
        self.ora.upload(self.local[ds], cur)

    def download(self, ds):
        """Gathered over every rank's owned box (logical points only); points
        outside every owned box stay NaN."""
        self.flush()
        g = self.sched.alloc_range(ds)
        la = self.ora.alloc_range(self.local[ds])
        mine = self.ora.download(self.local[ds])
        out = np.full(g.shape(), np.nan)
        parts = [None] * self.world
        own = self.owned[self.rank]
        lg = _lohi_pairs(self.sched.logical_range(ds))
        box = _inter(own, lg)
        dist.all_gather_object(parts, (box, mine[_box_slices(la, box)].copy()))
        for b, data in parts:
            if not _empty(b):
                out[_box_slices(g, b)] = data
        return out

    # -- execution ---------------------------------------------------------------
    def par_loop(self, kernel, rng, args, reduction=None):
        h = self.sched.par_loop(kernel, rng, args, reduction)
        self.pending.append((kernel, rng, args, reduction, h))
        return h

    def set_default_mode(self, mode):
        pass

    def periodic_fill(self, datasets, depth, logical=None):
        """Recorded by the product (a PeriodicMark in its queue): the flush's
        schedule carries the wraps the rewritten chain needs."""
        self.sched.periodic_fill(datasets, depth, logical)

    def _wrap(self, ds, g):
        """Periodic wrap of dataset ds to depth g, as Runtime::periodic_exchange
        does it: the faster dimensions inside this rank over the slabs it
        holds, the split (slowest) dimension as whole slabs between the end
        ranks (a self-exchange when there is one rank)."""
        s = self.dim - 1
        l = self.local[ds]
        la = self.ora.alloc_range(l)
        lg = self.sched.logical_range(ds)
        L = [lg.start(d) for d in range(self.dim)]
        H = [lg.end(d) for d in range(self.dim)]
        lo = [la.start(d) for d in range(self.dim)]
        arr = self.ora.download(l)
        z0, z1 = max(la.start(s), L[s]), min(la.end(s), H[s])

        def sl(d, a, b):
            idx = []
            for e in reversed(range(self.dim)):
                if e == d:
                    idx.append(slice(a - lo[e], b - lo[e]))
                elif e == s:
                    idx.append(slice(z0 - lo[e], z1 - lo[e]))
                elif e < d:
                    idx.append(slice(L[e] - g - lo[e], H[e] + g - lo[e]))
                else:
                    idx.append(slice(L[e] - lo[e], H[e] - lo[e]))
            return tuple(idx)

        if z1 > z0:
            for d in range(s):
                arr[sl(d, L[d] - g, L[d])] = arr[sl(d, H[d] - g, H[d])]
                arr[sl(d, H[d], H[d] + g)] = arr[sl(d, L[d], L[d] + g)]
        first, last = 0, self.world - 1

        def slab(a, b):
            idx = [slice(None)] * self.dim
            idx[0] = slice(a - lo[s], b - lo[s])   # numpy axis 0 = slowest dimension
            return tuple(idx)

        for src, dst, s0, d0 in ((last, first, H[s] - g, L[s] - g), (first, last, L[s], H[s])):
            if src == dst:
                if self.rank == src:
                    arr[slab(d0, d0 + g)] = arr[slab(s0, s0 + g)]
            elif self.rank == src:
                dist.send(torch.from_numpy(np.ascontiguousarray(arr[slab(s0, s0 + g)])), dst)
            elif self.rank == dst:
                buf = torch.empty(arr[slab(d0, d0 + g)].shape, dtype=torch.float64)
                dist.recv(buf, src)
                arr[slab(d0, d0 + g)] = buf.numpy()
            self.halo_messages += 1
        self.ora.upload(l, arr)

    def flush(self, mode=None):
        if not self.pending:
            return {}
        self._ensure_local()
        s = self.sched.schedule_pending()
        assert s["ranks"][self.rank]["owned"] == "x".join(f"[{a},{b})" for a, b in self.owned[self.rank])
        # Periodic chains: one wrap of the chain's inputs first.
        for ds, g in s.get("wraps", []):
            self._wrap(ds, g)
        # One exchange, in the schedule's global order (blocking send/recv
        # pairs: both ends walk the same list).
        for m in s["msgs"]:
            if self.rank not in (m["src"], m["dst"]):
                continue
            l = self.local[m["ds"]]
            la = self.ora.alloc_range(l)
            if m["src"] == self.rank:
                data = self.ora.download(l)[_box_slices(la, m["box"])]
                dist.send(torch.from_numpy(np.ascontiguousarray(data)), m["dst"])
            else:
                shape = tuple(b - a for a, b in reversed(m["box"]))
                buf = torch.empty(shape, dtype=torch.float64)
                dist.recv(buf, m["src"])
                cur = self.ora.download(l)
                cur[_box_slices(la, m["box"])] = buf.numpy()
                self.ora.upload(l, cur)
            self.halo_messages += 1
        # Rank-local chain with the owned reduction mask.
        mine = s["ranks"][self.rank]["loops"]
        own = self.owned[self.rank]
        self.ora.set_reduction_mask(Range(self.dim, sum(([a, b] for a, b in own), [])))
        partial = []
        for (kernel, rng, args, red, h), box in zip(self.pending, mine):
            if _empty(box):
                if red is not None:
                    partial.append(float(0.0 if int(red) == 0 else (np.inf if int(red) == 1 else -np.inf)))
                continue
            largs = [(self.local[ds], st, int(m)) for ds, st, m in
                     ((a.dataset, a.stencil, a.mode) if hasattr(a, "dataset") else tuple(a) for a in args)]
            lh = self.ora.par_loop(kernel, Range(self.dim, sum(([a, b] for a, b in box), [])), largs, red)
            if red is not None:
                partial.append(self.ora.fetch_reduction(lh))
        self.ora.set_reduction_mask(None)
        parts = [None] * self.world
        dist.all_gather_object(parts, partial)
        i = 0
        for kernel, rng, args, red, h in self.pending:
            if red is None:
                continue
            op = int(red)
            acc = 0.0 if op == 0 else (np.inf if op == 1 else -np.inf)
            for r in range(self.world):
                v = parts[r][i]
                acc = acc + v if op == 0 else (min(acc, v) if op == 1 else max(acc, v))
            self.values[h] = acc
            i += 1
        self.pending = []
        return {}

    def fetch_reduction(self, h):
        if h not in self.values:
            self.flush()
        return self.values.pop(h)

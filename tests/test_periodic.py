"""Periodic boundaries inside a chain (csrc/host/tcg_periodic.cpp): the
recorded periodic_fill marks of c5 keep the RK step one 22-loop chain; the
flush wraps the chain's inputs once and extends the producing loops into the
ghost layers (the deep-halo scheme of dist.cpp:617-689 for the wrap-around
neighbour the reference does not have, dist.cpp:135-140). Host-only checks of
the rewrite; GPU parity is in tests/test_gpu_periodic.py."""
import re

import pytest

from paper_1704_00693_b200 import (AccessMode, ArgSpec, KernelHandle, Range, Runtime, configs, kernels)
from paper_1704_00693_b200.runtime import PlanError

R, W = AccessMode.Read, AccessMode.Write


def _host_only(rt):
    rt.upload = lambda *a, **k: None
    rt.upload_box = lambda *a, **k: None
    return rt


def _ranges(text):
    return [tuple(int(v) for v in re.findall(r"-?\d+", l.split("range=")[1])) for l in text.splitlines()
            if l.startswith("loop=")]


def test_c5_step_is_one_chain_with_one_wrap(monkeypatch):
    monkeypatch.setattr(configs.NsC5, "_initial", lambda self, sb: {})
    rt = _host_only(Runtime(3))
    c = configs.NsC5(rt, 32)
    c.enqueue_step()
    assert rt.pending_loops() == 22  # the three periodic fills no longer flush
    text = rt.periodic_plan_pending()
    assert text.startswith("loops=22 marks=3 max_extension=6")
    rs = _ranges(text)
    # stage 1 prim over +-6, its RHS/update over +-4; stage 2 +-4 / +-2; stage 3 +-2 / 0
    ext = [-r[0] for r in rs]
    assert ext == [6] + [4] * 6 + [4] + [2] * 6 + [2] + [0] * 7
    assert all(r == (-e, 32 + e) * 3 for r, e in zip(rs, ext))
    wraps = dict((int(a), int(b)) for a, b in re.findall(r"wrap ds=(\d+) depth=(\d+)", text))
    f = c.f
    assert {wraps[f[n]] for n in ("rho", "mx", "my", "mz", "E")} == {6}
    assert {wraps[f[n]] for n in ("d_rho", "d_mx", "d_my", "d_mz", "d_E")} == {4}
    assert all(f[n] not in wraps for n in ("u", "v", "w", "p", "T"))  # produced inside the chain


def test_fill_deeper_than_marked_is_refused():
    rt = _host_only(Runtime(1))
    ident = rt.declare_stencil("id", [(0,)])
    wide = rt.declare_stencil("wide", [(-2,), (0,), (2,)])
    a = rt.declare_field("a", Range.d1(0, 16))
    b = rt.declare_field("b", Range.d1(0, 16))
    rt.par_loop(KernelHandle(0, "copy", kernels.COPY), Range.d1(0, 16), [ArgSpec(b, ident, R), ArgSpec(a, ident, W)])
    rt.periodic_fill([a], 1)
    rt.par_loop(KernelHandle(1, "sum", kernels.GEN_SUM, (0.5,)), Range.d1(0, 16), [ArgSpec(a, wide, R), ArgSpec(b, ident, W)])
    with pytest.raises(PlanError, match="ghost layers"):
        rt.periodic_plan_pending()


def test_unmarked_ghost_reads_are_left_alone():
    # Without a mark a read beyond the logical box is an ordinary read of the
    # padding (Dirichlet halos): no loop is extended, nothing is wrapped.
    rt = _host_only(Runtime(1))
    ident = rt.declare_stencil("id", [(0,)])
    three = rt.declare_stencil("three", [(-1,), (0,), (1,)])
    a = rt.declare_field("a", Range.d1(0, 16))
    b = rt.declare_field("b", Range.d1(0, 16))
    rt.par_loop(KernelHandle(0, "copy", kernels.COPY), Range.d1(0, 16), [ArgSpec(b, ident, R), ArgSpec(a, ident, W)])
    rt.par_loop(KernelHandle(1, "smooth", kernels.SMOOTH_1D), Range.d1(0, 16), [ArgSpec(a, three, R), ArgSpec(b, ident, W)])
    text = rt.periodic_plan_pending()
    assert "max_extension=0" in text and "wrap" not in text
    assert _ranges(text) == [(0, 16), (0, 16)]


def test_mark_extends_the_producer_and_wraps_its_input():
    rt = _host_only(Runtime(1))
    ident = rt.declare_stencil("id", [(0,)])
    three = rt.declare_stencil("three", [(-1,), (0,), (1,)])
    a = rt.declare_field("a", Range.d1(0, 16))
    b = rt.declare_field("b", Range.d1(0, 16))
    rt.par_loop(KernelHandle(0, "copy", kernels.COPY), Range.d1(0, 16), [ArgSpec(b, ident, R), ArgSpec(a, ident, W)])
    rt.periodic_fill([a], 1)
    rt.par_loop(KernelHandle(1, "smooth", kernels.SMOOTH_1D), Range.d1(0, 16), [ArgSpec(a, three, R), ArgSpec(b, ident, W)])
    text = rt.periodic_plan_pending()
    assert _ranges(text) == [(-1, 17), (0, 16)]
    assert re.findall(r"wrap ds=(\d+) depth=(\d+)", text) == [(str(b), "1")]


def test_c5_rank_grid_schedule_covers_the_extended_loops(monkeypatch):
    # Periodic box on a rank grid (host-only): the ghost layers join the
    # decomposed domain, so the union of the ranks' loop ranges is each
    # extended loop range of the rewritten chain (the end ranks compute the
    # ghost zones) and interior faces keep the usual deep-halo messages.
    from paper_1704_00693_b200 import RuntimeConfig
    monkeypatch.setattr(configs.NsC5, "_initial", lambda self, sb: {})
    rt = _host_only(Runtime(3, RuntimeConfig(skew_allowance=6)))
    rt.set_periodic_domain(True)
    rt.set_rank_grid((1, 1, 4))
    c = configs.NsC5(rt, 48)
    c.enqueue_step()
    sched = rt.schedule_pending()
    ext = [6] + [4] * 6 + [4] + [2] * 6 + [2] + [0] * 7
    assert len(sched["ranks"]) == 4
    # pad = 2 + 6 = 8: domain [-8, 56)^3, 16 planes per rank
    assert sched["ranks"][0]["owned"] == "[-8,56)x[-8,56)x[-8,8)"
    for l, e in enumerate(ext):
        zlo = min(r["loops"][l][2][0] for r in sched["ranks"].values() if r["loops"][l][2][1] > r["loops"][l][2][0])
        zhi = max(r["loops"][l][2][1] for r in sched["ranks"].values() if r["loops"][l][2][1] > r["loops"][l][2][0])
        assert (zlo, zhi) == (-e, 48 + e), (l, zlo, zhi)
        for r in sched["ranks"].values():
            (x0, x1), (y0, y1), _ = r["loops"][l]
            assert (x0, x1, y0, y1) == (-e, 48 + e, -e, 48 + e)
    assert all(m["dim"] == 2 for m in sched["msgs"]) and len(sched["msgs"]) > 0

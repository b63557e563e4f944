"""GPU parity of periodic boundaries kept inside the chain (tcg_periodic.cpp):
the product records periodic_fill and rewrites the chain at flush (one wrap,
extended loops); the oracle copies the ghost layers eagerly at every fill.
The logical boxes must agree bit for bit."""
import numpy as np
import pytest

from paper_1704_00693_b200 import (AccessMode, ArgSpec, ExecMode, KernelHandle, Range, ReduceOp, Runtime, configs,
                                   kernels, parse_report)

pytestmark = pytest.mark.gpu
R, W = AccessMode.Read, AccessMode.Write

MODES = {"untiled": ExecMode.untiled(), "stream": ExecMode.stream(), "auto": ExecMode.tiled_auto(),
         "tiled": ExecMode.tiled((0, 0, 0))}


def _interior(rt, ds, dom):
    al = rt.alloc_range(ds)
    a = rt.download(ds)
    sl = tuple(slice(dom.start(d) - al.start(d), dom.end(d) - al.start(d)) for d in reversed(range(dom.dim)))
    return np.ascontiguousarray(a[sl])


def _smooth_chain(rt, n, sweeps, seed):
    """a <-> b smoothing sweeps on a periodic n x n box, a ghost fill before
    every sweep, a Sum of the result at the end."""
    dom = Range.d2(0, n, 0, n)
    ident = rt.declare_stencil("id", [(0, 0)])
    star = rt.declare_stencil("star", [(0, 0), (-1, 0), (1, 0), (0, -1), (0, 1)])
    a, b = rt.declare_field("a", dom), rt.declare_field("b", dom)
    al = rt.alloc_range(a)
    rng = np.random.default_rng(seed)
    init = np.zeros(al.shape())
    lo = [dom.start(d) - al.start(d) for d in (1, 0)]
    init[lo[0]:lo[0] + n, lo[1]:lo[1] + n] = rng.random((n, n))
    rt.upload(a, init)
    rt.upload(b, np.zeros(al.shape()))
    src, dst = a, b
    for k in range(sweeps):
        rt.periodic_fill([src], 1, list(dom.lohi))
        rt.par_loop(KernelHandle(k, "smooth", kernels.SMOOTH_2D), dom, [ArgSpec(src, star, R), ArgSpec(dst, ident, W)])
        src, dst = dst, src
    h = rt.par_loop(KernelHandle(99, "sum", kernels.SUM_READ), dom, [ArgSpec(src, ident, R)], ReduceOp.Sum)
    return a, b, dom, h


@pytest.mark.parametrize("mode", list(MODES))
def test_periodic_smoothing_chain(oracle_lib, mode):
    ort = oracle_lib.OracleRuntime(2)
    oa, ob, dom, oh = _smooth_chain(ort, 40, 6, 5)
    want_sum = ort.fetch_reduction(oh)
    rt = Runtime(2)
    rt.set_default_mode(MODES[mode])
    a, b, dom, h = _smooth_chain(rt, 40, 6, 5)
    assert rt.pending_loops() == 7  # fills are recorded, not flushed
    got_sum = rt.fetch_reduction(h)
    rep = parse_report(rt.report_text())
    assert int(rep["halo_exchanges"]) == 1  # one wrap for the whole chain
    for g, o in ((a, oa), (b, ob)):
        assert np.array_equal(_interior(rt, g, dom), _interior(ort, o, dom))
    assert abs(got_sum - want_sum) <= 1e-12 * abs(want_sum)


def test_eager_periodic_fill_still_available(oracle_lib):
    ort = oracle_lib.OracleRuntime(2)
    oa, ob, dom, oh = _smooth_chain(ort, 24, 3, 9)
    want = ort.fetch_reduction(oh)
    rt = Runtime(2)
    rt.set_periodic_flush(True)
    a, b, dom, h = _smooth_chain(rt, 24, 3, 9)
    assert rt.pending_loops() == 2  # every fill flushed the loops before it (last sweep + the Sum remain)
    assert abs(rt.fetch_reduction(h) - want) <= 1e-12 * abs(want)
    # eager copies define the ghost layers too: whole allocations agree
    assert np.array_equal(rt.download(a), ort.download(oa))
    assert np.array_equal(rt.download(b), ort.download(ob))


@pytest.mark.parametrize("mode", ["untiled", "stream", "auto"])
def test_c5_step_runs_as_one_chain(oracle_lib, mode):
    def run(rt, steps=3):
        c = configs.NsC5(rt, 16)
        kes, loops = [], []
        for _ in range(steps):
            h = c.enqueue_step()
            loops.append(rt.pending_loops() if hasattr(rt, "pending_loops") else 22)
            kes.append(rt.fetch_reduction(h))
        return c.outputs(), kes, loops

    fo, ko, _ = run(oracle_lib.OracleRuntime(3))
    rt = Runtime(3)
    rt.set_default_mode(MODES[mode])
    fg, kg, loops = run(rt)
    assert loops == [22, 22, 22]
    for k in fo:
        assert np.array_equal(fg[k], fo[k]), k
    for a, b in zip(kg, ko):
        assert abs(a - b) <= 1e-12 * abs(b)


class _PeriodicGrid(Runtime):
    def __init__(self, dim, grid, skew=None):
        from paper_1704_00693_b200 import RuntimeConfig
        super().__init__(dim, RuntimeConfig(skew_allowance=skew) if skew is not None else RuntimeConfig())
        self.set_periodic_domain(True)
        self.set_rank_grid(grid)


@pytest.mark.parametrize("grid", [(1, 1, 1), (1, 2, 1), (1, 3, 1)])
@pytest.mark.parametrize("mode", ["untiled", "stream", "auto"])
def test_periodic_smoothing_chain_on_rank_grid(oracle_lib, mode, grid):
    # The wrap along the split dimension is a slab message between the end
    # ranks (a self-exchange at one rank), the other dimension wraps inside
    # every rank; ghost layers belong to the end ranks.
    ort = oracle_lib.OracleRuntime(2)
    oa, ob, dom, oh = _smooth_chain(ort, 40, 4, 5)
    want_sum = ort.fetch_reduction(oh)
    rt = _PeriodicGrid(2, grid, skew=7)
    rt.set_default_mode(MODES[mode])
    a, b, dom, h = _smooth_chain(rt, 40, 4, 5)
    got_sum = rt.fetch_reduction(h)
    for g, o in ((a, oa), (b, ob)):
        assert np.array_equal(_interior(rt, g, dom), _interior(ort, o, dom))
    assert abs(got_sum - want_sum) <= 1e-12 * abs(want_sum)


@pytest.mark.parametrize("grid", [(1, 1, 2), (1, 1, 4)])
@pytest.mark.parametrize("mode", ["untiled", "auto"])
def test_c5_z_split_with_periodic_wrap(oracle_lib, mode, grid):
    # BASELINE c5's decomposition: split along z, one deep-halo exchange per
    # RK step plus one periodic wrap; conserved fields bit-exact against the
    # single-rank oracle, kinetic energy (rank-order fold) to 1e-12.
    def run(rt, steps=2):
        c = configs.NsC5(rt, 48)
        kes = [rt.fetch_reduction(c.enqueue_step()) for _ in range(steps)]
        return c.outputs(), kes

    fo, ko = run(oracle_lib.OracleRuntime(3))
    rt = _PeriodicGrid(3, grid, skew=6)
    rt.set_default_mode(MODES[mode])
    fg, kg = run(rt)
    for k in fo:
        assert np.array_equal(fg[k], fo[k]), k
    for a, b in zip(kg, ko):
        assert abs(a - b) <= 1e-12 * abs(b)

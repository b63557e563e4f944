"""GPU parity: the B200 executors (untiled and windowed-tiled) against the
sequential oracle and the unmodified reference, through the C-ABI.

Bar (BASELINE north_star): per-point fp64 arithmetic bit-exact (-fmad=false on
the device, FMA-free host oracle); Sum reductions within 1e-12 relative of the
oracle's visit-order sum (the reference's own tolerance across thread counts,
test_executor.cpp:117-142); Min/Max exact."""
import numpy as np
import pytest

import chains as C
from paper_1704_00693_b200 import ExecMode, Runtime, RuntimeConfig, configs, parse_report

pytestmark = pytest.mark.gpu

MODES = {
    "untiled": lambda dim, seed: ExecMode.untiled(),
    # the reference's tile plans with random tile sizes, L2-resident executor
    "tiled": lambda dim, seed: ExecMode.tiled(C.random_tile_sizes(seed, dim)),
    "tiled_sizer": lambda dim, seed: ExecMode.tiled((0, 0, 0)),
    "windowed": lambda dim, seed: ExecMode.windowed(C.random_tile_sizes(seed, dim)),
    "auto": lambda dim, seed: ExecMode.tiled_auto(),
}


@pytest.mark.parametrize("mode", list(MODES))
@pytest.mark.parametrize("dim,seeds,kw", [
    (2, range(1, 41), {}),
    (1, range(5001, 5021), {"extent": (32, 96)}),
    (3, range(9001, 9013), {"extent": (8, 16)}),
])
def test_random_chains_match_oracle(oracle_lib, mode, dim, seeds, kw):
    for seed in seeds:
        gc = C.generate(seed, dim=dim, **kw)
        want = C.run(oracle_lib.OracleRuntime(dim), gc, None)
        got = C.run(Runtime(dim), gc, MODES[mode](dim, seed))
        C.assert_same(got, want, f"{mode} dim{dim} seed{seed}")


@pytest.mark.parametrize("segments", [1, 3])
def test_random_chains_stream_segments(oracle_lib, segments):
    # CTA segments along the stream dimension exercise the left-extension
    # (has_left) path of the rank plan (dist.cpp:300-310).
    for seed in range(101, 121):
        gc = C.generate(seed, dim=2)
        want = C.run(oracle_lib.OracleRuntime(2), gc, None)
        got = C.run(Runtime(2, RuntimeConfig(stream_segments=segments)), gc,
                    ExecMode.windowed(C.random_tile_sizes(seed, 2)))
        C.assert_same(got, want, f"segments{segments} seed{seed}")


@pytest.mark.parametrize("copy", [True, False])
@pytest.mark.parametrize("mode", [ExecMode.untiled(), ExecMode.tiled((16, 16, 1)), ExecMode.tiled((8, 4, 1)),
                                  ExecMode.windowed((16, 16, 1)), ExecMode.tiled_auto()])
def test_jacobi_app_matches_reference_app(ref_lib, copy, mode):
    want = ref_lib.ref_app_jacobi(64, 64, 10, copy)
    rt = Runtime(2)
    j = configs.Jacobi2D(rt, 64, 64)
    j.enqueue(10, copy)
    rt.flush(mode)
    got = np.stack([j.logical(j.a), j.logical(j.b)])
    assert np.array_equal(got, want)


@pytest.mark.parametrize("mode", [ExecMode.untiled(), ExecMode.tiled((8, 8, 1)), ExecMode.tiled((48, 16, 1)),
                                  ExecMode.windowed((48, 16, 1)), ExecMode.tiled_auto()])
def test_minihydro_app_matches_reference_app(ref_lib, mode):
    fields, monitors = ref_lib.ref_app_minihydro(48, 48, 3)
    rt = Runtime(2)
    rt.set_default_mode(mode)
    m = configs.MiniHydro(rt, 48, 48)
    got_mon = m.run(3)
    got = np.stack([m.logical(n) for n in ["rho", "e", "p", "u", "v", "fx", "fy", "w"]])
    assert np.array_equal(got, fields)
    for a, b in zip(got_mon, monitors):
        assert abs(a - b) <= 1e-12 * max(1.0, abs(b))


def _run_config(rt, cfg_cls, n, **kw):
    c = cfg_cls(rt, n)
    if cfg_cls is configs.HeatC1:
        for _ in range(kw.get("chains", 2)):
            c.enqueue_chain()
            rt.flush(kw.get("mode"))
        return c.outputs(), []
    if cfg_cls is configs.HydroC2:
        rt.set_default_mode(kw.get("mode") or ExecMode.untiled())
        mins = [rt.fetch_reduction(c.enqueue_step()) for _ in range(kw.get("steps", 3))]
        return c.outputs(), mins
    if cfg_cls is configs.Jacobi3DC3:
        c.enqueue_chain()
        rt.flush(kw.get("mode"))
        return c.outputs(), []
    raise ValueError(cfg_cls)


@pytest.mark.parametrize("cfg,n", [(configs.HeatC1, 64), (configs.HydroC2, 96), (configs.HydroC2, 90), (configs.Jacobi3DC3, 24)])
@pytest.mark.parametrize("mode", [ExecMode.untiled(), ExecMode.tiled((0, 0, 0)), ExecMode.windowed(),
                                  ExecMode.tiled_auto()])
def test_configs_small_match_oracle(oracle_lib, cfg, n, mode):
    want = _run_config(oracle_lib.OracleRuntime(3 if cfg is configs.Jacobi3DC3 else 2), cfg, n)
    got = _run_config(Runtime(3 if cfg is configs.Jacobi3DC3 else 2), cfg, n, mode=mode)
    for k in want[0]:
        assert np.array_equal(got[0][k], want[0][k]), k
    assert got[1] == want[1]


@pytest.mark.parametrize("mode", [ExecMode.untiled(), ExecMode.tiled((0, 0, 0)), ExecMode.tiled_auto()])
def test_cg_residual_history_matches_reference(ref_lib, mode):
    # c4 at 64^2: the residual history must agree to 1e-10 relative over the
    # window where the reference is self-consistent (SURVEY.md §7 hard parts).
    iters = 30
    ref = ref_lib.RefRuntime(2)
    cr = configs.CgC4(ref, 64)
    cr.start()
    for _ in range(iters):
        cr.iterate()
    rt = Runtime(2)
    rt.set_default_mode(mode)
    cg = configs.CgC4(rt, 64)
    cg.start()
    for _ in range(iters):
        cg.iterate()
    h, w = np.array(cg.history), np.array(cr.history)
    rel = np.abs(h - w) / np.maximum(np.abs(w), 1e-300)
    assert rel.max() <= 1e-10, rel


def test_fetch_reduction_flushes_prefix_only():
    from paper_1704_00693_b200 import ArgSpec, AccessMode, KernelHandle, Range, ReduceOp, kernels
    rt = Runtime(1)
    ident = rt.declare_stencil("id", [(0,)])
    f0 = rt.declare_field("f0", Range.d1(0, 8))
    f1 = rt.declare_field("f1", Range.d1(0, 8))
    rt.par_loop(KernelHandle(0, "iota", kernels.IOTA), Range.d1(0, 8), [ArgSpec(f0, ident, AccessMode.Write)])
    h = rt.par_loop(KernelHandle(1, "sum", kernels.SUM_READ), Range.d1(0, 8), [ArgSpec(f0, ident, AccessMode.Read)],
                    ReduceOp.Sum)
    rt.par_loop(KernelHandle(2, "copy", kernels.COPY), Range.d1(0, 8),
                [ArgSpec(f0, ident, AccessMode.Read), ArgSpec(f1, ident, AccessMode.Write)])
    assert rt.fetch_reduction(h) == 28.0
    assert rt.pending_loops() == 1
    with pytest.raises(Exception):
        rt.fetch_reduction(h)
    assert rt.get(f1, (5,)) == 5.0
    assert rt.pending_loops() == 0
    rt.put(f1, (5,), 2.5)
    assert rt.get(f1, (5,)) == 2.5
    rt.fill_logical(f1, 1.5)
    assert rt.get(f1, (0,)) == 1.5 and rt.get(f1, (-1,)) == 0.0


def test_tiled_auto_switches_executor_bit_exact(oracle_lib):
    # tiled_auto times the executors per chain signature (untiled and the
    # fused streaming executor, three times each) and keeps the fastest;
    # every flush bit-exact.
    steps = 12
    want = _run_config(oracle_lib.OracleRuntime(2), configs.HydroC2, 96, steps=steps)
    rt = Runtime(2)
    rt.set_default_mode(ExecMode.tiled_auto())
    c = configs.HydroC2(rt, 96)
    mins, used = [], []
    for _ in range(steps):
        mins.append(rt.fetch_reduction(c.enqueue_step()))
        used.append(parse_report(rt.report_text())["executor"])
    assert used[:6] == ["untiled", "stream"] * 3, used
    assert len(set(used[6:])) == 1, used
    got = c.outputs()
    for k in want[0]:
        assert np.array_equal(got[k], want[0][k]), k
    assert mins == want[1]


@pytest.mark.parametrize("mode", [ExecMode.untiled(), ExecMode.tiled((0, 0, 0)), ExecMode.windowed(),
                                  ExecMode.tiled_auto()], ids=["untiled", "tiled", "windowed", "auto"])
def test_empty_range_loops(oracle_lib, mode):
    # A loop with an empty range does nothing; a reducing one yields the
    # identity (reduce_identity, types.hpp:272-288).
    gc = C.generate(77, dim=2, min_loops=4, max_loops=6, extent=(40, 56))
    lohi, args, _ = gc.loops[1]
    gc.loops.insert(1, ([lohi[0], lohi[1], 9, 9], args, 1))
    gc.loops.insert(3, ([5, 5, lohi[2], lohi[3]], args, None))
    want = C.run(oracle_lib.OracleRuntime(2), gc, None)
    got = C.run(Runtime(2), gc, mode)
    C.assert_same(got, want, "empty loops")
    assert float("inf") in [v for v, _ in got[1]]


@pytest.mark.parametrize("mode", [ExecMode.untiled(), ExecMode.tiled((0, 0, 0)), ExecMode.tiled((16, 16, 4)),
                                  ExecMode.windowed(), ExecMode.tiled_auto()],
                         ids=["untiled", "tiled", "tiled_ts", "windowed", "auto"])
def test_ns_c5_matches_oracle(oracle_lib, mode):
    # c5 (3D Navier-Stokes-like TGV, 22 loops/step incl. periodic ghost fills)
    # at 16^3, 3 steps: conserved fields bit-exact, kinetic energy to 1e-12.
    def run(rt):
        rt.set_default_mode(mode)
        c = configs.NsC5(rt, 16)
        kes = [rt.fetch_reduction(c.enqueue_step()) for _ in range(3)]
        return c.outputs(), kes

    fo, ko = run(oracle_lib.OracleRuntime(3))
    fg, kg = run(Runtime(3))
    for k in fo:
        assert np.array_equal(fg[k], fo[k]), k
    for a, b in zip(kg, ko):
        assert abs(a - b) <= 1e-12 * abs(b)


@pytest.mark.parametrize("mode", [ExecMode.untiled(), ExecMode.tiled_auto(), ExecMode.stream()],
                         ids=["untiled", "auto", "stream"])
def test_hundred_reducing_loops_in_one_flush(mode):
    # A flush may hold any number of reducing loops (runtime.cpp:94-151): the
    # device / pinned result buffers grow with the chain.
    from paper_1704_00693_b200 import ArgSpec, AccessMode, KernelHandle, Range, ReduceOp, kernels
    rt = Runtime(2)
    ident = rt.declare_stencil("id", [(0, 0)])
    dom = Range.d2(0, 24, 0, 20)
    f0 = rt.declare_field("f0", dom)
    rt.par_loop(KernelHandle(0, "iota", kernels.IOTA), dom, [ArgSpec(f0, ident, AccessMode.Write)])
    handles, want = [], []
    for i in range(100):
        n = 1 + i % 24
        handles.append(rt.par_loop(KernelHandle(1 + i, "sum", kernels.SUM_READ), Range.d2(0, n, 0, 20),
                                   [ArgSpec(f0, ident, AccessMode.Read)], ReduceOp.Sum))
        want.append(20.0 * n * (n - 1) / 2)
    rt.flush(mode)
    assert [rt.fetch_reduction(h) for h in handles] == want


def test_step_templates_replay_equals_direct_calls(oracle_lib):
    # Runtime.record_begin / record_end / replay: the C++ host path re-issues
    # the recorded par_loop calls (new reduction handles, parameters replaced
    # in call order); results equal issuing every call from Python.
    def direct(rt, steps):
        c = configs.HydroC2(rt, 80)
        mins = [rt.fetch_reduction(c.enqueue_step()) for _ in range(steps)]
        return c.outputs(), mins

    want_f, want_m = direct(oracle_lib.OracleRuntime(2), 4)
    rt = Runtime(2)
    rt.set_default_mode(ExecMode.tiled_auto())
    c = configs.HydroC2(rt, 80)
    rt.record_begin()
    h = c.enqueue_step()
    tpl = rt.record_end()
    mins = [rt.fetch_reduction(h)]
    for _ in range(3):
        hs = rt.replay(tpl)
        assert len(hs) == 1 and rt.pending_loops() == 13
        mins.append(rt.fetch_reduction(hs[0]))
    got = c.outputs()
    for k in want_f:
        assert np.array_equal(got[k], want_f[k]), k
    assert mins == want_m

    # parameters replaced per replay (c4's alpha / beta), wrong counts refused
    from paper_1704_00693_b200.runtime import InvalidArgument
    cr = configs.CgC4(oracle_lib.OracleRuntime(2), 48)
    cr.start()
    for _ in range(5):
        cr.iterate()
    rt = Runtime(2)
    cg = configs.CgC4(rt, 48)
    cg.start()
    rt.record_begin()
    h = cg.enqueue_pq()
    t0 = rt.record_end()
    alpha = cg.rr / rt.fetch_reduction(h)
    rt.record_begin()
    h = cg.enqueue_update(alpha)
    t1 = rt.record_end()
    cg.finish_iteration(rt.fetch_reduction(h))
    with pytest.raises(InvalidArgument):
        rt.replay(t0, [1.0, 2.0])  # the template holds one scalar
    assert rt.pending_loops() == 0  # refused before anything was enqueued
    for _ in range(4):
        alpha = cg.rr / rt.fetch_reduction(rt.replay(t0, [cg.beta])[0])
        cg.finish_iteration(rt.fetch_reduction(rt.replay(t1, [alpha, alpha])[0]))
    rel = np.abs(np.array(cg.history) - np.array(cr.history)) / np.abs(np.array(cr.history))
    assert rel.max() <= 1e-10

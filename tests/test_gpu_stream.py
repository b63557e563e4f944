"""GPU parity of the fused streaming executor (ExecMode.stream(), one generated
kernel per chain signature) against the sequential oracle and
the unmodified reference, through the C-ABI.

Bar: per-point fp64 arithmetic bit-exact (-fmad=false, FMA-free oracle);
Min/Max exact; Sum within 1e-12 relative (fold order differs: per-thread
row order, warp tree, CTA order, like the reference's thread-count
tolerance, test_executor.cpp:117-142). Thread-block shapes, segment counts
and sub-chain lengths are forced through set_stream_choice so the small
cases exercise many CTAs, overlapped edges, stream segments and sub-chain
boundaries (with ping-pong buffers carried across kernels and flushes)."""
import numpy as np
import pytest

import chains as C
from paper_1704_00693_b200 import ExecMode, Runtime, configs, parse_report

pytestmark = pytest.mark.gpu

# (nt, bx, by, ntx, segments, max_loops, minb, prefetch)
CHOICES_2D = {
    "sizer": (0, 0, 0, 0, 0, 0, 0, -1),
    "narrow": (32, 1, 0, 0, 5, 0, 0, 2),
    "bx2_split3": (64, 2, 0, 0, 3, 3, 0, 0),
    "bx4_seg7": (32, 4, 0, 0, 7, 0, 0, 4),
}
CHOICES_3D = {
    "sizer": (0, 0, 0, 0, 0, 0, 0, -1),
    "t8x8": (64, 1, 1, 8, 3, 0, 0, 2),
    "bx2by2": (64, 2, 2, 16, 2, 2, 0, 0),
    "by4": (32, 1, 4, 16, 4, 0, 0, 3),
}


def _rt(dim, choice):
    rt = Runtime(dim)
    rt.set_stream_choice(*choice)
    return rt


@pytest.mark.parametrize("choice", list(CHOICES_2D))
def test_random_chains_2d(oracle_lib, choice):
    for seed in range(1, 41 if choice == "sizer" else 13):
        gc = C.generate(seed, dim=2)
        want = C.run(oracle_lib.OracleRuntime(2), gc, None)
        got = C.run(_rt(2, CHOICES_2D[choice]), gc, ExecMode.stream())
        C.assert_same(got, want, f"stream {choice} seed{seed}")


@pytest.mark.parametrize("choice", list(CHOICES_3D))
def test_random_chains_3d(oracle_lib, choice):
    for seed in range(9001, 9013 if choice == "sizer" else 9005):
        gc = C.generate(seed, dim=3, extent=(8, 16))
        want = C.run(oracle_lib.OracleRuntime(3), gc, None)
        got = C.run(_rt(3, CHOICES_3D[choice]), gc, ExecMode.stream())
        C.assert_same(got, want, f"stream3d {choice} seed{seed}")


def test_random_chains_repeated_flushes(oracle_lib):
    # The same chain flushed three times: ping-pong buffers swap every flush,
    # their dirty boxes must be synchronised before each kernel.
    for seed in range(201, 221):
        gc = C.generate(seed, dim=2)
        results = []
        for rt, mode in ((oracle_lib.OracleRuntime(2), None), (_rt(2, CHOICES_2D["narrow"]), ExecMode.stream())):
            ids = C.declare(rt, gc)
            reds = []
            for _ in range(3):
                hs = C.enqueue(rt, gc)
                if mode is not None:
                    rt.flush(mode)
                reds += [(rt.fetch_reduction(h), op) for h, op in hs]
            results.append(([rt.download(ds) for ds in ids], reds))
        C.assert_same(results[1], results[0], f"repeat seed{seed}")


def test_mixed_executors_keep_buffers_consistent(oracle_lib):
    # Alternating untiled and stream flushes: writes of the untiled executor
    # must be seen by the streaming kernels' second buffers.
    for seed in range(301, 311):
        gc = C.generate(seed, dim=2)
        results = []
        for rt, modes in ((oracle_lib.OracleRuntime(2), [None] * 4),
                          (Runtime(2), [ExecMode.stream(), ExecMode.untiled(), ExecMode.stream(), ExecMode.stream()])):
            ids = C.declare(rt, gc)
            reds = []
            for m in modes:
                hs = C.enqueue(rt, gc)
                if m is not None:
                    rt.flush(m)
                reds += [(rt.fetch_reduction(h), op) for h, op in hs]
            results.append(([rt.download(ds) for ds in ids], reds))
        C.assert_same(results[1], results[0], f"mixed seed{seed}")


@pytest.mark.parametrize("copy", [True, False])
def test_jacobi_app_matches_reference_app(ref_lib, copy):
    want = ref_lib.ref_app_jacobi(64, 64, 10, copy)
    rt = Runtime(2)
    j = configs.Jacobi2D(rt, 64, 64)
    j.enqueue(10, copy)
    rt.flush(ExecMode.stream())
    got = np.stack([j.logical(j.a), j.logical(j.b)])
    assert np.array_equal(got, want)


@pytest.mark.parametrize("choice", ["sizer", "narrow"])
def test_minihydro_app_matches_reference_app(ref_lib, choice):
    fields, monitors = ref_lib.ref_app_minihydro(48, 48, 3)
    rt = _rt(2, CHOICES_2D[choice])
    rt.set_default_mode(ExecMode.stream())
    m = configs.MiniHydro(rt, 48, 48)
    got_mon = m.run(3)
    got = np.stack([m.logical(n) for n in ["rho", "e", "p", "u", "v", "fx", "fy", "w"]])
    assert np.array_equal(got, fields)
    for a, b in zip(got_mon, monitors):
        assert abs(a - b) <= 1e-12 * max(1.0, abs(b))


def _executor(rt, mode):
    return parse_report(rt.report_text())["executor"] if mode is not None else None


def _run_config(rt, cfg_cls, n, mode, chains=2, steps=3):
    c = cfg_cls(rt, n)
    if cfg_cls is configs.HeatC1:
        for _ in range(chains):
            c.enqueue_chain()
            rt.flush(mode)
        ex = _executor(rt, mode)
        return c.outputs(), [], ex
    if cfg_cls is configs.HydroC2:
        rt.set_default_mode(mode)
        mins = [rt.fetch_reduction(c.enqueue_step()) for _ in range(steps)]
        ex = _executor(rt, mode)
        return c.outputs(), mins, ex
    if cfg_cls is configs.Jacobi3DC3:
        for _ in range(chains):
            c.enqueue_chain()
            rt.flush(mode)
        ex = _executor(rt, mode)
        return c.outputs(), [], ex
    raise ValueError(cfg_cls)


@pytest.mark.parametrize("cfg,n,choice", [
    (configs.HeatC1, 64, None), (configs.HeatC1, 100, (64, 2, 0, 0, 3, 0, 0, -1)),
    (configs.HydroC2, 96, None), (configs.HydroC2, 90, (64, 2, 0, 0, 4, 5, 0, -1)),
    (configs.Jacobi3DC3, 24, None), (configs.Jacobi3DC3, 30, (64, 2, 2, 16, 2, 3, 0, -1)),
])
def test_configs_small_match_oracle(oracle_lib, cfg, n, choice):
    dim = 3 if cfg is configs.Jacobi3DC3 else 2
    want = _run_config(oracle_lib.OracleRuntime(dim), cfg, n, None)
    rt = Runtime(dim)
    if choice:
        rt.set_stream_choice(*choice)
    got = _run_config(rt, cfg, n, ExecMode.stream())
    assert got[2] == "stream"
    for k in want[0]:
        assert np.array_equal(got[0][k], want[0][k]), k
    assert got[1] == want[1]


def test_cg_residual_history_matches_reference(ref_lib):
    iters = 30
    ref = ref_lib.RefRuntime(2)
    cr = configs.CgC4(ref, 64)
    cr.start()
    for _ in range(iters):
        cr.iterate()
    rt = Runtime(2)
    rt.set_default_mode(ExecMode.stream())
    cg = configs.CgC4(rt, 64)
    cg.start()
    for _ in range(iters):
        cg.iterate()
    h, w = np.array(cg.history), np.array(cr.history)
    rel = np.abs(h - w) / np.maximum(np.abs(w), 1e-300)
    assert rel.max() <= 1e-10, rel


def test_empty_range_loops(oracle_lib):
    gc = C.generate(77, dim=2, min_loops=4, max_loops=6, extent=(40, 56))
    lohi, args, _ = gc.loops[1]
    gc.loops.insert(1, ([lohi[0], lohi[1], 9, 9], args, 1))
    gc.loops.insert(3, ([5, 5, lohi[2], lohi[3]], args, None))
    want = C.run(oracle_lib.OracleRuntime(2), gc, None)
    got = C.run(Runtime(2), gc, ExecMode.stream())
    C.assert_same(got, want, "empty loops")


def test_tiled_auto_picks_among_untiled_and_stream(oracle_lib):
    steps = 9
    want = _run_config(oracle_lib.OracleRuntime(2), configs.HydroC2, 96, None, steps=steps)
    rt = Runtime(2)
    rt.set_default_mode(ExecMode.tiled_auto())
    c = configs.HydroC2(rt, 96)
    mins, used = [], []
    for _ in range(steps):
        mins.append(rt.fetch_reduction(c.enqueue_step()))
        used.append(parse_report(rt.report_text())["executor"])
    assert used[:6] == ["untiled", "stream"] * 3, used
    got = c.outputs()
    for k in want[0]:
        assert np.array_equal(got[k], want[0][k]), k
    assert mins == want[1]


@pytest.mark.parametrize("dim", [2, 3])
def test_horizontal_runs_with_own_point_dependencies_and_reductions(oracle_lib, dim):
    # A run of loops over one range in which written datasets are touched at
    # the iteration point only: fused point by point into one untiled-style
    # generated kernel (generate_horizontal) -- independent stencil loops, an
    # own-point read-modify-write of an earlier loop's output, an increment,
    # and Sum / Min reductions of values the run itself produced.
    from paper_1704_00693_b200 import AccessMode, ArgSpec, KernelHandle, Range, ReduceOp, kernels
    R_, W_, RW_, INC_ = AccessMode.Read, AccessMode.Write, AccessMode.ReadWrite, AccessMode.Increment
    n = (37, 29) if dim == 2 else (21, 13, 11)

    def run(rt, mode):
        ident = rt.declare_stencil("id", [(0,) * dim])
        star = rt.declare_stencil("star", [(0,) * dim] + [tuple((s if e == d else 0) for e in range(dim))
                                                          for d in range(dim) for s in (-1, 1, 2)])
        dom = Range(dim, sum(([0, e] for e in n), []))
        f = [rt.declare_field(f"f{i}", dom) for i in range(5)]
        rng = np.random.default_rng(11)
        for i in (0, 1):
            al = rt.alloc_range(f[i])
            rt.upload(f[i], rng.random(al.shape()))
        G = lambda i, s: KernelHandle(i, f"g{i}", kernels.GEN_SUM, (s,))
        rt.par_loop(G(0, 0.11), dom, [ArgSpec(f[0], star, R_), ArgSpec(f[2], ident, W_)])
        rt.par_loop(G(1, 0.07), dom, [ArgSpec(f[1], star, R_), ArgSpec(f[0], ident, R_), ArgSpec(f[3], ident, W_)])
        rt.par_loop(G(2, 0.5), dom, [ArgSpec(f[3], ident, R_), ArgSpec(f[2], ident, RW_)])
        h0 = rt.par_loop(G(3, 0.25), dom, [ArgSpec(f[2], ident, R_), ArgSpec(f[4], ident, INC_)], ReduceOp.Sum)
        h1 = rt.par_loop(KernelHandle(4, "min", kernels.GEN_SUM, (1.0,)), dom,
                         [ArgSpec(f[4], ident, R_), ArgSpec(f[3], ident, RW_)], ReduceOp.Min)
        rt.flush(mode) if mode is not None else rt.flush()
        rep = parse_report(rt.report_text()) if hasattr(rt, "report_text") else None
        return [rt.download(x) for x in f], [rt.fetch_reduction(h0), rt.fetch_reduction(h1)], rep

    want_f, want_r, _ = run(oracle_lib.OracleRuntime(dim), None)
    rt = Runtime(dim)
    got_f, got_r, rep = run(rt, ExecMode.stream())
    for a, b in zip(got_f, want_f):
        assert np.array_equal(a, b)
    assert abs(got_r[0] - want_r[0]) <= 1e-12 * abs(want_r[0])
    assert got_r[1] == want_r[1]
    assert rep["executor"] == "stream" and int(rep["subchains"]) == 1, rep  # one horizontal kernel

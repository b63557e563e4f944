"""Pins the CPU oracle restatement (oracle/tc_oracle.cpp) before any GPU
result is compared against it: the reference's own known answers and the
reference library's outputs (tests/golden/ref_*.json)."""
import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

import chains as C
from paper_1704_00693_b200 import AccessMode, ArgSpec, KernelHandle, Range, ReduceOp, configs, kernels

GOLD = Path(__file__).resolve().parent / "golden"


def sha(arrs):
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(a, dtype=np.float64).tobytes())
    return h.hexdigest()


def test_sequential_reference_kat(oracle_lib):
    # test_oracle.cpp:73-118: iota, neighbour sum, monitor -> sum = 42.0
    rt = oracle_lib.OracleRuntime(1, skew_allowance=0)
    ident = rt.declare_stencil("identity", [(0,)])
    pair = rt.declare_stencil("pair", [(-1,), (1,)])
    f0 = rt.declare_field("f0", Range.d1(0, 8))
    f1 = rt.declare_field("f1", Range.d1(0, 8))
    rt.par_loop(KernelHandle(0, "iota", kernels.IOTA), Range.d1(0, 8), [ArgSpec(f0, ident, AccessMode.Write)])
    rt.par_loop(KernelHandle(1, "nbrs", kernels.NBR_SUM), Range.d1(1, 7),
                [ArgSpec(f0, pair, AccessMode.Read), ArgSpec(f1, ident, AccessMode.Write)])
    h = rt.par_loop(KernelHandle(2, "monitor", kernels.SUM_READ), Range.d1(1, 7), [ArgSpec(f1, ident, AccessMode.Read)],
                    ReduceOp.Sum)
    f = rt.download(f1)
    assert [f[x + 1] for x in range(1, 7)] == [2.0 * x for x in range(1, 7)]
    assert rt.fetch_reduction(h) == 42.0
    with pytest.raises(Exception):
        rt.fetch_reduction(h)


def test_oracle_checked_access(oracle_lib):
    # kernel_ctx.hpp:58-73: reads outside the declared stencil are errors
    rt = oracle_lib.OracleRuntime(1)
    ident = rt.declare_stencil("identity", [(0,)])
    f0 = rt.declare_field("f0", Range.d1(0, 8))
    f1 = rt.declare_field("f1", Range.d1(0, 8))
    with pytest.raises(Exception, match="stencil"):
        rt.par_loop(KernelHandle(0, "c", kernels.CONSUME_1D), Range.d1(0, 8),
                    [ArgSpec(f0, ident, AccessMode.Read), ArgSpec(f1, ident, AccessMode.Write)])


def test_oracle_matches_reference_executions_golden(oracle_lib):
    data = json.loads((GOLD / "ref_exec.json").read_text())
    assert len(data) == 70
    for e in data:
        kw = {k: tuple(v) for k, v in e["kw"].items()}
        gc = C.generate(e["seed"], dim=e["dim"], **kw)
        fields, reds = C.run(oracle_lib.OracleRuntime(e["dim"]), gc, None)
        assert sha(fields) == e["fields_sha256"], (e["dim"], e["seed"])
        for (v, op), (w, wop) in zip(reds, e["reductions"]):
            assert op == wop and v == w  # sequential folds: bit-identical


def test_oracle_matches_reference_apps_golden(oracle_lib):
    gold = json.loads((GOLD / "ref_apps.json").read_text())
    for copy in (True, False):
        rt = oracle_lib.OracleRuntime(2)
        j = configs.Jacobi2D(rt, 64, 64)
        j.enqueue(10, copy)
        got = np.stack([j.logical(j.a), j.logical(j.b)])
        assert sha([got]) == gold[f"jacobi_64_10_{'copy' if copy else 'noncopy'}"]
    rt = oracle_lib.OracleRuntime(2)
    m = configs.MiniHydro(rt, 48, 48)
    mon = m.run(3)
    got = np.stack([m.logical(n) for n in ["rho", "e", "p", "u", "v", "fx", "fy", "w"]])
    assert sha([got]) == gold["minihydro_48_3"]
    assert mon == gold["minihydro_48_3_monitors"]


def test_oracle_matches_live_reference(ref_lib):
    for dim, seeds, kw in ((2, range(600, 625), {}), (3, range(700, 706), {"extent": (8, 14)})):
        for seed in seeds:
            gc = C.generate(seed, dim=dim, **kw)
            want = C.run(ref_lib.RefRuntime(dim, threads=1), gc, None)
            got = C.run(ref_lib.OracleRuntime(dim), gc, None)
            C.assert_same(got, want, f"dim{dim} seed{seed}")


def test_reference_self_consistent_across_tile_sizes(ref_lib):
    # acceptance.cpp:193-206 (criterion 3) on this project's chains: the
    # reference's tiled executor equals its untiled one bit for bit.
    for seed in range(800, 830):
        gc = C.generate(seed, dim=2)
        from paper_1704_00693_b200 import ExecMode
        want = C.run(ref_lib.RefRuntime(2), gc, ExecMode.untiled())
        got = C.run(ref_lib.RefRuntime(2, threads=3), gc, ExecMode.tiled(C.random_tile_sizes(seed, 2)))
        C.assert_same(got, want, f"seed{seed}")


def test_oracle_matches_reference_ns_c5(ref_lib):
    # c5 bodies (csrc/kernels/tc_ns.h) through the unmodified reference's
    # KernelCtx vs the restatement; periodic ghosts by host copy.
    def run(rt):
        c = configs.NsC5(rt, 12)
        kes = [rt.fetch_reduction(c.enqueue_step()) for _ in range(2)]
        return c.outputs(), kes

    import pyoracle

    (fo, ko), (fr, kr) = run(pyoracle.OracleRuntime(3)), run(ref_lib.RefRuntime(3))
    for k in fo:
        assert np.array_equal(fo[k], fr[k]), k
    assert ko == kr
    assert all(np.isfinite(ko)) and ko[0] > 0

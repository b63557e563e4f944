"""Host planner (construct_plan / construct_rank_plan / halo depths / sizer)
through the C-ABI, against the reference's golden known answers
(proj/tests/test_planner.cpp, test_dist.cpp, test_tile_sizer.cpp) and the
reference library's own output (tests/golden/*.json, tests/golden/make_golden.py)."""
import hashlib
import json
from pathlib import Path

import pytest

import chains as C
from paper_1704_00693_b200 import (AccessMode, ArgSpec, InvalidArgument, KernelHandle, PlanError, Range, Runtime,
                                   auto_tile_size, kernels)

GOLD = Path(__file__).resolve().parent / "golden"
R, W = AccessMode.Read, AccessMode.Write


def two_loop(rt, lo=0, hi=8):
    ident = rt.declare_stencil("identity", [(0,)])
    three = rt.declare_stencil("three", [(-1,), (0,), (1,)])
    f0 = rt.declare_field("f0", Range.d1(0, 8))
    f1 = rt.declare_field("f1", Range.d1(0, 8))
    rt.par_loop(KernelHandle(0, "produce", kernels.COPY), Range.d1(lo, hi), [ArgSpec(f0, ident, R), ArgSpec(f1, ident, W)])
    rt.par_loop(KernelHandle(1, "consume", kernels.CONSUME_1D), Range.d1(lo, hi),
                [ArgSpec(f1, three, R), ArgSpec(f0, ident, W)])
    return ident, three, f0, f1


def test_golden_two_loop_dump():
    # test_planner.cpp:40-52, acceptance.cpp:68-89 (SPEC Fig. 2)
    rt = Runtime(1)
    two_loop(rt)
    text = rt.plan_pending([4, 0, 0])
    assert text.startswith("tile=0 loop=0 d=0 [0,5)\n"
                           "tile=0 loop=1 d=0 [0,4)\n"
                           "tile=1 loop=0 d=0 [5,8)\n"
                           "tile=1 loop=1 d=0 [4,8)\n")
    assert "max_skew=1\n" in text


def test_skew_grows_with_chain_depth():
    # test_planner.cpp:140-164: k radius-1 consumers -> skew k-1
    rt = Runtime(1)
    ident = rt.declare_stencil("identity", [(0,)])
    three = rt.declare_stencil("three", [(-1,), (0,), (1,)])
    f = [rt.declare_field(f"f{i}", Range.d1(0, 32)) for i in range(2)]
    for l in range(5):
        rt.par_loop(KernelHandle(l, "s", kernels.SMOOTH_1D), Range.d1(0, 32),
                    [ArgSpec(f[l % 2], three, R), ArgSpec(f[(l + 1) % 2], ident, W)])
    text = rt.plan_pending([16, 0, 0])
    assert "max_skew=4\n" in text
    for l in range(5):
        assert f"tile=0 loop={l} d=0 [0,{16 + 4 - l})" in text
    assert "tile=1 loop=4 d=0 [16,32)" in text


def test_write_after_read_extension():
    # test_planner.cpp:244-273
    rt = Runtime(1)
    ident = rt.declare_stencil("identity", [(0,)])
    three = rt.declare_stencil("three", [(-1,), (0,), (1,)])
    f0 = rt.declare_field("f0", Range.d1(0, 8))
    f1 = rt.declare_field("f1", Range.d1(0, 8))
    rt.par_loop(KernelHandle(0, "c", kernels.CONSUME_1D), Range.d1(0, 8), [ArgSpec(f0, three, R), ArgSpec(f1, ident, W)])
    rt.par_loop(KernelHandle(1, "o", kernels.IOTA), Range.d1(0, 8), [ArgSpec(f0, ident, W)])
    text = rt.plan_pending([4, 0, 0])
    assert "tile=0 loop=0 d=0 [0,5)" in text
    assert "tile=0 loop=1 d=0 [0,4)" in text
    assert "tile=1 loop=0 d=0 [5,8)" in text
    assert "tile=1 loop=1 d=0 [4,8)" in text


def test_cartesian_product_leaves_independent_dim_unskewed():
    # test_planner.cpp:97-137
    rt = Runtime(2)
    ident = rt.declare_stencil("identity", [(0, 0)])
    xs = rt.declare_stencil("x3", [(-1, 0), (0, 0), (1, 0)])
    f0 = rt.declare_field("f0", Range.d2(0, 8, 0, 8))
    f1 = rt.declare_field("f1", Range.d2(0, 8, 0, 8))
    rt.par_loop(KernelHandle(0, "p", kernels.COPY), Range.d2(0, 8, 0, 8), [ArgSpec(f0, ident, R), ArgSpec(f1, ident, W)])
    rt.par_loop(KernelHandle(1, "c", kernels.GEN_SUM, (0.125,)), Range.d2(0, 8, 0, 8),
                [ArgSpec(f1, xs, R), ArgSpec(f0, ident, W)])
    text = rt.plan_pending([4, 4, 1])
    assert "max_skew=1,0\n" in text
    for t in range(4):
        ty = t % 2
        assert f"tile={t} loop=0 d=1 [{4 * ty},{4 * ty + 4})" in text
    assert "tile=0 loop=0 d=0 [0,5)" in text and "tile=2 loop=0 d=0 [5,8)" in text


def test_rank_plans_and_halo_depths_golden():
    # test_dist.cpp:117-158
    rt = Runtime(1)
    two_loop(rt)
    text = rt.rank_plans_pending([2, 1, 1], [4, 0, 0])
    r0, r1 = text.split("rank=1")
    assert "tile=0 loop=0 d=0 [0,5)\ntile=0 loop=1 d=0 [0,4)\n" in r0
    assert "tile=0 loop=0 d=0 [3,8)\ntile=0 loop=1 d=0 [4,8)\n" in r1
    assert "ds=0 needed=1 d0=0,1" in r0 and "ds=1 needed=0" in r0
    assert "ds=0 needed=1 d0=1,0" in r1


def test_pad_shortfall_is_plan_error():
    # planner.cpp:252-269: a tight allocation is a PlanError, never grown.
    # Fields declared before the stencils get pad = 0 (runtime.cpp:16-33).
    rt = Runtime(1, __import__("paper_1704_00693_b200").RuntimeConfig(skew_allowance=0))
    f0 = rt.declare_field("f0", Range.d1(0, 8))
    f1 = rt.declare_field("f1", Range.d1(0, 8))
    ident = rt.declare_stencil("identity", [(0,)])
    three = rt.declare_stencil("three", [(-1,), (0,), (1,)])
    rt.par_loop(KernelHandle(0, "produce", kernels.COPY), Range.d1(0, 8), [ArgSpec(f0, ident, R), ArgSpec(f1, ident, W)])
    rt.par_loop(KernelHandle(1, "consume", kernels.CONSUME_1D), Range.d1(0, 8),
                [ArgSpec(f1, three, R), ArgSpec(f0, ident, W)])
    with pytest.raises(PlanError):
        rt.gpu_plan_pending(__import__("paper_1704_00693_b200").ExecMode.tiled([4, 0, 0]))


def _replay_plan(entry, fn):
    kw = {k: tuple(v) for k, v in entry["kw"].items()}
    gc = C.generate(entry["seed"], dim=entry["dim"], **({"reads_within_logical": True} if "grid" in entry else {}),
                    **kw)
    import paper_1704_00693_b200.runtime as rtmod
    rt = Runtime(entry["dim"])
    rt.upload = lambda ds, a: None  # planning only: no device needed
    C.declare(rt, gc)
    C.enqueue(rt, gc)
    return fn(rt)


def test_plans_match_reference_golden():
    data = json.loads((GOLD / "ref_plans.json").read_text())
    assert len(data) == 140
    for e in data:
        text = _replay_plan(e, lambda rt: rt.plan_pending(e["ts"]))
        assert hashlib.sha256(text.encode()).hexdigest() == e["plan_sha256"], (e["seed"], e["dim"], e["ts"])
        if "plan" in e:
            assert text == e["plan"]


def test_rank_plans_match_reference_golden():
    data = json.loads((GOLD / "ref_rank_plans.json").read_text())
    assert len(data) == 150
    for e in data:
        text = _replay_plan(e, lambda rt: rt.rank_plans_pending(e["grid"], e["ts"]))
        assert hashlib.sha256(text.encode()).hexdigest() == e["text_sha256"], (e["seed"], e["dim"], e["grid"])


def test_plans_match_live_reference(ref_lib):
    for dim, seeds, kw in ((2, range(300, 340), {}), (1, range(400, 420), {"extent": (32, 96)}),
                           (3, range(500, 510), {"extent": (8, 16)})):
        for seed in seeds:
            gc = C.generate(seed, dim=dim, **kw)
            ts = C.random_tile_sizes(seed, dim)
            texts = []
            for rt in (Runtime(dim), ref_lib.RefRuntime(dim)):
                if isinstance(rt, Runtime):
                    rt.upload = lambda ds, a: None
                C.declare(rt, gc)
                C.enqueue(rt, gc)
                texts.append(rt.plan_pending(ts))
            assert texts[0] == texts[1], (dim, seed)


def test_sizer_matches_reference_golden():
    # tile_sizer.cpp:27-81, acceptance criterion 7 inputs
    for e in json.loads((GOLD / "ref_sizer.json").read_text()):
        got = auto_tile_size(e["dim"], e["cache"], e["threads"], e["bpp"], Range(e["dim"], e["extent"]))
        assert list(got) == e["ts"], e


def test_sizer_kats():
    # test_tile_sizer.cpp:19-65
    assert auto_tile_size(1, 64 << 10, 1, 16, Range.d1(0, 100000))[0] == 4096
    assert auto_tile_size(1, 64 << 10, 1, 16, Range.d1(0, 500))[0] == 500
    ts = auto_tile_size(2, 512 << 10, 4, 16, Range.d2(0, 4096, 0, 4096))
    assert ts[:2] == (256, 128)
    assert auto_tile_size(2, 512 << 10, 4, 16, Range.d2(0, 4096, 0, 6))[1] == 4
    assert auto_tile_size(2, 512 << 10, 4, 16, Range.d2(0, 4096, 0, 2))[1] == 2
    assert auto_tile_size(3, 1 << 20, 2, 8, Range.d3(0, 64, 0, 64, 0, 64)) == (64, 32, 32)


def test_signature_sensitivity():
    # test_mesh_core.cpp:204-225: identical structure -> identical signature;
    # bounds, ids and modes change it; scalar params do not (loop.cpp:20-41).
    def sig(hi=8, kid=1, params=(0.25,)):
        rt = Runtime(1)
        ident = rt.declare_stencil("identity", [(0,)])
        f0 = rt.declare_field("f0", Range.d1(0, 8))
        rt.par_loop(KernelHandle(kid, "k", kernels.GEN_SUM, params), Range.d1(0, hi),
                    [ArgSpec(f0, ident, AccessMode.ReadWrite)])
        return rt.signature_pending()
    assert sig() == sig()
    assert sig() != sig(hi=7)
    assert sig() != sig(kid=2)
    assert sig() == sig(params=(0.5,))


def test_par_loop_validation():
    # runtime.cpp:35-92, test_lazy_queue.cpp:134-180
    rt = Runtime(1)
    ident, three, f0, f1 = two_loop(rt)
    with pytest.raises(InvalidArgument):  # write through a multi-point stencil
        rt.par_loop(KernelHandle(2, "w", kernels.COPY), Range.d1(0, 8), [ArgSpec(f0, ident, R), ArgSpec(f1, three, W)])
    with pytest.raises(InvalidArgument):  # racy read-at-offset of a written dataset
        rt.par_loop(KernelHandle(3, "r", kernels.GEN_SUM, (0.1,)), Range.d1(0, 8),
                    [ArgSpec(f0, three, R), ArgSpec(f0, ident, W)])
    # one-point boundary loop reading outside itself is legal
    rt.par_loop(KernelHandle(4, "b", kernels.GEN_SUM, (0.1,)), Range.d1(0, 1), [ArgSpec(f0, rt.declare_stencil(
        "right", [(1,)]), R), ArgSpec(f0, ident, W)])
    with pytest.raises(InvalidArgument):
        rt.par_loop(KernelHandle(-1, "noid", kernels.COPY), Range.d1(0, 8), [ArgSpec(f0, ident, R)])
    with pytest.raises(InvalidArgument):  # unknown body: no CPU fallback
        rt.par_loop(KernelHandle(5, "nobody", 99999), Range.d1(0, 8), [ArgSpec(f0, ident, R)])
    with pytest.raises(InvalidArgument):
        rt.par_loop(KernelHandle(6, "badds", kernels.COPY), Range.d1(0, 8), [ArgSpec(17, ident, R)])
    with pytest.raises(InvalidArgument):
        rt.par_loop(KernelHandle(7, "baddim", kernels.COPY), Range.d2(0, 8, 0, 8), [ArgSpec(f0, ident, R)])
    assert rt.pending_loops() == 3
    with pytest.raises(InvalidArgument):
        rt.fetch_reduction(-1)
    with pytest.raises(InvalidArgument):
        rt.fetch_reduction(42)


def test_par_loop_checks_body_against_declaration():
    # KernelCtx's access checks (kernel_ctx.hpp:58-97) applied at enqueue time
    # by a host probe of the registered body: argument count, access modes,
    # offsets inside the declared stencil, contribute() without a reduction.
    from paper_1704_00693_b200.runtime import AccessError
    rt = Runtime(1)
    ident, three, f0, f1 = two_loop(rt)
    n0 = rt.pending_loops()
    with pytest.raises(AccessError, match="argument index"):  # COPY writes arg 1
        rt.par_loop(KernelHandle(20, "short", kernels.COPY), Range.d1(0, 8), [ArgSpec(f0, ident, R)])
    with pytest.raises(AccessError, match="write through read-only"):
        rt.par_loop(KernelHandle(21, "ro", kernels.COPY), Range.d1(0, 8), [ArgSpec(f0, ident, R), ArgSpec(f1, ident, R)])
    with pytest.raises(AccessError, match="read through write-only"):
        rt.par_loop(KernelHandle(22, "wo", kernels.COPY), Range.d1(0, 8), [ArgSpec(f0, ident, W), ArgSpec(f1, ident, W)])
    with pytest.raises(AccessError, match="offset not in declared stencil"):  # NBR_SUM reads x-1, x+1
        rt.par_loop(KernelHandle(23, "off", kernels.NBR_SUM), Range.d1(0, 8), [ArgSpec(f0, ident, R), ArgSpec(f1, ident, W)])
    with pytest.raises(AccessError, match="contribute"):
        rt.par_loop(KernelHandle(24, "nored", kernels.SUM_READ), Range.d1(0, 8), [ArgSpec(f0, ident, R)])
    assert rt.pending_loops() == n0
    rt.par_loop(KernelHandle(25, "ok", kernels.NBR_SUM), Range.d1(0, 8), [ArgSpec(f0, three, R), ArgSpec(f1, ident, W)])
    assert rt.pending_loops() == n0 + 1


def _plan_ranges(text, dim):
    """TilingPlan::dump text (planner.cpp:234-250) -> flat ranges, T, L."""
    rows = {}
    for line in text.splitlines():
        if not line.startswith("tile="):
            continue
        f = line.split()
        t, l, d = int(f[0][5:]), int(f[1][5:]), int(f[2][2:])
        s, e = f[3].strip("[)").split(",")
        rows[(t, l, d)] = (int(s), int(e))
    T = 1 + max(k[0] for k in rows)
    L = 1 + max(k[1] for k in rows)
    flat = []
    for t in range(T):
        for l in range(L):
            for d in range(3):
                flat += list(rows[(t, l, d)]) if d < dim else [0, 1]
    return flat, T, L


def test_reference_validators_accept_our_plans(ref_lib):
    # §8(f) row 3: the reference's own validate_dependencies and
    # validate_coverage (oracle.cpp:154-284) run on the plans this
    # repository's planner builds; a plan with one loop range shrunk is
    # rejected (the validators are live).
    checked = 0
    for dim, seeds, kw in ((2, range(600, 630), {}), (1, range(700, 710), {"extent": (32, 96)}),
                           (3, range(800, 806), {"extent": (8, 16)})):
        for seed in seeds:
            gc = C.generate(seed, dim=dim, **kw)
            ts = C.random_tile_sizes(seed, dim)
            rt = Runtime(dim)
            rt.upload = lambda ds, a: None
            C.declare(rt, gc)
            C.enqueue(rt, gc)
            flat, T, L = _plan_ranges(rt.plan_pending(ts), dim)
            ref = ref_lib.RefRuntime(dim)
            C.declare(ref, gc)
            C.enqueue(ref, gc)
            n, text = ref.validate_plan_pending(ts, flat, T, L)
            assert n == 0, (dim, seed, text)
            checked += 1
            if seed == seeds[0]:
                # Shrink the first non-empty range by one point: coverage gap.
                bad = list(flat)
                for i in range(0, len(bad), 6):
                    if all(bad[i + 2 * d] < bad[i + 2 * d + 1] for d in range(dim)):
                        bad[i + 1] -= 1
                        break
                ref2 = ref_lib.RefRuntime(dim)
                C.declare(ref2, gc)
                C.enqueue(ref2, gc)
                n2, _ = ref2.validate_plan_pending(ts, bad, T, L)
                assert n2 > 0, (dim, seed)
    assert checked == 46

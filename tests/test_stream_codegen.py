"""CPU checks of the streaming executor's planner and code generator
(csrc/host/tcg_stream.cpp): plans for the BASELINE configs at full size and
for random chains are generated and compiled with NVRTC for sm_100a (no GPU
needed). Catches codegen errors before a GPU run; parity is in
tests/test_gpu_stream.py."""
import re

import pytest

import chains as C
from paper_1704_00693_b200 import Range, Runtime, configs


def _host_only(rt):
    # Field uploads need a device; the plan only needs the declarations.
    rt.upload = lambda *a, **k: None
    rt.upload_box = lambda *a, **k: None
    return rt


def _kernels(text):
    return [l for l in text.splitlines() if l.startswith("kernel ")]


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4"])
def test_config_plans_compile(name):
    dim = 3 if name == "c3" else 2
    rt = _host_only(Runtime(dim))
    if name == "c1":
        configs.HeatC1(rt, 1024).enqueue_chain()
    elif name == "c2":
        configs.HydroC2(rt, 4096).enqueue_step()
    elif name == "c3":
        configs.Jacobi3DC3(rt, 512).enqueue_chain()
    else:
        cg = configs.CgC4(rt, 4096)
        # first chain of an iteration: p-update + matvec with p.q
        from paper_1704_00693_b200 import ArgSpec, KernelHandle, ReduceOp, kernels as K
        f, I = cg.f, cg.ident
        rt.par_loop(KernelHandle(K.CG_P_UPDATE, "p", K.CG_P_UPDATE, (0.5,)), cg.dom,
                    [ArgSpec(f["p"], I, 2), ArgSpec(f["r"], I, 0)])
        rt.par_loop(KernelHandle(K.CG_MATVEC, "mv", K.CG_MATVEC), cg.dom,
                    [ArgSpec(f["p"], cg.star, 0), ArgSpec(f["kx"], cg.west, 0), ArgSpec(f["ky"], cg.south, 0),
                     ArgSpec(f["q"], I, 1)], ReduceOp.Sum)
    out = rt.stream_plan_pending(compile=True)
    ks = _kernels(out)
    assert ks, out
    assert out.count("compiled kernel") == len(ks)
    assert "error" not in out.lower()
    if name == "c2":
        # the whole 13-loop step fuses into one kernel; every dataset is
        # written once per step (HBM traffic = inputs + outputs)
        assert len(ks) == 1 and "loops=[0,13)" in ks[0], ks


@pytest.mark.parametrize("dim,seeds,kw", [(2, range(1, 9), {}), (3, range(9001, 9005), {"extent": (8, 16)})])
def test_random_chain_plans_compile(dim, seeds, kw):
    for seed in seeds:
        gc = C.generate(seed, dim=dim, **kw)
        rt = _host_only(Runtime(dim))
        for i, pts in enumerate(gc.stencils):
            rt.declare_stencil(f"s{i}", [p[:dim] for p in pts])
        dom = Range(dim, sum(([0, e] for e in gc.extent), []))
        for i in range(gc.ndat):
            rt.declare_field(f"f{i}", dom)
        C.enqueue(rt, gc)
        out = rt.stream_plan_pending(compile=True)
        assert out.count("compiled kernel") == len(_kernels(out)), (seed, out[-2000:])


def test_plan_stats_are_consistent():
    rt = _host_only(Runtime(2))
    configs.HydroC2(rt, 4096).enqueue_step()
    k = _kernels(rt.stream_plan_pending())[0]
    computed = int(re.search(r"computed=(\d+)", k).group(1))
    recorded = int(re.search(r"recorded=(\d+)", k).group(1))
    # overlapped halos and pipeline warm-up recompute a few percent
    assert recorded == 13 * 4096 * 4096
    assert recorded <= computed <= 1.2 * recorded


def test_c5_plan_uses_horizontal_runs(monkeypatch):
    # c5's RK stage: [prim] [mass, momentum x3, energy] [update, prim of the
    # next stage]; the last stage ends with [update, kinetic-energy Sum]. The
    # runs are generated as untiled-style kernels (no shared memory); c2's
    # 13-loop step stays one vertically fused kernel.
    monkeypatch.setattr(configs.NsC5, "_initial", lambda self, sb: {})
    rt = _host_only(Runtime(3))
    configs.NsC5(rt, 64).enqueue_step()
    ks = _kernels(rt.stream_plan_pending(compile=True))
    spans = [re.search(r"loops=\[(\d+),(\d+)\)", k).groups() for k in ks]
    assert spans == [("0", "1"), ("1", "6"), ("6", "8"), ("8", "13"), ("13", "15"), ("15", "20"), ("20", "22")]
    assert all("smem=0 " in k for k in ks[1:])
    rt = _host_only(Runtime(2))
    configs.HydroC2(rt, 4096).enqueue_step()
    ks = _kernels(rt.stream_plan_pending())
    assert len(ks) == 1 and "loops=[0,13)" in ks[0]

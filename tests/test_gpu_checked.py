"""The checked executor build (libtcg_checked.so, -DTCG_CHECKED): the
reference's KernelCtx access checks (kernel_ctx.hpp:58-89 -- access mode,
stencil membership of every read offset, allocation bounds) evaluated on the
device by the untiled executor. Correct chains run bit-exact as in the
release build; a body that reads outside its declared stencil traps, where
the reference (and the oracle) raise AccessError. Runs in child processes:
the library is chosen once per process (TCG_LIB) and a trap ends the CUDA
context."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

REPO = Path(__file__).resolve().parent.parent
LIB = REPO / "paper_1704_00693_b200" / "_lib" / "libtcg_checked.so"

PRELUDE = r"""
import sys
sys.path.insert(0, {repo!r}); sys.path.insert(0, {repo!r} + "/oracle")
import numpy as np
import pyoracle
from paper_1704_00693_b200 import AccessMode, ArgSpec, CudaError, ExecMode, KernelHandle, Range, Runtime, configs
from paper_1704_00693_b200.runtime import AccessError
from paper_1704_00693_b200 import kernels as K
"""

GOOD = PRELUDE + r"""
def run(rt, cls, n, steps):
    rt.set_default_mode(ExecMode.untiled())
    c = cls(rt, n)
    reds = []
    for _ in range(steps):
        if hasattr(c, "enqueue_step"):
            reds.append(rt.fetch_reduction(c.enqueue_step()))
        elif hasattr(c, "iterate"):
            c.start() if not reds else None
            c.iterate(); reds.append(c.history[-1])
        else:
            c.enqueue_chain(); rt.flush()
    return c.outputs(), reds

for cls, n, dim, steps in ((configs.HydroC2, 64, 2, 2), (configs.HeatC1, 48, 2, 1), (configs.CgC4, 48, 2, 3),
                           (configs.Jacobi3DC3, 20, 3, 1), (configs.NsC5, 16, 3, 1)):
    fo, ro = run(pyoracle.OracleRuntime(dim), cls, n, steps)
    fg, rg = run(Runtime(dim), cls, n, steps)
    for k in fo:
        if cls is configs.CgC4:  # alpha / beta come from fold-order-dependent dot products
            assert np.allclose(fg[k], fo[k], rtol=1e-9, atol=1e-12), (cls.__name__, k)
        else:
            assert np.array_equal(fg[k], fo[k]), (cls.__name__, k)
    for a, b in zip(rg, ro):
        assert abs(a - b) <= 1e-10 * max(1.0, abs(b)), (cls.__name__, a, b)
print("ok")
"""

BAD = PRELUDE + r"""
def bad_loop(rt):
    dom = Range(2, [0, 32, 0, 32])
    pt = rt.declare_stencil("point", [(0, 0)])
    u = rt.declare_field("u", dom)
    v = rt.declare_field("v", dom)
    # heat_lap reads u at the 5-point star, but the loop declares a point.
    rt.par_loop(KernelHandle(K.HEAT_LAP, "heat_lap", K.HEAT_LAP), dom,
                [ArgSpec(u, pt, AccessMode.Read), ArgSpec(v, pt, AccessMode.Write)])
    rt.flush(ExecMode.untiled())
    if hasattr(rt, "synchronize"):
        rt.synchronize()

try:
    bad_loop(pyoracle.OracleRuntime(2))
    print("oracle did not raise")
except Exception as e:
    print("oracle raised:", e)
try:
    bad_loop(Runtime(2))
    print("device did not trap")
except CudaError as e:
    print("device trapped")
except AccessError as e:
    print("enqueue refused:", e)
"""


def _child(code, **extra):
    env = {**os.environ, "TCG_LIB": str(LIB), **extra}
    return subprocess.run([sys.executable, "-c", code.format(repo=str(REPO))], env=env, capture_output=True,
                          text=True, timeout=600)


def test_checked_build_runs_correct_chains_bit_exact():
    assert LIB.exists(), "checked library not built"
    r = _child(GOOD)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout[-2000:] + r.stderr[-4000:]


def test_checked_build_traps_read_outside_stencil():
    # With the host probe of par_loop switched off (test hook) the fault
    # reaches the device, where the checked build reports and traps it.
    r = _child(BAD, TCG_SKIP_BODY_PROBE="1")
    out = r.stdout + r.stderr
    assert "oracle raised: offset not in declared stencil" in r.stdout, out[-4000:]
    assert "device trapped" in r.stdout, out[-4000:]
    assert "offset is not a point of the argument's stencil" in out, out[-4000:]


def test_enqueue_refuses_read_outside_stencil():
    # Default: par_loop's host probe of the registered body raises the
    # reference's AccessError before anything is queued (kernel_ctx.hpp:58-73).
    r = _child(BAD)
    out = r.stdout + r.stderr
    assert "enqueue refused:" in r.stdout and "offset not in declared stencil" in r.stdout, out[-4000:]

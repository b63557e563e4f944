"""GPU parity of the opt-in executor variants that are selected once per
process by environment (so each case runs in a child process): the staged
2.5D 3D walk (TCG_STAGED3=1, shared-memory plane rings filled by bulk
copies), the item-graph form of the L2-tiled executor (TCG_L2_GRAPH=1), and
the untiled walk without CUDA graphs / L2 prefetch. Same bar as
test_gpu_parity.py: fields bit-exact against the oracle, Sum to 1e-12."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

REPO = Path(__file__).resolve().parent.parent

CHILD = r"""
import sys
sys.path.insert(0, {repo!r}); sys.path.insert(0, {repo!r} + "/oracle"); sys.path.insert(0, {repo!r} + "/tests")
import numpy as np
import pyoracle
import chains as C
from paper_1704_00693_b200 import ExecMode, Runtime, configs
mode = {{"untiled": ExecMode.untiled(), "tiled": ExecMode.tiled((0, 0, 0))}}[{mode!r}]

def c3(rt):
    rt.set_default_mode(mode)
    c = configs.Jacobi3DC3(rt, 29)
    c.enqueue_chain(); rt.flush()
    return c.outputs(), []

def c5(rt):
    rt.set_default_mode(mode)
    c = configs.NsC5(rt, 16)
    kes = [rt.fetch_reduction(c.enqueue_step()) for _ in range(2)]
    return c.outputs(), kes

def c2(rt):
    rt.set_default_mode(mode)
    c = configs.HydroC2(rt, 96)
    mins = [rt.fetch_reduction(c.enqueue_step()) for _ in range(2)]
    return c.outputs(), mins

for name, run in (("c3", c3), ("c5", c5), ("c2", c2)):
    fo, ro = run(pyoracle.OracleRuntime(3 if name != "c2" else 2))
    fg, rg = run(Runtime(3 if name != "c2" else 2))
    for k in fo:
        assert np.array_equal(fg[k], fo[k]), (name, k)
    for a, b in zip(rg, ro):
        assert abs(a - b) <= 1e-12 * abs(b), (name, a, b)
# random 3D chains (the reference's chain_gen shapes) on the same variant
for seed in range(9001, 9007):
    ch = C.generate(seed, 3, extent=(8, 16))
    want = C.run(pyoracle.OracleRuntime(3), ch, mode)
    got = C.run(Runtime(3), ch, mode)
    C.assert_same(got, want, f"seed {{seed}}")
print("ok")
"""


@pytest.mark.parametrize("env,mode", [
    ({"TCG_STAGED3": "1"}, "untiled"),
    ({"TCG_STAGED3": "1", "TCG_S3_D": "1", "TCG_S3_ZR": "5"}, "untiled"),
    ({"TCG_GRAPHS": "0", "TCG_PREFETCH_L2": "0"}, "untiled"),
    ({"TCG_L2_GRAPH": "1"}, "tiled"),
], ids=["staged3", "staged3_shallow", "no_graphs_no_prefetch", "l2_item_graph"])
def test_variant_matches_oracle(env, mode):
    code = CHILD.format(repo=str(REPO), mode=mode)
    r = subprocess.run([sys.executable, "-c", code], env={**os.environ, **env}, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout[-2000:] + r.stderr[-4000:]

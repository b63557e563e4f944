"""Tiny 3D chains through the untiled executor (staged walk) vs the oracle."""
import sys, time
from pathlib import Path
REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO)); sys.path.insert(0, str(REPO / "oracle"))
import numpy as np
import pyoracle
from paper_1704_00693_b200 import ExecMode, Runtime, configs
n = int(sys.argv[1]) if len(sys.argv) > 1 else 24
def run(rt):
    c = configs.Jacobi3DC3(rt, n)
    rt.set_default_mode(ExecMode.untiled())
    c.enqueue_chain(); rt.flush()
    return c.outputs()
t = time.time()
got = run(Runtime(3)); print("gpu done", time.time() - t, flush=True)
want = run(pyoracle.OracleRuntime(3))
print("equal", all(np.array_equal(got[k], want[k]) for k in want), flush=True)

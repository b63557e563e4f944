"""Host-side cost per chain (enqueue + flush) on a tiny grid, and device time."""
import sys, time
from pathlib import Path
REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
import bench
from paper_1704_00693_b200 import Runtime, ExecMode
for cfg_name, n in (("c1", 64), ("c1", 1024), ("c2", 96), ("c4", 96)):
    rt = Runtime(2)
    rt.set_default_mode(ExecMode.untiled())
    cfg = bench.make_config(cfg_name, rt, n=n)
    st = bench.Step(cfg_name, cfg, rt)
    for _ in range(5):
        st()
    rt.synchronize()
    t = time.perf_counter()
    for _ in range(200):
        st()
    host = (time.perf_counter() - t) / 200
    rt.synchronize()
    wall = (time.perf_counter() - t) / 200
    print(f"{cfg_name} n={n}: host {host*1e6:.1f} us/step, wall {wall*1e6:.1f} us/step", flush=True)

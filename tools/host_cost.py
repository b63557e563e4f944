"""Host-side cost per step split into enqueue (par_loop calls) and the flush
(fetch_reduction / flush incl. the device run) on tiny grids."""
import sys, time
from pathlib import Path
REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
import bench
from paper_1704_00693_b200 import Runtime, ExecMode
for cfg_name, n in (("c1", 64), ("c2", 96), ("c2", 4096), ("c4", 96)):
    rt = Runtime(2)
    rt.set_default_mode(ExecMode.untiled())
    cfg = bench.make_config(cfg_name, rt, n=n)
    st = bench.Step(cfg_name, cfg, rt)
    for _ in range(5):
        st()
    rt.synchronize()
    te = tf = 0.0
    N = 100 if n > 1000 else 300
    for _ in range(N):
        t0 = time.perf_counter()
        if cfg_name == "c2":
            h = cfg.enqueue_step(); t1 = time.perf_counter(); rt.fetch_reduction(h)
        elif cfg_name == "c1":
            cfg.enqueue_chain(); t1 = time.perf_counter(); rt.flush(); rt.synchronize()
        else:
            t1 = t0; cfg.iterate()
        t2 = time.perf_counter()
        te += t1 - t0; tf += t2 - t1
    print(f"{cfg_name} n={n}: enqueue {te/N*1e6:.1f} us, flush+run {tf/N*1e6:.1f} us per step", flush=True)

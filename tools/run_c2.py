"""Dev helper: time c2 (or other configs) through the Python API with CUDA events.
python tools/run_c2.py [untiled|tiled|auto] [n] [steps]"""
import sys, time
sys.path[:0] = ['.', 'oracle', 'tests']
import torch
from paper_1704_00693_b200 import ExecMode, Runtime, RuntimeConfig, configs
mode_name = sys.argv[1] if len(sys.argv) > 1 else "auto"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
mode = {"untiled": ExecMode.untiled(), "auto": ExecMode.tiled_auto()}.get(mode_name)
if mode is None:
    ts = [int(v) for v in mode_name.split(",")]
    mode = ExecMode.tiled(ts)
rt = Runtime(2)
rt.set_default_mode(mode)
h = configs.HydroC2(rt, n)
rt.fetch_reduction(h.enqueue_step())
rt.synchronize()
t = time.time()
for _ in range(steps):
    rt.fetch_reduction(h.enqueue_step())
rt.synchronize()
dt = (time.time() - t) / steps
print(mode_name, n, f"{dt*1e3:.3f} ms/step {h.cell_updates_per_step()/dt:.3e} cu/s {h.bytes_per_step()/dt/1e9:.1f} GB/s-eff")
print(rt.report_text().replace("\n", " ")[:400])

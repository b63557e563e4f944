"""Dev helper: time a config through the Python API (device time via CUDA events).
python tools/run_cfg.py CONFIG MODE [N] [STEPS]   CONFIG in c1,c2,c3,c4; MODE untiled|auto|X,Y[,Z]"""
import sys, time
sys.path[:0] = ['.', 'oracle', 'tests']
import torch
import bench
from paper_1704_00693_b200 import ExecMode, Runtime
cfg_name, mode_name = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3] != '-' else None
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
mode = {"untiled": ExecMode.untiled(), "auto": ExecMode.tiled_auto()}.get(mode_name)
if mode is None:
    mode = ExecMode.tiled([int(v) for v in mode_name.split(",")])
rt = Runtime(3 if cfg_name == "c3" else 2)
rt.set_default_mode(mode)
cfg = bench.make_config(cfg_name, rt, n)
st = bench.Step(cfg_name, cfg, rt)
st(); st()
ms = bench.time_steps(rt, st, steps) / steps
cu, by = st.cell_updates(), st.algorithmic_bytes()
rep = rt.report_text().replace("\n", " ")
print(f"{cfg_name} {mode_name} n={n} {ms:.3f} ms/step {cu/ms/1e-3:.3e} cu/s {by/ms/1e6:.0f} GB/s-eff | {rep[:220]}")

"""A/B timing of executor modes in one process (c2 by default)."""
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
import bench  # noqa: E402
import torch  # noqa: E402
from paper_1704_00693_b200 import Runtime  # noqa: E402

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "c2"
order = sys.argv[2].split(";") if len(sys.argv) > 2 else ["untiled", "auto", "untiled", "auto"]
steps = int(__import__("os").environ.get("AB_STEPS", "50"))
for mname in order:
    rt = Runtime(3 if cfg_name in ("c3", "c5") else 2)
    rt.set_default_mode(bench.parse_mode(mname))
    cfg = bench.make_config(cfg_name, rt)
    st = bench.Step(cfg_name, cfg, rt)
    for _ in range(6):
        st()
    ms = bench.time_steps(rt, st, steps)
    keys = ("executor", "tile_sizes", "subchains", "ctas", "grid_barriers", "max_skew")
    rep = {l.split("=")[0]: l.split("=")[1] for l in rt.report_text().splitlines() if "=" in l}
    print(f"{mname:12s} {ms / steps:.4f} ms/step  " + " ".join(f"{k}={rep.get(k)}" for k in keys), flush=True)
    del st, cfg, rt
    torch.cuda.empty_cache()

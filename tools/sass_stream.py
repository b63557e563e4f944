#!/usr/bin/env python
"""Offline look at a generated streaming kernel (no GPU): plans a config's
chain, compiles kernel K of the plan with nvcc for sm_100a and prints ptxas
resource usage plus the SASS instruction mix of the steady-state phase.

    python tools/sass_stream.py c3 [--kernel 0] [--choice nt,bx,by,ntx,seg,maxloops,minb,pf] [--dump out.sass]
Environment switches of the generator (TCG_STREAM_*) apply."""
import argparse, collections, os, re, subprocess, sys, tempfile
from pathlib import Path
REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO)); sys.path.insert(0, str(REPO / "tests"))
from paper_1704_00693_b200 import Runtime, configs

def plan(name, choice):
    dim = 3 if name in ("c3", "c5") else 2
    rt = Runtime(dim); rt.upload = lambda *a, **k: None; rt.upload_box = lambda *a, **k: None
    if choice: rt.set_stream_choice(*choice)
    if name == "c1": configs.HeatC1(rt, 1024).enqueue_chain()
    elif name == "c2": configs.HydroC2(rt, 4096).enqueue_step()
    elif name == "c3": configs.Jacobi3DC3(rt, 512).enqueue_chain()
    elif name == "c5": configs.NsC5.__init__ = _ns_init(configs.NsC5.__init__); configs.NsC5(rt, 768).enqueue_step()
    return rt.stream_plan_pending(source=True)

def _ns_init(orig):
    def init(self, rt, n=768, **kw):
        import numpy as np
        self._initial = lambda sb: {}
        orig(self, rt, n, **kw)
    return init

def main():
    ap = argparse.ArgumentParser(); ap.add_argument("config"); ap.add_argument("--kernel", type=int, default=0)
    ap.add_argument("--choice", default=""); ap.add_argument("--dump", default="")
    a = ap.parse_args()
    choice = [int(x) for x in a.choice.split(",")] if a.choice else None
    text = plan(a.config, choice)
    parts = re.split(r"----- source kernel (\d+)\n", text)
    print("\n".join(l for l in parts[0].splitlines() if l.startswith("kernel ")))
    srcs = {int(parts[i]): parts[i + 1] for i in range(1, len(parts), 2)}
    src = srcs[a.kernel]
    with tempfile.TemporaryDirectory() as td:
        cu = Path(td) / "k.cu"; cu.write_text(src)
        cubin = Path(td) / "k.cubin"
        r = subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-fmad=false", "-std=c++17", "-lineinfo",
                            "--extra-device-vectorization", "-Xptxas", "-v", "-cubin", "-o", str(cubin), str(cu),
                            f"-I{REPO / 'paper_1704_00693_b200/csrc/kernels'}"], capture_output=True, text=True)
        print("\n".join(l for l in (r.stdout + r.stderr).splitlines() if "registers" in l or "spill" in l or "error" in l))
        sass = subprocess.run(["cuobjdump", "-sass", str(cubin)], capture_output=True, text=True).stdout
    if a.dump: Path(a.dump).write_text(sass)
    ins = [l.split(";")[0].strip() for l in sass.splitlines() if re.match(r"\s+/\*[0-9a-f]{4,}\*/", l)]
    ins = [re.sub(r"/\*[0-9a-f]+\*/\s*", "", i).strip() for i in ins]
    bars = [i for i, s in enumerate(ins) if s.startswith("BAR.SYNC") or " BAR.SYNC" in s]
    print("instructions:", len(ins), "barriers at", bars[:12])
    if len(bars) >= 3:
        seg = ins[bars[1]:bars[2]]
        mix = collections.Counter(re.sub(r"^@!?U?P\d+\s+", "", s).split()[0].split(".")[0] for s in seg)
        print("phase 1:", len(seg), "instructions;", ", ".join(f"{k} {v}" for k, v in mix.most_common(16)))

if __name__ == "__main__":
    main()

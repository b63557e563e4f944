"""Builds an experiment variant of the executor library with extra nvcc
defines for one CUDA source: python tools/build_variant.py NAME SRC -DX=Y ..."""
import subprocess
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
from paper_1704_00693_b200 import build as b  # noqa: E402

name, src, defs = sys.argv[1], sys.argv[2], sys.argv[3:]
b.build()
objs = []
for s in b.HOST_SRCS + b.CUDA_SRCS:
    o = b.OBJ_DIR / (s.replace("/", "_") + ".o")
    if s == src:
        o = b.OBJ_DIR / (s.replace("/", "_") + f".{name}.o")
        subprocess.run([b.NVCC, *b.NVCCFLAGS, *defs, "-c", str(b.CSRC / s), "-o", str(o)], check=True,
                       capture_output=True)
    objs.append(str(o))
out = b.LIB_DIR / f"libtcg_{name}.so"
subprocess.run([b.NVCC, *b.ARCH, "-shared", "-o", str(out), *objs, "-lcuda", "-ldl"], check=True)
print(out)

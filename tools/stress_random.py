#!/usr/bin/env python
"""Ad-hoc GPU stress (not part of the suite): many random chains (the
reference's chain_gen shapes) under the streaming executor and tiled_auto vs
the CPU oracle.  python tools/stress_random.py [first_seed] [count]"""
import sys
from pathlib import Path
REPO = Path(__file__).resolve().parent.parent
sys.path[:0] = [str(REPO), str(REPO / "oracle"), str(REPO / "tests")]
import chains as C
import pyoracle
from paper_1704_00693_b200 import ExecMode, Runtime

first = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
count = int(sys.argv[2]) if len(sys.argv) > 2 else 200
pyoracle.load_oracle()
bad = 0
for i in range(count):
    seed = first + i
    dim = 3 if i % 4 == 3 else 2
    kw = {"extent": (8, 18)} if dim == 3 else {}
    gc = C.generate(seed, dim=dim, **kw)
    want = C.run(pyoracle.OracleRuntime(dim), gc, None)
    for name, mode in (("stream", ExecMode.stream()), ("auto", ExecMode.tiled_auto())):
        try:
            got = C.run(Runtime(dim), gc, mode)
            C.assert_same(got, want, f"{name} seed{seed}")
        except Exception as e:  # noqa: BLE001
            bad += 1
            print("FAIL", name, seed, dim, str(e)[:300], flush=True)
print(f"stress: {count} chains x 2 modes, {bad} failures")

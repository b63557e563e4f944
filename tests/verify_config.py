#!/usr/bin/env python
"""TEST INFRASTRUCTURE: the reference CLI's --verify / --report conventions
(proj/tools/tilechain_cli.cpp:85-92, :133-136) for the BASELINE configs.

    python tests/verify_config.py --config c2 [--mode auto|stream|untiled] [--n N] [--steps K] [--report]

Runs the config at a reduced size on the GPU (the product, through the C-ABI)
and on the CPU oracle, prints max_abs_diff / mismatched fields / reduction
max_rel and `verify=pass|fail` (exit code 3 on a mismatch), and with --report
the product's last ExecutionReport. Lives under tests/: it executes oracle/,
which the product path (and bench.py's timed legs) never does."""
from __future__ import annotations

import argparse
import sys
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent.parent
sys.path[:0] = [str(REPO), str(REPO / "oracle")]


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--mode", default="auto")
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--report", action="store_true")
    args = ap.parse_args()
    import pyoracle
    import bench
    from paper_1704_00693_b200 import Runtime

    n = args.n or {"c1": 128, "c2": 160, "c3": 40, "c4": 128, "c5": 24}[args.config]
    dim = 3 if args.config in ("c3", "c5") else 2

    def run(rt):
        c = bench.make_config(args.config, rt, n=n)
        st = bench.Step(args.config, c, rt, host="python")
        for _ in range(args.steps):
            st()
        return c.outputs(), list(getattr(c, "history", [])), rt

    pyoracle.load_oracle()
    fo, ro, _ = run(pyoracle.OracleRuntime(dim))
    rg = Runtime(dim)
    rg.set_default_mode(bench.parse_mode(args.mode))
    fg, rgv, _ = run(rg)
    # c4's fields depend on alpha / beta, quotients of Sum reductions whose fold
    # order differs from the sequential oracle's: compared to 1e-9 there;
    # everywhere else bit for bit.
    same = (lambda a, b: np.allclose(a, b, rtol=1e-9, atol=1e-12)) if args.config == "c4" else np.array_equal
    bad = [k for k in fo if not same(fo[k], fg[k])]
    max_abs = max(float(np.max(np.abs(fo[k] - fg[k]))) for k in fo)
    rel = max([abs(a - b) / max(abs(b), 1e-300) for a, b in zip(rgv, ro)], default=0.0)
    if args.report:
        sys.stdout.write(rg.report_text())
    print(f"config={args.config} n={n} steps={args.steps} mode={args.mode}")
    print(f"max_abs_diff={max_abs:.17g}")
    print(f"mismatched_fields={bad}")
    print(f"reduction_max_rel={rel:.17g}")
    ok = not bad and rel <= 1e-10
    print(f"verify={'pass' if ok else 'fail'}")
    return 0 if ok else 3


if __name__ == "__main__":
    sys.exit(main())

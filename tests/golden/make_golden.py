"""Generates tests/golden/*.json from the UNMODIFIED reference library
(oracle/_ref/libtcref.so, built from /root/reference by oracle/Makefile).

    python tests/golden/make_golden.py

Fixtures (small, committed) let the CPU tests pin this project's planner,
rank planner, halo analysis and sizer, and the oracle restatement, against
the reference on machines where /root/reference is absent (the GPU box).
"""
from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path[:0] = [str(REPO), str(REPO / "oracle"), str(REPO / "tests")]

import chains as C  # noqa: E402
import pyoracle as po  # noqa: E402


def sha(arrs) -> str:
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(a, dtype=np.float64).tobytes())
    return h.hexdigest()


def plans():
    out = []
    for dim, seeds, kw in ((1, range(5001, 5041), {"extent": (32, 96)}), (2, range(1, 81), {}),
                           (3, range(9001, 9021), {"extent": (8, 16)})):
        for seed in seeds:
            gc = C.generate(seed, dim=dim, **kw)
            ts = C.random_tile_sizes(seed, dim)
            rt = po.RefRuntime(dim)
            C.declare(rt, gc)
            C.enqueue(rt, gc)
            text = rt.plan_pending(ts)
            out.append({"seed": seed, "dim": dim, "kw": {k: list(v) for k, v in kw.items()}, "ts": ts,
                        "plan": text})
    return out


def rank_plans():
    out = []
    for dim, seeds, grids, kw in ((1, range(7001, 7021), ([2, 1, 1], [3, 1, 1]), {"extent": (32, 96)}),
                                  (2, range(7101, 7131), ([2, 1, 1], [2, 2, 1], [1, 3, 1]), {}),
                                  (3, range(7201, 7211), ([1, 1, 2], [2, 1, 2]), {"extent": (8, 16)})):
        for seed in seeds:
            gc = C.generate(seed, dim=dim, reads_within_logical=True, **kw)
            ts = C.random_tile_sizes(seed, dim)
            for g in grids:
                rt = po.RefRuntime(dim)
                C.declare(rt, gc)
                C.enqueue(rt, gc)
                out.append({"seed": seed, "dim": dim, "kw": {k: list(v) for k, v in kw.items()}, "ts": ts,
                            "grid": g, "text": rt.rank_plans_pending(g, ts)})
    return out


def sizer():
    g = np.random.Generator(np.random.PCG64(7))
    out = []
    for i in range(200):
        dim = int(g.integers(1, 4))
        cache = int(g.integers(2, 9)) << 20
        threads = [1, 2, 4, 6, 8, 12, 16][int(g.integers(0, 7))]
        bpp = 8 * int(g.integers(1, 7))
        if dim == 1:
            ext = [0, int(g.integers(1000, 1000001)), 0, 1, 0, 1]
        elif dim == 2:
            ext = [0, int(g.integers(2048, 6145)), 0, int(g.integers(1024, 4097)), 0, 1]
        else:
            ext = [0, int(g.integers(128, 513)), 0, int(g.integers(128, 513)), 0, int(g.integers(128, 513))]
        out.append({"dim": dim, "cache": cache, "threads": threads, "bpp": bpp, "extent": ext,
                    "ts": list(po.ref_auto_tile_size(dim, cache, threads, bpp, ext))})
    return out


def executions():
    """Reference runtime outputs (threads=1, untiled and tiled) on random chains."""
    out = []
    for dim, seeds, kw in ((1, range(5001, 5021), {"extent": (32, 96)}), (2, range(1, 41), {}),
                           (3, range(9001, 9011), {"extent": (8, 16)})):
        for seed in seeds:
            gc = C.generate(seed, dim=dim, **kw)
            fields, reds = C.run(po.RefRuntime(dim), gc, None)
            out.append({"seed": seed, "dim": dim, "kw": {k: list(v) for k, v in kw.items()},
                        "fields_sha256": sha(fields), "reductions": [[v, op] for v, op in reds]})
    return out


def apps():
    res = {}
    for copy in (True, False):
        res[f"jacobi_64_10_{'copy' if copy else 'noncopy'}"] = sha([po.ref_app_jacobi(64, 64, 10, copy)])
    f, mon = po.ref_app_minihydro(48, 48, 3)
    res["minihydro_48_3"] = sha([f])
    res["minihydro_48_3_monitors"] = mon.tolist()
    return res


def _hashed(entries, key, keep=6):
    """Keep full text for the first few entries, a SHA-256 for all."""
    for i, e in enumerate(entries):
        e[key + "_sha256"] = hashlib.sha256(e[key].encode()).hexdigest()
        if i >= keep:
            del e[key]
    return entries


if __name__ == "__main__":
    (HERE / "ref_plans.json").write_text(json.dumps(_hashed(plans(), "plan")))
    (HERE / "ref_rank_plans.json").write_text(json.dumps(_hashed(rank_plans(), "text")))
    (HERE / "ref_sizer.json").write_text(json.dumps(sizer()))
    (HERE / "ref_exec.json").write_text(json.dumps(executions()))
    (HERE / "ref_apps.json").write_text(json.dumps(apps(), indent=1))
    print("golden fixtures written to", HERE)

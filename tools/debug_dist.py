"""Debug: distributed tiled mismatch. Runs a random chain on a rank grid and,
per rank, the rank-local chain in isolation (fields declared over the owned
box so the allocation equals the rank allocation) tiled vs untiled."""
import sys
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent.parent
sys.path[:0] = [str(REPO), str(REPO / "tests"), str(REPO / "oracle")]
import chains as C  # noqa: E402
import pyoracle  # noqa: E402
from paper_1704_00693_b200 import ExecMode, KernelHandle, Range, Runtime, kernels  # noqa: E402

seed = int(sys.argv[1]) if len(sys.argv) > 1 else 31
grid = tuple(int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "1,2,1").split(","))
dim = int(sys.argv[3]) if len(sys.argv) > 3 else 2
gc = C.generate(seed, dim=dim, min_loops=2, max_loops=6, extent=(40, 72), max_radius=2)
print("extent", gc.extent, "loops", len(gc.loops))
for l in gc.loops:
    print("  loop", l)
want = C.run(pyoracle.OracleRuntime(dim), gc, None)
for mname, mode in [("untiled", ExecMode.untiled()), ("tiled", ExecMode.tiled((0, 0, 0)))]:
    rt = Runtime(dim)
    rt.set_rank_grid(grid)
    got = C.run(rt, gc, mode)
    for i, (a, b) in enumerate(zip(got[0], want[0])):
        bad = np.argwhere(a != b)
        if len(bad):
            print(mname, "dataset", i, "bad", len(bad), "rows(y idx)", sorted(set(bad[:, 0].tolist()))[:20],
                  "cols", sorted(set(bad[:, -1].tolist()))[:10])
    print(mname, "reds", got[1], want[1])

# Schedule (host only) and isolated rank-local chains.
sch = Runtime(dim)
sch.set_rank_grid(grid)
for i, pts in enumerate(gc.stencils):
    sch.declare_stencil(f"s{i}", [p[:dim] for p in pts])
dom = Range(dim, sum(([0, e] for e in gc.extent), []))
for i in range(gc.ndat):
    sch.declare_field(f"f{i}", dom)
C.enqueue(sch, gc)
s = sch.schedule_pending()
print("msgs", s["msgs"])
ora0 = pyoracle.OracleRuntime(dim)
ids0 = C.declare(ora0, gc)
init = [ora0.download(d) for d in ids0]
galloc = ora0.alloc_range(0)
for r, info in s["ranks"].items():
    own = sch.rank_owned(r)
    print("rank", r, "owned", own.lohi[:2 * dim], "loops", info["loops"])
    outs = {}
    for mname, mode in [("untiled", ExecMode.untiled()), ("tiled", ExecMode.tiled((0, 0, 0)))]:
        rt = Runtime(dim)
        for i, pts in enumerate(gc.stencils):
            rt.declare_stencil(f"s{i}", [p[:dim] for p in pts])
        ids = [rt.declare_field(f"f{i}", own) for i in range(gc.ndat)]
        for i, ds in enumerate(ids):
            al = rt.alloc_range(ds)
            arr = np.zeros(al.shape())
            sl_l, sl_g = [], []
            for d in reversed(range(dim)):
                lo, hi = max(al.start(d), galloc.start(d)), min(al.end(d), galloc.end(d))
                sl_l.append(slice(lo - al.start(d), hi - al.start(d)))
                sl_g.append(slice(lo - galloc.start(d), hi - galloc.start(d)))
            arr[tuple(sl_l)] = init[i][tuple(sl_g)]
            rt.upload(ds, arr)
        for l, ((lohi, args, red), box) in enumerate(zip(gc.loops, info["loops"])):
            if any(hi <= lo for lo, hi in box):
                continue
            total = sum(len(gc.stencils[st]) for ds, st, m in args if m == 0)
            scale = 1.0
            while scale * max(total, 1) > 0.5:
                scale *= 0.5
            rt.par_loop(KernelHandle(l, f"gen{l}", kernels.GEN_SUM, (scale,)),
                        Range(dim, sum(([a, b] for a, b in box), [])), args, red)
        rt.flush(mode)
        print("  ", mname, rt.report_text().replace("\n", " ")[:300])
        outs[mname] = [rt.download(ds) for ds in ids]
    for i, (a, b) in enumerate(zip(outs["tiled"], outs["untiled"])):
        bad = np.argwhere(a != b)
        if len(bad):
            print("   isolated rank", r, "dataset", i, "tiled!=untiled at", len(bad), "first", bad[:4].tolist())

"""Multi-process (gloo, world_size 2, CPU) tests of the distributed path's host
logic: the product's schedule (rank plans, halo depths, message list in the
reference's exchange order, reduction masks, rank-order fold) drives a rank of
the oracle per process (tests/dist_harness.py); the gathered result must equal
a single-process oracle run bit for bit (sums to 1e-12), as the reference's
DistContext must equal its shared-memory run (acceptance.cpp:263-344)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import chains as C


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from dist_harness import DistOracleRank

        out = case(lambda dim, grid, **kw: DistOracleRank(dim, grid, rank, world, **kw))
        q.put((rank, "ok", out if rank == 0 else None))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback

        q.put((rank, "err", traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def run_world(case, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        r, status, payload = q.get(timeout=240)
        res[r] = (status, payload)
    for p in procs:
        p.join(timeout=60)
    for r, (status, payload) in res.items():
        assert status == "ok", f"rank {r}:\n{payload}"
    return res[0][1]


# ---- cases (module-level so spawn can pickle them) ------------------------------

def _logical(arr, alloc, ext):
    sl = tuple(slice(-alloc.start(d), -alloc.start(d) + ext[d]) for d in reversed(range(len(ext))))
    return arr[sl]


def case_random_chains(make_rt, seeds=(1, 2, 3, 4, 5, 6), dim=2, split=1, repeats=2):
    outs = []
    for seed in seeds:
        gc = C.generate(seed, dim=dim, min_loops=2, max_loops=6, extent=(40, 64), max_radius=2)
        grid = [1, 1, 1]
        grid[split] = 2
        rt = make_rt(dim, grid)
        ids = C.declare(rt, gc)
        reds = []
        for _ in range(repeats):
            handles = C.enqueue(rt, gc)
            rt.flush()
            reds += [(rt.fetch_reduction(h), op) for h, op in handles]
        fields = [_logical(rt.download(ds), rt.alloc_range(ds), gc.extent) for ds in ids]
        outs.append((fields, reds, rt.halo_messages))
    return outs


def case_random_chains_3d(make_rt):
    return case_random_chains(make_rt, seeds=(11, 12, 13), dim=3, split=2)


def case_heat(make_rt):
    from paper_1704_00693_b200 import configs

    rt = make_rt(2, [1, 2, 1])
    h = configs.HeatC1(rt, 48)
    for _ in range(2):
        h.enqueue_chain(steps=4)
        rt.flush()
    return _logical(rt.download(h.u), rt.alloc_range(h.u), [48, 48]), rt.halo_messages


def case_hydro(make_rt):
    from paper_1704_00693_b200 import configs

    rt = make_rt(2, [1, 2, 1])
    hc = configs.HydroC2(rt, 64)
    mins = [rt.fetch_reduction(hc.enqueue_step()) for _ in range(2)]
    return {i: _logical(rt.download(ds), rt.alloc_range(ds), [64, 64]) for i, ds in enumerate(hc.d)}, mins


def _oracle_random(seeds, dim, repeats=2):
    import pyoracle

    outs = []
    for seed in seeds:
        gc = C.generate(seed, dim=dim, min_loops=2, max_loops=6, extent=(40, 64), max_radius=2)
        rt = pyoracle.OracleRuntime(dim)
        ids = C.declare(rt, gc)
        reds = []
        for _ in range(repeats):
            handles = C.enqueue(rt, gc)
            reds += [(rt.fetch_reduction(h), op) for h, op in handles]
        outs.append(([_logical(rt.download(ds), rt.alloc_range(ds), gc.extent) for ds in ids], reds))
    return outs


def _compare(got, want):
    for (gf, gr, _), (wf, wr) in zip(got, want):
        C.assert_same((gf, gr), (wf, wr), "dist")


def test_random_chains_2d_two_ranks(oracle_lib):
    got = run_world(case_random_chains)
    _compare(got, _oracle_random((1, 2, 3, 4, 5, 6), 2))
    assert sum(m for _, _, m in got) > 0  # halos actually moved


def test_random_chains_3d_two_ranks(oracle_lib):
    got = run_world(case_random_chains_3d)
    _compare(got, _oracle_random((11, 12, 13), 3))


def test_heat_two_ranks_one_exchange_per_chain(oracle_lib):
    from paper_1704_00693_b200 import configs

    u, msgs = run_world(case_heat)
    ora = oracle_lib.OracleRuntime(2)
    h = configs.HeatC1(ora, 48)
    for _ in range(2):
        h.enqueue_chain(steps=4)
    want = _logical(ora.download(h.u), ora.alloc_range(h.u), [48, 48])
    assert np.array_equal(u, want)
    # Deep halo: only u crosses the seam (v is written before it is read),
    # once per chain and direction (the reference's "fewer, larger messages",
    # acceptance.cpp:348-386): rank 0 sends one and receives one per chain.
    assert msgs == 4


def test_hydro_two_ranks(oracle_lib):
    from paper_1704_00693_b200 import configs

    fields, mins = run_world(case_hydro)
    ora = oracle_lib.OracleRuntime(2)
    hc = configs.HydroC2(ora, 64)
    want_mins = [ora.fetch_reduction(hc.enqueue_step()) for _ in range(2)]
    assert mins == want_mins
    for i, ds in enumerate(hc.d):
        assert np.array_equal(fields[i], _logical(ora.download(ds), ora.alloc_range(ds), [64, 64])), i


def _ref_msgs(text):
    out = []
    for line in text.splitlines():
        if line.startswith("msg "):
            kv = dict(x.split("=") for x in line.split()[1:])
            out.append((int(kv["from"]), int(kv["to"]), int(kv["ds"]), int(kv["dim"]), int(kv["dir"]),
                        int(kv["points"])))
    return out


@pytest.mark.parametrize("seed,dim,grid,ts", [
    (21, 2, (1, 2, 1), (1 << 20,) * 3), (22, 2, (1, 3, 1), (1 << 20,) * 3), (23, 2, (2, 2, 1), (1 << 20,) * 3),
    (24, 2, (1, 2, 1), (16, 8, 1)), (25, 3, (1, 1, 2), (1 << 20,) * 3), (26, 3, (1, 2, 2), (1 << 20,) * 3),
    (27, 1, (3, 1, 1), (1 << 20,) * 3), (28, 2, (1, 4, 1), (8, 8, 1))])
def test_schedule_messages_match_reference_log(ref_lib, seed, dim, grid, ts):
    """The product's exchange list (order, ranks, dataset, face, points) equals
    the message log of the reference's DistContext::run_tiled on the same
    chains (two flushes, so the write history feeds the second analysis)."""
    from paper_1704_00693_b200 import ExecMode, Runtime

    gc = C.generate(seed, dim=dim, min_loops=2, max_loops=5, extent=(48, 72), max_radius=2)
    ref = ref_lib.RefRuntime(dim)
    ref.set_rank_grid(grid)
    C.declare(ref, gc)
    rt = Runtime(dim)
    rt.set_rank_grid(grid)
    for i, pts in enumerate(gc.stencils):
        rt.declare_stencil(f"s{i}", [p[:dim] for p in pts])
    from paper_1704_00693_b200 import Range
    for i in range(gc.ndat):
        rt.declare_field(f"f{i}", Range(dim, sum(([0, e] for e in gc.extent), [])))
    seen = 0
    for _ in range(2):
        C.enqueue(ref, gc)
        ref.flush(ExecMode.tiled(list(ts)))
        want = _ref_msgs(ref.dist_info())[seen:]
        seen += len(want)
        C.enqueue(rt, gc)
        s = rt.schedule_pending()
        got = []
        for m in s["msgs"]:
            pts = 1
            for lo, hi in m["box"]:
                pts *= hi - lo
            got.append((m["src"], m["dst"], m["ds"], m["dim"], m["dir"], pts))
        assert got == want


# ---- periodic box on a rank grid (Runtime::periodic_exchange's schedule) --------

def case_ns_periodic(make_rt):
    from paper_1704_00693_b200 import configs
    rt = make_rt(3, [1, 1, 2], periodic=True, skew=6)
    c = configs.NsC5(rt, 24)
    kes = [rt.fetch_reduction(c.enqueue_step()) for _ in range(2)]
    return c.outputs(), kes, rt.halo_messages


def test_c5_periodic_z_split_two_ranks(oracle_lib):
    # c5 split along z over two processes: the product's schedule (rewritten
    # chain with extended loops, the wraps, the deep-halo messages) drives an
    # oracle rank per process; ghost layers belong to the end ranks, the wrap
    # along z is a slab exchange between them. Conserved fields bit-exact
    # against a single-process oracle that copies the ghosts eagerly.
    from paper_1704_00693_b200 import configs
    ort = oracle_lib.OracleRuntime(3)
    co = configs.NsC5(ort, 24)
    want_ke = [ort.fetch_reduction(co.enqueue_step()) for _ in range(2)]
    want = co.outputs()
    fields, kes, msgs = run_world(case_ns_periodic)
    for k in want:
        assert np.array_equal(fields[k], want[k]), k
    for a, b in zip(kes, want_ke):
        assert abs(a - b) <= 1e-12 * abs(b)
    assert msgs > 0

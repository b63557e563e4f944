"""GPU parity of the distributed path on one B200: every rank
of a grid hosted on the device (Runtime.set_rank_grid, the reference's
simulated DistContext), each rank's fields owned +- pad, one halo exchange per
chain through device staging buffers, per-rank execution by the untiled or
windowed executor, rank-order reduction fold. Results must equal the
single-process oracle bit for bit (sums 1e-12 relative) and the reference's
own distributed run; the exchange must move exactly the reference's
messages."""
import numpy as np
import pytest

import chains as C
from paper_1704_00693_b200 import ExecMode, Range, Runtime, comm_unique_id, configs, parse_report

pytestmark = pytest.mark.gpu

MODES = [ExecMode.untiled(), ExecMode.tiled((0, 0, 0)), ExecMode.windowed(), ExecMode.tiled_auto()]


class _GridRuntime(Runtime):
    def __init__(self, dim, grid):
        super().__init__(dim)
        self.set_rank_grid(grid)


@pytest.mark.parametrize("mode", MODES, ids=["untiled", "tiled", "windowed", "auto"])
@pytest.mark.parametrize("seed,dim,grid", [(31, 2, (1, 2, 1)), (32, 2, (1, 4, 1)), (33, 2, (2, 2, 1)),
                                           (34, 3, (1, 1, 2)), (35, 3, (1, 2, 2)), (36, 1, (3, 1, 1))])
def test_random_chains_on_rank_grid_match_oracle(oracle_lib, mode, seed, dim, grid):
    gc = C.generate(seed, dim=dim, min_loops=2, max_loops=6, extent=(40, 72), max_radius=2)
    want = C.run(oracle_lib.OracleRuntime(dim), gc, None)
    got = C.run(_GridRuntime(dim, grid), gc, mode)
    C.assert_same(got, want, f"seed {seed} grid {grid}")


@pytest.mark.parametrize("mode", MODES, ids=["untiled", "tiled", "windowed", "auto"])
def test_repeated_chains_use_write_history(oracle_lib, mode):
    # Second and third flushes see the first's writes in the history
    # (exchange_flags, dist.cpp:79-115): still exact.
    gc = C.generate(41, dim=2, min_loops=3, max_loops=6, extent=(48, 64), max_radius=2)
    ora = oracle_lib.OracleRuntime(2)
    ids_o = C.declare(ora, gc)
    rt = _GridRuntime(2, (1, 3, 1))
    ids = C.declare(rt, gc)
    for _ in range(3):
        ho = C.enqueue(ora, gc)
        hg = C.enqueue(rt, gc)
        rt.flush(mode)
        rep = parse_report(rt.report_text())
        assert rep["distributed"] == "1" and int(rep["halo_messages"]) > 0
        ro = [(ora.fetch_reduction(h), op) for h, op in ho]
        rg = [(rt.fetch_reduction(h), op) for h, op in hg]
        C.assert_same(([], rg), ([], ro), "reductions")
    C.assert_same(([rt.download(d) for d in ids], []), ([ora.download(d) for d in ids_o], []), "fields")


def test_hydro_on_four_ranks_matches_reference_dist(ref_lib):
    # c2 structure at 96^2 on a {1,4,1} grid against the reference's own
    # simulated ranks: fields exact, mins exact, same halo traffic.
    ref = ref_lib.RefRuntime(2)
    ref.set_rank_grid((1, 4, 1))
    ref.set_default_mode(ExecMode.tiled((1 << 20, 1 << 20, 1)))
    hr = configs.HydroC2(ref, 96)
    rt = _GridRuntime(2, (1, 4, 1))
    rt.set_default_mode(ExecMode.tiled_auto())
    hg = configs.HydroC2(rt, 96)
    for _ in range(4):
        assert rt.fetch_reduction(hg.enqueue_step()) == ref.fetch_reduction(hr.enqueue_step())
    got, want = hg.outputs(), hr.outputs()
    for k in want:
        n = 96
        sl = (slice(-hr.rt.alloc_range(0).start(1), n - hr.rt.alloc_range(0).start(1)),
              slice(-hr.rt.alloc_range(0).start(0), n - hr.rt.alloc_range(0).start(0)))
        assert np.array_equal(got[k][sl], want[k][sl]), k


def test_heat_on_rank_grid_host_access(oracle_lib):
    ora = oracle_lib.OracleRuntime(2)
    ho = configs.HeatC1(ora, 64)
    rt = _GridRuntime(2, (1, 2, 1))
    hg = configs.HeatC1(rt, 64)
    for rt_, h in ((ora, ho), (rt, hg)):
        h.enqueue_chain(steps=5)
        rt_.flush(ExecMode.tiled_auto())
    rep = parse_report(rt.report_text())
    assert int(rep["halo_messages"]) == 2  # u both ways once; v is written first
    assert np.array_equal(hg.outputs()["u"], ho.outputs()["u"])
    # get/put/fill_logical address the owning rank and every halo copy.
    want = ho.outputs()["u"]
    al = ora.alloc_range(ho.u)
    for p in [(0, 0), (63, 31), (5, 32), (17, 33), (-1, 32)]:
        assert rt.get(hg.u, p) == want[p[1] - al.start(1), p[0] - al.start(0)]
    rt.put(hg.u, (7, 32), 0.25)  # on the seam: owned by rank 1, halo of rank 0
    assert rt.get(hg.u, (7, 32)) == 0.25
    hg.enqueue_chain(steps=1)
    rt.flush(ExecMode.untiled())
    arr = want.copy()
    arr[32 - al.start(1), 7 - al.start(0)] = 0.25
    ora.upload(ho.u, arr)
    ho.enqueue_chain(steps=1)
    assert np.array_equal(hg.outputs()["u"], ho.outputs()["u"])
    rt.fill_logical(hg.v, 2.0)
    assert rt.get(hg.v, (3, 40)) == 2.0 and rt.get(hg.v, (-1, 40)) == 0.0


def test_process_rank_single_process_nccl():
    # One rank per process with a communicator of one (the NCCL transport's
    # init, all-gather and broadcast run; a grid of one has no messages).
    rt = Runtime(2)
    rt.set_process_rank((1, 1, 1), 0, comm_unique_id())
    h = configs.HydroC2(rt, 64)
    mins = [rt.fetch_reduction(h.enqueue_step()) for _ in range(2)]
    ref = Runtime(2)
    hr = configs.HydroC2(ref, 64)
    want = [ref.fetch_reduction(hr.enqueue_step()) for _ in range(2)]
    assert mins == want
    assert rt.get(h.d[0], (3, 3)) == ref.get(hr.d[0], (3, 3))


@pytest.mark.parametrize("grid", [(1, 2, 1), (2, 2, 1)])
def test_untiled_on_demand_exchange_matches_reference(ref_lib, grid):
    # DistContext::run_untiled (dist.cpp:691-788): a halo exchange before each
    # loop that reads stale faces. Same fields and the same message count and
    # bytes as the reference's own simulated ranks; the deep-halo (tiled)
    # schedule moves the chain's halos in one exchange of fewer, larger
    # messages (acceptance.cpp:348-386).
    steps = 5
    ref = ref_lib.RefRuntime(2)
    ref.set_rank_grid(grid)
    hr = configs.HeatC1(ref, 64)
    hr.enqueue_chain(steps=steps)
    rep_ref = ref.flush(ExecMode.untiled())
    rt = _GridRuntime(2, grid)
    hg = configs.HeatC1(rt, 64)
    hg.enqueue_chain(steps=steps)
    rep = rt.flush(ExecMode.untiled())
    assert int(rep["halo_messages"]) == int(rep_ref["halo_messages"]) > 0
    assert int(rep["halo_bytes"]) == int(rep_ref["halo_bytes"])
    assert int(rep["halo_exchanges"]) == steps  # one per Laplacian loop; the copies read at a point
    assert np.array_equal(hg.outputs()["u"], hr.outputs()["u"])
    # Deep halo on a fresh pair of runtimes: one exchange, fewer messages.
    rt2 = _GridRuntime(2, grid)
    h2 = configs.HeatC1(rt2, 64)
    h2.enqueue_chain(steps=steps)
    rep2 = rt2.flush(ExecMode.tiled((0, 0, 0)))
    assert int(rep2["halo_exchanges"]) == 1
    assert int(rep2["halo_messages"]) * steps == int(rep["halo_messages"])
    assert np.array_equal(h2.outputs()["u"], hr.outputs()["u"])


@pytest.mark.parametrize("mode", MODES, ids=["untiled", "tiled", "windowed", "auto"])
@pytest.mark.parametrize("seed,dim,grid", [(51, 2, (1, 3, 1)), (52, 2, (2, 2, 1)), (53, 3, (1, 1, 2))])
def test_poisoned_stale_halos_stay_exact(oracle_lib, monkeypatch, mode, seed, dim, grid):
    # TCG_POISON_HALOS=1: every halo point a chain (or an earlier one) writes
    # is NaN on every rank before the chain runs (dist.cpp:546-586); the
    # schedule must deliver or recompute every one it reads -- three flushes
    # of the chain still equal the oracle bit for bit.
    monkeypatch.setenv("TCG_POISON_HALOS", "1")
    gc = C.generate(seed, dim=dim, min_loops=3, max_loops=6, extent=(40, 64), max_radius=2)
    ora = oracle_lib.OracleRuntime(dim)
    ids_o = C.declare(ora, gc)
    rt = _GridRuntime(dim, grid)
    ids = C.declare(rt, gc)
    for _ in range(3):
        ho = C.enqueue(ora, gc)
        hg = C.enqueue(rt, gc)
        rt.flush(mode)
        ro = [(ora.fetch_reduction(h), op) for h, op in ho]
        rg = [(rt.fetch_reduction(h), op) for h, op in hg]
        C.assert_same(([], rg), ([], ro), "reductions")
    got = [rt.download(d) for d in ids]
    want = [ora.download(d) for d in ids_o]
    # Compare the logical (owned) points: poisoned halo copies are not part
    # of the global picture.
    for g, w, d in zip(got, want, ids):
        lg = rt.logical_range(d)
        al = rt.alloc_range(d)
        sl = tuple(slice(lg.start(k) - al.start(k), lg.end(k) - al.start(k)) for k in reversed(range(dim)))
        assert np.array_equal(g[sl], w[sl]), d

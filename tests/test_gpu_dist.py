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


_TWO_RANK = r"""
import os, sys
sys.path.insert(0, {repo!r}); sys.path.insert(0, {repo!r} + "/tests")
import numpy as np
import torch, torch.distributed as dist
rank = int(os.environ["RANK"]); world = int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo", rank=rank, world_size=world)
import paper_1704_00693_b200 as pkg
from paper_1704_00693_b200 import ExecMode, Runtime, configs
pkg.runtime.select_device(rank)
obj = [pkg.comm_unique_id() if rank == 0 else None]
dist.broadcast_object_list(obj, src=0)
rt = Runtime(3)
rt.set_process_rank((1, 1, world), rank, obj[0])
rt.set_default_mode(ExecMode.{mode}())
c = configs.Jacobi3DC3(rt, 48)
for _ in range(2):
    c.enqueue_chain()
    rt.flush()
box = rt.local_box(c.a)
mine = rt.download_box(c.a, box)
ref = Runtime(3)
ref.set_default_mode(ExecMode.untiled())
cr = configs.Jacobi3DC3(ref, 48)
for _ in range(2):
    cr.enqueue_chain()
    ref.flush()
want = ref.download_box(cr.a, box)
# compare the planes this rank owns
z0 = box.start(2); n = 48 // world
lo = rank * n - z0; hi = lo + n
assert np.array_equal(mine[lo:hi], want[lo:hi]), "rank %d differs" % rank
print("rank", rank, "ok", flush=True)
dist.destroy_process_group()
"""


@pytest.mark.parametrize("mode", ["tiled_auto", "untiled"])
def test_two_process_nccl_z_split(tmp_path, mode):
    # One rank per process / GPU, the deep-halo exchange carried by
    # ncclSend/ncclRecv straight from the field slabs. Needs two GPUs.
    import subprocess, sys, os
    # (torch must not be imported here: libtcg is linked against the system
    # NCCL and is already loaded; the children import torch first.)
    ngpu = subprocess.run(["nvidia-smi", "-L"], capture_output=True, text=True).stdout.count("GPU ")
    if ngpu < 2:
        pytest.skip("needs 2 GPUs")
    from pathlib import Path
    repo = str(Path(__file__).resolve().parent.parent)
    script = tmp_path / "two_rank.py"
    script.write_text(_TWO_RANK.format(repo=repo, mode=mode))
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr", "127.0.0.1", "--master-port", "29541", str(script)],
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and r.stdout.count(" ok") == 2, r.stdout[-2000:] + r.stderr[-4000:]


def test_depth_guard_refuses_halo_deeper_than_neighbour():
    # c3-shaped chain at N = 32 over 4 z-ranks: the 16-loop chain's halo depth
    # exceeds a neighbour's owned width (8 planes); the reference would read
    # stale values there, the schedule builder refuses.
    from paper_1704_00693_b200.runtime import PlanError
    rt = _GridRuntime(3, (1, 1, 4))
    rt.set_default_mode(ExecMode.tiled((0, 0, 0)))
    c = configs.Jacobi3DC3(rt, 32)
    c.enqueue_chain()
    with pytest.raises(PlanError):
        rt.flush()


@pytest.mark.parametrize("mode", [ExecMode.tiled_auto(), ExecMode.stream(), ExecMode.untiled()],
                         ids=["auto", "stream", "untiled"])
def test_c3_z_split_simulated_ranks_use_slab_copies(oracle_lib, mode):
    # BASELINE c3's decomposition (along z) on simulated ranks: the halo
    # messages are whole planes and move field to field (copy_slabs, the
    # peer-copy path), no staging pack.
    ort = oracle_lib.OracleRuntime(3)
    co = configs.Jacobi3DC3(ort, 40)
    rt = _GridRuntime(3, (1, 1, 2))
    rt.set_default_mode(mode)
    cg = configs.Jacobi3DC3(rt, 40)
    for _ in range(2):
        co.enqueue_chain()
        ort.flush()
        cg.enqueue_chain()
        rt.flush()
    rep = parse_report(rt.report_text())
    assert int(rep["halo_messages"]) > 0
    assert np.array_equal(cg.outputs()["a"], co.outputs()["a"])

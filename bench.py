#!/usr/bin/env python
"""Benchmark of the B200 lazy stencil-chain executor (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--config c2|c1|c3|c4] [--mode auto|untiled|tiled:X,Y,Z]

Workload (N=1): BASELINE.json configs[1], the c2 2D hydro-like chain at
4096^2 fp64 (8 datasets, 12 stencil loops + 1 min-reduction per step, one
chain per step closed by fetch_reduction). A step = one timestep of that
chain. Metric: cell-updates/s (one loop applied at one point of its recorded
range, bench_jacobi.cpp:26). Inputs (8 x 134 MB) exceed the 126 MB L2, so no
L2 flush is needed between steps.

value   device-resident whole-job throughput: K steps timed with CUDA events on
        the executor stream, max over ranks.
e2e     same metric through the public API with HOST buffers: the job uploads
        the 8 fields from pinned host memory, runs K steps (each step's
        min-reduction read back to the host), downloads the 8 fields; all
        copies inside the timed region.
--impl reference: the unmodified reference tilechain library
        (oracle/_ref/libtcref.so) on the host cores, same config and metric.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

METRIC = "stencil-chain cell-updates/s"
UNIT = "cell-updates/s"


def load_peaks():
    p = REPO / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def load_profile_traffic(key):
    p = REPO / "profiles" / "ncu_traffic.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d.get(key)
    return None


_SAMPLER = r"""
import sys, time, pynvml
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(int(sys.argv[1]))
print("max", pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM), flush=True)
while True:
    try:
        print(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
              pynvml.nvmlDeviceGetCurrentClocksEventReasons(h), flush=True)
    except Exception:
        pass
    time.sleep(0.01)
"""


class ClockSampler:
    """Samples SM clocks and throttle reasons via NVML during the timed region,
    from a child process (a sampling thread here would compete with the
    host-side launch loop for the GIL)."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index):
        self.index = index
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.proc = None

    def __enter__(self):
        import subprocess
        try:
            self.proc = subprocess.Popen([sys.executable, "-c", _SAMPLER, str(self.index)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            first = self.proc.stdout.readline().split()
            if first and first[0] == "max":
                self.max_mhz = int(first[1])
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if not self.proc:
            return
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        for line in out.splitlines():
            f = line.split()
            if len(f) != 2:
                continue
            self.samples.append(int(f[0]))
            mask = int(f[1])
            for bit, name in self.REASONS.items():
                if mask & bit and bit != 0x1:
                    self.reasons.add(name)

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def make_config(name, rt, n=None, ny=None):
    from paper_1704_00693_b200 import configs
    if name == "c2":
        return configs.HydroC2(rt, n or 4096, ny=ny)
    if name == "c1":
        return configs.HeatC1(rt, n or 1024)
    if name == "c3":
        return configs.Jacobi3DC3(rt, n or 512)
    if name == "c4":
        return configs.CgC4(rt, n or 4096)
    if name == "c5":
        return configs.NsC5(rt, n or 768)
    raise ValueError(name)


class Step:
    """One 'step' of each config through the Runtime API. The first call
    issues the par_loop calls from Python and records them as templates
    (Runtime.record_begin/record_end); later calls re-issue them through the
    C++ host path (Runtime.replay -> par_loop), the way the reference's C++
    apps drive it (apps.cpp:59-130). host="python" keeps every call in Python
    (2.3 us per enqueued loop)."""

    def __init__(self, name, cfg, rt, host="cxx"):
        self.name, self.cfg, self.rt = name, cfg, rt
        self.replay = host == "cxx" and hasattr(rt, "record_begin")
        self.tpl = None
        if name == "c4":
            cfg.start()

    def _python_step(self):
        c, rt = self.cfg, self.rt
        if self.name in ("c2", "c5"):
            rt.fetch_reduction(c.enqueue_step())
        elif self.name in ("c1", "c3"):
            c.enqueue_chain()
            rt.flush()
        elif self.name == "c4":
            c.iterate()

    def __call__(self):
        c, rt = self.cfg, self.rt
        if not self.replay:
            return self._python_step()
        if self.name == "c4":
            # two chains per iteration, scalars (beta / alpha) change every time
            if self.tpl is None:
                rt.record_begin()
                h = c.enqueue_pq()
                t0 = rt.record_end()
                pq = rt.fetch_reduction(h)
                alpha = c.rr / pq
                rt.record_begin()
                h = c.enqueue_update(alpha)
                t1 = rt.record_end()
                self.tpl = (t0, t1)
                c.finish_iteration(rt.fetch_reduction(h))
                return
            pq = rt.fetch_reduction(rt.replay(self.tpl[0], [c.beta])[0])
            alpha = c.rr / pq
            c.finish_iteration(rt.fetch_reduction(rt.replay(self.tpl[1], [alpha, alpha])[0]))
            return
        if self.tpl is None:
            rt.record_begin()
            h = c.enqueue_step() if self.name in ("c2", "c5") else c.enqueue_chain()
            self.tpl = rt.record_end()
            if self.name in ("c2", "c5"):
                rt.fetch_reduction(h)
            else:
                rt.flush()
            return
        hs = rt.replay(self.tpl)
        if self.name in ("c2", "c5"):
            rt.fetch_reduction(hs[-1])
        else:
            rt.flush()

    def cell_updates(self):
        c = self.cfg
        return {"c2": lambda: c.cell_updates_per_step(), "c1": lambda: c.cell_updates_per_chain(),
                "c3": lambda: c.cell_updates_per_chain(), "c4": lambda: c.cell_updates_per_iteration(),
                "c5": lambda: c.cell_updates_per_step()}[self.name]()

    def algorithmic_bytes(self):
        c = self.cfg
        return {"c2": lambda: c.bytes_per_step(), "c1": lambda: c.bytes_per_chain(), "c3": lambda: c.bytes_per_chain(),
                "c4": lambda: c.bytes_per_iteration(), "c5": lambda: c.bytes_per_step()}[self.name]()

    def compulsory_bytes(self):
        """Bytes a perfectly fused chain must move: each seeded dataset read
        once, each written dataset written once (over the recorded domain)."""
        c = self.cfg
        if self.name == "c2":
            return 16 * 8 * c.n * c.n
        if self.name == "c1":
            return 3 * 8 * c.n * c.n
        if self.name == "c3":
            return 3 * 8 * c.inner.volume()
        if self.name == "c5":
            # per RK stage every one of the 15 fields read once, 10 written once
            return 3 * (15 + 10) * 8 * c.n ** 3
        return 4 * 8 * c.n * c.n * 4 // 2


WORKLOAD_TEXT = {
    "c2": "c2_hydro2d: fp64 4096^2, 8 dats U[0.5,1.5) seed 7, 12 stencil loops (point/star5/box9/one-sided/star2) "
          "+ min-reduction per step, one chain per step closed by fetch_reduction",
    "c1": "c1_heat2d: fp64 1024^2, u U[0,1) seed 42, 20-loop chains (10 timesteps of lap + copy)",
    "c3": "c3_jacobi3d: fp64 512^3, 16-loop chains (8 sweeps a->b->a)",
    "c4": "c4_cg2d: fp64 4096^2 CG, 4 loops + 2 dot reductions per iteration",
    "c5": "c5_ns3d: fp64 768^3 periodic Taylor-Green vortex, 15 fields, 4th-order star2 differences, RK3: "
          "22 loops + 3 periodic ghost fills + kinetic-energy sum per step",
}


SHARDED = {"c2": 1, "c3": 2, "c5": 2}  # config -> dimension its domain is split along at N > 1


def workload_text(name, world):
    return WORKLOAD_TEXT[name]


def parse_mode(s):
    from paper_1704_00693_b200 import ExecMode
    if s == "auto":
        return ExecMode.tiled_auto()
    if s == "untiled":
        return ExecMode.untiled()
    if s.startswith("tiled:"):
        return ExecMode.tiled([int(v) for v in s[6:].split(",")])
    if s == "windowed":
        return ExecMode.windowed()
    if s == "stream":
        return ExecMode.stream()
    if s.startswith("windowed:"):
        return ExecMode.windowed([int(v) for v in s[9:].split(",")])
    raise ValueError(s)


def dist_setup(n_gpus):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch
        import torch.distributed as td
        torch.cuda.set_device(local)
        td.init_process_group("nccl", device_id=torch.device("cuda", local))
        dist = td
    return world, rank, local, dist


def max_over_ranks(v, dist):
    if dist is None:
        return v
    import torch
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def config_dict(name, world):
    """The workload description both arms print (identical by construction)."""
    sharded = world > 1 and name in SHARDED
    return {"workload": workload_text(name, world),
            "parallelism": (f"the BASELINE domain split into {world} slabs along {'xyz'[SHARDED[name]]} (strong "
                            "scaling), one rank per GPU, one deep-halo exchange per chain (NCCL send/recv of whole "
                            "rows / planes straight from the fields)" if sharded else
                            ("independent replicas" if world > 1 else "single GPU")),
            "l2": "inputs exceed the 126 MB L2; no flush needed"}


def barrier(dist):
    if dist is not None:
        dist.barrier()


def time_steps(rt, step, k):
    """Device time of k steps on the executor stream (CUDA events)."""
    import torch
    stream = torch.cuda.ExternalStream(rt.stream())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    rt.synchronize()
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(k):
        step()
    e1.record(stream)
    e1.synchronize()
    rt.synchronize()
    return e0.elapsed_time(e1)


def cpu_reference(cfg_name, k, warmup, budget_s=120.0, mode_pick=None, ny=None):
    """The unmodified reference (oracle/_ref) on the host cores: best of its
    untiled and tiled_auto modes, a bounded number of steps."""
    sys.path.insert(0, str(REPO / "oracle"))
    import pyoracle
    from paper_1704_00693_b200 import ExecMode
    if not pyoracle.ref_available():
        return None, "reference library oracle/_ref/libtcref.so not built"
    threads = os.cpu_count() or 1
    best = None
    modes = [("untiled", ExecMode.untiled()), ("tiled_auto", ExecMode.tiled_auto())]
    if mode_pick:
        modes = [m for m in modes if m[0] == mode_pick]
    for mname, mode in modes:
        rt = pyoracle.RefRuntime(3 if cfg_name in ("c3", "c5") else 2, threads=threads)
        rt.set_default_mode(mode)
        # c5 at 768^3 needs ~62 GB of host fields: the CPU sample runs 128^3.
        cfg = make_config(cfg_name, rt, n=128 if cfg_name == "c5" else None, ny=ny)
        st = Step(cfg_name, cfg, rt)
        t0 = time.perf_counter()
        st()  # probe step (also warm-up)
        t_step = time.perf_counter() - t0
        n = max(1, min(k, int(budget_s / max(t_step, 1e-3) / len(modes))))
        t0 = time.perf_counter()
        for _ in range(n):
            st()
        dt = time.perf_counter() - t0
        v = st.cell_updates() * n / dt
        if best is None or v > best[0]:
            best = (v, mname, n, dt)
        del rt
    v, mname, n, dt = best
    return {"value": v, "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": f"{n} full {cfg_name} steps at "
                      f"{'128^3 (BASELINE 768^3 does not fit host RAM)' if cfg_name == 'c5' else 'BASELINE size'} "
                      f"({dt:.1f} s), reference tilechain "
                      f"RuntimeConfig.threads={threads}, best of untiled/tiled_auto = {mname}"}, None


def run_reference_arm(args, world, rank, dist):
    if rank != 0:
        return 0
    # Same workload as the B200 arm: the BASELINE domain (split across the GPUs there).
    res, err = cpu_reference(args.config, args.steps + args.warmup, args.warmup, budget_s=args.ref_budget)
    if res is None:
        print(json.dumps({"impl": "reference", "unavailable": err}))
        return 0
    line = {"metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True,
            "scaling": "strong" if (world > 1 and args.config in SHARDED) else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE shapes)",
            "config": config_dict(args.config, world), "impl": "reference", "cpu_baseline": res,
            "e2e": {"value": res["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--mode", default="auto")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-untiled", action="store_true")
    ap.add_argument("--ref-budget", type=float, default=60.0)
    ap.add_argument("--shard", action="store_true", help="c2: use the sharded (NCCL) path even on one GPU")
    ap.add_argument("--report", action="store_true",
                    help="print the last flush's ExecutionReport to stderr (the reference CLI's --report, "
                         "tilechain_cli.cpp:133-136)")
    ap.add_argument("--host", default="cxx", choices=["cxx", "python"],
                    help="who re-issues the par_loop calls of a step: the C++ host path (step templates) or Python")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)  # the contract's minimum; --warmup is honoured above it
    # tiled_auto times each executor candidate three times per chain signature
    # before it settles: that is set-up, done before the warm-up steps.
    settle = 8 if args.mode == "auto" else 0

    # tiled_auto's per-chain executor choices persist here, so a profiler run
    # of the same command (kernels serialised, timings distorted) executes
    # the choices the timed run made.
    os.environ.setdefault("TCG_AUTOTUNE_FILE", str(REPO / f".tcg_autotune_{args.config}"))
    if os.environ.get("NCCL_DEBUG", "VERSION") == "VERSION":
        os.environ["NCCL_DEBUG"] = "WARN"  # keep stdout to the one JSON line
    if args.impl == "reference":
        # CPU arm: rank 0 alone works; no process group, no GPU.
        return run_reference_arm(args, int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), None)
    world, rank, local, dist = dist_setup(args.gpus)

    import torch
    import paper_1704_00693_b200 as pkg
    from paper_1704_00693_b200 import Runtime

    pkg.runtime.select_device(local)
    torch.cuda.set_device(local)
    mode = parse_mode(args.mode)

    # N > 1: c2 (along y), c3 and c5 (along z) split the BASELINE domain across
    # the GPUs -- strong scaling, one rank per process, one deep-halo exchange
    # per chain over NCCL (c5: plus one periodic wrap between the end ranks,
    # DESIGN.md §6); c1 / c4 run as independent replicas.
    sharded = (world > 1 or args.shard) and args.config in SHARDED

    def new_comm_id():
        # One NCCL unique id per communicator (every runtime gets its own).
        obj = [pkg.comm_unique_id() if rank == 0 else None]
        if dist is not None:
            dist.broadcast_object_list(obj, src=0)
        return obj[0]

    def build(m):
        rt = Runtime(3 if args.config in ("c3", "c5") else 2)
        if sharded:
            if args.config == "c5":
                rt.set_periodic_domain(True)  # ghost layers owned by the end ranks
            grid = [1, 1, 1]
            grid[SHARDED[args.config]] = world
            rt.set_process_rank(tuple(grid), rank, new_comm_id())
        rt.set_default_mode(m)
        cfg = make_config(args.config, rt)
        return rt, cfg, Step(args.config, cfg, rt, host=args.host)

    # ---- device-resident throughput (value) ----------------------------------
    rt, cfg, step = build(mode)
    for _ in range(settle + 1):  # set-up: template recording, plan construction / JIT, tiled_auto's trials
        step()
    for _ in range(args.warmup):
        step()
    barrier(dist)
    l0 = rt.launches()
    with ClockSampler(local) as clk:
        ms = time_steps(rt, step, args.steps)
    launches = rt.launches() - l0
    ms = max_over_ranks(ms, dist)
    # Whole-job cell-updates per step: the sharded domain counts once; each
    # replica counts its own.
    cu = step.cell_updates() if sharded else step.cell_updates() * world
    value = cu * args.steps / (ms / 1e3)
    report = pkg.parse_report(rt.report_text())
    if args.report and rank == 0:
        sys.stderr.write(rt.report_text())
    # Kernel durations for the roofline: the same K steps again with CUDA
    # events around every executor kernel on the executor stream (kept out of
    # the `value` run: the per-kernel event records cost host time per launch).
    rt.set_timing(True)
    ms_instr = time_steps(rt, step, args.steps)
    kt = rt.kernel_timing()
    rt.set_timing(False)
    # The dominant kernel: tiled_auto may settle on either executor per chain.
    tiled = kt["tiled_ms"] > kt["untiled_ms"]
    kname = "k_tiled" if tiled else "k_untiled"
    kms = kt["tiled_ms"] if tiled else kt["untiled_ms"]
    kn = kt["tiled_launches"] if tiled else kt["untiled_launches"]
    peak, peak_src = load_peaks()
    # Algorithmic bytes of this rank's share (kernel timing is per rank).
    alg = step.algorithmic_bytes() / (world if sharded else 1)
    comp = step.compulsory_bytes() / (world if sharded else 1)
    per_launch_alg = alg * args.steps / max(kn, 1)
    avg_ms = kms / max(kn, 1)
    achieved = per_launch_alg / (avg_ms / 1e3) / 1e9 if kn else None
    traffic = load_profile_traffic(f"{args.config}_{kname}")
    roofline = {"bound": "hbm", "kernel": kname, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak if achieved else None,
                "frac_nominal_8TBps": achieved / 8000.0 if achieved else None, "traffic": traffic,
                "traffic_source": "profiles/ncu_traffic.json: dram__bytes_read.sum + dram__bytes_write.sum per launch "
                                  "from a committed ncu --set full capture of this command (not measured in this run)",
                "peak_source": peak_src, "algorithmic_bytes_per_launch": per_launch_alg,
                "avg_launch_ms": avg_ms, "launches": kn,
                "kernel_share_of_step": kms / ms_instr if ms_instr else None,
                "timing": "per-kernel CUDA events on the executor stream over a repeat of the K timed steps "
                          f"({ms_instr / args.steps:.4f} ms/step instrumented)",
                "compulsory_bytes_per_launch": comp * args.steps / max(kn, 1),
                "frac_compulsory": (comp * args.steps / max(kn, 1)) / (avg_ms / 1e3) / 1e9 / peak if kn else None,
                "dram_GBps_from_traffic": (traffic / (avg_ms / 1e3) / 1e9) if (traffic and kn) else None,
                "frac_traffic": (traffic / (avg_ms / 1e3) / 1e9 / peak) if (traffic and kn) else None,
                "note": "achieved = untiled-chain (algorithmic) bytes / kernel time (SURVEY.md 8(d) effective GB/s); "
                        "a fused kernel keeps intermediates on chip, so frac > 1 is the fusion gain, not an HBM rate. "
                        "The HBM-side fractions of the same kernel: frac_compulsory (bytes a fully fused chain must "
                        "move / time / peak) and frac_traffic (committed ncu DRAM bytes per launch / time / peak)."}

    # ---- untiled executor on the same inputs (tiled-vs-untiled speedup) -------
    del rt, cfg, step
    fixed = {}
    plan_keys = ("executor", "tile_sizes", "cta_grid", "ctas", "max_skew", "grid_barriers", "subchains",
                 "computed_points", "halo_exchanges")
    plans = {args.mode: {k: report.get(k) for k in plan_keys}}
    if not args.no_untiled:
        for mname in ("untiled", "stream"):
            if mname == args.mode:
                continue
            rtu, cfgu, stepu = build(parse_mode(mname))
            for _ in range(args.warmup + 1):
                stepu()
            msu = time_steps(rtu, stepu, args.steps)
            fixed[mname] = cu * args.steps / (max_over_ranks(msu, dist) / 1e3)
            ru = pkg.parse_report(rtu.report_text())
            plans[mname] = {k: ru.get(k) for k in plan_keys}
            del rtu, cfgu, stepu
    # computed / recorded loop points of the last flush (overlapped tiles and
    # pipeline warm-up recompute points): the fused executors' redundancy.
    recorded = {"c4": 0.5}.get(args.config, 1.0) * (cu if sharded else cu / world)
    for pl in plans.values():
        try:
            cp = float(pl.get("computed_points") or 0)
        except (TypeError, ValueError):
            cp = 0.0
        pl["redundancy"] = cp / recorded if cp > 0 else None
    untiled_value = fixed.get("untiled", value if args.mode == "untiled" else None)
    tiled_value = fixed.get("stream", value if args.mode == "stream" else None)

    # ---- end-to-end through the public API with host buffers --------------------
    e2e = None
    if args.config == "c5" and not args.no_e2e:
        e2e = {"value": None, "note": "c5's five 4.2 GB conserved fields are generated slab by slab on the host; "
                                      "an end-to-end leg would need ~21 GB of pinned host copies -- skipped"}
    elif not args.no_e2e:
        rte, cfge, stepe = build(mode)
        ids = list(cfge.init.keys())
        boxes = getattr(cfge, "init_box", {})
        host = {}
        for ds in ids:
            t = torch.empty(cfge.init[ds].shape, dtype=torch.float64, pin_memory=True)
            t.numpy()[...] = cfge.init[ds]
            host[ds] = t.numpy()
        out = {ds: torch.empty(cfge.init[ds].shape, dtype=torch.float64, pin_memory=True).numpy() for ds in ids}
        for _ in range(settle + 1 + args.warmup):
            stepe()
        rte.synchronize()
        barrier(dist)
        t0 = time.perf_counter()
        for ds in ids:
            if ds in boxes and boxes[ds] != rte.alloc_range(ds):
                rte.upload_box(ds, host[ds], boxes[ds])
            else:
                rte.upload(ds, host[ds])
        for _ in range(args.steps):
            stepe()
        for ds in ids:
            if ds in boxes and boxes[ds] != rte.alloc_range(ds):
                rte.download_box(ds, boxes[ds], out=out[ds])
            else:
                rte.download(ds, out=out[ds])
        rte.synchronize()
        dt = max_over_ranks(time.perf_counter() - t0, dist)
        nbytes = sum(host[ds].nbytes for ds in ids) * world
        e2e = {"value": cu * args.steps / dt, "unit": UNIT,
               "h2d_bytes_per_step": nbytes / args.steps,
               "d2h_bytes_per_step": (nbytes + 8 * args.steps * (1 if args.config != "c4" else 2)) / args.steps,
               "definition": "job = upload all fields (pinned) + K steps (per-step reduction read back) + "
                             "download all fields; per-step bytes = job bytes / K"}
        del rte, cfge, stepe

    # ---- CPU baseline (reference library on the host cores) ----------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu, err = cpu_reference(args.config, 3, 0, budget_s=args.ref_budget / 2)
        if cpu is None:
            cpu = {"value": None, "unavailable": err}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
                "scaling": "strong" if (sharded and world > 1) else "weak",
                "vs_baseline": None, "dtype": "f64",
                "data": "synthetic: seeded PCG64 fields with the BASELINE config shapes and value ranges",
                "config": config_dict(args.config, world),
                "detail": {"mode": args.mode, "host": args.host,
                           "setup_steps": settle + 1,
                           "effective_GBps": alg * args.steps * world / (ms / 1e3) / 1e9,
                           "effective_frac_nominal_8TBps": alg * args.steps / (ms / 1e3) / 1e9 / 8000.0,
                           "halo": {k: report.get(k) for k in ("halo_messages", "halo_bytes")} if sharded else None,
                           "untiled_value": untiled_value, "tiled_value": tiled_value,
                           "speedup_vs_untiled": value / untiled_value if untiled_value else None,
                           "tiled_vs_untiled": tiled_value / untiled_value if tiled_value and untiled_value else None,
                           "plan": plans.get(args.mode), "plans": plans},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
                "clocks": clk.summary()}
        print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

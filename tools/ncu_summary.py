#!/usr/bin/env python
"""Summarise an ncu report (or a --metrics launch-list CSV) for profiles/.

    python tools/ncu_summary.py REPORT.ncu-rep [--key c2] [--traffic profiles/ncu_traffic.json]
    python tools/ncu_summary.py --launches LAUNCHES.csv

Prints a markdown table per kernel launch (duration, DRAM read/write bytes,
DRAM GB/s, SM throughput %, achieved occupancy, registers) and, with
--traffic, records the mean DRAM bytes per launch of each kernel family under
"<key>_<family>" (the `traffic` field of bench.py's roofline)."""
from __future__ import annotations

import argparse
import csv
import io
import json
import re
import subprocess
from collections import defaultdict
from pathlib import Path

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "nsecond": 1e-9, "usecond": 1e-6,
         "msecond": 1e-3, "second": 1, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1, "byte/second": 1, "Kbyte/second": 1e3, "Mbyte/second": 1e6,
         "Gbyte/second": 1e9, "Tbyte/second": 1e12, "%": 1, "": 1, "register/thread": 1, "inst": 1}
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "launch__registers_per_thread", "smsp__inst_executed.sum", "lts__t_bytes.sum"]


def family(name: str) -> str:
    m = re.search(r"(k_\w+)", name)
    if not m:
        return name[:40]
    return "k_untiled" if m.group(1) == "k_untiled2" else m.group(1)  # 2D instantiation, same executor


def val(row, units, idx, m):
    if m not in idx:
        return None
    v = row[idx[m]].replace(",", "")
    try:
        x = float(v)
    except ValueError:
        return None
    return x * SCALE.get(units[idx[m]], 1)


def read_report(path: Path):
    out = subprocess.run(["ncu", "-i", str(path), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = [r for r in csv.reader(io.StringIO(out))]
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    res = []
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        d = {m: val(r, units, idx, m) for m in METRICS}
        d["name"] = r[idx["Kernel Name"]]
        d["grid"] = r[idx.get("Grid Size", 0)] if "Grid Size" in idx else ""
        d["block"] = r[idx.get("Block Size", 0)] if "Block Size" in idx else ""
        res.append(d)
    return res


def table(res):
    lines = ["| # | kernel | grid | block | time (us) | DRAM read (MB) | DRAM write (MB) | DRAM GB/s | SM thru % | "
             "occupancy % | regs |", "|---|---|---|---|---|---|---|---|---|---|---|"]
    for i, d in enumerate(res):
        t = d["gpu__time_duration.sum"] or 0
        rd, wr = d["dram__bytes_read.sum"] or 0, d["dram__bytes_write.sum"] or 0
        bw = (rd + wr) / t / 1e9 if t else 0
        lines.append(f"| {i} | `{d['name'][:60]}` | {d['grid']} | {d['block']} | {t * 1e6:.1f} | {rd / 1e6:.1f} | "
                     f"{wr / 1e6:.1f} | {bw:.0f} | {d['sm__throughput.avg.pct_of_peak_sustained_elapsed'] or 0:.1f} | "
                     f"{d['sm__warps_active.avg.pct_of_peak_sustained_active'] or 0:.1f} | "
                     f"{int(d['launch__registers_per_thread'] or 0)} |")
    return "\n".join(lines)


def launches(path: Path):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr = [r for r in rows if r[0] == "ID"][0]
    idx = {h: i for i, h in enumerate(hdr)}
    agg = defaultdict(lambda: [0, 0.0])
    total = 0.0
    for r in rows:
        if not r[0].isdigit():
            continue
        t = float(r[idx["Metric Value"]].replace(",", "")) * SCALE.get(r[idx["Metric Unit"]], 1)
        f = family(r[idx["Kernel Name"]])
        agg[f][0] += 1
        agg[f][1] += t
        total += t
    lines = ["| kernel family | launches | total (us) | share of kernel time |", "|---|---|---|---|"]
    for f, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| `{f}` | {n} | {t * 1e6:.1f} | {t / total:.3f} |")
    return "\n".join(lines)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report", nargs="?")
    ap.add_argument("--launches")
    ap.add_argument("--key")
    ap.add_argument("--traffic")
    a = ap.parse_args()
    if a.launches:
        print(launches(Path(a.launches)))
        return
    res = read_report(Path(a.report))
    print(table(res))
    if a.traffic and a.key:
        fam = defaultdict(list)
        for d in res:
            fam[family(d["name"])].append((d["dram__bytes_read.sum"] or 0) + (d["dram__bytes_write.sum"] or 0))
        p = Path(a.traffic)
        cur = json.loads(p.read_text()) if p.exists() else {}
        for f, v in fam.items():
            cur[f"{a.key}_{f}"] = sum(v) / len(v)
        p.write_text(json.dumps(cur, indent=1, sort_keys=True) + "\n")
        print(f"\ntraffic per launch written to {p}: " + ", ".join(f"{a.key}_{f}" for f in fam))


if __name__ == "__main__":
    main()

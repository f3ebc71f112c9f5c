#!/usr/bin/env python
"""Summarise ncu evidence into profiles/ (run here, on the CPU box).

    python scripts/ncu_summary.py <tag> [gpurun_out]

Reads gpurun_out/launches_<tag>.csv (the --metrics gpu__time_duration.sum
launch list) and gpurun_out/prof_<tag>.ncu-rep (--set full capture) and
writes profiles/<tag>_launches.csv (per-kernel totals) and
profiles/<tag>_ncu.md (key metrics + the hottest source lines per kernel).
"""

import csv
import os
import subprocess
import sys
from collections import OrderedDict

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "L1/TEX Cache Throughput", "L2 Cache Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Executed Ipc Active", "Issue Slots Busy", "Achieved Occupancy",
        "Theoretical Occupancy", "Registers Per Thread", "Warp Cycles Per Issued Instruction",
        "Eligible Warps Per Scheduler", "No Eligible", "Executed Instructions",
        "Dynamic Shared Memory Per Block"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "sm__inst_executed_pipe_fp64.sum", "smsp__inst_executed.sum"]


def launch_totals(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    ni = h.index("Metric Name") if "Metric Name" in h else None
    tot = OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= mi or (ni is not None and r[ni] != "gpu__time_duration.sum"):
            continue
        v = float(r[mi].replace(",", ""))
        scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0,
                 "ms": 1e3}.get(r[ui], 1e-3)
        tot.setdefault(r[ki].split("(")[0], []).append(v * scale)
    return tot


def details(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    ki, mi, vi, ui = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"),
                      h.index("Metric Unit"))
    res = OrderedDict()
    for r in rows[1:]:
        k = r[ki].split("(")[0]
        if r[mi] in KEYS:
            res.setdefault(k, OrderedDict()).setdefault(r[mi], f"{r[vi]} {r[ui]}")
    return res


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    if len(rows) < 3:
        return {}
    h = rows[0]
    ki = h.index("Kernel Name")
    res = OrderedDict()
    for r in rows[2:]:
        k = r[ki].split("(")[0]
        d = res.setdefault(k, OrderedDict())
        for m in RAW:
            if m in h and m not in d:
                d[m] = r[h.index(m)]
    return res


def hot_lines(rep, kernel, n=12, launch=None):
    """Hottest source lines (by stall samples) of ONE launch of `kernel` (the
    launch-th matching launch: one size-bucket instantiation at a time)."""
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from ncu_lines import lines

    agg = lines(rep, kernel, launch)
    ts = sum(a[1] for a in agg.values()) or 1
    ti = sum(a[2] for a in agg.values()) or 1
    return [(f, ln, src, 100.0 * s / ts, 100.0 * i / ti)
            for (f, ln), (src, s, i, _t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:n]]


def main():
    tag = sys.argv[1]
    src = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out"
    os.makedirs("profiles", exist_ok=True)
    lines = [f"# ncu summary — {tag}", ""]
    lpath = os.path.join(src, f"launches_{tag}.csv")
    if os.path.exists(lpath):
        tot = launch_totals(lpath)
        with open(f"profiles/{tag}_launches.csv", "w") as f:
            f.write("kernel,launches,total_us,mean_us\n")
            for k, v in sorted(tot.items(), key=lambda x: -sum(x[1])):
                f.write(f"\"{k}\",{len(v)},{sum(v):.1f},{sum(v) / len(v):.1f}\n")
        lines += ["## Launch list (`--metrics gpu__time_duration.sum`, cold, serialised)", "",
                  "| kernel | launches | total µs | share |", "|---|---|---|---|"]
        grand = sum(sum(v) for v in tot.values())
        for k, v in sorted(tot.items(), key=lambda x: -sum(x[1]))[:14]:
            lines.append(f"| `{k}` | {len(v)} | {sum(v):.1f} | {100 * sum(v) / grand:.1f}% |")
        lines.append("")
    rep = os.path.join(src, f"prof_{tag}.ncu-rep")
    if os.path.exists(rep):
        det, rw = details(rep), raw(rep)
        for k, d in det.items():
            lines += [f"## `{k}` (`--set full`)", ""]
            for m, v in d.items():
                lines.append(f"- {m}: {v}")
            for m, v in rw.get(k, {}).items():
                lines.append(f"- {m}: {v}")
            short = k.split("<")[0].split("::")[-1].replace("void ", "").strip()
            same = [x for x in det if x.split("<")[0].split("::")[-1].replace(
                "void ", "").strip() == short]
            hl = hot_lines(rep, short, launch=same.index(k))
            if hl:
                lines += ["", "| file:line | stall samples | instructions | source |",
                          "|---|---|---|---|"]
                for f, ln, s, ps, pi in hl:
                    lines.append(f"| {f}:{ln} | {ps:.1f}% | {pi:.1f}% | `{s}` |")
            lines.append("")
    with open(f"profiles/{tag}_ncu.md", "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines[:60]))


if __name__ == "__main__":
    main()

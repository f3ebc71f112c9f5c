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
    tot = OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= mi:
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


def hot_lines(rep, kernel, n=12):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass", "-k", "regex:" + kernel], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    cur, hdr, agg = None, None, []
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr and r[0].isdigit():
            d = dict(zip(hdr, r))
            try:
                agg.append((cur, int(r[0]), r[1].strip()[:80],
                            int(d.get("Warp Stall Sampling (All Samples)") or 0),
                            int(d.get("Instructions Executed") or 0)))
            except ValueError:
                pass
    ts = sum(a[3] for a in agg) or 1
    ti = sum(a[4] for a in agg) or 1
    return [(f, ln, src, 100.0 * s / ts, 100.0 * i / ti)
            for f, ln, src, s, i in sorted(agg, key=lambda a: -a[3])[:n]]


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
            hl = hot_lines(rep, short)
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

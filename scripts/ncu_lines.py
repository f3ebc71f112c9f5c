#!/usr/bin/env python
"""Per-source-line instruction / stall table of one kernel in an ncu report.

    python scripts/ncu_lines.py REPORT KERNEL_REGEX [N] [--launch I]

KERNEL_REGEX matches the kernel's base name (e.g. k_build); --launch I
selects the I-th matching launch of the report (e.g. one size bucket)."""
import csv
import re
import subprocess
import sys


def lines(rep, regex, launch=None):
    args = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
            "-k", "regex:" + regex]
    if launch is not None:
        args += ["--launch-skip", str(launch), "--launch-count", "1"]
    out = subprocess.run(args, capture_output=True, text=True).stdout
    cur, hdr, agg = None, None, {}
    for r in csv.reader(out.splitlines()):
        if not r:
            continue
        if r[0] in ("File Name", "File Path"):
            cur = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr and r[0].isdigit():
            d = dict(zip(hdr[2:], r[2:]))
            try:
                s = int(d.get("Warp Stall Sampling (All Samples)") or 0)
                i = int(d.get("Instructions Executed") or 0)
                th = int(d.get("Thread Instructions Executed") or 0)
            except ValueError:
                continue
            key = (cur, int(r[0]))
            a = agg.setdefault(key, [r[1].strip()[:90], 0, 0, 0])
            a[1] += s
            a[2] += i
            a[3] += th
    return agg


def main():
    rep, regex = sys.argv[1], sys.argv[2]
    n = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3].isdigit() else 25
    launch = int(sys.argv[sys.argv.index("--launch") + 1]) if "--launch" in sys.argv else None
    agg = lines(rep, regex, launch)
    ts = sum(a[1] for a in agg.values()) or 1
    ti = sum(a[2] for a in agg.values()) or 1
    print(f"{regex}: {ti / 1e6:.1f}M warp instructions, {ts} stall samples")
    for by, col in (("instructions", 2), ("stalls", 1)):
        print(f"-- top by {by}")
        for (f, ln), (src, s, i, th) in sorted(agg.items(), key=lambda kv: -kv[1][col])[:n]:
            print(f"{f}:{ln:<5d} inst {100 * i / ti:5.1f}%  stall {100 * s / ts:5.1f}%  "
                  f"thr/inst {th / max(i, 1):4.1f} | {src}")


if __name__ == "__main__":
    main()

"""Per-kernel totals from an ncu launch-list CSV: python scripts/launch_table.py gpurun_out/launches_TAG.csv"""
import collections
import csv
import sys

for path in sys.argv[1:]:
    rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
    h = rows[0]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    agg = collections.defaultdict(lambda: [0.0, 0.0, 0])
    for r in rows[1:]:
        n = r[ki].split("(")[0][:60]
        v = float(r[vi].replace(",", ""))
        if r[mi] == "gpu__time_duration.sum":
            agg[n][0] += v
            agg[n][2] += 1
        else:
            agg[n][1] += v
    print(path)
    for n, (t, i, c) in sorted(agg.items(), key=lambda x: -x[1][0])[:12]:
        print(f"  {n:60s} {t / 1e3:9.1f}us {i / 1e6:8.1f}Minst n={c}")

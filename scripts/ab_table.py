"""Print the phases of gpurun_out/bench_TAG_*.json (A/B runs)."""
import glob
import json
import sys

for f in sorted(glob.glob(f"gpurun_out/bench_{sys.argv[1]}_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        p = d["phases_ms_per_step"]
        print(f.split("/")[-1][:-5].ljust(28), f"{d['value'] / 1e6:7.1f}M",
              " ".join(f"{k.replace('eager ', '')}={v:.3f}" for k, v in p.items()))
    except Exception as e:  # noqa: BLE001
        print(f, "ERR", e)

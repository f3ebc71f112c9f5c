"""Histogram of support sizes for a bench workload (GPU): python scripts/count_hist.py [C2]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2510_18838_b200 import device as D  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
    src, tgt, X, spec, desc = bench.workload(cfg, 0)
    src_d, tgt_d, X_d = D.to_device(src), D.to_device(tgt), D.to_device(X)
    marks = []
    Y, op, cnt, stats = bench.b200_step(src_d, tgt_d, X_d, spec, marks)
    torch.cuda.synchronize()
    c = cnt.counts.cpu().numpy()
    h = np.bincount(c)
    print(cfg, "nt", c.size, "mean", c.mean(), "max", c.max())
    for m in np.nonzero(h)[0]:
        print(f"  m={m:3d} {h[m]:8d} {h[m] / c.size:.4f}")


if __name__ == "__main__":
    main()

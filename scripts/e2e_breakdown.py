"""Wall-clock breakdown of the e2e path (host pinned buffers) for the C2 workload."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2510_18838_b200 import pointwise as P  # noqa: E402


def main():
    src, tgt, X, spec, desc = bench.workload("c2", 0)
    src_h = torch.from_numpy(src).pin_memory()
    tgt_h = torch.from_numpy(tgt).pin_memory()
    X_h = torch.from_numpy(X).pin_memory()
    for _ in range(3):
        P.PreparedTransfer(src_h, tgt_h, spec).apply(X_h)
    torch.cuda.synchronize()
    for rep in range(5):
        t0 = time.perf_counter()
        pt = P.PreparedTransfer(src_h, tgt_h, spec)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        Y = pt.apply(X_h)
        t3 = time.perf_counter()
        print(f"ctor {1e3*(t1-t0):.3f} ms (+sync {1e3*(t2-t1):.3f})  apply {1e3*(t3-t2):.3f} ms  "
              f"total {1e3*(t3-t0):.3f}")
    # raw copy rates
    d = torch.empty_like(X_h, device="cuda")
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        d.copy_(X_h, non_blocking=True)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        X_h.copy_(d, non_blocking=True)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
    nb = X_h.numel() * 8
    print(f"H2D {nb / (t1 - t0) / 1e9:.1f} GB/s  D2H {nb / (t2 - t1) / 1e9:.1f} GB/s ({nb / 1e6:.0f} MB)")
    # fit_point_cloud one-shot
    for rep in range(3):
        t0 = time.perf_counter()
        P.fit_point_cloud(src_h, X_h, tgt_h, spec)
        t1 = time.perf_counter()
        print(f"fit_point_cloud {1e3*(t1-t0):.3f} ms")


if __name__ == "__main__":
    main()

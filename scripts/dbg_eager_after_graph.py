"""Eager step timing before / after a GraphedTransfer exists in the process."""
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2510_18838_b200 import device as D  # noqa: E402

src, tgt, X, spec, desc = bench.workload("c2")
s_d, t_d, X_d = D.to_device(src), D.to_device(tgt), D.to_device(X)


def eager(tag):
    for i in range(4):
        m = []
        torch.cuda.synchronize()
        t = time.perf_counter()
        bench.b200_step(s_d, t_d, X_d, spec, m)
        torch.cuda.synchronize()
        ph = {b: round(ea.elapsed_time(eb), 3) for (a, ea), (b, eb) in zip(m[:-1], m[1:])}
        print(tag, i, round(1e3 * (time.perf_counter() - t), 3), ph, flush=True)


eager("before")
gt = D.GraphedTransfer(s_d, t_d, X_d, spec)
for _ in range(3):
    gt.run()
torch.cuda.synchronize()
print("graph check", gt.check(), flush=True)
eager("after")

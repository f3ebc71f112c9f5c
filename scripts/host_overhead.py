"""Host-side overhead of one device step (cProfile + per-phase wall clock)."""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, ".")
import torch

import bench
from paper_2510_18838_b200 import device as D

src, tgt, X, spec, desc = bench.workload("c2", 0)
src_d, tgt_d, X_d = D.to_device(src), D.to_device(tgt), D.to_device(X)
for _ in range(3):
    bench.b200_step(src_d, tgt_d, X_d, spec, [])
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    bench.b200_step(src_d, tgt_d, X_d, spec, [])
torch.cuda.synchronize()
print("wall per step ms", (time.perf_counter() - t0) * 100)
pr = cProfile.Profile()
pr.enable()
for _ in range(10):
    bench.b200_step(src_d, tgt_d, X_d, spec, [])
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)

"""Blocking overhead of distributed.map_gathered without communication: one
NCCL rank (the gather is a local copy), C2, B in {1, 2, 4, 8}; device time
per step (CUDA events, L2 flushed between steps)."""
import os
import socket
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2510_18838_b200 import device as D  # noqa: E402
from paper_2510_18838_b200.distributed import map_gathered  # noqa: E402

s = socket.socket()
s.bind(("127.0.0.1", 0))
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(s.getsockname()[1]))
s.close()
dist.init_process_group("nccl", rank=0, world_size=1)
src, tgt, X, spec, desc = bench.workload("c2")
src_d, tgt_d, X_d = D.to_device(src), D.to_device(tgt), D.to_device(X)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for B in (1, 2, 4, 8):
    for _ in range(3):
        map_gathered(src_d, tgt_d, X_d, spec, nblocks=B)
    tot = 0.0
    ph = {}
    for _ in range(10):
        flush.zero_()
        marks = []
        map_gathered(src_d, tgt_d, X_d, spec, nblocks=B, marks=marks)
        torch.cuda.synchronize()
        tot += marks[0][1].elapsed_time(marks[-1][1])
        for (a, ea), (b, eb) in zip(marks[:-1], marks[1:]):
            ph[b] = ph.get(b, 0.0) + ea.elapsed_time(eb) / 10
    print(f"B={B}: {tot / 10:.4f} ms/step", {k: round(v, 4) for k, v in ph.items()}, flush=True)
dist.destroy_process_group()

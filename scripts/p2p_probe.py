"""NVLink peer-copy bandwidth probe (one process, all visible GPUs): copy
engines (tensor.copy_ across devices, one or several streams) vs an SM copy
kernel writing straight into peer memory (torch elementwise copy with peer
access).  Prints GB/s per source GPU."""
import time

import torch

n = torch.cuda.device_count()
nbytes = 64 << 20
src = torch.empty(nbytes // 8, dtype=torch.float64, device="cuda:0").normal_()
dsts = [torch.empty_like(src, device=f"cuda:{q}") for q in range(1, n)]
for q in range(1, n):
    print("peer access 0->%d:" % q, torch.cuda.can_device_access_peer(0, q))


def timed(fn, reps=10):
    fn()
    for d in range(n):
        torch.cuda.synchronize(d)
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    for d in range(n):
        torch.cuda.synchronize(d)
    return (time.perf_counter() - t) / reps


streams = [torch.cuda.Stream(device="cuda:0") for _ in dsts]


def ce_one_stream():
    for d in dsts:
        d.copy_(src, non_blocking=True)


def ce_streams():
    for s, d in zip(streams, dsts):
        with torch.cuda.stream(s):
            d.copy_(src, non_blocking=True)


for name, fn in (("copy engines, 1 stream", ce_one_stream), ("copy engines, 1 stream/peer", ce_streams)):
    dt = timed(fn)
    print(f"{name}: {len(dsts) * nbytes / dt / 1e9:.0f} GB/s out of GPU 0 ({len(dsts)} peers)")
for q, d in enumerate(dsts, 1):
    dt = timed(lambda: d.copy_(src, non_blocking=True))
    print(f"single copy 0->{q}: {nbytes / dt / 1e9:.0f} GB/s")

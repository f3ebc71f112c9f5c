"""CPU (gloo, world_size 2): target sharding and the target-field all-gather
(paper_2510_18838_b200/distributed.py) -- the host logic of the N>1 path."""

import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2510_18838_b200.distributed import (gather_target_field, shard_bounds, shard_sizes,
                                               upload_replicated)


def test_shard_bounds_cover_exactly():
    for n in (0, 1, 7, 10, 1000003):
        for world in (1, 2, 3, 4, 8):
            b = [shard_bounds(n, r, world) for r in range(world)]
            assert b[0][0] == 0 and b[-1][1] == n
            assert all(b[r][1] == b[r + 1][0] for r in range(world - 1))
            assert max(shard_sizes(n, world)) - min(shard_sizes(n, world)) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, C, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        full = torch.arange(n * C, dtype=torch.float64).reshape(n, C) * 0.5 + 1.0
        lo, hi = shard_bounds(n, rank, world)
        got = gather_target_field(full[lo:hi].clone(), n)
        got1 = gather_target_field(full[lo:hi, 0].clone(), n)
        up = upload_replicated(full)  # every rank holds `full`; 1/world of it is copied
        q.put((rank, bool(torch.equal(got, full) and torch.equal(up, full)),
               bool(torch.equal(got1, full[:, 0]))))
    finally:
        dist.destroy_process_group()


def _run(world, n, C):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, C, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def test_gather_target_field_world2_even_and_ragged():
    for n, C in ((10, 3), (7, 8)):  # 7 rows over 2 ranks: padded block
        res = _run(2, n, C)
        assert all(ok and ok1 for _, ok, ok1 in res), res


def test_sharded_rows_equal_serial_rows_oracle():
    # target sharding is exact: a shard's rows equal the same rows of the
    # serial result (the property the rendezvous path relies on,
    # rendezvous.py:452-495); checked on the CPU oracle
    from oracle import oracle as O
    from paper_2510_18838_b200 import synth

    src = synth.square(40).coords
    tg = np.random.RandomState(3).uniform(0, 1, (999, 2))
    vals = np.sin(src[:, 0]) + src[:, 1]
    full, st, _ = O.transfer(src, vals, tg, 2, O.RBF_C4, 2.0, ("adaptive", 12, 0.02, 1.5))
    parts = []
    for r in range(3):
        lo, hi = shard_bounds(tg.shape[0], r, 3)
        # r_max depends on the target set; pass the global one as the caller does
        v, _, _ = O.transfer(src, vals, tg[lo:hi], 2, O.RBF_C4, 2.0,
                             ("adaptive", 12, 0.02, 1.5))
        parts.append(v)
    assert np.array_equal(np.concatenate(parts), full)

"""The distributed caller: rendezvous coupling of
two partitioned applications on real ranks (paper_2510_18838_b200.rendezvous)
against the reference's in-process coupled_transfer (tests/golden/
rendezvous.npz, written by the reference itself).

CPU: gloo world 1 and 2, the fit done by the CPU oracle (pinned bitwise to
the reference) -- routing, exchange and MessageStats must reproduce the
reference exactly and the values bitwise.  GPU (-m gpu): one NCCL rank
hosting every rendezvous rank, the fit on the B200: stats exact, values
within 1e-12 of the reference (what its own CLI demands of a coupled run,
cli.py:172-176)."""

import os
import socket
from types import SimpleNamespace

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import golden

CASES = ["4_2_3", "2_4_4", "1_1_1"]


def _objects(d, key):
    from paper_2510_18838_b200.rendezvous import build_rdv_partition

    na, nb, nr = (int(x) for x in key.split("_"))
    own_a, own_b = d[f"own_a_{key}"], d[f"own_b_{key}"]
    field = SimpleNamespace(dof_points=lambda: d["coords_a"], values=d["values_a"],
                            location="vertices")
    pa = SimpleNamespace(n_ranks=na, dof_owner=lambda loc: own_a)
    mb = SimpleNamespace(coords=d["coords_b"], nverts=d["coords_b"].shape[0])
    pb = SimpleNamespace(n_ranks=nb, dof_owner=lambda loc: own_b)
    g = d[f"grid_{key}"]
    rdv = build_rdv_partition((d["lo"], d["hi"]), int(g[0]), int(g[1]), nr)
    return field, pa, mb, pb, rdv


def _spec(d):
    from paper_2510_18838_b200 import pointwise as P

    return P.FitSpec(2, P.RadialBasisSpec(P.RbfKind.C4, a=2.0), P.FixedRadius(float(d["r_c"])))


def _oracle_fit(src, vals, tgt, spec):
    from oracle import oracle as O

    v, st, _ = O.transfer(src, vals, tgt, spec.degree, O.RBF_C4, spec.rbf.a,
                          ("fixed", spec.selection.r_c))
    assert (st == 0).all()
    return v


def _check(d, key, values, stats, exact):
    want = d[f"values_{key}"]
    if exact:
        assert np.array_equal(values, want)
    else:
        assert np.max(np.abs(values - want)) <= 1e-12
    got = np.array([row[2:] for row in stats.table()], dtype=np.int64)
    assert [f"{r[0]}:{r[1]}" for r in stats.table()] == list(d[f"stats_roles_{key}"])
    assert np.array_equal(got, d[f"stats_{key}"])


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2510_18838_b200.rendezvous import coupled_pointwise

        d = golden("rendezvous")
        for key in CASES:
            vals, stats = coupled_pointwise(*_objects(d, key), _spec(d), fit=_oracle_fit)
            _check(d, key, vals, stats, exact=True)
        q.put((rank, "ok"))
    except Exception as exc:  # report to the parent
        q.put((rank, repr(exc)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [1, 2])
def test_coupled_pointwise_gloo_vs_reference(world):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(msg == "ok" for _, msg in res), res


@pytest.mark.gpu
def test_coupled_pointwise_nccl_b200_fit():
    import torch

    from paper_2510_18838_b200.rendezvous import coupled_pointwise

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(s.getsockname()[1]))
    s.close()
    dist.init_process_group("nccl", rank=0, world_size=1,
                            device_id=torch.device("cuda", torch.cuda.current_device()))
    try:
        d = golden("rendezvous")
        for key in CASES:
            vals, stats = coupled_pointwise(*_objects(d, key), _spec(d))
            _check(d, key, vals, stats, exact=False)
    finally:
        dist.destroy_process_group()

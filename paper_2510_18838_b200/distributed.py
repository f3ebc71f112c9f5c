"""Target sharding across GPUs and the one collective of the path (§8(e)).

Per-target work is independent (pointwise.py:1-8; bitwise chunk-invariant,
reference test_pointwise.py:231-237; the reference's own sharded path,
rendezvous.py:452-495, equals serial), so the build shards by target with
the source cloud replicated on every rank and no data-path exchange.  The
only collective is the all-gather of the target field, for callers that need
the full field on every rank: NCCL over NVLink / NVSwitch (`nccl` backend),
or gloo for the CPU tests.

    lo, hi = shard_bounds(nt, rank, world)
    pt = PreparedTransfer(src, targets[lo:hi], spec)      # this rank's rows
    Y_full = gather_target_field(pt.apply(X), nt)         # (nt, C) on all ranks
"""

import ctypes

import torch
import torch.distributed as dist


def shard_bounds(n, rank, world):
    """Contiguous, near-equal target blocks (the first n % world get one more)."""
    base, rem = divmod(int(n), int(world))
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def shard_sizes(n, world):
    return [shard_bounds(n, r, world)[1] - shard_bounds(n, r, world)[0] for r in range(world)]


def gather_target_field(Y_local, n_total, group=None):
    """All-gather row blocks (in rank order) into the full (n_total, C) field.

    Blocks are padded to the largest shard so one all_gather_into_tensor
    (a single NCCL all-gather) moves everything; padding rows are dropped."""
    world = dist.get_world_size(group)
    squeeze = Y_local.ndim == 1
    Y2 = Y_local.reshape(Y_local.shape[0], -1)
    sizes = shard_sizes(n_total, world)
    cap = max(sizes)
    if Y2.shape[0] != sizes[dist.get_rank(group)]:
        raise ValueError("local block does not match shard_bounds")
    if Y2.shape[0] != cap:
        pad = torch.zeros((cap, Y2.shape[1]), dtype=Y2.dtype, device=Y2.device)
        pad[:Y2.shape[0]] = Y2
        Y2 = pad
    out = torch.empty((world * cap, Y2.shape[1]), dtype=Y2.dtype, device=Y2.device)
    dist.all_gather_into_tensor(out, Y2.contiguous(), group=group)
    if any(s != cap for s in sizes):
        out = torch.cat([out[r * cap:r * cap + sizes[r]] for r in range(world)])
    return out[:, 0] if squeeze else out


def upload_replicated(host, group=None):
    """Put a host array that every rank holds (the replicated source cloud or
    source field) on every rank's GPU: each rank copies only its 1/world row
    block over its own PCIe link (pinned host memory: asynchronous), and one
    NCCL all-gather over NVLink assembles the whole array on every GPU.  The
    ranks' PCIe links share the host's memory bandwidth, NVLink does not."""
    world = dist.get_world_size(group)
    lo, hi = shard_bounds(host.shape[0], dist.get_rank(group), world)
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    return gather_target_field(host[lo:hi].to(dev, non_blocking=True), host.shape[0], group)


class _RawCuda:
    """__cuda_array_interface__ view of library-allocated device memory."""

    def __init__(self, ptr, shape):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<f8",
                                         "data": (int(ptr), False), "version": 3,
                                         "strides": None}


class _Exchange:
    """Receive buffer (world, nt, C) of this rank, allocated by the library,
    exported over CUDA IPC, and the peers' buffers opened here: fm_build_apply
    _blocks pushes this rank's rows straight into every peer's copy."""

    def __init__(self, world, rank, nt, C, group):
        L = _lib()
        self.world, self.rank, self.nt, self.C = world, rank, nt, C
        nbytes = world * nt * C * 8
        base = ctypes.c_void_p()
        _check(L.fm_device_alloc(nbytes, ctypes.byref(base)), "fm_device_alloc")
        self.base = base.value
        self.full = torch.as_tensor(_RawCuda(self.base, (world, nt, C)),
                                    device=torch.device("cuda", torch.cuda.current_device()))
        self.peers = []
        if world > 1:
            hs = L.fm_ipc_handle_size()
            h = (ctypes.c_char * hs)()
            _check(L.fm_ipc_export(ctypes.c_void_p(self.base), h), "fm_ipc_export")
            handles = [None] * world
            dist.all_gather_object(handles, bytes(h), group=group)
            for q in range(world):
                if q == rank:
                    continue
                p = ctypes.c_void_p()
                hq = (ctypes.c_char * hs).from_buffer_copy(handles[q])
                _check(L.fm_ipc_open(hq, ctypes.byref(p)), "fm_ipc_open")
                self.peers.append(p.value)
        # this rank's slot in every peer's buffer
        off = rank * nt * C * 8
        self.peer_slots = (ctypes.c_void_p * max(1, len(self.peers)))(
            *[p + off for p in self.peers]) if self.peers else None

    def close(self):
        L = _lib()
        for p in self.peers:
            L.fm_ipc_close(ctypes.c_void_p(p))
        self.peers = []
        if self.base:
            torch.cuda.synchronize()
            L.fm_device_free(ctypes.c_void_p(self.base))
            self.base = None


_EXCHANGES = {}


def _exchange(world, rank, nt, C, group, slot=0):
    key = (torch.cuda.current_device(), world, rank, nt, C, id(group), slot)
    ex = _EXCHANGES.get(key)
    if ex is None:
        ex = _EXCHANGES[key] = _Exchange(world, rank, nt, C, group)
    return ex


_PARITY = {}


def map_gathered(src_d, tgt_d, X_d, fitspec, nblocks=4, group=None, marks=None,
                 pipelined=False):
    """Target-sharded transfer of this rank's targets with the full target
    field delivered to every rank WHILE the operator is built: one grid, one
    target order whose processing positions come block by block
    (`nblocks` contiguous target index blocks), ONE select pass (the only host
    sync), then fm_build_apply_blocks (fieldmap_dist.h): per block, operator
    rows built, applied into this rank's slot of the receive buffer, and
    pushed by copy engines over NVLink into every peer's buffer (CUDA IPC)
    under the next block's build.  A collective on the side stream closes the
    exchange.  Returns the full field (world * nt_local, C) in rank order --
    bitwise gather_target_field(fit_point_cloud(src, X, tgt_local, fitspec))
    (per-target work does not depend on the blocking; r_max comes from this
    rank's whole target set).  The result is a view of a receive buffer that
    the next call with the same shapes overwrites.

    Selection / fit failures raise the reference's exceptions naming the
    rank-local target.  `marks` (list) receives (name, cuda event) pairs.

    pipelined=True returns (field, done) without waiting for the exchange:
    the peers' rows keep arriving (copy engines) while the caller goes on --
    e.g. maps the next batch; `done.wait()` (a torch.distributed Work) makes
    the current stream wait until the field is complete.  Two receive buffers
    alternate, so a field stays valid until the call after next."""
    from . import device as D
    from . import pointwise as P
    from ._lib import FmRbf, ptr

    def mark(name):
        if marks is not None:
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            marks.append((name, e))

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    nt = int(tgt_d.shape[0])
    X2 = X_d.reshape(X_d.shape[0], -1).contiguous()
    C = X2.shape[1]
    main = torch.cuda.current_stream()
    comm = _comm_stream()
    mark("start")
    bs, bt = D.device_bboxes([src_d, tgt_d])
    cloud = D.SourceCloud(src_d, bbox=bs)
    sel = fitspec.selection
    if isinstance(sel, P.AdaptiveRadius):
        dsel = D.adaptive(sel.min_points, sel.r0, sel.growth, P._r_max_device(cloud, tgt_d, bt))
        need = 0
    else:
        dsel = D.fixed(sel.r_c)
        need = P.n_monomials(fitspec.degree, cloud.dim)
    mark("grid")
    nblocks = max(1, min(int(nblocks), nt)) if nt else 1
    perm = cloud.target_order(tgt_d, nblocks=nblocks)
    sl = D.select(cloud, tgt_d, dsel, perm, need)
    if sl.stats[2] > 0:
        i = int(sl.stats[3])
        raise P.UnderdeterminedError(
            f"target {i} of rank {rank} has {int(sl.counts[i].item())} support points inside "
            f"radius {sel.r_c:g}; a degree-{fitspec.degree} fit needs at least {need}")
    if sl.stats[4] > 0:
        i = int(sl.stats[5])
        raise P.InsufficientSourcesError(
            f"target {i} of rank {rank}: only {int(sl.counts[i].item())} sources in the whole "
            f"domain, min_points is {sel.min_points}")
    mark("select")
    slot = 0
    if pipelined:
        pk = (torch.cuda.current_device(), world, nt, C, id(group))
        slot = _PARITY.get(pk, 0)
        _PARITY[pk] = slot ^ 1
    ex = _exchange(world, rank, nt, C, group, slot)
    Y = ex.full[rank]
    dev = tgt_d.device
    nnz = sl.nnz
    col = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
    val = torch.empty(max(nnz, 1), dtype=torch.float64, device=dev)
    status = torch.empty(max(nt, 1), dtype=torch.uint8, device=dev)
    stride = max(1, max(nt * (b + 1) // nblocks - nt * b // nblocks for b in range(nblocks)))
    blist = torch.empty(D._lib.FM_NBUCKETS * stride, dtype=torch.int32, device=dev)
    bcount = torch.empty(D._lib.FM_NBUCKETS, dtype=torch.int32, device=dev)
    stats = torch.empty(2 * nblocks, dtype=torch.int32, device=dev)
    csel = sl.sel.to_ctypes()
    rbf = P._rbf_pair(fitspec.rbf)
    crbf = FmRbf(int(rbf[0]), 0, float(rbf[1]))
    cfit = D._fit_struct(cloud.dim, fitspec.degree, fitspec.lam, fitspec.centering)
    lists = sl.lists()
    comm.wait_stream(main)  # the receive buffer is free (previous exchange closed)
    _check(_lib().fm_build_apply_blocks(
        ctypes.byref(cloud.grid), ptr(cloud.cell_start), ptr(cloud.sorted_pts),
        ptr(cloud.sorted_ids), ptr(tgt_d), nt, ptr(perm), ctypes.byref(csel), ptr(sl.radii),
        ctypes.byref(lists), ptr(sl.offsets), max(sl.max_count, 1), ctypes.byref(crbf),
        ctypes.byref(cfit), ptr(col), ptr(val), ptr(status), ptr(blist), ptr(bcount),
        ptr(stats), nblocks, ptr(X2), C, ptr(Y), len(ex.peers), ex.peer_slots,
        ctypes.c_void_p(main.cuda_stream), ctypes.c_void_p(comm.cuda_stream)),
        "fm_build_apply_blocks")
    mark("blocks")
    work = None
    if world > 1:
        # every rank's pushes precede its contribution to this collective on
        # its side stream: once it completes here, all peers' rows have landed
        with torch.cuda.stream(comm):
            flag = torch.zeros(1, dtype=torch.float32, device=dev)
            work = dist.all_reduce(flag, group=group, async_op=pipelined)
        if not pipelined:
            main.wait_stream(comm)
    mark("exchange")
    st = stats.view(nblocks, 2)
    if int(st[:, 0].sum().item()) > 0:
        bad = int(st[:, 1].min().item())
        raise P.SingularFitError(f"target {bad} of rank {rank}: fit failed "
                                 f"(status {int(status[bad].item())})")
    out = ex.full.reshape(world * nt, C)
    out = out[:, 0] if X_d.ndim == 1 else out
    if pipelined:
        return out, (work if work is not None else _Done())
    return out


class _Done:
    def wait(self):
        return True


class GraphedGather:
    """map_gathered(pipelined=True) with the rank's compute replayed as a CUDA
    graph (device.GraphedTransfer writing straight into this rank's slot of
    the receive buffer): per step, the bbox/geometry check, the graph, then
    the copy-engine pushes of the rank's rows to every peer and the closing
    collective on the side stream.  Two receive buffers (and two graphs)
    alternate, so a step's exchange completes under the next step."""

    def __init__(self, src_d, tgt_d, X_d, fitspec, group=None):
        from . import device as D

        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.group = group
        self.nt = int(tgt_d.shape[0])
        self.C = X_d.reshape(X_d.shape[0], -1).shape[1]
        self.ex = [_exchange(self.world, self.rank, self.nt, self.C, group, slot)
                   for slot in (0, 1)]
        self.gt = [D.GraphedTransfer(src_d, tgt_d, X_d, fitspec, out=e.full[self.rank])
                   for e in self.ex]
        self.slot = 0

    def step(self):
        """One mapping of the current points/field; returns (field, done)."""
        slot = self.slot
        self.slot ^= 1
        ex, gt = self.ex[slot], self.gt[slot]
        main = torch.cuda.current_stream()
        comm = _comm_stream()
        comm.wait_stream(main)
        gt.run()
        work = None
        if self.world > 1:
            nbytes = self.nt * self.C * 8
            _check(_lib().fm_push_rows(ctypes.c_void_p(gt.Y.data_ptr()), nbytes,
                                       self.rank * nbytes, len(ex.peers),
                                       (ctypes.c_void_p * len(ex.peers))(*ex.peers),
                                       ctypes.c_void_p(main.cuda_stream),
                                       ctypes.c_void_p(comm.cuda_stream)), "fm_push_rows")
            with torch.cuda.stream(comm):
                flag = torch.zeros(1, dtype=torch.float32, device=gt.Y.device)
                work = dist.all_reduce(flag, group=self.group, async_op=True)
        out = ex.full.reshape(self.world * self.nt, self.C)
        return out, (work if work is not None else _Done())

    def check(self):
        return [gt.check() for gt in self.gt if gt.key is not None]


def _lib():
    from . import _lib as L

    return L.lib()


def _check(rc, what):
    from . import _lib as L

    L.check(rc, what)


_COMM_STREAMS = {}


def _comm_stream():
    dev = torch.cuda.current_device()
    if dev not in _COMM_STREAMS:
        _COMM_STREAMS[dev] = torch.cuda.Stream(device=dev)
    return _COMM_STREAMS[dev]

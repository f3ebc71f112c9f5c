"""Distributed caller of the hot path: rendezvous coupling on real ranks
(SURVEY.md §8(f) rank 4).

The reference couples two partitioned applications through a structured
rendezvous partition in ONE process (rendezvous.py: ranks are indexed
contexts with mailboxes).  Its pointwise branch (_coupled_pointwise,
rendezvous.py:452-495):

  1. application A sends each source dof (x, y, value) to the rendezvous
     owner of its point and to every owner of a cell its r_c halo box
     overlaps (_scatter_with_halo, 423-440);
  2. application B sends each target request (x, y) to its anchor owner
     (_scatter_once, 443-447);
  3. each rendezvous rank fits its requested targets from its deduplicated
     local source cloud (_dedupe_sorted + fit_point_cloud, 462-483);
  4. the values go back to B's ranks, one message per (rdv, B) pair, ids
     ascending.

Here every torch.distributed rank hosts the rendezvous ranks r with
r % world == rank (and the application ranks likewise); messages between
ranks travel in two all_to_all exchanges per step (int64 ids + float64
payload, NCCL over NVLink with CUDA tensors, gloo on the CPU), and step 3 is
the B200 fit (pointwise.fit_point_cloud).  Routing, message grouping and the
MessageStats byte accounting (rendezvous.py:318-372: one message per
(src, dst) pair, 8 bytes per id and per payload value) are the reference's;
every rank ends with the same global stats table and the full target field.
"""

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from .errors import ExchangeError, FieldError

__all__ = ["RdvPartition", "build_rdv_partition", "AppPartition", "MessageStats",
           "coupled_pointwise"]


@dataclass(frozen=True)
class RdvPartition:
    """Structured rendezvous decomposition (rendezvous.py:43-103): cells
    half-open (lo, hi] per axis, closed at the bbox minimum edge; owner per
    cell."""

    bbox: np.ndarray
    nx: int
    ny: int
    n_ranks: int
    cell_owner: np.ndarray

    def _axis_cells(self, v, axis):  # rendezvous.py:65-71
        lo = self.bbox[0][axis]
        hi = self.bbox[1][axis]
        n = self.nx if axis == 0 else self.ny
        d = (hi - lo) / n
        c = np.ceil((np.asarray(v, dtype=np.float64) - lo) / d).astype(np.int64) - 1
        return np.clip(c, 0, n - 1)

    def cell_index_of(self, points):
        pts = np.asarray(points, dtype=np.float64).reshape(-1, 2)
        return self._axis_cells(pts[:, 1], 1) * self.nx + self._axis_cells(pts[:, 0], 0)

    def owner_of_points(self, points):
        return np.asarray(self.cell_owner)[self.cell_index_of(points)]

    def owners_in_box(self, lo_x, lo_y, hi_x, hi_y):
        ix0, ix1 = self._axis_cells([lo_x, hi_x], 0)
        iy0, iy1 = self._axis_cells([lo_y, hi_y], 1)
        cells = (np.arange(iy0, iy1 + 1)[:, None] * self.nx
                 + np.arange(ix0, ix1 + 1)[None, :]).reshape(-1)
        return np.unique(np.asarray(self.cell_owner)[cells])

    def contains_box(self, bbox):
        b = np.asarray(self.bbox)
        return (b[0] <= bbox[0] + 1e-30).all() and (bbox[1] <= b[1] + 1e-30).all()


def build_rdv_partition(bbox, nx, ny, n_ranks):
    """Round-robin row-major cell ownership (rendezvous.py:106-114)."""
    owner = np.arange(nx * ny, dtype=np.int64) % n_ranks
    return RdvPartition(np.asarray(bbox, dtype=np.float64).reshape(2, 2), int(nx), int(ny),
                        int(n_ranks), owner)


@dataclass(frozen=True)
class AppPartition:
    """Element ownership of one application's mesh (rendezvous.py:117-136):
    vertex dofs belong to the rank of their lowest-id incident element."""

    mesh: object
    elem_owner: np.ndarray
    n_ranks: int

    def vertex_owner(self):
        first = np.full(self.mesh.nverts, self.mesh.nelems, dtype=np.int64)
        np.minimum.at(first, np.asarray(self.mesh.tris).reshape(-1),
                      np.repeat(np.arange(self.mesh.nelems, dtype=np.int64), 3))
        return np.asarray(self.elem_owner)[first]

    def dof_owner(self, location):
        return self.vertex_owner() if location == "vertices" else np.asarray(self.elem_owner)


class MessageStats:
    """Per-(role, rank) message and byte counters of one transfer round
    (rendezvous.py:318-361), same rows and table()."""

    ROLES = ("app_a", "app_b", "rdv")
    _COLS = {"msgs_sent": 0, "msgs_recv": 1, "bytes_sent": 2, "bytes_recv": 3}

    def __init__(self, rank_counts):
        self.rank_counts = dict(rank_counts)
        self.rows = {(role, r): [0, 0, 0, 0] for role in self.ROLES
                     for r in range(self.rank_counts.get(role, 0))}

    def sent(self, role, rank, nbytes):
        row = self.rows[(role, rank)]
        row[0] += 1
        row[2] += nbytes

    def received(self, role, rank, nbytes):
        row = self.rows[(role, rank)]
        row[1] += 1
        row[3] += nbytes

    def total(self, role, column):
        c = self._COLS[column]
        return sum(v[c] for (role_, _), v in self.rows.items() if role_ == role)

    def table(self):
        return [(role, r) + tuple(self.rows[(role, r)]) for role in self.ROLES
                for r in range(self.rank_counts.get(role, 0))]

    def _as_tensor(self, device):
        keys = sorted(self.rows)
        return keys, torch.tensor([self.rows[k] for k in keys], dtype=torch.int64, device=device)


# ------------------------------------------------------------- messages
def _group(ids, srcs, dsts, payload):
    """One message per (src, dst), entities ascending by id
    (_group_messages, rendezvous.py:364-381): list of (src, dst, ids, rows)."""
    if ids.size == 0:
        return []
    order = np.lexsort((ids, dsts, srcs))
    ids, srcs, dsts, payload = ids[order], srcs[order], dsts[order], payload[order]
    brk = np.nonzero((srcs[1:] != srcs[:-1]) | (dsts[1:] != dsts[:-1]))[0] + 1
    b = np.concatenate([[0], brk, [ids.size]])
    return [(int(srcs[a]), int(dsts[a]), ids[a:e], payload[a:e]) for a, e in zip(b[:-1], b[1:])]


def _halo_pairs(rdv, pts, r_c, rows):
    """(row, destination) pairs of _scatter_with_halo (rendezvous.py:423-440)
    for the given rows: every owner of a cell the point's r_c box overlaps,
    plus its anchor owner, each once -- vectorised over the cells."""
    p = pts[rows]
    ix0 = rdv._axis_cells(p[:, 0] - r_c, 0)
    ix1 = rdv._axis_cells(p[:, 0] + r_c, 0)
    iy0 = rdv._axis_cells(p[:, 1] - r_c, 1)
    iy1 = rdv._axis_cells(p[:, 1] + r_c, 1)
    owners = np.asarray(rdv.cell_owner)
    sx = int((ix1 - ix0).max()) + 1 if rows.size else 0
    sy = int((iy1 - iy0).max()) + 1 if rows.size else 0
    rr, dd = [], []
    for dy in range(sy):
        for dx in range(sx):
            ok = (ix0 + dx <= ix1) & (iy0 + dy <= iy1)
            cells = (iy0 + dy) * rdv.nx + (ix0 + dx)
            rr.append(rows[ok])
            dd.append(owners[cells[ok]])
    rr.append(rows)
    dd.append(rdv.owner_of_points(p))
    r = np.concatenate(rr) if rr else np.empty(0, np.int64)
    d = np.concatenate(dd) if dd else np.empty(0, np.int64)
    key = np.unique(r * np.int64(rdv.n_ranks) + d)
    return key // rdv.n_ranks, key % rdv.n_ranks


def _exchange(msgs, ncols, world, group, device):
    """all_to_all of messages (src, dst, ids, payload rows) to the ranks
    hosting dst (dst % world).  Returns the received messages."""
    per = [[] for _ in range(world)]
    for m in msgs:
        per[m[1] % world].append(m)
    hdr, ids, val = [], [], []
    nh, ni = [], []
    for q in range(world):
        nh.append(3 * len(per[q]))
        ni.append(sum(m[2].size for m in per[q]))
        for src, dst, mid, mval in per[q]:
            hdr += [src, dst, mid.size]
            ids.append(mid)
            val.append(np.asarray(mval, dtype=np.float64).reshape(mid.size, ncols))
    i64 = lambda a: torch.as_tensor(np.asarray(a, dtype=np.int64), device=device)  # noqa: E731
    cnt = i64(np.column_stack([nh, ni]).reshape(-1))  # (header, id) counts per destination
    rcnt = torch.empty_like(cnt)
    dist.all_to_all_single(rcnt, cnt, group=group)
    rc = rcnt.cpu().numpy().reshape(world, 2)
    rh, ri = rc[:, 0].tolist(), rc[:, 1].tolist()
    h_in = torch.empty(sum(rh), dtype=torch.int64, device=device)
    dist.all_to_all_single(h_in, i64(hdr), output_split_sizes=rh, input_split_sizes=nh,
                           group=group)
    id_out = i64(np.concatenate(ids) if ids else np.empty(0))
    id_in = torch.empty(sum(ri), dtype=torch.int64, device=device)
    dist.all_to_all_single(id_in, id_out, output_split_sizes=ri, input_split_sizes=ni,
                           group=group)
    v_out = torch.as_tensor(np.concatenate(val).reshape(-1) if val else np.empty(0),
                            dtype=torch.float64, device=device)
    v_in = torch.empty(sum(ri) * ncols, dtype=torch.float64, device=device)
    dist.all_to_all_single(v_in, v_out, output_split_sizes=[n * ncols for n in ri],
                           input_split_sizes=[n * ncols for n in ni], group=group)
    h, idv, vv = h_in.cpu().numpy(), id_in.cpu().numpy(), v_in.cpu().numpy()
    out, o = [], 0
    for k in range(0, h.size, 3):
        src, dst, n = int(h[k]), int(h[k + 1]), int(h[k + 2])
        out.append((src, dst, idv[o:o + n], vv[o * ncols:(o + n) * ncols].reshape(n, ncols)))
        o += n
    return out


def _inbox(msgs, rank, ncols):
    """_inbox_concat (rendezvous.py:450-459): messages to `rank` in (src,
    dst) order."""
    mine = sorted((m for m in msgs if m[1] == rank), key=lambda m: (m[0], m[1]))
    if not mine:
        return np.empty(0, np.int64), np.empty((0, ncols)), np.empty(0, np.int64)
    return (np.concatenate([m[2] for m in mine]),
            np.concatenate([m[3].reshape(-1, ncols) for m in mine]),
            np.concatenate([np.full(m[2].size, m[0], np.int64) for m in mine]))


def _count(stats, msgs, src_role, dst_role, ncols):
    for src, dst, ids, _v in msgs:
        nbytes = 8 * (ids.size + ids.size * ncols)  # Message.nbytes, rendezvous.py:285-287
        stats.sent(src_role, src, nbytes)
        stats.received(dst_role, dst, nbytes)


def coupled_pointwise(source_field, source_partition, target_mesh, target_partition, rdv,
                      fitspec, group=None, fit=None, device=None):
    """coupled_transfer's pointwise branch (rendezvous.py:452-495, 601-629)
    across the ranks of `group`.  Returns (values on target_mesh vertices,
    full array on every rank, MessageStats with the global counts).

    `fit(src_xy, src_vals, targets, fitspec)` defaults to the B200
    pointwise.fit_point_cloud; `device` is where the exchanged tensors live
    (CUDA for NCCL, CPU for gloo; default: CUDA if available)."""
    from . import pointwise as P

    if not isinstance(fitspec.selection, P.FixedRadius):
        raise FieldError(
            "coupled pointwise transfer needs a fixed-radius selection; the "
            "halo width must be known from the method configuration")
    fit = fit or P.fit_point_cloud
    world = dist.get_world_size(group)
    me = dist.get_rank(group)
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device()) \
            if dist.get_backend(group) == "nccl" else torch.device("cpu")
    stats = MessageStats({"app_a": source_partition.n_ranks, "app_b": target_partition.n_ranks,
                          "rdv": rdv.n_ranks})
    r_c = fitspec.selection.r_c
    # 1. application A (hosted ranks): dof data to anchor + halo owners
    src_pts = np.asarray(source_field.dof_points(), dtype=np.float64)
    src_owner = np.asarray(source_partition.dof_owner(source_field.location))
    vals = np.asarray(source_field.values, dtype=np.float64).reshape(src_pts.shape[0])
    rows = np.flatnonzero(src_owner % world == me)
    hr, hd = _halo_pairs(rdv, src_pts, r_c, rows)
    payload = np.column_stack([src_pts, vals])
    msgs_a = _group(hr.astype(np.int64), src_owner[hr], hd, payload[hr])
    _count(stats, msgs_a, "app_a", "rdv", 3)
    in_a = _exchange(msgs_a, 3, world, group, device)
    # 2. application B (hosted ranks): target requests to anchor owners
    tgt = np.asarray(target_mesh.coords, dtype=np.float64)
    tgt_owner = np.asarray(target_partition.dof_owner("vertices"))
    rows_b = np.flatnonzero(tgt_owner % world == me)
    msgs_b = _group(rows_b.astype(np.int64), tgt_owner[rows_b],
                    rdv.owner_of_points(tgt[rows_b]), tgt[rows_b])
    _count(stats, msgs_b, "app_b", "rdv", 2)
    in_b = _exchange(msgs_b, 2, world, group, device)
    # 3. hosted rendezvous ranks fit their targets from deduped local clouds
    out_msgs = []
    for r in range(me, rdv.n_ranks, world):
        req_ids, req_xy, req_srcs = _inbox(in_b, r, 2)
        if req_ids.size == 0:
            continue
        sids, sdata, _s = _inbox(in_a, r, 3)
        order = np.argsort(sids, kind="stable")  # _dedupe_sorted, rendezvous.py:462-470
        sids, sdata = sids[order], sdata[order]
        keep = np.ones(sids.size, dtype=bool)
        keep[1:] = sids[1:] != sids[:-1]
        sdata = sdata[keep]
        values = np.asarray(fit(np.ascontiguousarray(sdata[:, :2]),
                                np.ascontiguousarray(sdata[:, 2]), req_xy, fitspec))
        for b_rank in np.unique(req_srcs):
            sel = req_srcs == b_rank
            o = np.argsort(req_ids[sel], kind="stable")
            out_msgs.append((r, int(b_rank), req_ids[sel][o], values[sel][o]))
    _count(stats, out_msgs, "rdv", "app_b", 1)
    in_v = _exchange(out_msgs, 1, world, group, device)
    # 4. B's hosted ranks place their values; every rank gets the full field
    out = torch.zeros(target_mesh.nverts, dtype=torch.float64, device=device)
    for src, dst, ids, v in in_v:
        if dst % world != me:
            raise ExchangeError(f"rank {me} received a message for B rank {dst}")
        out[torch.as_tensor(ids, device=device)] = torch.as_tensor(v.reshape(-1), device=device)
    dist.all_reduce(out, group=group)  # each target is delivered exactly once
    keys, t = stats._as_tensor(device)
    dist.all_reduce(t, group=group)
    for k, row in zip(keys, t.cpu().numpy().tolist()):
        stats.rows[k] = row
    return out.cpu().numpy(), stats

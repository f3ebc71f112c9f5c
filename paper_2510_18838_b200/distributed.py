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

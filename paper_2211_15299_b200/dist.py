"""Batch sharding over GPUs.

Signals are independent: rank g owns the contiguous slice
[g*B/G, (g+1)*B/G) of the batch (and of the per-signal supports), with no
data-path collective.  The only exchange is the optional final gather of
the B x k coefficients to every rank, one all_gather over NCCL (NVLink /
NVSwitch on a B200 node; gloo in the CPU tests).
"""

from __future__ import annotations


def shard_range(B: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced [start, stop) of B items for `rank` of `world`."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    base, extra = divmod(B, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def gather_rows(local, B: int, group=None):
    """All-gather row shards (each rank's contiguous slice) into (B, ...)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    sizes = [shard_range(B, r, world) for r in range(world)]
    width = max(b - a for a, b in sizes)
    pad = torch.zeros((width,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    if local.is_complex():
        pad = torch.view_as_real(pad)
    buf = torch.empty((world * width,) + tuple(pad.shape[1:]), dtype=pad.dtype, device=pad.device)
    dist.all_gather_into_tensor(buf, pad.contiguous(), group=group)
    buf = buf.view((world, width) + tuple(pad.shape[1:]))
    if local.is_complex():
        buf = torch.view_as_complex(buf)
    return torch.cat([buf[r, : b - a] for r, (a, b) in enumerate(sizes)], dim=0)

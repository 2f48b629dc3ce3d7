"""Multi-GPU plumbing for the split-linear path (one process per GPU).

The forward is row-parallel: per-token quantization (quantizer.py:95-101)
and the row-local MAC branch (layer.py:157-166) make any row sharding exact,
so the forward runs as token-sharded replicas with no collective. Only the
MOCD calibration statistics need collectives (see mocd_gpu): a MAX
all-reduce of the per-channel absmax statistics and an all-gather of the
integer rank counts.
"""

from __future__ import annotations


def token_shard(tokens: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced row range [lo, hi) of `rank`."""
    base, extra = divmod(tokens, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def gather_rows(local, tokens: int, group=None):
    """All-gather row shards (token_shard layout) into the full [tokens, ...]
    tensor on every rank (for callers that need the output on one device;
    the forward itself never calls it)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    sizes = [token_shard(tokens, r, world) for r in range(world)]
    width = max(h - l for l, h in sizes)
    pad = torch.zeros((width,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    return torch.cat([b[: h - l] for b, (l, h) in zip(bufs, sizes)], dim=0)

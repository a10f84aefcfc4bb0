"""Sharded d >= 2 applies across processes: marshalling and
the collective only -- every product step runs in libgpmatern.so (gp_kmvm_partial).

One process per GPU, each with the whole plan (its own gp_setup of the same points) and
all of v in rank order; rank r computes shard r of world_size (gp_kmvm_partial) and the
shards are summed with one all-reduce (NCCL on GPUs, gloo on the host)."""
from __future__ import annotations


def sharded_kmvm_rank(plan, v_rank, group=None, out=None, stream=None):
    """K v_rank (rank order, d >= 2) as the sum over the process group's shards."""
    import torch.distributed as dist
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    part = plan.kmvm_partial(v_rank, rank, world, out=out, stream=stream)
    dist.all_reduce(part, op=dist.ReduceOp.SUM, group=group)
    return part


def shard_plan(n: int, d: int, world: int):
    """The work split of every shard: [((tile_lo, tile_hi), (item_lo, item_hi)), ...]."""
    from . import shard_ranges
    return [shard_ranges(n, d, r, world) for r in range(world)]
